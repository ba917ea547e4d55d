"""CPU arm of bench.py: the REAL reference package (`localmap`, installed unmodified into
baseline/_ref by `pip install --target baseline/_ref`) timed on this host's cores.

Bench infrastructure, not product: nothing in paper_2511_02036_b200/ imports it.

The timed quantity is the reference's own per-stage clock, `StageTimings.triangulation_ms
+ fusion_ms` (pipeline.py:174-195), i.e. exactly the `create_map_points` + `run_fusion`
calls that the device path replaces, on the reference's stock `LocalMappingPipeline`:
  * mode="optimized": engine="batch" on `WorkerPool(os.cpu_count())` (config.py:141-143,
    parallel.py:41-69), the reference's own data-parallel path;
  * mode="baseline": engine="reference", one thread (the oracle engine).
LBA and keyframe culling are force-skipped on both sides (config.py:113-114), as on the
device, so the map evolves identically.

Steady state: the reference's cost per keyframe grows with the map (~4x between keyframes
0-11 and 100+ on C2), so the window timed is keyframes 100.. of C2, resumed from the
reference pipeline's own state after 100 keyframes. That state is pickled by
tests/golden/make_golden_steady.py (`--pickle-at 100`) into baseline/_state/ (git-ignored;
it travels to the GPU box with the snapshot). Unpickling breaks the `scale_counts` <->
counter-matrix view aliasing, so the views are rebound after loading.
When the reference or the state is missing, the NumPy port (oracle/) from an empty map is
timed instead and labelled "port".
"""

from __future__ import annotations

import os
import pickle
import platform
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(ROOT, "baseline", "_ref")
STATE_DIR = os.path.join(ROOT, "baseline", "_state")


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def reference_available() -> bool:
    return os.path.isfile(os.path.join(REF_DIR, "localmap", "pipeline.py"))


def _import_reference():
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import localmap  # noqa: F401
    from localmap import synth
    from localmap.config import FuseConfig, MatchConfig, PipelineConfig
    from localmap.pipeline import LocalMappingPipeline

    return synth, FuseConfig, MatchConfig, PipelineConfig, LocalMappingPipeline


class ReferenceWindow:
    """A reference LocalMappingPipeline resumed at keyframe `start` of a BASELINE config.

    `step()` processes the next keyframe and returns its (triangulation_ms, fusion_ms)."""

    def __init__(self, name: str, mode: str, start: int = 100, workers: int | None = None):
        from paper_2511_02036_b200.workload import BENCH_CONFIGS, BENCH_STAGE

        synth, FuseConfig, MatchConfig, PipelineConfig, LocalMappingPipeline = _import_reference()
        self.name, self.mode = name, mode
        kw = dict(BENCH_CONFIGS[name])
        n_nbr, n1, n2 = BENCH_STAGE[name]
        self.workers = 1 if mode == "baseline" else (workers or host_threads())
        self.seq = synth.generate_sequence(synth.WorldConfig(**kw))
        self.kfs = self.seq.to_keyframes()
        pc = PipelineConfig(mode=mode, worker_count=self.workers, force_skip_lba=True, force_skip_culling=True,
                            match=MatchConfig(neighbor_count=n_nbr), fuse=FuseConfig(n1=n1, n2=n2))
        self.pipe = LocalMappingPipeline(pc, num_levels=self.seq.intrinsics().num_levels)
        self.start = 0
        path = os.path.join(STATE_DIR, f"{name}_kf{start}.pkl")
        self.resumed = False
        if start and os.path.isfile(path):
            with open(path, "rb") as fh:
                blob = pickle.load(fh)
            st = blob["state"]
            m = st["model"]
            for mp in m.points.values():  # pickling breaks the view aliasing
                mp.scale_counts = m._counters[mp.mp_id]
            p = self.pipe
            p.model, p.store, p._recent, p._processed = m, st["store"], st["recent"], st["processed"]
            p.creation_stats, p.fusion_totals, p.culled_points = st["creation_stats"], st["fusion_totals"], st[
                "culled_points"]
            p._last_admitted_frame = self.kfs[start - 1].frame_index
            self.start = start
            self.resumed = True
        self.next = self.start

    def step(self) -> tuple[float, float]:
        kf = self.kfs[self.next]
        self.next += 1
        self.pipe.enqueue_keyframe(kf)
        t = self.pipe.process_one()
        return t.triangulation_ms, t.fusion_ms

    def close(self):
        self.pipe.close()


def time_reference(name: str = "c2", budget_s: float = 20.0, start: int = 100, modes=("optimized", "baseline"),
                   max_kfs: int = 4) -> dict:
    """Both reference modes on a steady-state window, each bounded by budget_s/len(modes)
    seconds of stage time (at least one keyframe). Returns the cpu_baseline record."""
    out = {"kind": "reference", "cpu": cpu_model(), "host_threads": host_threads(), "modes": {}}
    per_mode = budget_s / len(modes)
    for mode in modes:
        t_load = time.perf_counter()
        w = ReferenceWindow(name, mode, start)
        load_s = time.perf_counter() - t_load
        ms, kfs = [], []
        try:
            while w.next < len(w.kfs) and len(ms) < max_kfs:
                tri, fus = w.step()
                ms.append(tri + fus)
                kfs.append(w.next - 1)
                if sum(ms) * 1e-3 >= per_mode:
                    break
        finally:
            w.close()
        out["modes"][mode] = {"keyframes_per_s": len(ms) / (sum(ms) * 1e-3), "ms_per_keyframe": sum(ms) / len(ms),
                              "keyframes": [kfs[0], kfs[-1]], "threads": w.workers, "resumed_from_state": w.resumed,
                              "per_keyframe_ms": [round(x, 1) for x in ms], "setup_s": round(load_s, 1)}
    best = max(out["modes"], key=lambda m: out["modes"][m]["keyframes_per_s"])
    b = out["modes"][best]
    origin = (f"resumed from its own state after {start} keyframes" if b["resumed_from_state"]
              else "from an empty map (no pickled state)")
    out.update({"value": b["keyframes_per_s"], "unit": "keyframes/s", "cores": b["threads"], "best_mode": best,
                "window": b["keyframes"],
                "sample": f"real reference (baseline/_ref localmap) {name} keyframes {b['keyframes'][0]}-"
                          f"{b['keyframes'][1]} {origin}; StageTimings.triangulation_ms + fusion_ms; faster of "
                          f"modes {list(modes)} ({best}, {b['threads']} threads) on {out['cpu']}"})
    return out


def time_port(seq, name: str, budget_s: float) -> dict:
    """Fallback: the NumPy port (oracle/) from an empty map, one thread."""
    sys.path.insert(0, ROOT)
    from oracle import lm_oracle as O
    from paper_2511_02036_b200.workload import BENCH_STAGE

    n, n1, n2 = BENCH_STAGE["c2" if name == "c5" else name]
    c = seq.config
    cam = O.Cam(c.fx, c.fy, c.cx, c.cy, c.width, c.height, c.num_levels, c.scale_factor)
    pipe = O.OraclePipeline(c.num_levels, n, fc=O.FuseCfg(n1=n1, n2=n2))
    t0 = time.perf_counter()
    done = 0
    for rec in seq.records:
        pipe.step(O.okf_from_record(rec, cam))
        done += 1
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    return {"value": done / dt, "unit": "keyframes/s", "cores": 1, "kind": "port", "cpu": cpu_model(),
            "window": [0, done - 1],
            "sample": f"oracle (NumPy port; reference not installed in baseline/_ref or no pickled state) keyframes "
                      f"0..{done - 1} of the same sequence from an empty map, {dt:.1f} s"}
