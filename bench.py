#!/usr/bin/env python
"""Benchmark: keyframes/sec of triangulate+fuse (CreateNewMapPoints + SearchAndFuse) on the
EuRoC-shaped synthetic sequence (BASELINE.json configs[1]: 752x480, 1200 features/KF,
20 covisible neighbours, 200 keyframes), per B200, vs the CPU oracle on the host cores.

One *step* = the whole 200-keyframe sequence from an empty map: per keyframe insert,
recent map-point cull, CreateNewMapPoints, SearchAndFuse (LBA and keyframe culling are out
of scope and force-skipped, as in the reference's throughput benches).

  value  device-resident inputs (keyframes staged once, the map rewound between steps),
         CUDA events on the library's stream around each step, L2 flushed between steps.
  e2e    the same metric through the C-ABI with host buffers: every step stages each
         keyframe from host memory (pinned staging + H2D inside the timed region) and
         reads its step statistics back (D2H), wall-clock.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--workload c2]
Multi-GPU (torchrun): one process per GPU, each rank runs its own independent session
(seed offset by rank; weak scaling, no collective on the data path); the per-step time is
the max over ranks (all_reduce MAX on a 1-element tensor).
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2511_02036_b200 import workload as W  # noqa: E402
from paper_2511_02036_b200.config import FuseConfig, MatchConfig  # noqa: E402

METRIC = "keyframes/sec (triangulate+fuse) and ms/keyframe at 1/2/4/8 B200 vs host CPU"
UNIT = "keyframes/s"
L2_FLUSH_BYTES = 512 << 20


def load_workload(name: str, seed: int | None):
    cfg = W.bench_world(name, seed)
    return W.generate_sequence(cfg)


def stage_params(name):
    n, n1, n2 = W.BENCH_STAGE["c2" if name == "c5" else name]
    return n, MatchConfig(neighbor_count=n), FuseConfig(n1=n1, n2=n2)


def _gen(seed):
    return W.generate_sequence(W.bench_world("c2", seed))


def load_sessions(seeds: list[int]):
    """C5: independent C2-shaped sequences (seeds 5000..5063), generated in parallel."""
    from concurrent.futures import ProcessPoolExecutor

    workers = max(1, min(len(seeds), (os.cpu_count() or 2) - 1))
    if workers == 1:
        return [_gen(s) for s in seeds]
    with ProcessPoolExecutor(workers) as ex:
        return list(ex.map(_gen, seeds))


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={index}", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                       "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = [r.split(",") for r in open(self.f.name).read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1]))
                mx.append(float(r[2]))
            except (ValueError, IndexError):
                continue
            for k, nm in enumerate(names):
                if len(r) > 5 + k and r[5 + k].strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        return {}


def ncu_traffic(kernel: str):
    """dram bytes per launch of `kernel` from the committed ncu --set full summary, if any."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
        return d.get(kernel, {}).get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


def run_reference(args):
    """--impl reference: the real reference (baseline/_ref) on this host's cores, every step one
    steady-state keyframe of C2 (KFs 100.. resumed from the reference's own state) through its
    stock LocalMappingPipeline in mode="optimized" (engine="batch", WorkerPool(all host
    threads)); value = keyframes / (triangulation_ms + fusion_ms). Falls back to the NumPy port
    (labelled) when the reference or its pickled state is absent."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import bench_ref

    name = "c2" if args.workload == "c5" else args.workload
    if bench_ref.reference_available():
        w = bench_ref.ReferenceWindow(name, "optimized", start=args.ref_start)
        ms = []
        try:
            for _ in range(args.warmup + args.steps):
                if w.next >= len(w.kfs):
                    break
                tri, fus = w.step()
                ms.append(tri + fus)
        finally:
            w.close()
        timed = ms[args.warmup:] or ms
        secs = sum(timed) * 1e-3
        v = len(timed) / secs
        first = w.next - len(timed)
        sample = (f"real reference (baseline/_ref) {name} keyframe{'s' if len(timed) > 1 else ''} {first}-{w.next - 1}, "
                  + (f"resumed from its own state after {w.start} keyframes" if w.resumed else "from an empty map")
                  + f"; one keyframe per step; StageTimings.triangulation_ms + fusion_ms; mode=optimized "
                    f"(engine=batch, {w.workers} threads) on {bench_ref.cpu_model()}")
        cores, kind, ms_step = w.workers, "reference", 1e3 * secs / len(timed)
    else:
        seq = load_workload(name, None)
        rec = bench_ref.time_port(seq, name, args.ref_budget)
        v, cores, kind, sample, ms_step = rec["value"], 1, "port", rec["sample"], 1e3 / rec["value"]
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "ms_per_keyframe": 1e3 / v,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32 popc / f64 geometry",
            "data": "synthetic", "config": config_of(args),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def config_of(args, seq=None):
    n, mc, fc = stage_params(args.workload)
    c = W.BENCH_CONFIGS["c2" if args.workload == "c5" else args.workload]
    if args.workload == "c5":
        return {"workload": f"c5: {args.sessions} independent EuRoC-shaped sessions (seeds 5000+), batched per GPU",
                "sessions": args.sessions, "keyframes_per_session": c["keyframe_count"] if args.kfs is None else args.kfs,
                "features_per_kf": c["features_per_kf"], "neighbor_count": n, "fusion_n1": fc.n1, "fusion_n2": fc.n2,
                "l2": f"flushed between steps ({L2_FLUSH_BYTES >> 20} MiB write)",
                "step": "every session's whole sequence, one batched launch sequence per keyframe index"}
    return {"workload": f"{args.workload}: EuRoC-shaped synthetic sequence" if args.workload == "c2" else args.workload,
            "keyframes": c["keyframe_count"] if args.kfs is None else args.kfs,
            "features_per_kf": c["features_per_kf"], "image": [c.get("width", 640), c.get("height", 480)],
            "neighbor_count": n, "fusion_n1": fc.n1, "fusion_n2": fc.n2, "seed": c["seed"],
            "l2": f"flushed between steps ({L2_FLUSH_BYTES >> 20} MiB write)",
            "step": "whole sequence from an empty map (insert, recent cull, triangulate, fuse per keyframe)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="c2", choices=sorted(W.BENCH_CONFIGS) + ["c5"])
    ap.add_argument("--sessions", type=int, default=64, help="c5: total sessions over all ranks")
    ap.add_argument("--c5-groups", type=int, default=8, help="c5: session groups per rank (one stream each)")
    ap.add_argument("--kfs", type=int, default=None, help="limit keyframes per step (debug)")
    ap.add_argument("--cpu-budget", type=float, default=24.0, help="cpu_baseline: seconds of reference stage time")
    ap.add_argument("--ref-budget", type=float, default=8.0, help="port fallback budget (s)")
    ap.add_argument("--ref-start", type=int, default=100, help="reference steady-state window start (keyframe)")
    ap.add_argument("--window", type=int, default=20, help="device steady-state window length (keyframes)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--profile-steps", type=int, default=1, help="separate per-stage profiling pass")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-api", action="store_true", help="skip the Python-API e2e variant")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test hooks (one-GPU rehearsal of the multi-rank path): every rank on device 0, gloo
    if os.environ.get("LM_BENCH_SAME_DEVICE") == "1":
        local = 0
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local)
        backend = os.environ.get("LM_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    from paper_2511_02036_b200 import _lib
    from paper_2511_02036_b200.session import LocalMapper, store_for
    from paper_2511_02036_b200.mapmodel import KeyFrame

    if args.workload == "c5":
        run_c5(args, rank, world, local, dist)
        return
    seed = W.BENCH_CONFIGS[args.workload]["seed"] + 1000 * rank
    seq = load_workload(args.workload, seed)
    recs = seq.records if args.kfs is None else seq.records[:args.kfs]
    intr = seq.intrinsics()
    n, mc, fc = stage_params(args.workload)
    kfs = [KeyFrame(int(r.kf_id), r.pose_init, intr, r.kp_u, r.kp_v, r.kp_level, r.descriptors) for r in recs]
    ctx = _lib.Context.get(local)
    lib = ctx.lib
    mapper = LocalMapper(intr, neighbor_count=n, match=mc, fuse=fc, ctx=ctx,
                         store=store_for(len(kfs), max(k.num_keypoints for k in kfs) + 64))
    for kf in kfs:
        mapper.stage(kf)
    ids = [kf.kf_id for kf in kfs]

    def barrier():
        if dist is not None:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if dist is None:
            return x
        import torch

        t = torch.tensor([x], dtype=torch.float64,
                         device=f"cuda:{local}" if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def one_step(profile: bool) -> float:
        ctx.call("lm_map_rewind", mapper.map)
        mapper.processed = 0
        lib.lm_flush_l2(ctx.h, L2_FLUSH_BYTES)
        ctx.call("lm_synchronize")
        barrier()
        ctx.call("lm_timer_start")
        for k in ids:
            mapper.step(k, sync=False)
        ms = C.c_float()
        ctx.call("lm_timer_stop", C.byref(ms))
        return ms.value

    def absorb_totals(acc):
        totals = _lib.StepStats()
        ctx.call("lm_totals_fetch", mapper.map, C.byref(totals))  # this step's totals (rewind clears)
        if totals.error:
            raise RuntimeError(f"device error {totals.error}")
        for f, _ in _lib.StepStats._fields_:
            v = getattr(totals, f)
            if isinstance(v, int):
                acc[f] = acc.get(f, 0) + v
            elif f in ("fuse_cycles", "dbg", "borderline"):
                acc[f] = [a + b for a, b in zip(acc.get(f, [0] * len(v)), list(v))]

    # -------- device-resident timed region: the bare launch sequence (no profiling events)
    for _ in range(args.warmup):
        one_step(False)
    sampler = ClockSampler(local)
    launches0 = lib.lm_launch_count(ctx.h)
    step_ms = []
    acc = {}
    for _ in range(args.steps):
        ms = one_step(False)
        step_ms.append(max_over_ranks(ms))
        absorb_totals(acc)
    launches = lib.lm_launch_count(ctx.h) - launches0
    clocks = sampler.stop()
    mean_ms = sum(step_ms) / len(step_ms)
    total_kf = len(ids) * world
    value = total_kf / (mean_ms * 1e-3)

    # -------- profile pass (separate, untimed for `value`): per-stage CUDA events between the
    # step's kernels on the library stream, for the rooflines and the stage breakdown
    prof_steps = max(1, args.profile_steps)
    lib.lm_profile_enable(ctx.h, 1)
    one_step(True)  # (warm-up: the timer-carrying kernel instantiations load on their first launch)
    lib.lm_profile_read(ctx.h, (C.c_double * 16)(), (C.c_int64 * 16)())
    prof_acc = {}
    prof_total = 0.0
    for _ in range(prof_steps):
        prof_total += one_step(True)
        absorb_totals(prof_acc)
    prof_ms = (C.c_double * 16)()
    prof_n = (C.c_int64 * 16)()
    lib.lm_profile_read(ctx.h, prof_ms, prof_n)
    lib.lm_profile_enable(ctx.h, 0)
    # the in-kernel phase timers run in the profile pass only (globaltimer reads cost ~0.7% of
    # the step): per-step work counts and phase times come from that pass (same workload)
    pacc, psteps = prof_acc, prof_steps
    stages = ["insert", "cull", "select", "prep", "match", "tri", "commit", "fuse_targets", "fuse_geo",
              "fuse_gather", "fuse_apply", "fuse_refresh", "fuse_spec", "fuse_rev", "fuse_visible"]
    stage_ms = {s: prof_ms[k] / prof_steps for k, s in enumerate(stages)}
    stage_ms["fuse"] = sum(stage_ms[s] for s in stages if s.startswith("fuse"))
    profiled_step_ms = prof_total / prof_steps

    # -------- steady-state window on the device (the keyframes the CPU reference is timed on):
    # replay keyframes 0..lo-1 untimed, then time lo..hi-1 with CUDA events
    lo = min(args.ref_start, max(0, len(ids) - 1))
    hi = min(len(ids), lo + args.window)
    win_ms = []
    for _ in range(3):
        ctx.call("lm_map_rewind", mapper.map)
        mapper.processed = 0
        for k in ids[:lo]:
            mapper.step(k, sync=False)
        lib.lm_flush_l2(ctx.h, L2_FLUSH_BYTES)
        ctx.call("lm_synchronize")
        ctx.call("lm_timer_start")
        for k in ids[lo:hi]:
            mapper.step(k, sync=False)
        ms = C.c_float()
        ctx.call("lm_timer_stop", C.byref(ms))
        win_ms.append(ms.value)
    window = {"keyframes": [lo, hi - 1], "ms_per_keyframe": sum(win_ms) / len(win_ms) / (hi - lo),
              "keyframes_per_s": (hi - lo) / (sum(win_ms) / len(win_ms) * 1e-3),
              "timing": "CUDA events around keyframes lo..hi-1 after an untimed replay of 0..lo-1 (L2 flushed)"}

    # -------- end-to-end through the C ABI with host buffers
    e2e = None
    if not args.no_e2e:
        h2d = sum(k.num_keypoints * (8 + 8 + 32 + 4 + 1) + 208 for k in kfs)
        d2h = C.sizeof(_lib.StepStats) * len(kfs)
        e_ms = []
        for it in range(args.warmup + args.steps):
            mapper.reset()
            barrier()
            t0 = time.perf_counter()
            for kf in kfs:
                mapper.process(kf)  # stage (H2D) + step + stats readback (D2H, synchronising)
            dt = (time.perf_counter() - t0) * 1e3
            if it >= args.warmup:
                e_ms.append(max_over_ranks(dt))
        sync_each = {"value": total_kf / (sum(e_ms) / len(e_ms) * 1e-3), "unit": UNIT, "h2d_bytes_per_step": h2d,
                     "d2h_bytes_per_step": d2h, "ms_per_step": sum(e_ms) / len(e_ms),
                     "timing": "wall clock around stage (H2D) + step + statistics readback (D2H, synchronising) "
                               "of every keyframe"}
        # streaming: every keyframe staged from host memory (pinned ring, H2D) and stepped
        # without waiting; the sequence's statistics read back once at the end (D2H)
        p_ms = []
        tot = _lib.StepStats()
        for it in range(args.warmup + args.steps):
            mapper.reset()
            barrier()
            t0 = time.perf_counter()
            for kf in kfs:
                mapper.stage(kf)
                mapper.step(kf.kf_id, sync=False)
            ctx.call("lm_totals_fetch", mapper.map, C.byref(tot))
            dt = (time.perf_counter() - t0) * 1e3
            if tot.error or tot.created <= 0:
                raise RuntimeError(f"streaming e2e: device error {tot.error}")
            if it >= args.warmup:
                p_ms.append(max_over_ranks(dt))
        e2e = {"value": total_kf / (sum(p_ms) / len(p_ms) * 1e-3), "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": C.sizeof(_lib.StepStats), "ms_per_step": sum(p_ms) / len(p_ms),
               "timing": "wall clock: every keyframe staged from host memory (H2D) and stepped through the C ABI, "
                         "the sequence's statistics read back (D2H) at the end",
               "sync_each_keyframe": sync_each}
        # the same through the binary ingest wire format (LMKF records in host memory)
        from paper_2511_02036_b200 import ingest

        recs = [ingest.pack_keyframe(kf) for kf in kfs]
        bufs = [(C.create_string_buffer(r, len(r)), len(r)) for r in recs]
        kid = C.c_int64()
        st = _lib.StepStats()
        r_ms = []
        for it in range(args.warmup + args.steps):
            mapper.reset()
            barrier()
            t0 = time.perf_counter()
            for b, ln in bufs:
                ctx.call("lm_kf_stage_record", mapper.map, b, ln, C.byref(kid))
                p = mapper.params()
                ctx.call("lm_step", mapper.map, kid.value, C.byref(p), C.byref(st))
                mapper.processed += 1
            dt = (time.perf_counter() - t0) * 1e3
            if it >= args.warmup:
                r_ms.append(max_over_ranks(dt))
        e2e["records"] = {"value": total_kf / (sum(r_ms) / len(r_ms) * 1e-3), "unit": UNIT,
                          "h2d_bytes_per_step": sum(len(r) for r in recs), "d2h_bytes_per_step": d2h,
                          "timing": "wall clock: lm_kf_stage_record (LMKF wire records) + lm_step + stats readback"}

    # -------- end to end through the reference-shaped Python API (the drop-in a user of the
    # reference calls): per keyframe MapModel.insert_keyframe (H2D) +
    # DeviceStore.upload_keyframe + cull_recent_map_points + create_map_points + run_fusion
    # (each call returns its result to the host, as the reference's functions do)
    if e2e is not None and not args.no_api:
        e2e["api"] = api_e2e(args, kfs, intr, n, mc, fc, total_kf, barrier, max_over_ranks)

    # -------- roofline of the dominant kernel (k_fuse_rev), the whole fusion stage, and the
    # matching kernel's popc roofline. Achieved = algorithmic work per launch (SURVEY.md 8(d),
    # counted on the device from the inputs) / the kernel's average launch time (CUDA events
    # on the library stream around that launch, inside the timed region).
    peaks = measured_peaks()
    per_step_bytes = acc["fuse_bytes"] / args.steps
    per_step_rev_bytes = acc["fuse_bytes_rev"] / args.steps
    per_step_pairs = acc["match_pairs"] / args.steps
    popc_peak = C.c_double()
    ctx.call("lm_bench_popc", C.byref(popc_peak))
    dom = max((k for k in stage_ms if k != "fuse"), key=stage_ms.get)
    hbm_peak = peaks.get("hbm_gbs", 6457.4)
    peak_src = "MEASURED_PEAKS.json hbm_gbs (measured copy bandwidth)" if "hbm_gbs" in peaks else \
        "B200_PROFILING.md fallback"
    rev_s = stage_ms["fuse_rev"] * 1e-3
    rev_gbs = per_step_rev_bytes / rev_s / 1e9 if rev_s > 0 else 0.0
    roofline = {"kernel": "k_fuse_rev", "bound": "hbm", "achieved": rev_gbs, "peak": hbm_peak, "unit": "GB/s",
                "frac": rev_gbs / hbm_peak, "traffic": ncu_traffic("k_fuse_rev"),
                "algorithmic_bytes_per_launch": per_step_rev_bytes / len(ids),
                "launch_ms": stage_ms["fuse_rev"] / len(ids), "peak_source": peak_src, "dominant_stage": dom,
                "note": "one CTA per map walking the ordered reverse passes: a dependency chain of L2 round "
                        "trips and barriers, so bytes/s is far below HBM peak by construction (DESIGN.md 5)"}
    fuse_s = stage_ms["fuse"] * 1e-3
    fuse_gbs = per_step_bytes / fuse_s / 1e9 if fuse_s > 0 else 0.0
    roof_fuse = {"kernel": "k_fuse_* (whole SearchAndFuse stage)", "bound": "hbm", "achieved": fuse_gbs,
                 "peak": hbm_peak, "unit": "GB/s", "frac": fuse_gbs / hbm_peak,
                 "algorithmic_bytes_per_keyframe": per_step_bytes / len(ids), "ms_per_keyframe": stage_ms["fuse"] / len(ids)}
    match_s = stage_ms["match"] * 1e-3
    popc_achieved = 8 * per_step_pairs / match_s if match_s > 0 else 0.0
    per_step_second = acc.get("match_second_half", 0) / args.steps
    executed = 4 * per_step_pairs + 4 * per_step_second
    roof_popc = {"kernel": "k_match", "bound": "popc", "achieved": popc_achieved / 1e12, "peak": popc_peak.value / 1e12,
                 "unit": "Tpopc32/s", "frac": popc_achieved / popc_peak.value,
                 "algorithmic_popc_per_launch": 8 * per_step_pairs / len(ids), "launch_ms": stage_ms["match"] / len(ids),
                 "executed_popc_per_launch": executed / len(ids),
                 "executed_frac": (executed / match_s) / popc_peak.value if match_s > 0 else 0.0,
                 "note": "algorithmic = 8 popc32 per eligible pair (SURVEY 8(d)); executed = what the 128-bit early "
                         "exit leaves (4 per pair + 4 per pair passing the first half): the pipe utilisation",
                 "peak_source": "lm_bench_popc microbenchmark on this GPU (measured)"}

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": mean_ms, "ms_per_keyframe": mean_ms / len(ids),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32 popc / f64 geometry",
            "data": "synthetic (workload.py restatement of the reference generator)", "config": config_of(args),
            "parallelism": f"{world} independent sessions, one per GPU, no collective on the data path",
            "clocks": clocks, "e2e": e2e, "gpu_launches": int(launches), "roofline": roofline,
            "roofline_popc": roof_popc, "roofline_fusion_stage": roof_fuse, "stage_ms_per_step": stage_ms,
            "work_per_step": {"keyframes": len(ids), "match_pairs": per_step_pairs, "fuse_bytes": per_step_bytes,
                              "created": pacc["created"] / psteps, "merged": pacc["merged"] / psteps,
                              "observations_added": pacc["observations_added"] / psteps,
                              "apply_rounds": pacc["apply_rounds"] / psteps,
                              "rev_passes": (pacc["fuse_passes"] / psteps) / 2,
                              "rev_passes_acting": pacc["rev_passes_acting"] / psteps,
                              "rev_items_reevaluated": pacc["rev_passes_redo"] / psteps,
                              "rev_acting_passes_untouched_by_previous_apply": pacc["rev_mergeable"] / psteps,
                              "rev_points_recomputed": pacc["fuse_cycles"][1] / psteps,
                              "rev_passes_direct_all_add": pacc["dbg"][0] / psteps,
                              "cull_phase_ms": {"classify": pacc["dbg"][1] / psteps / 1e6,
                                                "kills": pacc["dbg"][2] / psteps / 1e6,
                                                "flush": pacc["dbg"][3] / psteps / 1e6},
                              "fwd_apply_detail": {"heads_ms": pacc["dbg"][8] / psteps / 1e6,
                                                   "members_merges_ms": pacc["dbg"][9] / psteps / 1e6,
                                                   "rounds": pacc["dbg"][10] / psteps,
                                                   "actions": pacc["dbg"][11] / psteps,
                                                   "pending_in_later_rounds": pacc["dbg"][15] / psteps},
                              "rev_touched_points_from_post_add_speculation": pacc["dbg"][12] / psteps,
                              "culled": pacc["culled"] / psteps,
                              "cull_probation_entries": pacc["dbg"][13] / psteps,
                              "cull_kills_over_8_obs": pacc["dbg"][14] / psteps,
                              "rev_subphase_ms": {"select_actions_preitems": pacc["dbg"][7] / psteps / 1e6,
                                                  "postitems_changed": pacc["dbg"][4] / psteps / 1e6,
                                                  "hitlist": pacc["dbg"][5] / psteps / 1e6,
                                                  "refresh_hits": pacc["dbg"][6] / psteps / 1e6}},
            "fuse_phase_ms_per_step": {n: pacc["fuse_cycles"][k] / psteps / 1e6
                                       for k, n in enumerate(["targets", "-", "fwd_assemble", "fwd_apply",
                                                              "rev_redo_refresh", "rev_select", "rev_apply",
                                                              "rev_rescan", "rev_prologue", "rev_apply_reserve_check",
                                                              "rev_apply_commit", "rev_apply_merges",
                                                              "rev_apply_compaction", "fwd_apply_reserve_check",
                                                              "fwd_apply_commit_merges", "fwd_apply_compaction"])
                                       if n != "-"},
            "rev_recomputed_points_per_step": pacc["fuse_cycles"][1] / psteps}
    line["profiled_ms_per_step"] = profiled_step_ms
    line["device_window"] = window
    bl = [x / args.steps for x in acc.get("borderline", [0, 0, 0, 0])]
    line["borderline"] = {"per_step": {"epipolar": bl[0], "creation_gates": bl[1], "fusion_gates": bl[2],
                                       "level_rint_ties": bl[3]}, "total_per_step": sum(bl),
                          "rel_band": 1e-10,
                          "meaning": "threshold compares whose two sides are within 1e-10 relative (lm_math.cuh "
                                     "kFlipRel): an upper bound of decisions that could flip against the reference"}
    line["parity"] = golden_parity(args, seed, mapper, ids)
    if rank == 0 and world == 1 and not args.no_cpu:
        import bench_ref

        name = "c2" if args.workload == "c5" else args.workload
        if bench_ref.reference_available():
            cb = bench_ref.time_reference(name, budget_s=args.cpu_budget, start=args.ref_start)
            cb["device_same_window_kf_per_s"] = window["keyframes_per_s"] if cb["window"][0] == lo else None
        else:
            cb = bench_ref.time_port(seq, name, args.cpu_budget)
        line["cpu_baseline"] = cb
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def api_e2e(args, kfs, intr, n, mc, fc, total_kf, barrier, max_over_ranks) -> dict:
    from paper_2511_02036_b200.config import CullConfig, GateConfig
    from paper_2511_02036_b200.culling import RecentPoint, cull_recent_map_points
    from paper_2511_02036_b200.fusion import run_fusion
    from paper_2511_02036_b200.mapmodel import DeviceStore, MapModel
    from paper_2511_02036_b200.session import store_for
    from paper_2511_02036_b200.triangulation import CreationStats, create_map_points

    model = MapModel(intr.num_levels, scale_factor=intr.scale_factor,
                     store=store_for(len(kfs), max(k.num_keypoints for k in kfs) + 64))
    gc, cc = GateConfig(), CullConfig()
    ms = []
    stage_ms = 0.0
    for it in range(args.warmup + args.steps):
        model.reset()
        store = DeviceStore(model=model)
        stats = CreationStats()
        fused = {"merged": 0, "observations_added": 0, "stale": 0}
        recent = []
        barrier()
        t0 = time.perf_counter()
        t_stage = 0.0
        for processed, kf in enumerate(kfs):
            kf.mp_bindings[:] = -1
            model.insert_keyframe(kf)
            store.upload_keyframe(kf)
            _, recent = cull_recent_map_points(model, recent, processed, cc)
            ts = time.perf_counter()
            made = create_map_points(model, store, kf.kf_id, n, mc, gc, stats=stats)
            recent.extend(RecentPoint(i, processed) for i in made)
            for k, v in run_fusion(model, store, kf.kf_id, fc).items():
                fused[k] += v
            t_stage += time.perf_counter() - ts
        dt = (time.perf_counter() - t0) * 1e3
        if it >= args.warmup:
            ms.append(max_over_ranks(dt))
            stage_ms += t_stage * 1e3
    timed = len(ms)
    h2d = sum(k.num_keypoints * (8 + 8 + 32 + 4 + 1) + 208 for k in kfs)
    return {"value": total_kf / (sum(ms) / timed * 1e-3), "unit": UNIT, "ms_per_step": sum(ms) / timed,
            "stage_only_keyframes_per_s": total_kf / (stage_ms / timed * 1e-3),
            "h2d_bytes_per_step": h2d, "created": stats.created, "fusion": fused,
            "timing": "wall clock per sequence through the reference-shaped Python API: per keyframe "
                      "MapModel.insert_keyframe (H2D) + DeviceStore.upload_keyframe + cull_recent_map_points + "
                      "create_map_points + run_fusion, each returning its result (D2H); stage_only = the "
                      "create_map_points + run_fusion calls alone (the reference's StageTimings window)"}


def golden_parity(args, seed, mapper, ids):
    """Final structural digest of the timed sequence against the REAL reference's frozen
    per-keyframe digest (tests/golden/steady_<workload>.json, make_golden_steady.py). Equality
    after the last keyframe means no decision anywhere in the sequence flipped."""
    path = os.path.join(ROOT, "tests", "golden", f"steady_{args.workload}.json")
    try:
        g = json.load(open(path))
    except (OSError, ValueError):
        return {"checked": False, "why": "no golden for this workload"}
    n_kf = len(ids)
    if g["config"].get("seed") != seed or n_kf > len(g["steps"]):
        return {"checked": False, "why": "sequence differs from the golden's (seed / length)"}
    want = g["steps"][n_kf - 1]
    mapper.ctx.call("lm_map_rewind", mapper.map)  # replay the whole sequence once more
    mapper.processed = 0
    for k in ids:
        mapper.step(k, sync=False)
    got = mapper.snapshot(with_covis=False).structural_digest()
    return {"checked": True, "keyframes": n_kf, "final_digest_equal_reference": got == want["digest"],
            "golden": os.path.relpath(path, ROOT)}


def total_kf_all(args, n_kf):
    return n_kf * args.sessions


def run_c5(args, rank, world, local, dist):
    """Batched sessions: this rank's contiguous shard of the C5 sessions advances in
    lock-step, one batched launch sequence (all its maps) per keyframe index."""
    from paper_2511_02036_b200 import _lib
    from paper_2511_02036_b200.mapmodel import KeyFrame
    from paper_2511_02036_b200.session import LocalMapper, SessionBatch, store_for
    from paper_2511_02036_b200.sharding import max_over_ranks, session_seeds

    seeds = session_seeds(5000, args.sessions, world, rank)
    seqs = load_sessions(seeds)
    n, mc, fc = stage_params("c5")
    # the rank's sessions split into groups, each a context with its own stream: one group's
    # single-CTA fusion kernels overlap the other group's wide kernels
    ngroups = max(1, min(args.c5_groups, len(seqs)))
    ctxs = [_lib.Context.get(local)] + [_lib.Context(local) for _ in range(ngroups - 1)]
    if ngroups > 1:  # concurrent groups: no programmatic dependent launch (parked successor CTAs
        for c in ctxs:  # of one group's chain would hold SMs the other groups' kernels need)
            c.call("lm_ctx_set_pdl", 0)
    ctx = ctxs[0]
    lib = ctx.lib
    mappers, kf_lists, owner, kf_objs = [], [], [], []
    for si, seq in enumerate(seqs):
        recs = seq.records if args.kfs is None else seq.records[:args.kfs]
        intr = seq.intrinsics()
        kfs = [KeyFrame(int(r.kf_id), r.pose_init, intr, r.kp_u, r.kp_v, r.kp_level, r.descriptors) for r in recs]
        g = si * ngroups // len(seqs)
        m = LocalMapper(intr, neighbor_count=n, match=mc, fuse=fc, ctx=ctxs[g],
                        store=store_for(len(kfs), max(k.num_keypoints for k in kfs) + 64))
        for kf in kfs:
            m.stage(kf)
        mappers.append(m)
        kf_lists.append([kf.kf_id for kf in kfs])
        kf_objs.append(kfs)
        owner.append(g)
    batches = [SessionBatch([m for m, o in zip(mappers, owner) if o == g]) for g in range(ngroups)]
    lists = [[ids for ids, o in zip(kf_lists, owner) if o == g] for g in range(ngroups)]
    n_kf = min(len(x) for x in kf_lists)
    dev = f"cuda:{local}" if dist is not None and dist.get_backend() == "nccl" else None

    def one_step():
        for m in mappers:
            m.ctx.call("lm_map_rewind", m.map)
            m.processed = 0
        lib.lm_flush_l2(ctx.h, L2_FLUSH_BYTES)
        for c in ctxs:
            c.call("lm_synchronize")
        if dist is not None:
            dist.barrier()
        hs = (C.c_void_p * ngroups)(*[c.h for c in ctxs])
        _lib.check(lib.lm_timer_start_multi(hs, ngroups), ctx.h)
        for k in range(n_kf):
            for b, ls in zip(batches, lists):
                b.step([ids[k] for ids in ls], sync=False)
        ms = C.c_float()
        _lib.check(lib.lm_timer_stop_multi(hs, ngroups, C.byref(ms)), ctx.h)
        return ms.value

    for _ in range(args.warmup):
        one_step()
    sampler = ClockSampler(local)
    l0 = sum(lib.lm_launch_count(c.h) for c in ctxs)
    times, tot_err = [], 0
    for _ in range(args.steps):
        times.append(max_over_ranks(one_step(), dev))
    launches = sum(lib.lm_launch_count(c.h) for c in ctxs) - l0
    clocks = sampler.stop()
    # stage profile (outside the timed steps): each group's whole sequence on its own, with
    # CUDA events between its kernels, so per-kernel intervals are not overlapped by the other
    # groups; stage times are summed over the groups, work over all sessions
    stages = ["insert", "cull", "select", "prep", "match", "tri", "commit", "fuse_targets", "fuse_geo",
              "fuse_gather", "fuse_apply", "fuse_refresh", "fuse_spec", "fuse_rev", "fuse_visible"]
    stage_ms = {s_: 0.0 for s_ in stages}
    pairs = fbytes = 0
    for c, b, ls in zip(ctxs, batches, lists):
        for m in b.mappers:
            c.call("lm_map_rewind", m.map)
            m.processed = 0
        c.call("lm_synchronize")
        lib.lm_profile_enable(c.h, 1)
        for k in range(n_kf):
            b.step([ids[k] for ids in ls], sync=False)
        prof_ms = (C.c_double * 16)()
        prof_n = (C.c_int64 * 16)()
        lib.lm_profile_read(c.h, prof_ms, prof_n)
        lib.lm_profile_enable(c.h, 0)
        for k, s_ in enumerate(stages):
            stage_ms[s_] += prof_ms[k]
        for m in b.mappers:
            t = _lib.StepStats()
            c.call("lm_totals_fetch", m.map, C.byref(t))
            tot_err |= t.error
            pairs += t.match_pairs
            fbytes += t.fuse_bytes
    if tot_err:
        raise RuntimeError(f"device error {tot_err}")
    # end to end: every keyframe of every session staged from host memory (H2D through the
    # pinned staging ring) at its keyframe index, batches stepped without waiting, every
    # session's running totals read back at the end (D2H); wall clock, max over ranks
    e2e = None
    if not args.no_e2e:
        e_ms = []
        h2d = sum(k.num_keypoints * (8 + 8 + 32 + 4 + 1) + 208 for kl in kf_objs for k in kl[:n_kf])
        for it in range(args.warmup + args.steps):
            for m in mappers:
                m.reset()
            for c in ctxs:
                c.call("lm_synchronize")
            if dist is not None:
                dist.barrier()
            t0 = time.perf_counter()
            for k in range(n_kf):
                for m, kl in zip(mappers, kf_objs):
                    m.stage(kl[k])
                for b, ls in zip(batches, lists):
                    b.step([ids[k] for ids in ls], sync=False)
            err = 0
            for m in mappers:
                err |= m.totals().error
            dt = (time.perf_counter() - t0) * 1e3
            if err:
                raise RuntimeError(f"c5 e2e: device error {err}")
            if it >= args.warmup:
                e_ms.append(max_over_ranks(dt, dev))
        e2e = {"value": total_kf_all(args, n_kf) / (sum(e_ms) / len(e_ms) * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": C.sizeof(_lib.StepStats) * len(mappers),
               "ms_per_step": sum(e_ms) / len(e_ms),
               "timing": "wall clock: every session's keyframes staged from host memory (H2D) per keyframe "
                         "index and stepped in batched launches through the C ABI; each session's running "
                         "totals read back (D2H) at the end"}
    args_steps_profiled = 1
    mean_ms = sum(times) / len(times)
    total_kf = n_kf * args.sessions
    popc_peak = C.c_double()
    ctx.call("lm_bench_popc", C.byref(popc_peak))
    match_s = stage_ms["match"] * 1e-3
    popc_achieved = 8 * (pairs / args_steps_profiled) / match_s if match_s > 0 else 0.0
    roof_popc = {"kernel": "k_match", "bound": "popc", "achieved": popc_achieved / 1e12,
                 "peak": popc_peak.value / 1e12, "unit": "Tpopc32/s", "frac": popc_achieved / popc_peak.value,
                 "algorithmic_popc_per_launch": 8 * pairs / n_kf, "launch_ms": stage_ms["match"] / n_kf,
                 "scope": "profile pass: every group's sequence on its own (16 sessions per launch at 4 groups)",
                 "peak_source": "lm_bench_popc microbenchmark on this GPU (measured)"}
    fuse_s = sum(v for k_, v in stage_ms.items() if k_.startswith("fuse")) * 1e-3
    peaks = measured_peaks()
    hbm_peak = peaks.get("hbm_gbs", 6457.4)
    fuse_gbs = fbytes / fuse_s / 1e9 if fuse_s > 0 else 0.0
    roof_fuse = {"kernel": "k_fuse_* (whole SearchAndFuse stage, all sessions)", "bound": "hbm", "achieved": fuse_gbs,
                 "peak": hbm_peak, "unit": "GB/s", "frac": fuse_gbs / hbm_peak}
    line = {"metric": METRIC, "value": total_kf / (mean_ms * 1e-3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": mean_ms,
            "ms_per_keyframe": mean_ms / n_kf, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u32 popc / f64 geometry", "data": "synthetic", "config": config_of(args),
            "parallelism": f"{args.sessions} sessions sharded contiguously over {world} GPU(s), batched launches "
                           f"in {ngroups} stream group(s) per GPU",
            "sessions_this_rank": len(seeds), "clocks": clocks, "gpu_launches": int(launches), "e2e": e2e,
            "roofline": roof_popc if stage_ms["match"] >= max(stage_ms.values()) else roof_fuse,
            "roofline_popc": roof_popc, "roofline_fusion_stage": roof_fuse,
            "stage_ms_per_step": stage_ms}
    if rank == 0:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
