"""Freeze the REAL reference's per-keyframe outputs on the headline configs at their
BASELINE neighbour counts (steady state, not a short prefix), so the GPU path can be
gated on every keyframe of C2 and on long windows of C3 / C4 / C5.

    OPENBLAS_NUM_THREADS=1 PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden_steady.py c2            # 200 KFs, ~25 min
    ... c3 (KFs 0-59), c4 (KFs 0-9), c5_5000 .. c5_5003 (60 KFs each)

Writes tests/golden/steady_<name>.json (+ steady_<name>_positions.npz). Per keyframe:
running creation / gate / fusion / cull counters (as the reference pipeline keeps them,
`pipeline.py:175-195`), the structural map digest (`make_golden.ref_digest`: bindings,
live ids, found/visible, representative descriptors, observation lists, live counter
rows), the `TransferLedger.as_dict()` (`devicestore.py:32-48`) and the reference's own
stage timings (`StageTimings.triangulation_ms + fusion_ms`). Metadata records the NumPy
and OpenBLAS build (core type) that produced the file: the reference's F and P matrices
come out of OpenBLAS dgemm, whose accumulation order is core-specific.

With --pickle-at K (C2 uses 100) the reference pipeline state after K keyframes
(model, store, probation list, counters) is pickled to baseline/_state/<name>_kf<K>.pkl
(git-ignored; it travels to the GPU box with the snapshot) so bench.py's reference arm can
time a steady-state window without replaying K keyframes first.

The pipeline runs mode="baseline" (engine="reference", the oracle engine) with LBA and
keyframe culling force-skipped, like the device session (`config.py:113-114`).
"""

from __future__ import annotations

import argparse
import json
import os
import pickle
import platform
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

from make_golden import REF, record_digest, ref_digest  # noqa: E402

from paper_2511_02036_b200.workload import BENCH_CONFIGS, BENCH_STAGE  # noqa: E402

# name -> (bench config, seed override, keyframes processed)
STEADY = {
    "c2": ("c2", None, 200),
    "c3": ("c3", None, 60),
    "c4": ("c4", None, 10),
    "c5_5000": ("c2", 5000, 60),
    "c5_5001": ("c2", 5001, 60),
    "c5_5002": ("c2", 5002, 60),
    "c5_5003": ("c2", 5003, 60),
}


def blas_info() -> dict:
    try:
        import threadpoolctl

        info = [{k: d.get(k) for k in ("internal_api", "version", "architecture", "threading_layer")}
                for d in threadpoolctl.threadpool_info() if d.get("user_api") == "blas"]
    except Exception as e:  # pragma: no cover
        info = [{"error": repr(e)}]
    return {"numpy": np.__version__, "blas": info, "machine": platform.machine(),
            "cpu": _cpu_model(), "python": platform.python_version()}


def _cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def pipeline_state(pipe) -> dict:
    """What a pipeline needs to resume: the map, the store, the probation list and the
    running counters (`pipeline.py:92-107`). The pool is recreated by the loader."""
    return {"model": pipe.model, "store": pipe.store, "recent": pipe._recent,
            "processed": pipe._processed, "creation_stats": pipe.creation_stats,
            "fusion_totals": pipe.fusion_totals, "culled_points": pipe.culled_points}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("name", choices=sorted(STEADY))
    ap.add_argument("--pickle-at", type=int, default=None)
    ap.add_argument("--kfs", type=int, default=None, help="override the keyframe count")
    args = ap.parse_args()
    sys.path.insert(0, REF)
    from localmap import synth
    from localmap.config import FuseConfig, MatchConfig, PipelineConfig
    from localmap.pipeline import LocalMappingPipeline

    base, seed, n_kf = STEADY[args.name]
    n_kf = args.kfs or n_kf
    kw = dict(BENCH_CONFIGS[base])
    if seed is not None:
        kw["seed"] = seed
    n_nbr, n1, n2 = BENCH_STAGE[base]
    seq = synth.generate_sequence(synth.WorldConfig(**kw))
    pc = PipelineConfig(mode="baseline", force_skip_lba=True, force_skip_culling=True,
                        match=MatchConfig(neighbor_count=n_nbr), fuse=FuseConfig(n1=n1, n2=n2))
    steps = []
    t_start = time.time()
    with LocalMappingPipeline(pc, num_levels=seq.intrinsics().num_levels) as pipe:
        for kf in seq.to_keyframes()[:n_kf]:
            pipe.admit(kf)
            while pipe.queue:
                t = pipe.process_one()
            cs = pipe.creation_stats
            steps.append({"kf": kf.kf_id, "created": cs.created, "conflicts": cs.conflicts,
                          "degenerate": cs.degenerate, "gates": dict(cs.gate_failures),
                          "fusion": dict(pipe.fusion_totals), "culled": len(pipe.culled_points),
                          "digest": ref_digest(pipe.model), "ledger": pipe.store.ledger.as_dict(),
                          "tri_ms": round(t.triangulation_ms, 3), "fusion_ms": round(t.fusion_ms, 3),
                          "live_points": t.n_points})
            print(args.name, kf.kf_id, f"{t.triangulation_ms + t.fusion_ms:.0f} ms", t.n_points, flush=True)
            if args.pickle_at is not None and kf.kf_id + 1 == args.pickle_at:
                d = os.path.join(ROOT, "baseline", "_state")
                os.makedirs(d, exist_ok=True)
                with open(os.path.join(d, f"{args.name}_kf{args.pickle_at}.pkl"), "wb") as fh:
                    pickle.dump({"state": pipeline_state(pipe), "digest": steps[-1]["digest"],
                                 "config": kw, "stage": [n_nbr, n1, n2]}, fh, protocol=pickle.HIGHEST_PROTOCOL)
        live = sorted(p.mp_id for p in pipe.model.live_points())
        pos = np.stack([pipe.model.points[i].position for i in live]) if live else np.zeros((0, 3))
    out = {"name": args.name, "config": kw, "neighbor_count": n_nbr, "n1": n1, "n2": n2,
           "keyframes": n_kf, "record_digest": record_digest(seq.records[:n_kf]),
           "meta": {**blas_info(), "seconds": round(time.time() - t_start, 1), "mode": "baseline"},
           "steps": steps}
    with open(os.path.join(HERE, f"steady_{args.name}.json"), "w") as fh:
        json.dump(out, fh, indent=0, sort_keys=True)
    np.savez_compressed(os.path.join(HERE, f"steady_{args.name}_positions.npz"),
                        ids=np.array(live, np.int64), pos=pos)


if __name__ == "__main__":
    main()
