"""Where the reference-shaped Python API spends its time per keyframe (GPU box).

    python tools/api_profile.py [--workload c2]

Runs bench.py's API e2e loop (MapModel.insert_keyframe + DeviceStore.upload_keyframe +
cull_recent_map_points + create_map_points + run_fusion) once to warm up, then once timing
each call kind with perf_counter, then once under cProfile (top functions by own time)."""

from __future__ import annotations

import argparse
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2")
    args = ap.parse_args()
    import bench
    from paper_2511_02036_b200.config import CullConfig, GateConfig
    from paper_2511_02036_b200.culling import RecentPoint, cull_recent_map_points
    from paper_2511_02036_b200.fusion import run_fusion
    from paper_2511_02036_b200.mapmodel import DeviceStore, KeyFrame, MapModel
    from paper_2511_02036_b200.session import store_for
    from paper_2511_02036_b200.triangulation import CreationStats, create_map_points

    seq = bench.load_workload(args.workload, bench.W.BENCH_CONFIGS[args.workload]["seed"])
    intr = seq.intrinsics()
    kfs = [KeyFrame(int(r.kf_id), r.pose_init, intr, r.kp_u, r.kp_v, r.kp_level, r.descriptors) for r in seq.records]
    n, mc, fc = bench.stage_params(args.workload)
    model = MapModel(intr.num_levels, scale_factor=intr.scale_factor,
                     store=store_for(len(kfs), max(k.num_keypoints for k in kfs) + 64))
    gc, cc = GateConfig(), CullConfig()
    acc = {}

    def timed(name, f, *a, **k):
        t = time.perf_counter()
        r = f(*a, **k)
        acc[name] = acc.get(name, 0.0) + time.perf_counter() - t
        return r

    def run(timing):
        model.reset()
        store = DeviceStore(model=model)
        stats = CreationStats()
        recent = []
        call = timed if timing else (lambda name, f, *a, **k: f(*a, **k))
        t0 = time.perf_counter()
        for processed, kf in enumerate(kfs):
            kf.mp_bindings[:] = -1
            call("insert_keyframe", model.insert_keyframe, kf)
            call("upload_keyframe", store.upload_keyframe, kf)
            _, recent = call("cull_recent_map_points", cull_recent_map_points, model, recent, processed, cc)
            made = call("create_map_points", create_map_points, model, store, kf.kf_id, n, mc, gc, stats=stats)
            t = time.perf_counter()
            recent.extend(RecentPoint(i, processed) for i in made)
            acc["caller: recent.extend"] = acc.get("caller: recent.extend", 0.0) + time.perf_counter() - t
            call("run_fusion", run_fusion, model, store, kf.kf_id, fc)
        return (time.perf_counter() - t0) * 1e3

    run(False)
    acc.clear()
    ms = run(True)
    print(f"sequence {ms:.1f} ms ({len(kfs) / ms * 1e3:.0f} KF/s), per keyframe:")
    for k, v in sorted(acc.items(), key=lambda kv: -kv[1]):
        print(f"  {k:28s} {v / len(kfs) * 1e6:8.1f} us")
    pr = cProfile.Profile()
    pr.enable()
    run(False)
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)


if __name__ == "__main__":
    main()
