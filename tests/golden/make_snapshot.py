"""Freeze REAL-reference map states mid-sequence, for per-step parity from a reference
state (SURVEY.md §5 checkpoint row / §8(c) comparator caveat): the device imports the
reference's own map after K keyframes (lm_import_snapshot) and must then reproduce the
reference's next keyframes bit for bit, so no earlier low-bit position drift can cascade.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_snapshot.py

Writes tests/golden/snap_<name>_kf<K>.npz = paper_2511_02036_b200.snapshot.state_arrays(...,
keypoints=False) of the reference LocalMappingPipeline (mode="baseline", LBA + keyframe
culling force-skipped) after K keyframes, plus `processed` and the running counters. The
keypoints/descriptors are not stored (the workload generator reproduces them, pinned by
its digest) and neither are representative descriptors (the import recomputes them: a pure
function of the observation lists). C2 at K=100 is taken from the pickled state that
make_golden_steady.py --pickle-at 100 wrote (baseline/_state/c2_kf100.pkl) when present.
"""

from __future__ import annotations

import os
import pickle
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

from make_golden import REF, WORKLOADS  # noqa: E402

from paper_2511_02036_b200.snapshot import state_arrays  # noqa: E402
from paper_2511_02036_b200.workload import BENCH_CONFIGS, BENCH_STAGE  # noqa: E402

# name -> (config, neighbour count, n1, K)
SNAPS = {
    "line14dup": (WORKLOADS["line14dup"], 10, 20, 7),
    "c2": (BENCH_CONFIGS["c2"], *BENCH_STAGE["c2"][:2], 100),
}


def counters(pipe) -> dict:
    cs = pipe.creation_stats
    return {"created": cs.created, "conflicts": cs.conflicts, "degenerate": cs.degenerate,
            "gates": dict(cs.gate_failures), "fusion": dict(pipe.fusion_totals), "culled": len(pipe.culled_points)}


def save(name, k, model, store, recent, processed, ctr):
    a = state_arrays(model, store, recent, keypoints=False)
    del a["rep"]
    a["processed"] = np.array(processed, np.int64)
    a["counters"] = np.frombuffer(repr(ctr).encode(), np.uint8)
    path = os.path.join(HERE, f"snap_{name}_kf{k}.npz")
    np.savez_compressed(path, **a)
    print(path, os.path.getsize(path), "bytes", len(a["pos"]), "points")


def main():
    sys.path.insert(0, REF)
    from localmap import synth
    from localmap.config import FuseConfig, MatchConfig, PipelineConfig
    from localmap.pipeline import LocalMappingPipeline

    names = sys.argv[1:] or list(SNAPS)
    for name in names:
        kw, n_nbr, n1, k = SNAPS[name]
        pk = os.path.join(ROOT, "baseline", "_state", f"{name}_kf{k}.pkl")
        if os.path.isfile(pk):
            st = pickle.load(open(pk, "rb"))["state"]
            ctr = {"created": st["creation_stats"].created, "conflicts": st["creation_stats"].conflicts,
                   "degenerate": st["creation_stats"].degenerate, "gates": dict(st["creation_stats"].gate_failures),
                   "fusion": dict(st["fusion_totals"]), "culled": len(st["culled_points"])}
            save(name, k, st["model"], st["store"], st["recent"], st["processed"], ctr)
            continue
        seq = synth.generate_sequence(synth.WorldConfig(**kw))
        pc = PipelineConfig(mode="baseline", force_skip_lba=True, force_skip_culling=True,
                            match=MatchConfig(neighbor_count=n_nbr), fuse=FuseConfig(n1=n1))
        with LocalMappingPipeline(pc, num_levels=seq.intrinsics().num_levels) as pipe:
            for kf in seq.to_keyframes()[:k]:
                pipe.admit(kf)
                while pipe.queue:
                    pipe.process_one()
            save(name, k, pipe.model, pipe.store, pipe._recent, pipe._processed, counters(pipe))


if __name__ == "__main__":
    main()
