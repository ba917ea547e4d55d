"""Freeze the REAL reference pipeline WITH keyframe culling (culling.py:127-154, pipeline.py:
210-223; LBA still force-skipped) so the device keyframe-cull fast path (§8(f) row 4) is
pinned on whole sequences: per keyframe the culled keyframe list, counters, structural digest
(make_golden.ref_digest) and ledger (evictions included).

    OPENBLAS_NUM_THREADS=1 PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_kfcull.py

Writes tests/golden/kfcull.json. mode="baseline" (observation-walk redundancy); the
reference guarantees the "fast" counter path gives identical maps.
"""

from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

from make_golden import REF, WORKLOADS, ref_digest  # noqa: E402

from paper_2511_02036_b200.workload import BENCH_CONFIGS  # noqa: E402

# name -> (config, neighbours, n1, keyframes, LBA on); "default_*" runs are the reference's
# default pipeline (LBA + keyframe culling), whose LBA writes poses and positions back
RUNS = {
    "default_line14dup": (WORKLOADS["line14dup"], 10, 20, 14, True),
    "default_orbit20": (WORKLOADS["orbit20"], 10, 20, 20, True),
    "line14dup": (WORKLOADS["line14dup"], 10, 20, 14, False),
    "orbit20": (WORKLOADS["orbit20"], 10, 20, 20, False),
    "corridor12": (WORKLOADS["corridor12"], 6, 20, 12, False),
    "c2_60": (BENCH_CONFIGS["c2"], 20, 20, 60, False),
}


def main():
    sys.path.insert(0, REF)
    from localmap import synth
    from localmap.config import FuseConfig, MatchConfig, PipelineConfig
    from localmap.pipeline import LocalMappingPipeline

    names = sys.argv[1:] or list(RUNS)
    out = {}
    path = os.path.join(HERE, "kfcull.json")
    if sys.argv[1:] and os.path.isfile(path):
        out = json.load(open(path))
    for name in names:
        kw, n_nbr, n1, n_kf, lba = RUNS[name]
        seq = synth.generate_sequence(synth.WorldConfig(**kw))
        pc = PipelineConfig(mode="baseline", force_skip_lba=not lba, force_skip_culling=False,
                            match=MatchConfig(neighbor_count=n_nbr), fuse=FuseConfig(n1=n1))
        steps = []
        with LocalMappingPipeline(pc, num_levels=seq.intrinsics().num_levels) as pipe:
            for kf in seq.to_keyframes()[:n_kf]:
                pipe.admit(kf)
                while pipe.queue:
                    pipe.process_one()
                cs = pipe.creation_stats
                steps.append({"kf": kf.kf_id, "created": cs.created, "conflicts": cs.conflicts,
                              "gates": dict(cs.gate_failures), "fusion": dict(pipe.fusion_totals),
                              "culled": len(pipe.culled_points), "culled_keyframes": list(pipe.culled_keyframes),
                              "digest": ref_digest(pipe.model), "ledger": pipe.store.ledger.as_dict()})
        out[name] = {"config": kw, "neighbor_count": n_nbr, "n1": n1, "keyframes": n_kf, "lba": lba, "steps": steps}
        print(name, "culled keyframes", steps[-1]["culled_keyframes"], flush=True)
    with open(path, "w") as fh:
        json.dump(out, fh, indent=0, sort_keys=True)


if __name__ == "__main__":
    main()
