"""Freeze golden outputs of the REAL reference package (importable only in the build
container, from /root/reference/pkg/src) so the oracle can be pinned on any machine.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Writes tests/golden/golden.json (+ golden_positions.npz):
  * workload digests: sha256 of every record the reference generator emits for each
    config in WORKLOADS (pins paper_2511_02036_b200/workload.py);
  * search: candidate tuples of reference search_for_triangulation(engine="reference")
    for keyframe pairs of those workloads;
  * fuse: reference fuse_pass(engine="reference") actions/visible ids on maps built by
    the reference pipeline;
  * pipeline: per keyframe, the reference LocalMappingPipeline (mode=baseline, LBA and
    keyframe culling force-skipped) creation/fusion counters and a structural digest of
    the map (bindings, live ids, found/visible, rep descriptors, observations, counters),
    plus the final live point positions.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))

WORKLOADS = {
    "orbit7": dict(seed=300, landmark_count=180, keyframe_count=7, features_per_kf=110, pixel_noise_sigma=0.7,
                   descriptor_flip_bits=2, trajectory="orbit"),
    "orbit20": dict(seed=11, landmark_count=300, keyframe_count=20, features_per_kf=220, pixel_noise_sigma=1.0,
                    descriptor_flip_bits=3, trajectory="orbit", pose_noise_trans=0.03, pose_noise_rot_deg=0.3),
    "line14dup": dict(seed=41, landmark_count=2000, keyframe_count=14, features_per_kf=400, pixel_noise_sigma=0.8,
                      descriptor_flip_bits=3, trajectory="line", extent=6.0, duplicate_injection_rate=0.05,
                      twin_flip_bits=20),
    "corridor12": dict(seed=6, landmark_count=300, keyframe_count=12, features_per_kf=150, min_covisible=5,
                       trajectory="corridor-loop", extent=10.0, spurious_feature_fraction=0.1,
                       duplicate_injection_rate=0.05, pixel_noise_sigma=0.5),
    "c1": dict(seed=101, landmark_count=6000, keyframe_count=11, features_per_kf=1000, trajectory="line",
               extent=4.0, min_covisible=50, descriptor_flip_bits=3, pixel_noise_sigma=0.8),
}
PIPELINES = {"orbit7": 10, "orbit20": 10, "line14dup": 10, "corridor12": 6, "c1": 10}


def record_digest(records) -> str:
    h = hashlib.sha256()
    for r in records:
        for a in (r.pose_init.quat, r.pose_init.trans, r.pose_gt.quat, r.pose_gt.trans, r.kp_u, r.kp_v,
                  r.kp_level, r.descriptors, r.landmark_ids):
            h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def ref_digest(m) -> str:
    h = hashlib.sha256()
    for k in sorted(kf.kf_id for kf in m.live_keyframes()):
        h.update(f"kf {k} ".encode())
        h.update(m.keyframes[k].mp_bindings.astype(np.int64).tobytes())
    for p in sorted(m.live_points(), key=lambda p: p.mp_id):
        h.update(f"mp {p.mp_id} {p.found_count} {p.visible_count} ".encode())
        h.update(p.rep_descriptor.tobytes())
        h.update(str(sorted(p.observations.items())).encode())
        # the live counter row (mp.scale_counts views go stale when the matrix grows)
        h.update(m.counter_matrix[p.mp_id].astype(np.int64).tobytes())
    return h.hexdigest()


def main():
    sys.path.insert(0, REF)
    from localmap import synth
    from localmap.config import MatchConfig, PipelineConfig
    from localmap.fusion import fuse_pass
    from localmap.pipeline import LocalMappingPipeline
    from localmap.triangulation import search_for_triangulation

    out = {"workloads": {}, "search": {}, "fuse": {}, "pipeline": {}}
    positions = {}
    for name, kw in WORKLOADS.items():
        seq = synth.generate_sequence(synth.WorldConfig(**kw))
        out["workloads"][name] = {"config": kw, "digest": record_digest(seq.records), "n": len(seq.records)}
        kfs = seq.to_keyframes()
        pairs = [(1, 0), (3, 1), (len(kfs) - 1, len(kfs) - 3)]
        out["search"][name] = {
            f"{a},{b}": [[c.kp_index_current, c.kp_index_neighbor, c.distance]
                         for c in search_for_triangulation(kfs[a], kfs[b], engine="reference")]
            for a, b in pairs}
        n_nbr = PIPELINES[name]
        pc = PipelineConfig(mode="baseline", force_skip_lba=True, force_skip_culling=True,
                            match=MatchConfig(neighbor_count=n_nbr))
        steps = []
        with LocalMappingPipeline(pc, num_levels=seq.intrinsics().num_levels) as pipe:
            for kf in seq.to_keyframes():
                pipe.admit(kf)
                while pipe.queue:
                    pipe.process_one()
                cs = pipe.creation_stats
                steps.append({"kf": kf.kf_id, "created": cs.created, "conflicts": cs.conflicts,
                              "degenerate": cs.degenerate, "gates": dict(cs.gate_failures),
                              "fusion": dict(pipe.fusion_totals), "culled": len(pipe.culled_points),
                              "digest": ref_digest(pipe.model)})
                if kf.kf_id == len(kfs) // 2:  # a fuse_pass snapshot mid-sequence
                    m = pipe.model
                    cur = kf.kf_id
                    fw = m.bound_points_of(cur)
                    tgts = m.covisible_neighbors(cur, 3)
                    out["fuse"][name] = {
                        "after_kf": cur,
                        "passes": [{"points": "bound_of_current", "target": t,
                                    "actions": [[a.target_kf_id, a.mp_id_projected, a.kp_index_hit,
                                                 a.existing_mp_id, a.kind] for a in fuse_pass(m, fw, t)[0]],
                                    "visible": fuse_pass(m, fw, t)[1]} for t in tgts]}
            live = sorted(p.mp_id for p in pipe.model.live_points())
            positions[f"{name}_ids"] = np.array(live, np.int64)
            positions[f"{name}_pos"] = np.stack([pipe.model.points[i].position for i in live]) if live else np.zeros((0, 3))
        out["pipeline"][name] = {"neighbor_count": n_nbr, "steps": steps}
        print(name, "done", steps[-1]["created"], steps[-1]["fusion"], flush=True)
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
    np.savez_compressed(os.path.join(HERE, "golden_positions.npz"), **positions)


if __name__ == "__main__":
    main()
