"""Pins the CPU oracle (oracle/lm_oracle.py) and the workload generator against golden
outputs of the real reference package (tests/golden/make_golden.py). CPU only."""

from __future__ import annotations

import json
import os

import numpy as np
import pytest

from helpers import cam_of
from oracle import lm_oracle as O
from paper_2511_02036_b200 import workload as W

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "golden.json")))
POS = np.load(os.path.join(HERE, "golden", "golden_positions.npz"))


def record_digest(records) -> str:
    import hashlib

    h = hashlib.sha256()
    for r in records:
        for a in (r.pose_init.quat, r.pose_init.trans, r.pose_gt.quat, r.pose_gt.trans, r.kp_u, r.kp_v,
                  r.kp_level, r.descriptors, r.landmark_ids):
            h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


_SEQ = {}


def seq(name):
    if name not in _SEQ:
        _SEQ[name] = W.generate_sequence(W.WorldConfig(**GOLD["workloads"][name]["config"]))
    return _SEQ[name]


@pytest.mark.parametrize("name", sorted(GOLD["workloads"]))
def test_workload_generator_matches_reference(name):
    assert record_digest(seq(name).records) == GOLD["workloads"][name]["digest"]


@pytest.mark.parametrize("name", sorted(GOLD["search"]))
def test_oracle_search_matches_reference(name):
    s = seq(name)
    cam = cam_of(s)
    for key, want in GOLD["search"][name].items():
        a, b = map(int, key.split(","))
        oa, ob = O.okf_from_record(s.records[a], cam), O.okf_from_record(s.records[b], cam)
        f = O.fundamental(oa.quat, oa.trans, oa.cam, ob.quat, ob.trans, ob.cam)
        got = [] if f is None else O.search_pairs(oa, ob, f, 3.84, 50, 1, np.ones(oa.n, bool), np.ones(ob.n, bool))
        assert [list(t) for t in got] == want, key


@pytest.mark.parametrize("name", sorted(GOLD["pipeline"]))
def test_oracle_pipeline_matches_reference(name):
    s = seq(name)
    cam = cam_of(s)
    g = GOLD["pipeline"][name]
    pipe = O.OraclePipeline(cam.num_levels, g["neighbor_count"])
    fuse_gold = GOLD["fuse"].get(name)
    for rec, want in zip(s.records, g["steps"]):
        pipe.step(O.okf_from_record(rec, cam))
        st = pipe.stats
        assert (st.created, st.conflicts, st.degenerate) == (want["created"], want["conflicts"], want["degenerate"])
        assert st.gate_failures == want["gates"]
        assert pipe.fused == want["fusion"]
        assert len(pipe.culled) == want["culled"]
        assert O.structural_digest(pipe.map) == want["digest"], rec.kf_id
        if fuse_gold and rec.kf_id == fuse_gold["after_kf"]:
            fw = pipe.map.bound_points(rec.kf_id)
            for ps in fuse_gold["passes"]:
                acts, vis = O.fuse_gather(pipe.map, fw, ps["target"])
                assert [list(a) for a in acts] == ps["actions"]
                assert vis == ps["visible"]
    ids = sorted(p.mp_id for p in pipe.map.live_points())
    assert ids == POS[f"{name}_ids"].tolist()
    got = np.stack([pipe.map.pts[i].pos for i in ids]) if ids else np.zeros((0, 3))
    assert np.array_equal(got, POS[f"{name}_pos"])  # the oracle uses the same LAPACK: bitwise


def test_oracle_audit_clean_after_pipeline():
    s = seq("orbit7")
    cam = cam_of(s)
    pipe = O.OraclePipeline(cam.num_levels, 10)
    for rec in s.records:
        pipe.step(O.okf_from_record(rec, cam))
    assert pipe.map.audit() == []


KFCULL = json.load(open(os.path.join(HERE, "golden", "kfcull.json")))


@pytest.mark.parametrize("name", ["line14dup", "orbit20", "corridor12"])
def test_oracle_keyframe_cull_matches_reference_pipeline(name):
    """Pins the oracle's keyframe cull (kill_keyframe + is_redundant_baseline + cull_keyframes,
    culling.py:60-154, mapmodel.py:275-283) to the real reference pipeline with keyframe culling
    (tests/golden/kfcull.json): culled keyframes and structural digest after every keyframe."""
    g = KFCULL[name]
    s = W.generate_sequence(W.WorldConfig(**g["config"]))
    cam = cam_of(s)
    pipe = O.OraclePipeline(s.config.num_levels, g["neighbor_count"], fc=O.FuseCfg(n1=g["n1"]))
    culled = []
    for rec, want in zip(s.records[:g["keyframes"]], g["steps"]):
        kf = O.okf_from_record(rec, cam)
        pipe.step(kf)
        cand = [k for k in pipe.map.neighbors(kf.kf_id) if k != kf.kf_id]
        culled += O.cull_keyframes(pipe.map, cand)
        assert culled == want["culled_keyframes"], (name, rec.kf_id)
        assert O.structural_digest(pipe.map) == want["digest"], (name, rec.kf_id)
