"""The reference's own pipeline driving this package (SURVEY.md §8(b) drop-in): the stock
``localmap.pipeline.LocalMappingPipeline`` (from baseline/_ref, or /root/reference in the
build container) with ``MapModel``, ``DeviceStore``, ``create_map_points``, ``run_fusion``
and ``cull_recent_map_points`` rebound to this package (pipeline.py:20-28 binds them at
import), must reproduce the reference's frozen per-keyframe outputs:
running counters and the reference's own structural digest (``make_golden.ref_digest``,
computed through the MapModel API: live_keyframes, keyframes[k].mp_bindings, live_points,
counter_matrix) after every keyframe, and the ledger (TransferLedger.as_dict) where frozen.

Also: per-step parity from an imported reference state (lm_import_snapshot), and the
LBA write-back calls (lm_kf_set_pose / lm_mp_patch_positions) against the reference's
geometry after the same write-back.
"""

from __future__ import annotations

import contextlib
import json
import os
import sys

import numpy as np
import pytest

from helpers import device_kf

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, os.path.join(HERE, "golden"))
from make_golden import ref_digest  # noqa: E402

GOLD = json.load(open(os.path.join(HERE, "golden", "golden.json")))


def reference():
    for p in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isfile(os.path.join(p, "localmap", "pipeline.py")):
            if p not in sys.path:
                sys.path.insert(0, p)
            import localmap.pipeline  # noqa: F401

            return localmap
    pytest.skip("reference package not installed (baseline/_ref)")


@contextlib.contextmanager
def device_bound(store_cfg, own_cull=True):
    """Rebind the reference pipeline's collaborators to this package (what a maintainer's
    integration does)."""
    lm = reference()
    import localmap.pipeline as P

    from paper_2511_02036_b200 import culling, fusion, triangulation
    from paper_2511_02036_b200.mapmodel import DeviceStore, MapModel

    saved = {k: getattr(P, k) for k in ("MapModel", "DeviceStore", "create_map_points", "run_fusion",
                                        "cull_recent_map_points", "cull_keyframes")}
    P.MapModel = lambda num_levels=8, config=None: MapModel(num_levels, config, store=store_cfg)
    P.DeviceStore = DeviceStore
    P.create_map_points = triangulation.create_map_points
    P.run_fusion = fusion.run_fusion
    if own_cull:
        P.cull_recent_map_points = culling.cull_recent_map_points
    P.cull_keyframes = culling.cull_keyframes
    try:
        yield lm
    finally:
        for k, v in saved.items():
            setattr(P, k, v)


def run_reference_pipeline(lm, cfg_kw, n_nbr, n1, n_kf, check, kf_cull=False, lba=False):
    from localmap import synth
    from localmap.config import FuseConfig, MatchConfig, PipelineConfig
    from localmap.pipeline import LocalMappingPipeline

    seq = synth.generate_sequence(synth.WorldConfig(**cfg_kw))
    pc = PipelineConfig(mode="optimized", worker_count=2, force_skip_lba=not lba, force_skip_culling=not kf_cull,
                        match=MatchConfig(neighbor_count=n_nbr), fuse=FuseConfig(n1=n1))
    with LocalMappingPipeline(pc, num_levels=seq.intrinsics().num_levels) as pipe:
        for k, kf in enumerate(seq.to_keyframes()[:n_kf]):
            pipe.admit(kf)
            while pipe.queue:
                pipe.process_one()
            check(k, pipe)
    return pipe


def counters(pipe):
    cs = pipe.creation_stats
    return {"created": cs.created, "conflicts": cs.conflicts, "degenerate": cs.degenerate,
            "gates": dict(cs.gate_failures), "fusion": dict(pipe.fusion_totals), "culled": len(pipe.culled_points)}


@pytest.mark.parametrize("name,own_cull", [("orbit7", False), ("line14dup", True), ("corridor12", True),
                                           ("c1", True), ("orbit20", False)])
def test_reference_pipeline_on_device_matches_golden(name, own_cull):
    from paper_2511_02036_b200.session import store_for

    g = GOLD["pipeline"][name]
    cfg_kw = GOLD["workloads"][name]["config"]
    steps = g["steps"]

    def check(k, pipe):
        want = steps[k]
        got = counters(pipe)
        for key in ("created", "conflicts", "degenerate", "gates", "fusion", "culled"):
            assert got[key] == want[key], (name, k, key)
        assert ref_digest(pipe.model) == want["digest"], (name, k)
        assert pipe.model.audit() == [], (name, k)

    with device_bound(store_for(len(steps), cfg_kw["features_per_kf"] * 2), own_cull) as lm:
        run_reference_pipeline(lm, cfg_kw, g["neighbor_count"], 20, len(steps), check)


def test_reference_pipeline_on_device_c5_session_with_ledger():
    """60 keyframes of a C5 session (EuRoC shape, 20 neighbours) through the reference's
    pipeline, digest + ledger after every keyframe."""
    from paper_2511_02036_b200.session import store_for

    path = os.path.join(HERE, "golden", "steady_c5_5000.json")
    if not os.path.isfile(path):
        pytest.skip("no steady golden")
    g = json.load(open(path))
    n = 30

    def check(k, pipe):
        want = g["steps"][k]
        got = counters(pipe)
        for key in ("created", "conflicts", "degenerate", "gates", "fusion", "culled"):
            assert got[key] == want[key], (k, key)
        assert ref_digest(pipe.model) == want["digest"], k
        assert pipe.store.ledger.as_dict() == want["ledger"], (k, pipe.store.ledger.as_dict(), want["ledger"])

    with device_bound(store_for(g["keyframes"], g["config"]["features_per_kf"] + 64)) as lm:
        run_reference_pipeline(lm, g["config"], g["neighbor_count"], g["n1"], n, check)


def test_import_reference_state_then_native_steps_match_golden():
    """Per-step parity from a reference state: import the reference's map after 7 keyframes
    of line14dup (tests/golden/snap_line14dup_kf7.npz), step the rest natively, compare with
    the reference's frozen per-keyframe digests."""
    from paper_2511_02036_b200 import workload as W
    from paper_2511_02036_b200.session import LocalMapper, store_for

    name, k0 = "line14dup", 7
    snap = dict(np.load(os.path.join(HERE, "golden", f"snap_{name}_kf{k0}.npz")))
    g = GOLD["pipeline"][name]
    seq = W.generate_sequence(W.WorldConfig(**GOLD["workloads"][name]["config"]))
    intr = seq.intrinsics()
    recs = seq.records
    # keypoints from the generator (pinned by its digest), map state from the snapshot
    snap["cam"] = np.array([[intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height]] * k0)
    snap["u"] = np.concatenate([r.kp_u for r in recs[:k0]])
    snap["v"] = np.concatenate([r.kp_v for r in recs[:k0]])
    snap["level"] = np.concatenate([r.kp_level for r in recs[:k0]])
    snap["desc"] = np.concatenate([r.descriptors for r in recs[:k0]])
    snap["rep"] = np.zeros((len(snap["pos"]), 32), np.uint8)  # recomputed by the import
    dev = LocalMapper(intr, neighbor_count=g["neighbor_count"], store=store_for(len(recs), 800))
    dev.import_state(snap, processed=int(snap["processed"]))
    assert dev.snapshot(with_covis=False).structural_digest() == g["steps"][k0 - 1]["digest"]
    base = g["steps"][k0 - 1]
    for k in range(k0, len(recs)):
        r = dev.process(device_kf(recs[k], intr))
        want = g["steps"][k]
        assert dev.snapshot(with_covis=False).structural_digest() == want["digest"], k
        assert dev.stats.created == want["created"] - base["created"], k
        del r


def test_lba_write_back_pose_and_positions():
    """lm_kf_set_pose / lm_mp_patch_positions: after an LBA-style write-back the device's
    fusion geometry equals a fresh map built from the written-back state (the cached view
    geometry and hits are invalidated, not reused)."""
    from paper_2511_02036_b200 import workload as W
    from paper_2511_02036_b200.geometry import SE3Pose
    from paper_2511_02036_b200.mapmodel import MapModel
    from paper_2511_02036_b200.session import store_for

    seq = W.generate_sequence(W.WorldConfig(**GOLD["workloads"]["line14dup"]["config"]))
    intr = seq.intrinsics()
    kfs = [device_kf(r, intr) for r in seq.records[:8]]
    from paper_2511_02036_b200.fusion import fuse_pass, run_fusion
    from paper_2511_02036_b200.mapmodel import DeviceStore
    from paper_2511_02036_b200.triangulation import create_map_points

    def build(kfs, patch):
        m = MapModel(intr.num_levels, store=store_for(16, 800))
        st = DeviceStore()
        for kf in kfs[:-1]:
            m.insert_keyframe(kf)
            st.upload_keyframe(kf)
            create_map_points(m, st, kf.kf_id, 5)
            run_fusion(m, st, kf.kf_id)
        patch(m)
        m.insert_keyframe(kfs[-1])
        st.upload_keyframe(kfs[-1])
        return m

    rng = np.random.default_rng(7)

    def patch(m):
        ids = [p.mp_id for p in m.live_points()]
        pos = np.array([m.points[i].position for i in ids]) + rng.normal(0, 0.01, (len(ids), 3))
        m.patch_positions(ids, pos)
        kf = m.keyframes[3]
        m.set_pose(3, SE3Pose(kf.pose.quat, kf.pose.trans + np.array([0.01, -0.02, 0.005])))
        return ids, pos

    m1 = build([device_kf(r, intr) for r in seq.records[:8]], patch)
    a1 = fuse_pass(m1, [p.mp_id for p in m1.live_points()], 3)
    # the same map, rebuilt from the written-back state through the import path
    from paper_2511_02036_b200.snapshot import import_reference

    m2 = MapModel(intr.num_levels, store=store_for(16, 800))
    import_reference(m2, m1, None, None, keyframes=list(m1.keyframes.values()))
    a2 = fuse_pass(m2, [p.mp_id for p in m2.live_points()], 3)
    assert a1 == a2


KFCULL = os.path.join(HERE, "golden", "kfcull.json")


@pytest.mark.parametrize("name", sorted(json.load(open(KFCULL))) if os.path.isfile(KFCULL) else [])
def test_reference_pipeline_with_keyframe_culling_on_device(name):
    """§8(f) row 4 end to end: the reference pipeline with keyframe culling enabled
    (pipeline.py:210-223) and cull_keyframes bound to the device fast path must cull the same
    keyframes and leave the same map (digest, ledger incl. evictions) after every keyframe as
    the reference's own run (tests/golden/kfcull.json, make_golden_kfcull.py). The "default_*"
    cases are the reference's DEFAULT pipeline: its own LBA (out of scope, run on the host)
    reads the device map through the MapModel API and writes poses and positions back
    (localba.py:571-574), which the device takes over (lm_kf_set_pose,
    lm_mp_patch_positions) before the next stage."""
    from paper_2511_02036_b200.session import store_for

    g = json.load(open(KFCULL))[name]

    def check(k, pipe):
        want = g["steps"][k]
        assert list(pipe.culled_keyframes) == want["culled_keyframes"], (name, k)
        got = counters(pipe)
        for key in ("created", "conflicts", "gates", "fusion", "culled"):
            assert got[key] == want[key], (name, k, key)
        assert ref_digest(pipe.model) == want["digest"], (name, k)
        assert pipe.store.ledger.as_dict() == want["ledger"], (name, k)

    with device_bound(store_for(g["keyframes"], g["config"]["features_per_kf"] + 64)) as lm:
        run_reference_pipeline(lm, g["config"], g["neighbor_count"], g["n1"], g["keyframes"], check, kf_cull=True,
                               lba=g.get("lba", False))
