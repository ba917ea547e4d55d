"""Device map bookkeeping against the oracle, op for op.

A restatement of the reference's long random-operation test (pkg/tests/test_mapmodel.py:
257-298), widened to every bookkeeping op the device exposes: insert_keyframe with pre-bound
slots, new_map_point + add_observation, erase_observation (with the min_obs_keep kill),
kill_map_point, replace_map_point and kill_keyframe. The same seeded op stream drives the
device MapModel and the oracle's OracleMap (oracle/lm_oracle.py, the reference's
mapmodel.py:113-353 restated); the op choices are drawn from the oracle's state, so the
device is read only at checkpoints: structural digest (bindings, live ids, representative
descriptors, observations, counters) and covisibility neighbour lists every 500 ops, and
the device audit (lm_audit) clean at the end. Plus the reference's audit fault-injection
tests (test_mapmodel.py:238-255) on the device audit.
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import lm_oracle as O
from paper_2511_02036_b200.geometry import CameraIntrinsics, SE3Pose
from paper_2511_02036_b200.mapmodel import UNBOUND, KeyFrame, MapModel
from paper_2511_02036_b200.session import store_for

pytestmark = pytest.mark.gpu

CAM = CameraIntrinsics(fx=460.0, fy=460.0, cx=320.0, cy=240.0, width=640, height=480)


def make_pair(rng, kf_id, n, bind=None):
    u = rng.uniform(0, 640, n)
    v = rng.uniform(0, 480, n)
    lev = rng.integers(0, CAM.num_levels, n)
    desc = rng.integers(0, 256, (n, 32), dtype=np.uint8)
    pose = SE3Pose(np.array([0.0, 0.0, 0.0, 1.0]), np.array([0.1 * kf_id, 0.0, 0.0]))
    b = np.full(n, UNBOUND, np.int64) if bind is None else bind.copy()
    kf = KeyFrame(kf_id, pose, CAM, u, v, lev, desc, mp_bindings=b.copy())
    cam = O.Cam(CAM.fx, CAM.fy, CAM.cx, CAM.cy, CAM.width, CAM.height, CAM.num_levels, CAM.scale_factor)
    okf = O.OKF(kf_id, pose.quat, pose.trans, cam, u, v, lev, desc, b.copy())
    return kf, okf


def neighbours_equal(m: MapModel, o: O.OracleMap) -> bool:
    for k, kf in o.kfs.items():
        if not kf.alive:
            continue
        if m.covisible_neighbors(k) != o.neighbors(k):
            return False
    return True


def test_long_random_sequence_matches_oracle():
    rng = np.random.default_rng(2025)
    n_kf0, n_slots, n_ops = 12, 40, 10000
    m = MapModel(CAM.num_levels, store=store_for(400, n_slots, points=1 << 15))
    o = O.OracleMap(CAM.num_levels)
    next_kf = 0
    for _ in range(n_kf0):
        kf, okf = make_pair(rng, next_kf, n_slots)
        m.insert_keyframe(kf)
        o.insert_keyframe(okf)
        next_kf += 1
    counts = dict.fromkeys(["new", "add", "erase", "kill", "replace", "insert_bound", "kill_kf"], 0)
    for step in range(n_ops):
        op = int(rng.integers(0, 100))
        live = [p for p in o.pts.values() if p.alive]
        live_kfs = [k for k, kf in o.kfs.items() if kf.alive]
        if op < 30 or not live:  # new point + first observation
            k = int(rng.choice(live_kfs))
            free = np.flatnonzero(o.kfs[k].bind == UNBOUND)
            if len(free) == 0:
                continue
            i = int(rng.choice(free))
            pos = rng.normal(0, 5, 3)
            p = o.new_point(pos, o.kfs[k].desc[i], k)
            mp = m.new_map_point(pos, o.kfs[k].desc[i], k)
            assert mp.mp_id == p.mp_id
            o.add_obs(p.mp_id, k, i)
            m.add_observation(p.mp_id, k, i)
            counts["new"] += 1
        elif op < 62:  # add an observation
            p = live[int(rng.integers(0, len(live)))]
            k = int(rng.choice(live_kfs))
            if k in p.obs:
                continue
            free = np.flatnonzero(o.kfs[k].bind == UNBOUND)
            if len(free) == 0:
                continue
            i = int(rng.choice(free))
            o.add_obs(p.mp_id, k, i)
            m.add_observation(p.mp_id, k, i)
            counts["add"] += 1
        elif op < 82:  # erase one (kills below min_obs_keep)
            p = live[int(rng.integers(0, len(live)))]
            if not p.obs:
                continue
            k = int(rng.choice(sorted(p.obs)))
            o.erase_obs(p.mp_id, k)
            m.erase_observation(p.mp_id, k)
            counts["erase"] += 1
        elif op < 87:  # kill a point
            p = live[int(rng.integers(0, len(live)))]
            o.kill_point(p.mp_id)
            m.kill_map_point(p.mp_id)
            counts["kill"] += 1
        elif op < 97:  # merge two points
            if len(live) < 2:
                continue
            a, b = rng.choice(len(live), size=2, replace=False)
            lo, wi = live[int(a)], live[int(b)]
            if len(lo.obs) > len(wi.obs):
                lo, wi = wi, lo
            o.replace(lo.mp_id, wi.mp_id)
            m.replace_map_point(lo.mp_id, wi.mp_id)
            counts["replace"] += 1
        elif op < 99:  # a new keyframe with pre-bound slots (insert_keyframe registers them)
            bind = np.full(n_slots, UNBOUND, np.int64)
            for q in rng.permutation(len(live))[: int(rng.integers(1, 8))]:
                bind[int(rng.integers(0, n_slots))] = live[int(q)].mp_id
            # one slot per point and no duplicates
            _, first = np.unique(bind, return_index=True)
            keep = np.full(n_slots, UNBOUND, np.int64)
            keep[first] = bind[first]
            kf, okf = make_pair(rng, next_kf, n_slots, keep)
            o.insert_keyframe(okf)
            m.insert_keyframe(kf)
            next_kf += 1
            counts["insert_bound"] += 1
        else:  # kill a keyframe (keep a few alive)
            if len(live_kfs) <= 4:
                continue
            k = int(rng.choice(live_kfs))
            o.kill_keyframe(k)
            m.kill_keyframe(k)
            counts["kill_kf"] += 1
        if step % 500 == 499:
            assert m._snapshot().structural_digest() == O.structural_digest(o), step
            assert neighbours_equal(m, o), step
    assert m._snapshot().structural_digest() == O.structural_digest(o)
    assert neighbours_equal(m, o)
    assert m.audit() == []
    assert o.audit() == []
    assert min(counts.values()) > 0, counts


def _small_world():
    rng = np.random.default_rng(5)
    m = MapModel(CAM.num_levels, store=store_for(16, 64, points=1024))
    kfs = []
    for k in range(3):
        kf, _ = make_pair(rng, k, 20)
        m.insert_keyframe(kf)
        kfs.append(kf)
    return m, kfs


def test_device_audit_clean_and_fault_injection():
    m, kfs = _small_world()
    mp = m.new_map_point([0, 0, 5.0], kfs[0].descriptors[0], 0)
    m.add_observation(mp.mp_id, 0, 0)
    m.add_observation(mp.mp_id, 1, 0)
    assert m.audit() == []
    # test_corrupted_scale_counts_detected
    m.ctx.call("lm_debug_corrupt", m.map, 0, mp.mp_id, 0, 1)
    m.invalidate()
    v = m.audit()
    assert f"scale_counts mismatch for map point {mp.mp_id}" in v
    assert f"scale_counts sum mismatch for map point {mp.mp_id}" in v
    m.ctx.call("lm_debug_corrupt", m.map, 0, mp.mp_id, 0, -1)
    m.invalidate()
    assert m.audit() == []
    # test_corrupted_edge_detected
    m.ctx.call("lm_debug_corrupt", m.map, 1, 0, 1, 1)
    m.invalidate()
    v = m.audit()
    assert v and any("(0, 1)" in x for x in v)


def test_kill_keyframe_matches_oracle_on_a_pipeline_map():
    """kill_keyframe on a map built by the hot path (thousands of bindings, points dying
    below min_obs_keep) against the oracle on the same map."""
    from helpers import cam_of, device_kf
    from paper_2511_02036_b200 import workload as W
    from paper_2511_02036_b200.session import LocalMapper

    seq = W.generate_sequence(W.WorldConfig(seed=41, landmark_count=2000, keyframe_count=10, features_per_kf=400,
                                            pixel_noise_sigma=0.8, descriptor_flip_bits=3, trajectory="line",
                                            extent=6.0))
    intr, cam = seq.intrinsics(), cam_of(seq)
    dev = LocalMapper(intr, neighbor_count=6, store=store_for(16, 512))
    ora = O.OraclePipeline(intr.num_levels, 6)
    for rec in seq.records:
        dev.process(device_kf(rec, intr))
        ora.step(O.okf_from_record(rec, cam))
    for k in (4, 7, 0):
        dev.ctx.call("lm_kf_kill", dev.map, k)
        ora.map.kill_keyframe(k)
        assert dev.snapshot(with_covis=False).structural_digest() == O.structural_digest(ora.map), k


def test_cull_keyframes_matches_oracle_on_a_pipeline_map():
    """§8(f) row 4: the device keyframe cull (counter prefix, lm_cull_keyframes) against the
    oracle's observation-walk restatement (is_redundant_baseline) on the same hot-path map,
    candidates = every live keyframe's covisible neighbours in turn (pipeline.py:215-221)."""
    from helpers import cam_of, device_kf
    from paper_2511_02036_b200 import workload as W
    from paper_2511_02036_b200.config import CullConfig
    from paper_2511_02036_b200.culling import cull_keyframes
    from paper_2511_02036_b200.mapmodel import DeviceStore
    from paper_2511_02036_b200.session import LocalMapper

    seq = W.generate_sequence(W.WorldConfig(seed=41, landmark_count=2000, keyframe_count=14, features_per_kf=400,
                                            pixel_noise_sigma=0.8, descriptor_flip_bits=3, trajectory="line",
                                            extent=6.0))
    intr, cam = seq.intrinsics(), cam_of(seq)
    ora = O.OraclePipeline(intr.num_levels, 8)
    m = MapModel(intr.num_levels, store=store_for(16, 512))
    st = DeviceStore()
    from paper_2511_02036_b200.culling import RecentPoint, cull_recent_map_points
    from paper_2511_02036_b200.fusion import run_fusion
    from paper_2511_02036_b200.triangulation import create_map_points

    recent, total = [], []
    for processed, rec in enumerate(seq.records):
        kf = device_kf(rec, intr)
        m.insert_keyframe(kf)
        st.upload_keyframe(kf)
        _, recent = cull_recent_map_points(m, recent, processed)
        recent += [RecentPoint(i, processed) for i in create_map_points(m, st, kf.kf_id, 8)]
        run_fusion(m, st, kf.kf_id)
        ora.step(O.okf_from_record(rec, cam))
        cand = [k for k in m.covisible_neighbors(kf.kf_id) if k != kf.kf_id]
        assert cand == [k for k in ora.map.neighbors(kf.kf_id) if k != kf.kf_id]
        cc = CullConfig(redundancy_ratio=0.6)  # a looser ratio so this short run culls
        got = cull_keyframes(m, st, cand, impl="fast", cfg=cc)
        want = O.cull_keyframes(ora.map, cand, O.KfCullCfg(redundancy_ratio=0.6))
        assert got == want, processed
        total += got
        for k in got:
            assert not st.is_resident(k)
        assert m._snapshot().structural_digest() == O.structural_digest(ora.map), processed
    assert total, "the run should cull at least one keyframe"
    assert st.ledger.evictions == len(total)


def test_cull_recent_skips_unknown_ids_and_rejects_repeats():
    """cull_recent_map_points (culling.py:28-59) skips an entry whose point the model cannot
    find (``mp is None``: neither removed nor kept). Two identical device maps, one culled
    with the pipeline's probation list and one with that list plus entries naming no point
    (negative, past the arena, not created yet): same removed ids, same kept entries (the
    caller's own objects), same map afterwards. A point listed twice is rejected."""
    from helpers import device_kf
    from paper_2511_02036_b200 import workload as W
    from paper_2511_02036_b200.culling import RecentPoint, cull_recent_map_points
    from paper_2511_02036_b200.errors import InvalidArgumentError
    from paper_2511_02036_b200.fusion import run_fusion
    from paper_2511_02036_b200.mapmodel import DeviceStore
    from paper_2511_02036_b200.triangulation import create_map_points

    seq = W.generate_sequence(W.WorldConfig(seed=43, landmark_count=2000, keyframe_count=8, features_per_kf=400,
                                            pixel_noise_sigma=0.8, descriptor_flip_bits=3, trajectory="line",
                                            extent=6.0))
    intr = seq.intrinsics()
    maps = [MapModel(intr.num_levels, store=store_for(16, 512)) for _ in range(2)]
    stores = [DeviceStore(), DeviceStore()]
    recent = [[], []]
    checked = 0
    for processed, rec in enumerate(seq.records):
        out = []
        for side in range(2):
            m, st = maps[side], stores[side]
            kf = device_kf(rec, intr)
            m.insert_keyframe(kf)
            st.upload_keyframe(kf)
            lst = recent[side]
            if side == 1 and lst:
                nxt = m._next_id()
                lst = [RecentPoint(-3, processed)] + lst[: len(lst) // 2] + [RecentPoint(nxt + 50, processed),
                                                                               RecentPoint(10 ** 9, 0)] + lst[len(lst) // 2:]
            removed, kept = cull_recent_map_points(m, lst, processed)
            assert all(any(k is e for e in lst) for k in kept)  # the caller's own entries
            out.append((removed, [(k.mp_id, k.created_at) for k in kept]))
            made = create_map_points(m, st, kf.kf_id, 6)
            recent[side] = kept + [RecentPoint(i, processed) for i in made]
            run_fusion(m, st, kf.kf_id)
        assert out[0] == out[1], processed
        checked += bool(out[0][0]) or bool(out[0][1])
        assert maps[0]._snapshot().structural_digest() == maps[1]._snapshot().structural_digest(), processed
    assert checked
    lst = recent[0]
    assert lst
    with pytest.raises(InvalidArgumentError):
        cull_recent_map_points(maps[0], lst + [lst[0]], len(seq.records))


@pytest.mark.parametrize("n_obs", [3, 31, 33, 64, 65, 128, 129, 300, 513, 700])
def test_representative_descriptor_every_refresh_path(n_obs):
    """_refresh_rep_descriptor (mapmodel.py:165-181) on one point observed n times, through
    every device path: register symmetric (<= 64), lane rows (<= 128), per-row distance
    array (<= 512) and the radix select without a size limit (> 512). Descriptors share a
    few prototypes plus bit flips, so the medians have many ties (first row wins)."""
    from helpers import rep_descriptor

    rng = np.random.default_rng(n_obs)
    protos = rng.integers(0, 256, (3, 32), dtype=np.uint8)
    m = MapModel(CAM.num_levels, store=store_for(n_obs + 8, 8, points=64))
    descs = []
    for k in range(n_obs):
        d = protos[rng.integers(0, 3)].copy()
        for _ in range(int(rng.integers(0, 12))):
            b = int(rng.integers(0, 256))
            d[b >> 3] ^= np.uint8(1 << (b & 7))
        desc = np.vstack([d, rng.integers(0, 256, (1, 32), dtype=np.uint8)])
        kf = KeyFrame(k, SE3Pose(np.array([0.0, 0.0, 0.0, 1.0]), np.array([0.01 * k, 0.0, 0.0])), CAM,
                      np.array([100.0, 200.0]), np.array([100.0, 200.0]), np.zeros(2, np.int64), desc)
        m.insert_keyframe(kf)
        descs.append(d)
    p = m.new_map_point([0.0, 0.0, 5.0], descs[0], 0)
    for k in range(n_obs):
        m.add_observation(p.mp_id, k, 0)
    got = m.points[p.mp_id].rep_descriptor
    want = rep_descriptor(np.stack(descs))
    assert np.array_equal(got, want)
