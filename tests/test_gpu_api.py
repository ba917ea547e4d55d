"""Drop-in API behaviour on the GPU, mirroring the reference's unit tests
(pkg/tests/test_triangulation.py, test_fusion.py, test_mapmodel.py) against this
package's device-backed MapModel and stage functions."""

from __future__ import annotations

import numpy as np
import pytest

from scenes import CAM, views
from paper_2511_02036_b200 import (DeviceStore, InvalidArgumentError, InvalidStateError, KeyFrame, MapModel,
                                   SE3Pose, SlotConflictError)
from paper_2511_02036_b200.config import FuseConfig, MatchConfig
from paper_2511_02036_b200.fusion import (ADD_OBSERVATION, MERGE, FuseAction, apply_fusion, collect_fusion_targets,
                                          fuse_pass, run_fusion)
from paper_2511_02036_b200.geometry import flip_descriptor_bits, project, random_descriptors
from paper_2511_02036_b200.triangulation import CreationStats, create_map_points, search_for_triangulation

pytestmark = pytest.mark.gpu


def small_store():
    from paper_2511_02036_b200.session import store_for

    return store_for(16, 512, points=4096)


def model_of(kfs, cam=CAM):
    m = MapModel(num_levels=cam.num_levels, store=small_store())
    st = DeviceStore()
    for kf in kfs:
        m.insert_keyframe(kf)
        st.upload_keyframe(kf)
    return m, st


# ----------------------------------------------------------------------------- search


class TestSearch:
    def test_exact_scene_recovers_every_landmark(self):
        kfs, truth, _ = views(np.random.default_rng(31))
        got = search_for_triangulation(kfs[0], kfs[1])
        assert len(got) == 50
        for c in got:
            assert truth[0][c.kp_index_current] == truth[1][c.kp_index_neighbor] and c.distance == 0

    def test_unrelated_descriptors_give_nothing(self):
        kfs, _, _ = views(np.random.default_rng(33), n_landmarks=30)
        kfs[1].descriptors = np.random.default_rng(999).integers(0, 256, kfs[1].descriptors.shape, dtype=np.uint8)
        assert search_for_triangulation(kfs[0], kfs[1]) == []

    def test_tie_goes_to_lowest_current_index(self):
        kfs, truth, _ = views(np.random.default_rng(35), n_landmarks=12)
        j = next(i for i, lm in truth[1].items() if lm == truth[0][0])
        kfs[0].descriptors[1] = kfs[1].descriptors[j].copy()
        winners = [c for c in search_for_triangulation(kfs[0], kfs[1]) if c.kp_index_neighbor == j]
        assert len(winners) == 1 and winners[0].kp_index_current == 0

    def test_zero_baseline_pair_skipped(self):
        kfs, _, _ = views(np.random.default_rng(37), centers=((0, 0, 0), (0, 0, 0)))
        assert search_for_triangulation(kfs[0], kfs[1]) == []

    def test_bound_keypoints_are_excluded(self):
        kfs, _, _ = views(np.random.default_rng(39), n_landmarks=20)
        mask = np.ones(kfs[0].num_keypoints, dtype=bool)
        mask[:10] = False
        got = search_for_triangulation(kfs[0], kfs[1], unbound_current=mask)
        assert len(got) == 10 and all(c.kp_index_current >= 10 for c in got)

    def test_engine_aliases_identical_and_unknown_rejected(self):
        kfs, _, _ = views(np.random.default_rng(40), n_landmarks=40, desc_noise=4)
        ref = search_for_triangulation(kfs[0], kfs[1], engine="b200")
        assert search_for_triangulation(kfs[0], kfs[1], engine="reference") == ref
        assert search_for_triangulation(kfs[0], kfs[1], MatchConfig(chunk_size=16), engine="batch") == ref
        with pytest.raises(ValueError):
            search_for_triangulation(kfs[0], kfs[1], engine="cpu")

    def test_larger_threshold_only_adds_pairs(self):
        kfs, _, _ = views(np.random.default_rng(41), n_landmarks=40, desc_noise=12)

        def pairs(d):
            return {(c.kp_index_current, c.kp_index_neighbor)
                    for c in search_for_triangulation(kfs[0], kfs[1], MatchConfig(match_max_distance=d))}

        assert pairs(20) <= pairs(60)


# ----------------------------------------------------------------------------- creation


class TestCreate:
    def test_noise_free_pair_creates_every_point(self):
        kfs, truth, _ = views(np.random.default_rng(51), centers=((0, 0, 0), (0.6, 0, 0)))
        m, st = model_of(kfs)
        stats = CreationStats()
        made = create_map_points(m, st, 1, 1, stats=stats)
        assert len(made) == 50 and stats.created == 50
        for mp_id in made:
            mp = m.points[mp_id]
            assert len(mp.observations) == 2 and int(mp.scale_counts.sum()) == 2
            for k, idx in mp.observations.items():
                kf = m.keyframes[k]
                pix = project(CAM, kf.pose.transform(mp.position))
                assert abs(pix[0] - kf.kp_u[idx]) < 1e-6 and abs(pix[1] - kf.kp_v[idx]) < 1e-6
        assert m.audit() == []
        assert st.ledger.naive_bytes_up == st.payload_bytes(kfs[0].num_keypoints)

    def test_points_behind_both_cameras_fail_the_depth_gate(self):
        rng = np.random.default_rng(53)
        n = 50
        lm = np.column_stack([rng.uniform(-1.5, 1.5, n), rng.uniform(-1.0, 1.0, n), rng.uniform(-8.0, -4.0, n)])
        desc = random_descriptors(rng, n)
        poses = [SE3Pose.identity(), SE3Pose(np.array([0, 0, 0, 1.0]), np.array([-0.6, 0.0, 0.0]))]
        kfs = []
        for k, pose in enumerate(poses):
            pc = np.stack([pose.transform(p) for p in lm])
            u = CAM.fx * (pc[:, 0] / pc[:, 2]) + CAM.cx
            v = CAM.fy * (pc[:, 1] / pc[:, 2]) + CAM.cy
            kfs.append(KeyFrame(k, pose, CAM, u, v, np.zeros(n, np.int64), desc))
        m, st = model_of(kfs)
        stats = CreationStats()
        assert create_map_points(m, st, 1, 1, stats=stats) == []
        assert stats.gate_failures.get("positive-depth", 0) == 50

    def test_zero_neighbours(self):
        kfs, _, _ = views(np.random.default_rng(51))
        m, st = model_of(kfs)
        assert create_map_points(m, st, 1, 0) == []

    def test_conflicts_are_counted_not_raised(self):
        kfs, _, _ = views(np.random.default_rng(55), n_landmarks=30, centers=((0, 0, 0), (0.5, 0, 0), (-0.5, 0, 0)))
        m, st = model_of(kfs)
        stats = CreationStats()
        assert len(create_map_points(m, st, 0, 2, stats=stats)) == 30
        assert stats.conflicts == 30
        assert m.audit() == []


# ----------------------------------------------------------------------------- fusion


def chain_map(weights):
    rng = np.random.default_rng(0)
    n = len(weights) + 1
    kfs, _, _ = views(rng, n_landmarks=sum(weights) + 4, centers=[(0.1 * i, 0, 0) for i in range(n)])
    m, _ = model_of(kfs)
    slot = 0
    for a, w in enumerate(weights):
        for _ in range(w):
            mp = m.new_map_point([0, 0, 8.0], kfs[a].descriptors[slot], a)
            m.add_observation(mp.mp_id, a, slot)
            m.add_observation(mp.mp_id, a + 1, slot)
            slot += 1
    return m, kfs


def fused_scene(seed=71, n=40):
    kfs, truth, pts = views(np.random.default_rng(seed), n_landmarks=n, centers=((0, 0, 0), (0.5, 0, 0), (1.0, 0.1, 0)))
    m, st = model_of(kfs)
    assert len(create_map_points(m, st, 2, 1)) == n  # pads with the most recent keyframe: 1
    return m, st, kfs, truth, pts


def true_slot(truth, k, lm):
    return next(i for i, x in truth[k].items() if x == lm)


class TestTargets:
    def test_chain_walk(self):
        m, _ = chain_map([3, 2])
        assert collect_fusion_targets(m, 0, n1=1, n2=1) == [1, 2]

    def test_isolated_keyframe_has_no_targets(self):
        m, kfs = chain_map([3])
        k = kfs[0]
        m.insert_keyframe(KeyFrame(99, k.pose, CAM, k.kp_u, k.kp_v, k.kp_level, k.descriptors))
        assert collect_fusion_targets(m, 99, 5, 5) == []

    def test_first_and_second_order_dedup(self):
        m, _ = chain_map([3, 2])
        assert collect_fusion_targets(m, 1, 2, 2) == [0, 2]


class TestFusePass:
    def test_injected_twin_yields_one_merge(self):
        m, st, kfs, truth, _ = fused_scene()
        donor = next(p for p in m.points.values() if p.alive)
        lm = truth[1][donor.observations[1]]
        j0 = true_slot(truth, 0, lm)
        twin = m.new_map_point(donor.position.copy(), kfs[0].descriptors[j0], 0)
        m.add_observation(twin.mp_id, 0, j0)
        acts, vis = fuse_pass(m, [twin.mp_id], 1)
        merges = [a for a in acts if a.kind == MERGE]
        assert len(merges) == 1 and merges[0].existing_mp_id == donor.mp_id
        assert merges[0].mp_id_projected == twin.mp_id and twin.mp_id in vis

    def test_point_out_of_view(self):
        m, st, kfs, _, _ = fused_scene()
        p = m.new_map_point([0, 0, -50.0], kfs[0].descriptors[0], 0)
        m.add_observation(p.mp_id, 0, 0)
        assert fuse_pass(m, [p.mp_id], 1) == ([], [])

    def test_unbound_hits_add_at_the_true_slot(self):
        m, st, kfs, truth, _ = fused_scene()
        pts = m.bound_points_of(2)
        acts, _ = fuse_pass(m, pts, 0)
        adds = [a for a in acts if a.kind == ADD_OBSERVATION]
        assert len(adds) == len(pts)
        for a in adds:
            assert truth[0][a.kp_index_hit] == truth[2][m.points[a.mp_id_projected].observations[2]]


class TestApply:
    def test_two_merges_sharing_a_loser(self):
        m, st, kfs, truth, _ = fused_scene()
        pts = m.bound_points_of(1)
        a, b = pts[0], pts[1]
        twin = m.new_map_point(m.points[a].position.copy(), m.points[a].rep_descriptor, 0)
        m.add_observation(twin.mp_id, 0, 0)
        batch = [FuseAction(1, twin.mp_id, m.points[a].observations[1], a, MERGE),
                 FuseAction(1, twin.mp_id, m.points[b].observations[1], b, MERGE)]
        c = apply_fusion(m, batch)
        assert c["merged"] == 1 and c["stale"] == 1
        assert m.audit() == []

    def test_empty_batch(self):
        m, _, _, _, _ = fused_scene()
        assert apply_fusion(m, []) == {"merged": 0, "observations_added": 0, "stale": 0}

    def test_merge_then_add(self):
        m, st, kfs, truth, _ = fused_scene()
        before = len(m.live_points())
        pts = m.bound_points_of(1)
        a, b = pts[0], pts[1]
        twin = m.new_map_point(m.points[a].position.copy(), m.points[a].rep_descriptor, 0)
        m.add_observation(twin.mp_id, 0, 1)
        jb = true_slot(truth, 0, truth[1][m.points[b].observations[1]])
        c = apply_fusion(m, [FuseAction(1, twin.mp_id, m.points[a].observations[1], a, MERGE),
                             FuseAction(0, b, jb, None, ADD_OBSERVATION)])
        assert c == {"merged": 1, "observations_added": 1, "stale": 0}
        assert len(m.live_points()) == before
        assert len(m.points[b].observations) == 3
        assert m.audit() == []


class TestRunFusion:
    def test_clean_map_keeps_its_points(self):
        m, st, _, _, _ = fused_scene()
        before = len(m.live_points())
        c = run_fusion(m, st, 2)
        assert c["merged"] == 0 and len(m.live_points()) == before and m.audit() == []

    def test_every_injected_twin_merges(self):
        m, st, kfs, truth, _ = fused_scene(n=40)
        rng = np.random.default_rng(1)
        pts = m.bound_points_of(2)
        for mp_id in pts[:10]:
            m.add_observation(mp_id, 0, true_slot(truth, 0, truth[2][m.points[mp_id].observations[2]]))
        for mp_id in pts[10:15]:
            p = m.points[mp_id]
            t = m.new_map_point(p.position.copy(), flip_descriptor_bits(rng, p.rep_descriptor, 5), 0)
            m.add_observation(t.mp_id, 0, true_slot(truth, 0, truth[2][p.observations[2]]))
        before = len(m.live_points())
        c = run_fusion(m, st, 0)
        assert c["merged"] == 5 and len(m.live_points()) == before - 5 and m.audit() == []

    def test_second_run_is_idempotent(self):
        m, st, _, _, _ = fused_scene()
        run_fusion(m, st, 2)
        assert run_fusion(m, st, 2)["merged"] == 0 and m.audit() == []

    def test_never_increases_points(self):
        for seed in range(3):
            m, st, _, _, _ = fused_scene(seed=300 + seed)
            before = len(m.live_points())
            run_fusion(m, st, 2)
            assert len(m.live_points()) <= before


# ----------------------------------------------------------------------------- map model


class TestMapModel:
    def test_prebound_keyframe_registers_observations(self):
        kfs, _, _ = views(np.random.default_rng(3), n_landmarks=16, centers=((0, 0, 0), (0.3, 0, 0)))
        m = MapModel(num_levels=CAM.num_levels, store=small_store())
        m.insert_keyframe(kfs[0])
        ids = []
        for i in range(12):
            p = m.new_map_point(np.zeros(3), kfs[0].descriptors[i], 0)
            m.add_observation(p.mp_id, 0, i)
            ids.append(p.mp_id)
        kfs[1].mp_bindings[:12] = ids
        m.insert_keyframe(kfs[1])
        assert m.graph.weight(0, 1) == 12 and m.audit() == []

    def test_errors_match_reference(self):
        kfs, _, _ = views(np.random.default_rng(4), n_landmarks=8)
        m, _ = model_of(kfs)
        with pytest.raises(InvalidArgumentError):
            m.insert_keyframe(kfs[0])
        p = m.new_map_point(np.zeros(3), kfs[0].descriptors[0], 0)
        m.add_observation(p.mp_id, 0, 0)
        with pytest.raises(SlotConflictError):
            m.add_observation(p.mp_id, 0, 1)  # already observes keyframe 0
        q = m.new_map_point(np.zeros(3), kfs[0].descriptors[0], 0)
        with pytest.raises(SlotConflictError):
            m.add_observation(q.mp_id, 0, 0)  # slot bound to p
        with pytest.raises(InvalidArgumentError):
            m.add_observation(q.mp_id, 0, 10_000)
        m.kill_map_point(q.mp_id)
        with pytest.raises(InvalidStateError):
            m.add_observation(q.mp_id, 1, 0)
        with pytest.raises(InvalidArgumentError):
            m.replace_map_point(p.mp_id, p.mp_id)

    def test_replace_migrates_and_unbinds_shared_keyframes(self):
        kfs, _, _ = views(np.random.default_rng(5), n_landmarks=8, centers=((0, 0, 0), (0.3, 0, 0), (0.6, 0, 0)))
        m, _ = model_of(kfs)
        a = m.new_map_point(np.zeros(3), kfs[0].descriptors[0], 0)
        b = m.new_map_point(np.zeros(3), kfs[0].descriptors[1], 0)
        m.add_observation(a.mp_id, 0, 0)
        m.add_observation(a.mp_id, 1, 0)
        m.add_observation(b.mp_id, 1, 1)
        m.add_observation(b.mp_id, 2, 1)
        m.add_observation(b.mp_id, 0, 1)
        mig = m.replace_map_point(a.mp_id, b.mp_id)  # both see kf0, kf1: nothing migrates
        assert mig == 0
        assert m.points[b.mp_id].observations == {0: 1, 1: 1, 2: 1}
        assert not m.points[a.mp_id].alive
        assert m.keyframes[0].mp_bindings[0] == -1 and m.audit() == []

    def test_rep_descriptor_is_median_minimiser(self):
        kfs, _, _ = views(np.random.default_rng(6), n_landmarks=6,
                          centers=tuple((0.2 * i, 0, 0) for i in range(5)))
        m, _ = model_of(kfs)
        base = kfs[0].descriptors[0]
        rng = np.random.default_rng(7)
        for k in range(5):
            kfs[k].descriptors[0] = flip_descriptor_bits(rng, base, 2 + 6 * k)
        m2, _ = model_of([KeyFrame(k, kf.pose, CAM, kf.kp_u, kf.kp_v, kf.kp_level, kf.descriptors)
                          for k, kf in enumerate(kfs)])
        p = m2.new_map_point(np.zeros(3), base, 0)
        for k in range(5):
            m2.add_observation(p.mp_id, k, 0)
        descs = [kf.descriptors[0] for kf in kfs]
        d = np.array([[int(np.bitwise_count(a ^ b).sum()) for b in descs] for a in descs], float)
        np.fill_diagonal(d, np.nan)
        best = int(np.argmin(np.nanmedian(d, axis=1)))
        assert np.array_equal(m2.points[p.mp_id].rep_descriptor, kfs[best].descriptors[0])
