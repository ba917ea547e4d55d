"""GPU path at BASELINE.json's full sizes and in batched form.

* C2 (EuRoC shape, 1200 features, 20 neighbours): the first keyframes compared with the
  oracle after every keyframe (bitwise structure, positions within 1e-4 relative), then
  the whole 200-keyframe sequence checked through size-independent properties of the map
  the reference's own audit checks (mapmodel.py:304-353): binding <-> observation
  bijection, per-level counters, covisibility weight == shared bound points for every
  keyframe pair, and representative descriptor == median-Hamming minimiser of the
  observing descriptors (sampled points); plus determinism (two runs, identical digests).
* Batched sessions (C5's form): several independent maps advanced in lock-step with one
  launch sequence per keyframe index give exactly the results of running each alone.
* Edge cases: a keyframe without keypoints, and a keyframe whose descriptors match nothing.
"""

from __future__ import annotations

import numpy as np
import pytest

from helpers import audit_snapshot, cam_of, compare_state, device_kf, first_difference
from oracle import lm_oracle as O
from paper_2511_02036_b200 import workload as W
from paper_2511_02036_b200.config import FuseConfig, MatchConfig
from paper_2511_02036_b200.mapmodel import KeyFrame
from paper_2511_02036_b200.session import LocalMapper, SessionBatch, store_for

pytestmark = pytest.mark.gpu

_C2 = {}


def c2():
    if "s" not in _C2:
        _C2["s"] = W.generate_sequence(W.bench_world("c2"))
    return _C2["s"]


def c2_mapper(seq):
    n, n1, n2 = W.BENCH_STAGE["c2"]
    return LocalMapper(seq.intrinsics(), neighbor_count=n, match=MatchConfig(neighbor_count=n),
                       fuse=FuseConfig(n1=n1, n2=n2), store=store_for(len(seq.records), seq.config.features_per_kf + 64))


def test_c2_prefix_matches_oracle_every_keyframe():
    s = c2()
    intr, cam = s.intrinsics(), cam_of(s)
    n, n1, n2 = W.BENCH_STAGE["c2"]
    dev = c2_mapper(s)
    ora = O.OraclePipeline(intr.num_levels, n, fc=O.FuseCfg(n1=n1, n2=n2))
    for rec in s.records[:12]:
        dev.process(device_kf(rec, intr))
        ora.step(O.okf_from_record(rec, cam))
        snap = dev.snapshot(with_covis=False)
        cmp = compare_state(snap, ora.map)
        assert (dev.stats.created, dev.stats.conflicts) == (ora.stats.created, ora.stats.conflicts), rec.kf_id
        assert dev.fused == ora.fused, rec.kf_id
        assert cmp["structural_equal"], (rec.kf_id, first_difference(snap, ora.map))
        assert cmp["pos_ok"], (rec.kf_id, cmp["pos_worst_rel"])


def test_c2_full_sequence_properties_and_determinism():
    s = c2()
    intr = s.intrinsics()
    kfs = [device_kf(r, intr) for r in s.records]
    digests = []
    for run in range(2):
        dev = c2_mapper(s)
        for kf in kfs:
            dev.process(kf)
        snap = dev.snapshot(with_covis=True)
        digests.append(snap.structural_digest())
        if run == 0:
            assert dev.stats.created > 100_000 and dev.fused["merged"] > 1000  # the workload is exercised
            bad = audit_snapshot(snap, kfs, sample_rep=3000)
            assert bad == [], bad[:10]
    assert digests[0] == digests[1]


SESS = [dict(seed=11, landmark_count=300, keyframe_count=12, features_per_kf=220, trajectory="orbit"),
        dict(seed=41, landmark_count=2000, keyframe_count=12, features_per_kf=400, trajectory="line", extent=6.0,
             duplicate_injection_rate=0.05, twin_flip_bits=20),
        dict(seed=6, landmark_count=300, keyframe_count=12, features_per_kf=150, min_covisible=5,
             trajectory="corridor-loop", extent=10.0, spurious_feature_fraction=0.1)]


def test_batched_sessions_equal_independent_runs_and_oracle():
    seqs = [W.generate_sequence(W.WorldConfig(**c)) for c in SESS]
    mk = lambda q: LocalMapper(q.intrinsics(), neighbor_count=10,  # noqa: E731
                               store=store_for(len(q.records), q.config.features_per_kf * 2))
    batch_m = [mk(q) for q in seqs]
    batch = SessionBatch(batch_m)
    for q, m in zip(seqs, batch_m):
        for r in q.records:
            m.stage(device_kf(r, q.intrinsics()))
    nk = min(len(q.records) for q in seqs)
    for k in range(nk):
        batch.step([int(q.records[k].kf_id) for q in seqs])
    for q, m in zip(seqs, batch_m):
        alone = mk(q)
        ora = O.OraclePipeline(q.intrinsics().num_levels, 10)
        for r in q.records[:nk]:
            alone.process(device_kf(r, q.intrinsics()))
            ora.step(O.okf_from_record(r, cam_of(q)))
        sb, sa = m.snapshot(), alone.snapshot()
        assert sb.structural_digest() == sa.structural_digest()
        assert np.array_equal(sb.pos, sa.pos)
        assert m.fused == alone.fused == ora.fused
        cmp = compare_state(sb, ora.map)
        assert cmp["structural_equal"] and cmp["pos_ok"]


def _orbit(n_kf=6, feats=150, seed=300):
    return W.generate_sequence(W.WorldConfig(seed=seed, landmark_count=200, keyframe_count=n_kf,
                                             features_per_kf=feats, trajectory="orbit"))


def test_empty_keyframe_and_unmatched_descriptors():
    s = _orbit()
    intr, cam = s.intrinsics(), cam_of(s)
    dev = LocalMapper(intr, neighbor_count=10, store=store_for(len(s.records) + 2, 300))
    ora = O.OraclePipeline(intr.num_levels, 10)
    recs = list(s.records)
    for r in recs[:3]:
        dev.process(device_kf(r, intr))
        ora.step(O.okf_from_record(r, cam))
    # a keyframe with no keypoints: nothing to search or fuse, the map is unchanged
    r = recs[3]
    empty = KeyFrame(int(r.kf_id), r.pose_init, intr, np.zeros(0), np.zeros(0), np.zeros(0, np.int64),
                     np.zeros((0, 32), np.uint8))
    res = dev.process(empty)
    assert res.created == 0 and res.merged == 0 and res.observations_added == 0
    assert audit_snapshot(dev.snapshot(), None) == []
    # a keyframe whose descriptors match nothing: no new points, no fusion actions
    r = recs[4]
    rng = np.random.default_rng(7)
    noise = KeyFrame(int(r.kf_id), r.pose_init, intr, r.kp_u, r.kp_v, r.kp_level,
                     rng.integers(0, 256, r.descriptors.shape, dtype=np.uint8))
    res = dev.process(noise)
    assert res.created == 0 and res.merged == 0 and res.observations_added == 0


def _stage_mapper(name, seq):
    n, n1, n2 = W.BENCH_STAGE[name]
    return LocalMapper(seq.intrinsics(), neighbor_count=n, match=MatchConfig(neighbor_count=n),
                       fuse=FuseConfig(n1=n1, n2=n2), store=store_for(len(seq.records), seq.config.features_per_kf + 64))


@pytest.mark.parametrize("name,prefix", [("c3", 8), ("c4", 3)])
def test_large_configs_prefix_match_oracle(name, prefix):
    """TUM-VI shape (1500 features, 30 neighbours) and the stress shape (5000 features, 50
    neighbours, up to 300 fusion targets): the first keyframes against the oracle."""
    s = W.generate_sequence(W.bench_world(name))
    intr, cam = s.intrinsics(), cam_of(s)
    n, n1, n2 = W.BENCH_STAGE[name]
    dev = _stage_mapper(name, s)
    ora = O.OraclePipeline(intr.num_levels, n, fc=O.FuseCfg(n1=n1, n2=n2))
    for rec in s.records[:prefix]:
        dev.process(device_kf(rec, intr))
        ora.step(O.okf_from_record(rec, cam))
        snap = dev.snapshot(with_covis=False)
        cmp = compare_state(snap, ora.map)
        assert (dev.stats.created, dev.stats.conflicts) == (ora.stats.created, ora.stats.conflicts), rec.kf_id
        assert dev.fused == ora.fused, rec.kf_id
        assert cmp["structural_equal"], (rec.kf_id, first_difference(snap, ora.map))
        assert cmp["pos_ok"], (rec.kf_id, cmp["pos_worst_rel"])


@pytest.mark.parametrize("name", ["c3", "c4"])
def test_large_configs_full_run_audit(name):
    """Whole C3 (500 keyframes) / C4 (60 keyframes, 5000 features) sequences: map audit."""
    s = W.generate_sequence(W.bench_world(name))
    intr = s.intrinsics()
    kfs = [device_kf(r, intr) for r in s.records]
    dev = _stage_mapper(name, s)
    for kf in kfs:
        dev.process(kf)
    snap = dev.snapshot(with_covis=True)
    bad = audit_snapshot(snap, kfs, sample_rep=2000)
    assert bad == [], bad[:10]


def test_stream_groups_equal_independent_runs():
    """C5's multi-stream form: sessions in two contexts (one stream each), steps issued
    without synchronisation and interleaved, equal independent runs."""
    from paper_2511_02036_b200 import _lib

    seqs = [W.generate_sequence(W.WorldConfig(**c)) for c in SESS]
    ctxs = [_lib.Context.get(0), _lib.Context(0)]
    groups = [[0, 2], [1]]
    mk = lambda q, ctx: LocalMapper(q.intrinsics(), neighbor_count=10, ctx=ctx,  # noqa: E731
                                    store=store_for(len(q.records), q.config.features_per_kf * 2))
    mappers = {}
    batches = []
    for g, members in enumerate(groups):
        ms = [mk(seqs[i], ctxs[g]) for i in members]
        for i, m in zip(members, ms):
            mappers[i] = m
            for r in seqs[i].records:
                m.stage(device_kf(r, seqs[i].intrinsics()))
        batches.append((SessionBatch(ms), members))
    nk = min(len(q.records) for q in seqs)
    for k in range(nk):
        for b, members in batches:
            b.step([int(seqs[i].records[k].kf_id) for i in members], sync=False)
    for c in ctxs:
        c.call("lm_synchronize")
    for i, q in enumerate(seqs):
        alone = mk(q, None)
        for r in q.records[:nk]:
            alone.process(device_kf(r, q.intrinsics()))
        sb, sa = mappers[i].snapshot(), alone.snapshot()
        assert sb.structural_digest() == sa.structural_digest()
        assert np.array_equal(sb.pos, sa.pos)
