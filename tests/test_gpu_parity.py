"""GPU parity: the CUDA path (through the C ABI) against the NumPy oracle on the same
seeded inputs. Integer/index outputs are compared bit for bit; triangulated positions
within 1e-4 relative (BASELINE.json north_star)."""

from __future__ import annotations

import numpy as np
import pytest

from helpers import cam_of, compare_state, device_kf, first_difference
from oracle import lm_oracle as O
from paper_2511_02036_b200 import workload as W
from paper_2511_02036_b200.config import FuseConfig, MatchConfig
from paper_2511_02036_b200.session import LocalMapper, store_for
from paper_2511_02036_b200.triangulation import search_for_triangulation

pytestmark = pytest.mark.gpu

SEQS = {
    "orbit20": dict(seed=11, landmark_count=300, keyframe_count=20, features_per_kf=220, pixel_noise_sigma=1.0,
                    descriptor_flip_bits=3, trajectory="orbit", pose_noise_trans=0.03, pose_noise_rot_deg=0.3),
    "line14dup": dict(seed=41, landmark_count=2000, keyframe_count=14, features_per_kf=400, pixel_noise_sigma=0.8,
                      descriptor_flip_bits=3, trajectory="line", extent=6.0, duplicate_injection_rate=0.05,
                      twin_flip_bits=20),
    "orbit7": dict(seed=300, landmark_count=180, keyframe_count=7, features_per_kf=110, pixel_noise_sigma=0.7,
                   descriptor_flip_bits=2, trajectory="orbit"),
}


def _seq(name):
    return W.generate_sequence(W.WorldConfig(**SEQS[name]))


@pytest.mark.parametrize("name", ["orbit7", "line14dup"])
def test_search_pairs_match_oracle(name):
    seq = _seq(name)
    intr = seq.intrinsics()
    cam = cam_of(seq)
    recs = seq.records
    mism = 0
    for a, b in [(1, 0), (3, 1), (5, 4), (len(recs) - 1, len(recs) - 3)]:
        ka, kb = device_kf(recs[a], intr), device_kf(recs[b], intr)
        got = [(c.kp_index_current, c.kp_index_neighbor, c.distance) for c in search_for_triangulation(ka, kb)]
        oa, ob = O.okf_from_record(recs[a], cam), O.okf_from_record(recs[b], cam)
        f = O.fundamental(oa.quat, oa.trans, oa.cam, ob.quat, ob.trans, ob.cam)
        want = O.search_pairs(oa, ob, f, 3.84, 50, 1, np.ones(oa.n, bool), np.ones(ob.n, bool))
        mism += got != want
    assert mism == 0


@pytest.mark.parametrize("name", ["orbit7", "orbit20", "line14dup"])
def test_sequence_matches_oracle(name):
    seq = _seq(name)
    intr = seq.intrinsics()
    cam = cam_of(seq)
    n = 10
    dev = LocalMapper(intr, neighbor_count=n, store=store_for(len(seq.records), seq.config.features_per_kf * 2))
    ora = O.OraclePipeline(intr.num_levels, n)
    for rec in seq.records:
        r = dev.process(device_kf(rec, intr))
        ora.step(O.okf_from_record(rec, cam))
        snap = dev.snapshot()
        cmp = compare_state(snap, ora.map)
        assert (dev.stats.created, dev.stats.conflicts) == (ora.stats.created, ora.stats.conflicts), rec.kf_id
        assert dev.fused == ora.fused, (rec.kf_id, dev.fused, ora.fused)
        assert cmp["structural_equal"], (rec.kf_id, first_difference(snap, ora.map))
        assert cmp["pos_ok"], (rec.kf_id, cmp["pos_worst_rel"])
