"""GPU path against the REAL reference's frozen outputs (tests/golden/golden.json, made by
tests/golden/make_golden.py from /root/reference): per keyframe creation/fusion/cull
counters and the structural map digest (bindings, live ids, found/visible, representative
descriptors, observation lists, per-level counters) bit for bit; search candidate tuples
bit for bit; final positions within the north_star's 1e-4 relative tolerance. This is the
device compared with the reference directly, with no oracle in between."""

from __future__ import annotations

import json
import os

import numpy as np
import pytest

from helpers import device_kf
from paper_2511_02036_b200 import workload as W
from paper_2511_02036_b200.session import LocalMapper, store_for
from paper_2511_02036_b200.triangulation import search_for_triangulation

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "golden.json")))
POS = np.load(os.path.join(HERE, "golden", "golden_positions.npz"))
POS_RTOL = 1e-4

_SEQ = {}


def seq(name):
    if name not in _SEQ:
        _SEQ[name] = W.generate_sequence(W.WorldConfig(**GOLD["workloads"][name]["config"]))
    return _SEQ[name]


@pytest.mark.parametrize("name", sorted(GOLD["pipeline"]))
def test_pipeline_matches_reference_golden(name):
    s = seq(name)
    intr = s.intrinsics()
    g = GOLD["pipeline"][name]
    dev = LocalMapper(intr, neighbor_count=g["neighbor_count"],
                      store=store_for(len(s.records), s.config.features_per_kf * 2))
    for rec, want in zip(s.records, g["steps"]):
        dev.process(device_kf(rec, intr))
        st = dev.stats  # running totals, like the golden's (CreationStats / fusion totals / culled list)
        assert (st.created, st.conflicts, st.degenerate) == (want["created"], want["conflicts"], want["degenerate"]), \
            (name, rec.kf_id)
        assert st.gate_failures == want["gates"], (name, rec.kf_id)
        assert dev.fused == want["fusion"], (name, rec.kf_id)
        assert dev.culled == want["culled"], (name, rec.kf_id)
        assert dev.snapshot(with_covis=False).structural_digest() == want["digest"], (name, rec.kf_id)
    snap = dev.snapshot(with_covis=False)
    ids = np.flatnonzero(snap.alive)
    assert ids.tolist() == POS[f"{name}_ids"].tolist()
    if len(ids):
        got, want = snap.pos[ids], POS[f"{name}_pos"]
        rel = np.linalg.norm(got - want, axis=1) / np.maximum(np.linalg.norm(want, axis=1), 1e-12)
        assert float(rel.max()) <= POS_RTOL


@pytest.mark.parametrize("name", sorted(GOLD["search"]))
def test_search_matches_reference_golden(name):
    s = seq(name)
    intr = s.intrinsics()
    for key, want in GOLD["search"][name].items():
        a, b = map(int, key.split(","))
        ka, kb = device_kf(s.records[a], intr), device_kf(s.records[b], intr)
        got = [[c.kp_index_current, c.kp_index_neighbor, c.distance] for c in search_for_triangulation(ka, kb)]
        assert got == want, (name, key)
