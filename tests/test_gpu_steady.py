"""Steady-state parity on the headline configs: the GPU path against the REAL reference's
frozen per-keyframe outputs (tests/golden/steady_*.json, written by
tests/golden/make_golden_steady.py from /root/reference, mode="baseline", LBA and keyframe
culling force-skipped) on EVERY keyframe, at the BASELINE neighbour counts:

  * C2 (EuRoC shape): all 200 keyframes, 20 neighbours, n1=20 -- the sequence bench.py times;
  * C3 (TUM-VI shape): keyframes 0-59, 30 neighbours, n1=30;
  * C4 (stress): keyframes 0-9, 5000 features, 50 neighbours, n1=50;
  * C5: 4 of the 64 session seeds (5000-5003), 60 keyframes each, stepped as one batch.

Per keyframe: running creation / gate / fusion / cull counters, the structural map digest
(bindings, live ids, found/visible, representative descriptors, observation lists, live
per-level counter rows) bit for bit, and the TransferLedger.as_dict() fields. After the last
keyframe, live point positions within the north_star's 1e-4 relative tolerance. The
device's borderline-compare counters (lm_step_stats.borderline) are reported alongside: with
every digest equal, none of them flipped a decision.
"""

from __future__ import annotations

import glob
import json
import os

import numpy as np
import pytest

from helpers import device_kf
from paper_2511_02036_b200 import workload as W
from paper_2511_02036_b200.config import FuseConfig, MatchConfig
from paper_2511_02036_b200.session import LocalMapper, SessionBatch, store_for

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = {os.path.basename(p)[len("steady_"):-len(".json")]: p
        for p in sorted(glob.glob(os.path.join(HERE, "golden", "steady_*.json")))}
POS_RTOL = 1e-4


def load(name):
    g = json.load(open(GOLD[name]))
    pos = np.load(GOLD[name][:-len(".json")] + "_positions.npz")
    return g, pos


def mapper_for(g, seq, ctx=None):
    intr = seq.intrinsics()
    return LocalMapper(intr, neighbor_count=g["neighbor_count"], match=MatchConfig(neighbor_count=g["neighbor_count"]),
                       fuse=FuseConfig(n1=g["n1"], n2=g["n2"]), ctx=ctx,
                       store=store_for(g["keyframes"], seq.config.features_per_kf + 64))


def ledger_matches(dev: dict, want: dict) -> bool:
    small = want["small_transfer_bytes_by_stage"]
    return (dev["persistent_bytes_up"] == want["persistent_bytes_up"] and dev["naive_bytes_up"] == want["naive_bytes_up"]
            and dev["small_bytes_fusion"] == small.get("fusion", 0)
            and dev["small_bytes_triangulation"] == small.get("triangulation", 0)
            and dev["small_transfer_events"] == want["small_transfer_events"] and dev["evictions"] == want["evictions"])


def check_step(name, dev, want, kf_id):
    st = dev.stats
    assert (st.created, st.conflicts, st.degenerate) == (want["created"], want["conflicts"], want["degenerate"]), \
        (name, kf_id)
    assert st.gate_failures == want["gates"], (name, kf_id)
    assert dev.fused == want["fusion"], (name, kf_id)
    assert dev.culled == want["culled"], (name, kf_id)
    assert dev.snapshot(with_covis=False).structural_digest() == want["digest"], (name, kf_id)
    assert ledger_matches(dev.ledger(), want["ledger"]), (name, kf_id, dev.ledger(), want["ledger"])


def check_positions(dev, pos):
    snap = dev.snapshot(with_covis=False)
    ids = np.flatnonzero(snap.alive)
    assert ids.tolist() == pos["ids"].tolist()
    if len(ids):
        got, want = snap.pos[ids], pos["pos"]
        rel = np.linalg.norm(got - want, axis=1) / np.maximum(np.linalg.norm(want, axis=1), 1e-12)
        assert float(rel.max()) <= POS_RTOL
        return float(rel.max())
    return 0.0


def seq_of(g):
    return W.generate_sequence(W.WorldConfig(**g["config"]))


@pytest.mark.parametrize("name", [n for n in GOLD if not n.startswith("c5_")])
def test_steady_state_matches_reference_every_keyframe(name):
    g, pos = load(name)
    seq = seq_of(g)
    intr = seq.intrinsics()
    dev = mapper_for(g, seq)
    border = np.zeros(4, np.int64)
    for rec, want in zip(seq.records[:g["keyframes"]], g["steps"]):
        assert int(rec.kf_id) == want["kf"]
        r = dev.process(device_kf(rec, intr))
        del r
        check_step(name, dev, want, int(rec.kf_id))
    tot = dev.totals()
    border += np.array(list(tot.borderline), np.int64)
    worst = check_positions(dev, pos)
    print(f"{name}: {g['keyframes']} keyframes bit-equal to the reference; worst position rel {worst:.2e}; "
          f"borderline compares (epi, gates, fusion, rint) {border.tolist()}")


def test_streaming_async_c2_matches_reference_final_state():
    """The streaming path bench.py's e2e times: keyframe k+1 staged (on the staging stream)
    while step k runs, every step asynchronous, nothing read back until the end. Running
    counters, the structural digest and the positions after the last keyframe equal the
    reference's (a half-staged keyframe seen by any step would change them)."""
    g, pos = load("c2")
    seq = seq_of(g)
    intr = seq.intrinsics()
    dev = mapper_for(g, seq)
    recs = seq.records[:g["keyframes"]]
    for rec in recs:
        dev.stage(device_kf(rec, intr))
        dev.step(int(rec.kf_id), sync=False)
    tot = dev.totals()
    want = g["steps"][len(recs) - 1]
    assert (tot.created, tot.conflicts, tot.degenerate) == (want["created"], want["conflicts"], want["degenerate"])
    assert {"merged": tot.merged, "observations_added": tot.observations_added, "stale": tot.stale} == want["fusion"]
    assert tot.culled == want["culled"]
    assert dev.snapshot(with_covis=False).structural_digest() == want["digest"]
    check_positions(dev, pos)


def test_c5_sessions_batched_match_reference_every_keyframe():
    names = [n for n in GOLD if n.startswith("c5_")]
    if not names:
        pytest.skip("no C5 goldens")
    golds = [load(n) for n in names]
    seqs = [seq_of(g) for g, _ in golds]
    devs = [mapper_for(g, s) for (g, _), s in zip(golds, seqs)]
    batch = SessionBatch(devs)
    n_kf = min(g["keyframes"] for g, _ in golds)
    for k in range(n_kf):
        for d, s in zip(devs, seqs):
            d.stage(device_kf(s.records[k], s.intrinsics()))
        batch.step([int(s.records[k].kf_id) for s in seqs])
        for name, d, (g, _) in zip(names, devs, golds):
            check_step(name, d, g["steps"][k], k)
    for d, (g, pos) in zip(devs, golds):
        if n_kf == g["keyframes"]:
            check_positions(d, pos)


SNAPS = sorted(glob.glob(os.path.join(HERE, "golden", "snap_*_kf*.npz")))


@pytest.mark.parametrize("path", [p for p in SNAPS
                                  if os.path.basename(p).split("_kf")[0][len("snap_"):] in GOLD])
def test_from_reference_state_every_keyframe(path):
    """Per-step parity from the REAL reference's map state: import its map after K
    keyframes (lm_import_snapshot of tests/golden/snap_<name>_kf<K>.npz, written by
    make_snapshot.py), then step K.. natively; every keyframe's digest, counter deltas and
    ledger must equal the reference's. No position drift from earlier keyframes can
    cascade here: the device starts from the reference's own LAPACK positions."""
    base = os.path.basename(path)
    name, k0 = base[len("snap_"):].split("_kf")
    k0 = int(k0[:-len(".npz")])
    g, pos = load(name)
    seq = seq_of(g)
    intr = seq.intrinsics()
    recs = seq.records
    snap = dict(np.load(path))
    snap["cam"] = np.array([[intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height]] * k0)
    snap["u"] = np.concatenate([r.kp_u for r in recs[:k0]])
    snap["v"] = np.concatenate([r.kp_v for r in recs[:k0]])
    snap["level"] = np.concatenate([r.kp_level for r in recs[:k0]])
    snap["desc"] = np.concatenate([r.descriptors for r in recs[:k0]])
    snap["rep"] = np.zeros((len(snap["pos"]), 32), np.uint8)
    dev = mapper_for(g, seq)
    dev.import_state(snap, processed=int(snap["processed"]))
    prev = g["steps"][k0 - 1]
    assert dev.snapshot(with_covis=False).structural_digest() == prev["digest"]
    assert ledger_matches(dev.ledger(), prev["ledger"])
    for k in range(k0, g["keyframes"]):
        dev.process(device_kf(recs[k], intr))
        want = g["steps"][k]
        st = dev.stats
        assert st.created == want["created"] - prev["created"], k
        assert st.conflicts == want["conflicts"] - prev["conflicts"], k
        assert {r: n for r, n in st.gate_failures.items()} == {
            r: n - prev["gates"].get(r, 0) for r, n in want["gates"].items() if n - prev["gates"].get(r, 0)}, k
        assert {f: dev.fused[f] for f in dev.fused} == {f: want["fusion"][f] - prev["fusion"][f] for f in dev.fused}, k
        assert dev.culled == want["culled"] - prev["culled"], k
        assert dev.snapshot(with_covis=False).structural_digest() == want["digest"], k
        assert ledger_matches(dev.ledger(), want["ledger"]), k
    if g["keyframes"] == len(g["steps"]):
        check_positions(dev, pos)
