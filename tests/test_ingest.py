"""Binary keyframe ingest: LMKF records and LMSQ files, and the
reference's own JSONL sequence format (tests/golden/orbit7_reference.jsonl, written by the
real reference's synth.write_sequence via tests/golden/make_jsonl.py) read without the
reference. CPU tests use the library's host entry point only; staging runs under -m gpu."""

from __future__ import annotations

import hashlib
import json
import os

import numpy as np
import pytest

from helpers import device_kf
from paper_2511_02036_b200 import _lib, ingest
from paper_2511_02036_b200 import workload as W
from paper_2511_02036_b200.errors import InvalidArgumentError

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "golden.json")))
JSONL = os.path.join(HERE, "golden", "orbit7_reference.jsonl")


def _seq():
    return W.generate_sequence(W.WorldConfig(**GOLD["workloads"]["orbit7"]["config"]))


def test_record_round_trip_and_size():
    s = _seq()
    intr = s.intrinsics()
    lib = _lib.load()
    for rec in s.records:
        kf = device_kf(rec, intr)
        buf = ingest.pack_keyframe(kf)
        assert len(buf) == ingest.record_bytes(kf.num_keypoints) == lib.lm_kf_record_bytes(kf.num_keypoints, 0)
        back = ingest.unpack_keyframe(buf).keyframe
        assert back.kf_id == kf.kf_id and back.frame_index == kf.frame_index
        for a in ("kp_u", "kp_v", "kp_level", "descriptors"):
            assert np.array_equal(getattr(back, a), getattr(kf, a)), a
        assert np.array_equal(back.pose.quat, kf.pose.quat) and np.array_equal(back.pose.trans, kf.pose.trans)
        assert back.intrinsics == kf.intrinsics


def test_record_with_bindings():
    s = _seq()
    kf = device_kf(s.records[2], s.intrinsics())
    kf.mp_bindings = np.full(kf.num_keypoints, -1, np.int64)
    kf.mp_bindings[[1, 5]] = [7, 9]
    buf = ingest.pack_keyframe(kf)
    assert len(buf) == _lib.load().lm_kf_record_bytes(kf.num_keypoints, ingest.REC_BINDINGS)
    assert np.array_equal(ingest.unpack_keyframe(buf).keyframe.mp_bindings, kf.mp_bindings)


def test_bad_records_rejected():
    s = _seq()
    buf = ingest.pack_keyframe(device_kf(s.records[0], s.intrinsics()))
    with pytest.raises(InvalidArgumentError):
        ingest.unpack_keyframe(b"XXXX" + buf[4:])
    with pytest.raises(InvalidArgumentError):
        ingest.unpack_keyframe(buf[:-1])
    with pytest.raises(InvalidArgumentError):
        ingest.unpack_keyframe(buf[:100])


def test_sequence_file_round_trip(tmp_path):
    s = _seq()
    recs = [ingest.pack_keyframe(device_kf(r, s.intrinsics())) for r in s.records]
    p = str(tmp_path / "seq.lmsq")
    ingest.write_sequence_bin(p, recs)
    assert ingest.read_sequence_bin(p) == recs


def test_reference_jsonl_matches_generator_and_golden_digest():
    """The reference's own file, read by the restated reader, is the generator's sequence
    (the golden digest pins both to the real reference)."""
    cfg, rows = ingest.read_reference_jsonl(JSONL)
    s = _seq()
    assert len(rows) == len(s.records)
    h = hashlib.sha256()
    for (kid, fi, pose, u, v, lv, desc, gt, lm), r in zip(rows, s.records):
        assert kid == r.kf_id and fi == r.frame_index
        for a in (pose.quat, pose.trans, gt.quat, gt.trans, u, v, lv, desc, lm):
            h.update(np.ascontiguousarray(a).tobytes())
    assert h.hexdigest() == GOLD["workloads"]["orbit7"]["digest"]
    recs = ingest.reference_jsonl_to_records(JSONL)
    want = [ingest.pack_keyframe(device_kf(r, s.intrinsics())) for r in s.records]
    assert recs == want


@pytest.mark.gpu
def test_staging_records_equals_staging_arrays():
    from paper_2511_02036_b200.session import LocalMapper, store_for

    s = _seq()
    intr = s.intrinsics()
    a = LocalMapper(intr, neighbor_count=10, store=store_for(len(s.records), 256))
    b = LocalMapper(intr, neighbor_count=10, store=store_for(len(s.records), 256))
    for rec in s.records:
        kf = device_kf(rec, intr)
        a.process(kf)
        kid = ingest.stage_record(b.ctx, b.map, ingest.pack_keyframe(kf))
        b.step(kid)
    sa, sb = a.snapshot(), b.snapshot()
    assert sa.structural_digest() == sb.structural_digest()
    assert np.array_equal(sa.pos, sb.pos)
    assert a.fused == b.fused


@pytest.mark.gpu
def test_stage_record_validation():
    from paper_2511_02036_b200.geometry import CameraIntrinsics
    from paper_2511_02036_b200.session import LocalMapper, store_for

    s = _seq()
    intr = s.intrinsics()
    m = LocalMapper(intr, neighbor_count=10, store=store_for(4, 256))
    kf = device_kf(s.records[0], intr)
    buf = ingest.pack_keyframe(kf)
    with pytest.raises(InvalidArgumentError):
        ingest.stage_record(m.ctx, m.map, b"XXXX" + buf[4:])
    with pytest.raises(InvalidArgumentError):
        ingest.stage_record(m.ctx, m.map, buf[:-8])
    other = CameraIntrinsics(intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height,
                             num_levels=intr.num_levels, scale_factor=1.3)
    kf2 = device_kf(s.records[1], other)
    with pytest.raises(InvalidArgumentError):
        ingest.stage_record(m.ctx, m.map, ingest.pack_keyframe(kf2))
    assert ingest.stage_record(m.ctx, m.map, buf) == kf.kf_id
