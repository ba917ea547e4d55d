"""Binary keyframe ingest.

The reference moves keyframes as JSON: the service's ``KeyframePayload`` with hex
descriptors (``service/schemas.py:111-126``, consumed at ``service/app.py:197-226``) and
the JSONL sequence files (``synth.py:376-439``). Here a keyframe is one little-endian
"LMKF" v1 record (layout in ``include/lm_b200.h``: ``lm_kf_record_hdr``, then u, v, level,
descriptors, optional bindings) that ``lm_kf_stage_record`` validates and stages straight
into the device store, and a sequence is an "LMSQ" file of length-prefixed records.

``read_reference_jsonl`` restates the reference's ``read_sequence`` (synth.py:407-439) so a
reference sequence file converts to records without importing the reference.
"""

from __future__ import annotations

import ctypes as C
import json
import struct
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import Context, check
from .errors import InvalidArgumentError
from .geometry import CameraIntrinsics, SE3Pose
from .mapmodel import UNBOUND, KeyFrame

REC_MAGIC = 0x464B4D4C  # "LMKF"
REC_VERSION = 1
REC_BINDINGS = 1
HDR = struct.Struct("<IHHII qq 4d 3d 4d iiii d 2d")  # lm_kf_record_hdr, 160 bytes
assert HDR.size == 160
SEQ_MAGIC = b"LMSQ"
SEQ_VERSION = 1
REFERENCE_SEQUENCE_FORMAT = 1  # synth.SEQUENCE_FORMAT (synth.py:32)


def record_bytes(n: int, flags: int = 0) -> int:
    pad = (n + 7) & ~7
    return HDR.size + 16 * n + pad + 32 * n + (8 * n if flags & REC_BINDINGS else 0)


def pack_keyframe(kf: KeyFrame, frame_index: int | None = None) -> bytes:
    """One keyframe as an LMKF v1 record (bindings included when any slot is bound)."""
    n = kf.num_keypoints
    k = kf.intrinsics
    bind = None
    if kf.mp_bindings is not None and (np.asarray(kf.mp_bindings) != UNBOUND).any():
        bind = np.ascontiguousarray(kf.mp_bindings, dtype=np.int64)
    flags = REC_BINDINGS if bind is not None else 0
    lv = np.asarray(kf.kp_level)
    if n and (lv.min() < 0 or lv.max() > 255):
        raise InvalidArgumentError("keypoint level outside 0..255")
    q, t = np.asarray(kf.pose.quat, np.float64), np.asarray(kf.pose.trans, np.float64)
    fi = kf.frame_index if frame_index is None else frame_index
    parts = [HDR.pack(REC_MAGIC, REC_VERSION, flags, n, HDR.size, int(kf.kf_id), int(fi), *q.tolist(), *t.tolist(),
                      float(k.fx), float(k.fy), float(k.cx), float(k.cy), int(k.width), int(k.height),
                      int(k.num_levels), 0, float(k.scale_factor), 0.0, 0.0),
             np.ascontiguousarray(kf.kp_u, np.float64).tobytes(), np.ascontiguousarray(kf.kp_v, np.float64).tobytes()]
    lvb = np.zeros((n + 7) & ~7, np.uint8)
    lvb[:n] = lv.astype(np.uint8)
    parts += [lvb.tobytes(), np.ascontiguousarray(kf.descriptors, np.uint8).reshape(n, 32).tobytes()]
    if bind is not None:
        parts.append(bind.tobytes())
    out = b"".join(parts)
    assert len(out) == record_bytes(n, flags)
    return out


@dataclass
class RecordView:
    kf_id: int
    frame_index: int
    keyframe: KeyFrame


def unpack_keyframe(buf: bytes) -> RecordView:
    """Inverse of pack_keyframe (host-side checks mirror lm_kf_stage_record's)."""
    if len(buf) < HDR.size:
        raise InvalidArgumentError("record shorter than its header")
    (magic, ver, flags, n, hb, kf_id, fi, qx, qy, qz, qw, tx, ty, tz, fx, fy, cx, cy, w, h, nl, _pad, sf, _r0,
     _r1) = HDR.unpack_from(buf, 0)
    if magic != REC_MAGIC or ver != REC_VERSION or hb != HDR.size:
        raise InvalidArgumentError("not an LMKF v1 keyframe record")
    if flags & ~REC_BINDINGS or len(buf) != record_bytes(n, flags):
        raise InvalidArgumentError("record size does not match its keypoint count")
    o = HDR.size
    u = np.frombuffer(buf, np.float64, n, o).copy()
    o += 8 * n
    v = np.frombuffer(buf, np.float64, n, o).copy()
    o += 8 * n
    lv = np.frombuffer(buf, np.uint8, n, o).astype(np.int64)
    o += (n + 7) & ~7
    desc = np.frombuffer(buf, np.uint8, 32 * n, o).reshape(n, 32).copy()
    o += 32 * n
    cam = CameraIntrinsics(fx, fy, cx, cy, int(w), int(h), num_levels=int(nl), scale_factor=sf)
    kf = KeyFrame(int(kf_id), SE3Pose(np.array([qx, qy, qz, qw]), np.array([tx, ty, tz])), cam, u, v, lv, desc,
                  frame_index=int(fi))
    if flags & REC_BINDINGS:
        kf.mp_bindings = np.frombuffer(buf, np.int64, n, o).copy()
    return RecordView(int(kf_id), int(fi), kf)


def stage_record(ctx: Context, map_idx: int, record: bytes) -> int:
    """lm_kf_stage_record: validate + stage one record; returns its keyframe id."""
    out = C.c_int64()
    buf = C.create_string_buffer(record, len(record))
    check(ctx.lib.lm_kf_stage_record(ctx.h, map_idx, buf, len(record), C.byref(out)), ctx.h)
    return int(out.value)


def write_sequence_bin(path: str, records: list[bytes]):
    with open(path, "wb") as fh:
        fh.write(SEQ_MAGIC + struct.pack("<II", SEQ_VERSION, len(records)))
        for r in records:
            fh.write(struct.pack("<Q", len(r)))
            fh.write(r)


def read_sequence_bin(path: str) -> list[bytes]:
    with open(path, "rb") as fh:
        data = fh.read()
    if data[:4] != SEQ_MAGIC:
        raise InvalidArgumentError(f"{path} is not an LMSQ file")
    ver, count = struct.unpack_from("<II", data, 4)
    if ver != SEQ_VERSION:
        raise InvalidArgumentError(f"{path}: LMSQ version {ver}")
    o, out = 12, []
    for _ in range(count):
        (ln,) = struct.unpack_from("<Q", data, o)
        o += 8
        if o + ln > len(data):
            raise InvalidArgumentError(f"{path}: truncated record")
        out.append(data[o:o + ln])
        o += ln
    return out


def read_reference_jsonl(path: str):
    """The reference's sequence file (synth.write_sequence, synth.py:376-404) -> (config dict,
    list of (kf_id, frame_index, pose_init, kp_u, kp_v, kp_level, descriptors, pose_gt,
    landmark_ids)); a restatement of synth.read_sequence (synth.py:407-439)."""
    with open(path) as fh:
        header = json.loads(fh.readline())
        if header.get("type") != "header" or header.get("format") != REFERENCE_SEQUENCE_FORMAT:
            raise InvalidArgumentError(f"{path} is not a sequence file")
        rows = []
        for line in fh:
            if not line.strip():
                continue
            d = json.loads(line)
            desc = np.frombuffer(bytes.fromhex(d["descriptors"]), dtype=np.uint8).reshape(-1, 32).copy()
            pose = lambda p: SE3Pose(np.array(p["q"], np.float64), np.array(p["t"], np.float64))  # noqa: E731
            rows.append((int(d["kf_id"]), int(d["frame_index"]), pose(d["pose_init"]),
                         np.array(d["kp_u"], np.float64), np.array(d["kp_v"], np.float64),
                         np.array(d["kp_level"], np.int64), desc, pose(d["truth"]["pose_gt"]),
                         np.array(d["truth"]["landmark_ids"], np.int64)))
    return header["config"], rows


def intrinsics_of_config(cfg: dict) -> CameraIntrinsics:
    """The sequence camera (WorldConfig fields width/height/fx/fy/cx/cy/num_levels/scale_factor)."""
    return CameraIntrinsics(float(cfg["fx"]), float(cfg["fy"]), float(cfg["cx"]), float(cfg["cy"]),
                            int(cfg["width"]), int(cfg["height"]), num_levels=int(cfg["num_levels"]),
                            scale_factor=float(cfg["scale_factor"]))


def reference_jsonl_to_records(path: str) -> list[bytes]:
    cfg, rows = read_reference_jsonl(path)
    cam = intrinsics_of_config(cfg)
    return [pack_keyframe(KeyFrame(kid, pose, cam, u, v, lv, desc, frame_index=fi))
            for kid, fi, pose, u, v, lv, desc, _gt, _lm in rows]


__all__ = ["pack_keyframe", "unpack_keyframe", "stage_record", "write_sequence_bin", "read_sequence_bin",
           "read_reference_jsonl", "reference_jsonl_to_records", "record_bytes", "RecordView", "_lib"]
