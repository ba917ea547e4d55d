"""Snapshot import: a reference map state (``localmap.mapmodel.MapModel`` + its
``DeviceStore`` + the pipeline's probation list) into a device map (lm_import_snapshot).

This is the SURVEY.md §5 checkpoint row: the reference has no map serialisation
(SPEC.md:273), so per-step parity from a reference state needs an importer. Duck-typed on
the reference's public attributes (``keyframes``, ``points``, ``store.ledger``,
``RecentPoint``), so any MapModel-shaped object works, including this package's own.

``state_arrays`` flattens a state to plain arrays (the form tests/golden stores, minus the
keypoints, which the workload generator reproduces); ``import_arrays`` loads such arrays.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import ptr

UNBOUND = -1


def state_arrays(ref_model, ref_store=None, recent=None, keypoints: bool = True) -> dict:
    kfs = list(ref_model.keyframes.values())
    a = {
        "kf_id": np.array([kf.kf_id for kf in kfs], np.int64),
        "kf_alive": np.array([bool(kf.alive) for kf in kfs], np.uint8),
        "kf_resident": np.array([bool(ref_store.is_resident(kf.kf_id)) if ref_store is not None else True
                                 for kf in kfs], np.uint8),
        "quat": np.array([np.asarray(kf.pose.quat, np.float64) for kf in kfs]).reshape(-1, 4),
        "trans": np.array([np.asarray(kf.pose.trans, np.float64) for kf in kfs]).reshape(-1, 3),
        "kp_n": np.array([kf.num_keypoints for kf in kfs], np.int32),
        "bindings": np.concatenate([np.where(kf.alive, np.asarray(kf.mp_bindings, np.int64), UNBOUND)
                                    for kf in kfs]) if kfs else np.zeros(0, np.int64),
    }
    if keypoints:
        a["cam"] = np.array([[kf.intrinsics.fx, kf.intrinsics.fy, kf.intrinsics.cx, kf.intrinsics.cy,
                              kf.intrinsics.width, kf.intrinsics.height] for kf in kfs], np.float64).reshape(-1, 6)
        a["u"] = np.concatenate([np.asarray(kf.kp_u, np.float64) for kf in kfs]) if kfs else np.zeros(0)
        a["v"] = np.concatenate([np.asarray(kf.kp_v, np.float64) for kf in kfs]) if kfs else np.zeros(0)
        a["level"] = np.concatenate([np.asarray(kf.kp_level, np.int64) for kf in kfs]) if kfs else np.zeros(0, np.int64)
        a["desc"] = np.concatenate([np.asarray(kf.descriptors, np.uint8) for kf in kfs]) if kfs else np.zeros((0, 32),
                                                                                                           np.uint8)
    pts = sorted(ref_model.points.values(), key=lambda p: p.mp_id)
    if [p.mp_id for p in pts] != list(range(len(pts))):
        raise ValueError("map point ids must be 0..n-1")
    a["pos"] = np.array([np.asarray(p.position, np.float64) for p in pts]).reshape(-1, 3)
    a["rep"] = np.array([np.asarray(p.rep_descriptor, np.uint8) for p in pts]).reshape(-1, 32)
    a["alive"] = np.array([bool(p.alive) for p in pts], np.uint8)
    a["found"] = np.array([p.found_count for p in pts], np.int32)
    a["visible"] = np.array([p.visible_count for p in pts], np.int32)
    a["first_kf"] = np.array([p.first_kf_id for p in pts], np.int64)
    recent = recent or []
    a["recent_id"] = np.array([r.mp_id for r in recent], np.int64)
    a["recent_born"] = np.array([r.created_at for r in recent], np.int32)
    lg = np.zeros(6, np.int64)
    if ref_store is not None:
        d = ref_store.ledger.as_dict()
        small = d["small_transfer_bytes_by_stage"]
        lg[:] = [d["persistent_bytes_up"], d["naive_bytes_up"], small.get("triangulation", 0), small.get("fusion", 0),
                 d["small_transfer_events"], d["evictions"]]
    a["ledger"] = lg
    return a


def import_arrays(model, a: dict):
    """Load state arrays (state_arrays' layout) into the empty device map of `model`."""
    keep = {}

    def arr(name, dtype, shape_tail=()):
        x = np.ascontiguousarray(a[name], dtype=dtype)
        keep[name] = x
        return x

    s = _lib.Snapshot()
    kf_id = arr("kf_id", np.int64)
    s.n_kf = len(kf_id)
    s.kf_id = ptr(kf_id, C.c_int64)
    s.kf_alive = ptr(arr("kf_alive", np.uint8), C.c_uint8)
    s.kf_resident = ptr(arr("kf_resident", np.uint8), C.c_uint8)
    s.quat = ptr(arr("quat", np.float64), C.c_double)
    s.trans = ptr(arr("trans", np.float64), C.c_double)
    s.cam = ptr(arr("cam", np.float64), C.c_double)
    s.kp_n = ptr(arr("kp_n", np.int32), C.c_int32)
    s.u = ptr(arr("u", np.float64), C.c_double)
    s.v = ptr(arr("v", np.float64), C.c_double)
    s.level = ptr(arr("level", np.int64), C.c_int64)
    s.desc = ptr(arr("desc", np.uint8), C.c_uint8)
    s.bindings = ptr(arr("bindings", np.int64), C.c_int64)
    pos = arr("pos", np.float64)
    s.n_points = len(pos)
    s.pos = ptr(pos, C.c_double)
    s.rep = ptr(arr("rep", np.uint8), C.c_uint8)
    s.alive = ptr(arr("alive", np.uint8), C.c_uint8)
    s.found = ptr(arr("found", np.int32), C.c_int32)
    s.visible = ptr(arr("visible", np.int32), C.c_int32)
    s.first_kf = ptr(arr("first_kf", np.int64), C.c_int64)
    rid = arr("recent_id", np.int64)
    s.n_recent = len(rid)
    s.recent_id = ptr(rid, C.c_int64)
    s.recent_born = ptr(arr("recent_born", np.int32), C.c_int32)
    lg = np.asarray(a["ledger"], np.int64)
    s.ledger = _lib.Ledger(*[int(x) for x in lg])
    model._call("lm_import_snapshot", model.map, C.byref(s))
    del keep


def import_reference(model, ref_model, ref_store=None, recent=None, keyframes=None):
    """Import a reference state into `model` (a paper_2511_02036_b200 MapModel). The
    keyframe objects are registered with the model (``keyframes`` overrides which objects
    represent them, e.g. this package's KeyFrame copies)."""
    a = state_arrays(ref_model, ref_store, recent)
    import_arrays(model, a)
    kfs = keyframes if keyframes is not None else list(ref_model.keyframes.values())
    from .mapmodel import _HOME
    import weakref

    for kf in kfs:
        model._kfs[kf.kf_id] = kf
        model._pose_ref[kf.kf_id] = kf.pose
        _HOME[id(kf)] = (weakref.ref(model), kf.kf_id)
    model.invalidate()
