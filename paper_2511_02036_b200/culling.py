"""Recent map-point culling drop-in (reference: pkg/src/localmap/culling.py:20-59).

``cull_recent_map_points(model, recent, current_index, cfg)`` with the reference's
signature and return value ``(removed ids, points still under probation)``, run by the
device cull (k_cull, csrc/lm_kernels.cuh) on a device-backed MapModel: the probation list
is loaded into the map (lm_recent_import), culled on the device (lm_cull_recent) and read
back (lm_recent_export); removed ids are the entries that were alive before and are dead
after, in probation-list order (the reference's kill order). Keyframe culling
(culling.py:62-154) is out of scope (BASELINE.json north_star).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import ptr
from .config import CullConfig


@dataclass
class RecentPoint:
    mp_id: int
    created_at: int  # processed-keyframe counter at creation time


def _alive(model, ids: np.ndarray) -> np.ndarray:
    out = np.zeros(max(len(ids), 1), np.uint8)
    if len(ids):
        model.ctx.call("lm_mp_alive", model.map, len(ids), ptr(ids, C.c_int64), ptr(out, C.c_uint8))
    return out[:len(ids)].astype(bool)


def cull_recent_map_points(model, recent: list, current_index: int, cfg: CullConfig | None = None):
    cfg = cfg or CullConfig()
    if not recent:
        return [], []
    kind = type(recent[0])  # keep the caller's RecentPoint class (the reference's or this one)
    ids = np.array([r.mp_id for r in recent], np.int64)
    born = np.array([r.created_at for r in recent], np.int32)
    before = _alive(model, ids)
    model._call("lm_recent_import", model.map, ptr(ids, C.c_int64), ptr(born, C.c_int32), len(ids))
    culled = C.c_int32()
    cc = _lib.CullCfg(float(cfg.found_ratio_min), int(cfg.probation_kfs), int(cfg.min_obs_graduate))
    model._call("lm_cull_recent", model.map, int(current_index), C.byref(cc), C.byref(culled))
    cap = len(ids)
    kid = np.zeros(max(cap, 1), np.int64)
    kborn = np.zeros(max(cap, 1), np.int32)
    n = C.c_int32()
    model.ctx.call("lm_recent_export", model.map, ptr(kid, C.c_int64), ptr(kborn, C.c_int32), cap, C.byref(n))
    after = _alive(model, ids)
    removed = [int(i) for i, b, a in zip(ids, before, after) if b and not a]
    keep = [kind(int(kid[k]), int(kborn[k])) for k in range(n.value)]
    return removed, keep
