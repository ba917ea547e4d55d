"""Recent map-point culling drop-in (reference: pkg/src/localmap/culling.py:20-59).

``cull_recent_map_points(model, recent, current_index, cfg)`` with the reference's
signature and return value ``(removed ids, points still under probation)``, run by the
device cull (k_cull, csrc/lm_kernels.cuh) on a device-backed MapModel: the probation list
is loaded into the map, culled on the device and read back in one call
(lm_cull_recent_list); removed ids are the entries that were alive before and are dead
after, in probation-list order (the reference's kill order).

``cull_keyframes(model, store, candidate_ids, impl, cfg)`` (culling.py:127-154, §8(f) row 4):
the counter fast path on the device (lm_cull_keyframes): per candidate, in id order, the
per-level counter prefix of every bound live point (is_redundant_fast 95-117, identical to
the observation-list walk of is_redundant_baseline 60-92, so both ``impl`` values run it),
removal immediate, eviction from the store when resident.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from operator import attrgetter

import numpy as np

from . import _lib
from ._lib import ptr
from .config import CullConfig


@dataclass
class RecentPoint:
    mp_id: int
    created_at: int  # processed-keyframe counter at creation time


_MP_ID, _BORN = attrgetter("mp_id"), attrgetter("created_at")


def cull_recent_map_points(model, recent: list, current_index: int, cfg: CullConfig | None = None):
    cfg = cfg or CullConfig()
    if not recent:
        return [], []
    kind = type(recent[0])  # keep the caller's RecentPoint class (the reference's or this one)
    n = len(recent)
    ids = np.fromiter(map(_MP_ID, recent), np.int64, n)
    born = np.fromiter(map(_BORN, recent), np.int32, n)
    rem = np.zeros(n, np.int64)
    kid = np.zeros(n, np.int64)
    kborn = np.zeros(n, np.int32)
    nr, nk = C.c_int32(), C.c_int32()
    cc = _lib.CullCfg(float(cfg.found_ratio_min), int(cfg.probation_kfs), int(cfg.min_obs_graduate))
    model._call("lm_cull_recent_list", model.map, int(current_index), C.byref(cc), n, ptr(ids, C.c_int64),
                ptr(born, C.c_int32), ptr(rem, C.c_int64), C.byref(nr), ptr(kid, C.c_int64), ptr(kborn, C.c_int32),
                C.byref(nk))
    kid, kborn = kid[:nk.value], kborn[:nk.value]
    # the kept entries are a subsequence of the list (the device keeps list order): hand back
    # the caller's own entries, as the reference does (culling.py:58 keep.append(entry)); a
    # list whose kept ids cannot be located unambiguously (repeated ids) gets new entries
    at = np.flatnonzero(np.isin(ids, kid))
    if len(at) == len(kid) and np.array_equal(ids[at], kid) and np.array_equal(born[at], kborn):
        return rem[:nr.value].tolist(), [recent[i] for i in at.tolist()]
    return rem[:nr.value].tolist(), [kind(k, b) for k, b in zip(kid.tolist(), kborn.tolist())]


_IMPLS = ("baseline", "fast")


def _kc(cfg: CullConfig) -> _lib.KfCullCfg:
    return _lib.KfCullCfg(float(cfg.redundancy_ratio), int(cfg.min_redundant_observers),
                          int(cfg.scale_tolerance_levels))


def cull_keyframes(model, store, candidate_ids, impl: str = "baseline", cfg: CullConfig | None = None) -> list[int]:
    if impl not in _IMPLS:
        raise KeyError(impl)  # the reference indexes a dict of impls
    cfg = cfg or CullConfig()
    own = model._use_store(store)
    cand = np.ascontiguousarray(list(candidate_ids), dtype=np.int64)
    out = np.zeros(max(len(cand), 1), np.int64)
    n = C.c_int32()
    model._call("lm_cull_keyframes", model.map, ptr(cand, C.c_int64), len(cand), C.byref(_kc(cfg)),
                ptr(out, C.c_int64), C.byref(n))
    removed = out[:n.value].tolist()
    for k in removed:
        model._kfs[k].alive = False
        if not own and store is not None and store.is_resident(k):  # a foreign store evicts itself
            store.evict_keyframe(k)
    return removed


def _redundancy(model, kf_id: int, cfg: CullConfig | None):
    """(redundant, redundant_points, considered) of one keyframe from the device counters."""
    cfg = cfg or CullConfig()
    kf = model.keyframes[kf_id]
    b = np.asarray(kf.mp_bindings)
    bound = np.flatnonzero(b != -1)
    if len(bound) == 0:
        return False, 0, 0
    ids = b[bound]
    alive = np.array([model.points[int(m)].alive for m in ids], dtype=bool)
    bound, ids = bound[alive], ids[alive]
    considered = len(bound)
    if considered == 0:
        return False, 0, 0
    counters = np.stack([model.points[int(m)].scale_counts for m in ids])
    limits = np.minimum(np.asarray(kf.kp_level)[bound] + cfg.scale_tolerance_levels, model.num_levels - 1)
    others = np.cumsum(counters, axis=1)[np.arange(considered), limits] - 1
    red = int((others >= cfg.min_redundant_observers).sum())
    return red >= cfg.redundancy_ratio * considered, red, considered


def is_redundant_fast(model, kf_id: int, cfg: CullConfig | None = None):
    """culling.py:95-117 on a device-backed MapModel (reads one record per bound point)."""
    return _redundancy(model, kf_id, cfg)


def is_redundant_baseline(model, kf_id: int, cfg: CullConfig | None = None):
    """culling.py:60-92: identical output to the fast path (the reference's own contract)."""
    return _redundancy(model, kf_id, cfg)
