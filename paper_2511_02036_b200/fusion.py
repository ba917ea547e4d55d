"""SearchAndFuse drop-in (reference: pkg/src/localmap/fusion.py).

Same names, dataclasses, constants and signatures as the reference module. The gather
(projection, gates, grid-cell window search, best-distance pick, action build) and the
ordered apply run in k_fuse / k_op (csrc/lm_kernels.cuh); ``engine`` follows the same
alias rule as triangulation.py.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import ACT_ADD, ACT_MERGE, ptr
from .config import FuseConfig
from .mapmodel import MapModel
from .triangulation import ENGINES

MERGE = "merge"
ADD_OBSERVATION = "add-observation"


@dataclass(frozen=True)
class FuseAction:
    target_kf_id: int
    mp_id_projected: int
    kp_index_hit: int
    existing_mp_id: int | None
    kind: str


def _check_engine(engine: str):
    if engine not in ENGINES:
        raise ValueError(f"unknown fuse engine {engine!r}")


def fuse_cfg_c(cfg: FuseConfig) -> _lib.FuseCfg:
    return _lib.FuseCfg(int(cfg.match_max_distance), float(cfg.fuse_radius), float(cfg.min_view_cos),
                        float(cfg.dist_band_slack), int(cfg.level_window), int(cfg.n1), int(cfg.n2))


def collect_fusion_targets(model: MapModel, current_kf_id: int, n1: int, n2: int) -> list[int]:
    """First-order neighbours by weight, then up to n2 unseen second-order ones each (fusion.py:38-54)."""
    model._require_kf(current_kf_id)
    buf = np.zeros(_lib.MAX_TARGETS, np.int64)
    n = C.c_int32()
    model.ctx.call("lm_fusion_targets", model.map, int(current_kf_id), int(n1), int(n2), ptr(buf, C.c_int64),
                   len(buf), C.byref(n))
    return [int(x) for x in buf[:n.value]]


def fuse_pass(model: MapModel, point_ids: list[int], target_kf_id: int, cfg: FuseConfig | None = None, *,
              engine: str = "b200", pool=None) -> tuple[list[FuseAction], list[int]]:
    """Project each live point into the target and pick the best hit in its window (fusion.py:132-175)."""
    _check_engine(engine)
    cfg = cfg or FuseConfig()
    model._require_kf(target_kf_id)
    if not point_ids:
        return [], []
    ids = np.ascontiguousarray(point_ids, dtype=np.int64)
    n = len(ids)
    acts = (_lib.FuseActionC * n)()
    vis = np.zeros(n, np.int64)
    na, nv = C.c_int32(), C.c_int32()
    model.ctx.call("lm_fuse_pass", model.map, ptr(ids, C.c_int64), n, int(target_kf_id),
                   C.byref(fuse_cfg_c(cfg)), acts, n, C.byref(na), ptr(vis, C.c_int64), C.byref(nv))
    out = []
    for k in range(na.value):
        a = acts[k]
        kind = MERGE if a.kind == ACT_MERGE else ADD_OBSERVATION
        out.append(FuseAction(int(a.target_kf_id), int(a.mp_id_projected), int(a.kp_index_hit),
                              int(a.existing_mp_id) if a.kind == ACT_MERGE else None, kind))
    return out, [int(x) for x in vis[:nv.value]]


def apply_fusion(model: MapModel, actions: list[FuseAction]) -> dict[str, int]:
    """Apply gathered actions in list order; stale ones are skipped and counted (fusion.py:249-292)."""
    counts = {"merged": 0, "observations_added": 0, "stale": 0}
    if not actions:
        return counts
    arr = (_lib.FuseActionC * len(actions))()
    for k, a in enumerate(actions):
        arr[k].target_kf_id = int(a.target_kf_id)
        arr[k].mp_id_projected = int(a.mp_id_projected)
        arr[k].kp_index_hit = int(a.kp_index_hit)
        arr[k].kind = ACT_MERGE if a.kind == MERGE else ACT_ADD
        arr[k].existing_mp_id = -1 if a.existing_mp_id is None else int(a.existing_mp_id)
    c = np.zeros(3, np.int32)
    model._call("lm_apply_fusion", model.map, arr, len(actions), ptr(c, C.c_int32))
    counts["merged"], counts["observations_added"], counts["stale"] = int(c[0]), int(c[1]), int(c[2])
    return counts


def run_fusion(model: MapModel, store, current_kf_id: int, cfg: FuseConfig | None = None, *,
               engine: str = "b200", pool=None) -> dict[str, int]:
    """Forward pass (current keyframe's points into every target), then reverse (fusion.py:307-347).

    With this map's DeviceStore the kernels keep the ledger (neighbour access, one small
    transfer per pass). A foreign store (e.g. the reference's DeviceStore) gets the same
    calls the reference makes: record_neighbor_access("fusion", targets), then one
    record_small_transfer("fusion", len(points) * its map_point_record_bytes) per pass, read
    back from the device's per-pass log."""
    _check_engine(engine)
    cfg = cfg or FuseConfig()
    model._require_kf(current_kf_id)
    own = model._use_store(store)
    foreign = not own and store is not None
    if foreign:
        targets = collect_fusion_targets(model, current_kf_id, cfg.n1, cfg.n2)
        if not targets:
            return {"merged": 0, "observations_added": 0, "stale": 0}
        store.record_neighbor_access("fusion", targets)
        before = _lib.Ledger()
        model.ctx.call("lm_ledger", model.map, C.byref(before))
    st = _lib.StepStats()
    model._call("lm_run_fusion", model.map, int(current_kf_id), C.byref(fuse_cfg_c(cfg)), C.byref(st))
    if foreign:
        after = _lib.Ledger()
        model.ctx.call("lm_ledger", model.map, C.byref(after))
        n = int(after.small_transfer_events - before.small_transfer_events)
        log = np.zeros(max(n, 1), np.int64)
        got = C.c_int32()
        model.ctx.call("lm_ledger_log", model.map, int(before.small_transfer_events), ptr(log, C.c_int64), n,
                       C.byref(got))
        per_point = model.store_config.map_point_record_bytes
        for b in log[:got.value]:
            store.record_small_transfer("fusion", int(b) // per_point * store.config.map_point_record_bytes)
    return {"merged": st.merged, "observations_added": st.observations_added, "stale": st.stale}
