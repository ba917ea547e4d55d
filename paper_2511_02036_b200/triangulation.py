"""CreateNewMapPoints drop-in (reference: pkg/src/localmap/triangulation.py).

Same names, signatures, return types and error behaviour as the reference module; the
work runs in the sm_100a kernels k_select / k_prep / k_match / k_tri / k_commit
(csrc/lm_kernels.cuh). ``engine`` is the reference's plugin point (triangulation.py:108-113):
"b200" selects this implementation; "reference" and "batch" are accepted as aliases
because all engines are byte-identical by contract and this package ships exactly one.
Anything else raises ValueError like the reference.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import ptr
from .config import GateConfig, MatchConfig
from .mapmodel import UNBOUND, KeyFrame, MapModel, stage_keyframe, create_map
from .config import MapConfig, StoreConfig

ENGINES = ("b200", "reference", "batch")


@dataclass(frozen=True)
class MatchCandidate:
    neighbor_kf_id: int
    kp_index_current: int
    kp_index_neighbor: int
    distance: int


@dataclass
class CreationStats:
    """Per-stage outcome counters; failures are values, not errors (triangulation.py:49-60)."""

    created: int = 0
    conflicts: int = 0
    degenerate: int = 0
    gate_failures: dict = field(default_factory=dict)
    degenerate_neighbors: list = field(default_factory=list)

    def count_gate(self, reason: str, n: int = 1):
        if n:
            self.gate_failures[reason] = self.gate_failures.get(reason, 0) + n

    def absorb(self, st: _lib.StepStats):
        absorb_stats(self, st)


def absorb_stats(stats, st: _lib.StepStats):
    """Add one device step's creation outcome to any CreationStats-shaped object (this
    package's or the reference's, triangulation.py:49-60)."""
    stats.created += st.created
    stats.conflicts += st.conflicts
    stats.degenerate += st.degenerate
    for reason, n in (("parallax", st.gate_parallax), ("positive-depth", st.gate_depth),
                      ("reprojection", st.gate_reprojection), ("scale", st.gate_scale)):
        if n:
            stats.gate_failures[reason] = stats.gate_failures.get(reason, 0) + n
    stats.degenerate_neighbors.extend(int(st.degenerate_neighbors[k]) for k in range(st.n_degenerate_neighbors))


def _check_engine(engine: str):
    if engine not in ENGINES:
        raise ValueError(f"unknown search engine {engine!r}")


def match_cfg_c(cfg: MatchConfig) -> _lib.MatchCfg:
    return _lib.MatchCfg(int(cfg.match_max_distance), float(cfg.chi2_epi), int(cfg.level_window))


def gate_cfg_c(cfg: GateConfig) -> _lib.GateCfg:
    return _lib.GateCfg(float(cfg.cos_parallax_max), float(cfg.chi2_mono), float(cfg.scale_ratio_slack))


class _Scratch:
    """Per-context scratch map for searches on keyframes that are not in a device map."""

    maps: dict = {}

    @classmethod
    def get(cls, ctx, kfs: list[KeyFrame]):
        k = kfs[0].intrinsics
        key = (id(ctx), k.num_levels, k.scale_factor)
        ent = cls.maps.get(key)
        need = sum(kf.num_keypoints for kf in kfs)
        maxkp = max(kf.num_keypoints for kf in kfs)
        if ent is None or ent["used_kf"] + len(kfs) > ent["kf_cap"] or ent["used_kp"] + need > ent["kp_cap"] \
                or maxkp > ent["kpkf"]:
            kpkf = max(4096, maxkp)
            store = StoreConfig(max_keyframes=256, max_keypoints=max(1 << 18, 8 * kpkf), max_keypoints_per_kf=kpkf,
                                max_points=16, obs_pool_entries=64)
            if ent is None:
                idx = create_map(ctx, k.num_levels, k.scale_factor, store, MapConfig())
            else:
                idx = ent["map"]
                ctx.call("lm_map_reset", idx)
            ent = {"map": idx, "kf_cap": store.max_keyframes, "kp_cap": store.max_keypoints, "kpkf": kpkf,
                   "used_kf": 0, "used_kp": 0, "next_id": 0}
            cls.maps[key] = ent
        ids = []
        for kf in kfs:
            fake = ent["next_id"]
            ent["next_id"] += 1
            ids.append(fake)
            tmp = KeyFrame(fake, kf.pose, kf.intrinsics, kf.kp_u, kf.kp_v, kf.kp_level, kf.descriptors)
            stage_keyframe(ctx, ent["map"], tmp, bindings=False)
            ent["used_kf"] += 1
            ent["used_kp"] += kf.num_keypoints
        return ent["map"], ids


def search_for_triangulation(current: KeyFrame, neighbor: KeyFrame, cfg: MatchConfig | None = None, *,
                             engine: str = "b200", pool=None, unbound_current: np.ndarray | None = None,
                             unbound_neighbor: np.ndarray | None = None) -> list[MatchCandidate]:
    """Best epipolar-consistent descriptor match in `neighbor` for each unbound current
    keypoint; one-to-one; sorted by current index (triangulation.py:80-114)."""
    _check_engine(engine)
    cfg = cfg or MatchConfig()
    ctx = _lib.Context.get(0)
    if unbound_current is None:
        unbound_current = current.mp_bindings == UNBOUND
    if unbound_neighbor is None:
        unbound_neighbor = neighbor.mp_bindings == UNBOUND
    mc = np.ascontiguousarray(unbound_current, dtype=np.uint8)
    mn = np.ascontiguousarray(unbound_neighbor, dtype=np.uint8)
    m, (ci, ni) = _Scratch.get(ctx, [current, neighbor])
    cap = max(current.num_keypoints, 1)
    out = (_lib.Candidate * cap)()
    n = C.c_int32()
    ctx.call("lm_search", m, ci, ni, C.byref(match_cfg_c(cfg)), ptr(mc, C.c_uint8), ptr(mn, C.c_uint8), out, cap,
             C.byref(n))
    return [MatchCandidate(int(neighbor.kf_id), out[k].kp_index_current, out[k].kp_index_neighbor, out[k].distance)
            for k in range(n.value)]


def create_map_points(model: MapModel, store, current_kf_id: int, neighbor_count: int,
                      match_cfg: MatchConfig | None = None, gate_cfg: GateConfig | None = None, *,
                      engine: str = "b200", pool=None, stats: CreationStats | None = None) -> list[int]:
    """Triangulate new map points against the top covisible neighbours (triangulation.py:195-300).

    Returns the new map point ids in creation order."""
    _check_engine(engine)
    match_cfg = match_cfg or MatchConfig()
    gate_cfg = gate_cfg or GateConfig()
    stats = stats if stats is not None else CreationStats()
    model._require_kf(current_kf_id)
    if neighbor_count <= 0:
        return []
    own = model._use_store(store)  # this map's DeviceStore: k_select accounts the neighbour access
    st = _lib.StepStats()
    model._call("lm_create_map_points", model.map, int(current_kf_id), int(neighbor_count),
                C.byref(match_cfg_c(match_cfg)), C.byref(gate_cfg_c(gate_cfg)), C.byref(st))
    nbrs = [int(st.neighbors[k]) for k in range(st.n_neighbors)]
    if not nbrs:
        return []
    if not own and store is not None:  # a foreign store keeps its own ledger (triangulation.py:232)
        store.record_neighbor_access("triangulation", nbrs)
    absorb_stats(stats, st)
    return list(range(int(st.first_new_id), int(st.first_new_id) + st.created))
