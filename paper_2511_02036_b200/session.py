"""Native local-mapping sessions: the whole per-keyframe hot path in one device call.

``LocalMapper`` owns one device map and runs, per keyframe, what the reference pipeline
does between upload and LBA (pipeline.py:152-195): insert, recent map-point cull,
CreateNewMapPoints, SearchAndFuse. LBA and keyframe culling are out of scope
(BASELINE.json north_star); the reference's throughput benches force-skip them too.
``SessionBatch`` advances many independent maps in lock-step with one batched launch
sequence per step (BASELINE config C5).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import Context, ptr
from .config import CullConfig, FuseConfig, GateConfig, MapConfig, MatchConfig, StoreConfig
from .fusion import fuse_cfg_c
from .geometry import CameraIntrinsics
from .mapmodel import KeyFrame, MapSnapshot, create_map, export_snapshot, stage_keyframe
from .triangulation import CreationStats, gate_cfg_c, match_cfg_c


def params_c(neighbor_count: int, match: MatchConfig, gates: GateConfig, fuse: FuseConfig, cull: CullConfig,
             processed: int, do_cull=True, do_create=True, do_fuse=True) -> _lib.StepParams:
    p = _lib.StepParams()
    p.neighbor_count = int(neighbor_count)
    p.do_cull, p.do_create, p.do_fuse = int(do_cull), int(do_create), int(do_fuse)
    p.processed_index = int(processed)
    p.match = match_cfg_c(match)
    p.gate = gate_cfg_c(gates)
    p.fuse = fuse_cfg_c(fuse)
    p.cull = _lib.CullCfg(float(cull.found_ratio_min), int(cull.probation_kfs), int(cull.min_obs_graduate))
    return p


def store_for(n_keyframes: int, kp_per_kf: int, points: int | None = None) -> StoreConfig:
    """Arena sizes for a session of n keyframes with at most kp_per_kf keypoints each."""
    kp_per_kf = max(64, int(kp_per_kf))
    pts = points or max(1 << 14, n_keyframes * kp_per_kf)
    return StoreConfig(capacity=max(4096, n_keyframes + 8), max_keyframes=max(16, n_keyframes + 8),
                       max_keypoints=max(1 << 12, (n_keyframes + 8) * kp_per_kf), max_keypoints_per_kf=kp_per_kf,
                       max_points=pts, obs_pool_entries=max(1 << 16, 16 * pts))


@dataclass
class StepResult:
    kf_id: int
    created: int
    first_new_id: int
    conflicts: int
    degenerate: int
    merged: int
    observations_added: int
    stale: int
    culled: int
    n_neighbors: int
    n_targets: int


def _result(kf_id, st: _lib.StepStats) -> StepResult:
    return StepResult(kf_id, st.created, st.first_new_id, st.conflicts, st.degenerate, st.merged,
                      st.observations_added, st.stale, st.culled, st.n_neighbors, st.n_targets)


class LocalMapper:
    """One device-resident map processed keyframe by keyframe."""

    def __init__(self, cam: CameraIntrinsics, neighbor_count: int = 10, match: MatchConfig | None = None,
                 gates: GateConfig | None = None, fuse: FuseConfig | None = None, cull: CullConfig | None = None,
                 store: StoreConfig | None = None, map_config: MapConfig | None = None, device: int = 0,
                 ctx: Context | None = None):
        self.ctx = ctx or Context.get(device)
        self.cam = cam
        self.neighbor_count = neighbor_count
        self.match, self.gates = match or MatchConfig(), gates or GateConfig()
        self.fuse, self.cull = fuse or FuseConfig(), cull or CullConfig()
        self.store = store or StoreConfig()
        self.map = create_map(self.ctx, cam.num_levels, cam.scale_factor, self.store, map_config or MapConfig())
        self.processed = 0
        self.stats = CreationStats()
        self.fused = {"merged": 0, "observations_added": 0, "stale": 0}
        self.culled = 0

    def _call(self, name, *args):
        self.ctx.call(name, *args)

    def close(self):
        """Free the device map (lm_map_destroy)."""
        if self.map is not None and self.ctx.h:
            self.ctx.call("lm_map_destroy", self.map)
        self.map = None

    def import_state(self, arrays: dict, processed: int = 0):
        """Start from an imported map state (snapshot.import_arrays layout, e.g. a reference
        MapModel after k keyframes): the map is reset first; `processed` is the pipeline's
        keyframe counter at that point (probation ages)."""
        from .snapshot import import_arrays

        self.reset()
        import_arrays(self, arrays)
        self.processed = int(processed)

    def reset(self):
        self.ctx.call("lm_map_reset", self.map)
        self.processed = 0
        self.stats = CreationStats()
        self.fused = {"merged": 0, "observations_added": 0, "stale": 0}
        self.culled = 0

    def stage(self, kf: KeyFrame):
        stage_keyframe(self.ctx, self.map, kf)

    def params(self) -> _lib.StepParams:
        return params_c(self.neighbor_count, self.match, self.gates, self.fuse, self.cull, self.processed)

    def step(self, kf_id: int, sync: bool = True) -> StepResult | None:
        """insert (if staged) -> cull -> create -> fuse for keyframe kf_id."""
        p = self.params()
        if sync:
            st = _lib.StepStats()
            self.ctx.call("lm_step", self.map, int(kf_id), C.byref(p), C.byref(st))
            self._absorb(st)
        else:
            maps = (C.c_int32 * 1)(self.map)
            ids = (C.c_int64 * 1)(int(kf_id))
            self.ctx.call("lm_step_batch", 1, maps, ids, C.byref(p), None)
        self.processed += 1
        return _result(kf_id, st) if sync else None

    def _absorb(self, st):
        self.stats.absorb(st)
        for k in self.fused:
            self.fused[k] += getattr(st, k)
        self.culled += st.culled

    def process(self, kf: KeyFrame) -> StepResult:
        self.stage(kf)
        return self.step(kf.kf_id)

    def synchronize(self):
        self.ctx.call("lm_synchronize")

    def snapshot(self, with_covis: bool = True) -> MapSnapshot:
        return export_snapshot(self.ctx, self.map, with_covis)

    def totals(self) -> _lib.StepStats:
        """Running totals on the device since creation / reset / rewind (lm_totals_fetch);
        first_new_id holds the number of steps accumulated. Covers async steps too."""
        st = _lib.StepStats()
        self.ctx.call("lm_totals_fetch", self.map, C.byref(st))
        if st.error:
            _lib.check(int(st.error))
        return st

    def ledger(self) -> dict:
        lg = _lib.Ledger()
        self.ctx.call("lm_ledger", self.map, C.byref(lg))
        return {f: getattr(lg, f) for f, _ in _lib.Ledger._fields_}

    def recent(self) -> list[tuple[int, int]]:
        cap = 1 << 20
        ids = np.zeros(cap, np.int64)
        born = np.zeros(cap, np.int32)
        n = C.c_int32()
        self.ctx.call("lm_recent_export", self.map, ptr(ids, C.c_int64), ptr(born, C.c_int32), cap, C.byref(n))
        return list(zip(ids[:n.value].tolist(), born[:n.value].tolist()))


class SessionBatch:
    """Independent maps (same context) advanced in lock-step, one batched launch per step."""

    def __init__(self, mappers: list[LocalMapper]):
        if len({id(m.ctx) for m in mappers}) != 1:
            raise ValueError("all sessions of a batch must share one context")
        if len({m.map for m in mappers}) != len(mappers):
            raise ValueError("a map may appear only once in a batch")
        self.mappers = mappers
        self.ctx = mappers[0].ctx
        self._maps = (C.c_int32 * len(mappers))(*[m.map for m in mappers])

    def step(self, kf_ids: list[int], sync: bool = True):
        n = len(self.mappers)
        params = (_lib.StepParams * n)(*[m.params() for m in self.mappers])
        ids = (C.c_int64 * n)(*[int(k) for k in kf_ids])
        out = (_lib.StepStats * n)() if sync else None
        self.ctx.call("lm_step_batch", n, self._maps, ids, params, out)
        for m in self.mappers:
            m.processed += 1
        if sync:
            for m, st in zip(self.mappers, out):
                m._absorb(st)
            return [_result(k, st) for k, st in zip(kf_ids, out)]
        return None
