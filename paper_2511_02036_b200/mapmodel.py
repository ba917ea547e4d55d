"""Device-backed map with the reference's MapModel interface, and the DeviceStore /
TransferLedger of the persistent keyframe store as views of the device ledger.

The state lives on the GPU (csrc/lm_map.cuh); this module is the host handle. Every read
costs O(what it returns), never a whole-map export, except the reads that are O(map) in the
reference too (``live_points``, ``counter_matrix``, ``audit``, iterating ``points``):
  * ``keyframes[k]`` refreshes that keyframe's ``mp_bindings`` (one D2H of its slots) only
    when the map changed since it was last read; keyframe liveness is tracked host-side;
  * ``points[i]`` / ``points.get(i)`` export one point record (lm_mp_get), cached until the
    next mutation;
  * ``graph`` reads one covisibility row (lm_covis_row); ``bound_points_of`` is a device
    compaction (lm_bound_points).
Mutations are single-op kernels that run the same device code as the hot-path stages.
Mirrors pkg/src/localmap/mapmodel.py (KeyFrame 24-62, MapPoint 65-77, CovisibilityGraph
80-110, MapModel 113-353) and devicestore.py (TransferLedger 25-48, DeviceStore 51-109).
"""

from __future__ import annotations

import ctypes as C
import weakref
from collections.abc import Mapping
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import Context, check, ptr
from .config import MapConfig, StoreConfig
from .errors import InvalidArgumentError, InvalidStateError, StoreCapacityError
from .geometry import DESCRIPTOR_BYTES, CameraIntrinsics, SE3Pose

UNBOUND = -1


@dataclass
class KeyFrame:
    """A retained frame: pose, camera, pyramid keypoints, descriptors, slot bindings."""

    kf_id: int
    pose: SE3Pose
    intrinsics: CameraIntrinsics
    kp_u: np.ndarray
    kp_v: np.ndarray
    kp_level: np.ndarray
    descriptors: np.ndarray
    frame_index: int = 0
    alive: bool = True
    mp_bindings: np.ndarray = None

    def __post_init__(self):
        self.kp_u = np.ascontiguousarray(self.kp_u, dtype=np.float64)
        self.kp_v = np.ascontiguousarray(self.kp_v, dtype=np.float64)
        self.kp_level = np.ascontiguousarray(self.kp_level, dtype=np.int64)
        self.descriptors = np.ascontiguousarray(self.descriptors, dtype=np.uint8)
        n = len(self.kp_u)
        if not (len(self.kp_v) == len(self.kp_level) == n and self.descriptors.shape == (n, DESCRIPTOR_BYTES)):
            raise InvalidArgumentError("keypoint arrays and descriptors must have matching lengths")
        if n and (self.kp_level.min() < 0 or self.kp_level.max() >= self.intrinsics.num_levels):
            raise InvalidArgumentError("keypoint level outside pyramid")
        if self.mp_bindings is None:
            self.mp_bindings = np.full(n, UNBOUND, dtype=np.int64)
        else:
            self.mp_bindings = np.asarray(self.mp_bindings, dtype=np.int64)
            if self.mp_bindings.shape != (n,):
                raise InvalidArgumentError("mp_bindings length mismatch")

    @property
    def num_keypoints(self) -> int:
        return len(self.kp_u)


@dataclass
class MapPoint:
    """Snapshot of one device map point. Assigning ``position``, ``found_count`` or
    ``visible_count`` on a point read from a MapModel writes through to the device (batched,
    before the model's next device call): the reference's LBA writes positions back this way
    (localba.py:573-574)."""

    mp_id: int
    position: np.ndarray
    rep_descriptor: np.ndarray
    first_kf_id: int
    observations: dict = field(default_factory=dict)
    found_count: int = 1
    visible_count: int = 1
    alive: bool = True
    scale_counts: np.ndarray = None

    def __setattr__(self, name, value):
        object.__setattr__(self, name, value)
        m = self.__dict__.get("_model")
        if m is not None and name in _WRITE_THROUGH:
            m._pending[self.mp_id] = self


_WRITE_THROUGH = ("position", "found_count", "visible_count")


def stage_keyframe(ctx: Context, map_idx: int, kf: KeyFrame, bindings: bool = True):
    """Copy a keyframe into a device map's pool (lm_kf_stage)."""
    q = np.ascontiguousarray(kf.pose.quat, dtype=np.float64)
    t = np.ascontiguousarray(kf.pose.trans, dtype=np.float64)
    k = kf.intrinsics
    cam = np.array([k.fx, k.fy, k.cx, k.cy, k.width, k.height], dtype=np.float64)
    b = None
    if bindings and kf.mp_bindings is not None and (kf.mp_bindings != UNBOUND).any():
        b = np.ascontiguousarray(kf.mp_bindings, dtype=np.int64)
    lib = ctx.lib
    check(lib.lm_kf_stage(ctx.h, map_idx, int(kf.kf_id), ptr(q, C.c_double), ptr(t, C.c_double),
                          ptr(cam, C.c_double), kf.num_keypoints, ptr(kf.kp_u, C.c_double),
                          ptr(kf.kp_v, C.c_double), ptr(kf.kp_level, C.c_int64),
                          ptr(kf.descriptors, C.c_uint8), ptr(b, C.c_int64) if b is not None else None), ctx.h)


def map_caps(num_levels: int, scale_factor: float, store: StoreConfig, cfg: MapConfig) -> _lib.MapCaps:
    c = _lib.MapCaps()
    c.max_keyframes = store.max_keyframes
    c.max_keypoints = store.max_keypoints
    c.max_keypoints_per_kf = store.max_keypoints_per_kf
    c.max_points = store.max_points
    c.obs_pool_entries = store.obs_pool_entries
    c.num_levels = num_levels
    c.scale_factor = scale_factor
    c.min_covis_weight = cfg.min_covis_weight
    c.min_obs_keep = cfg.min_obs_keep
    c.keypoint_record_bytes = store.keypoint_record_bytes
    c.descriptor_bytes = store.descriptor_bytes
    c.map_point_record_bytes = store.map_point_record_bytes
    c.store_capacity = store.capacity
    return c


@dataclass
class MapSnapshot:
    """Exported device state, in the reference's terms (ids, bindings, observations)."""

    kf_ids: np.ndarray          # per slot
    kf_state: np.ndarray        # 1 staged, 2 live, 3 dead
    kp_off: np.ndarray
    kp_n: np.ndarray
    bindings: np.ndarray        # whole keypoint pool
    pos: np.ndarray             # [n_points, 3]
    rep: np.ndarray             # [n_points, 32]
    alive: np.ndarray
    found: np.ndarray
    visible: np.ndarray
    nobs: np.ndarray
    counts: np.ndarray          # [n_points, L]
    obs_kf: np.ndarray
    obs_kp: np.ndarray
    covis: np.ndarray | None    # [kf_cap, kf_cap] by slot

    def slot_of(self) -> dict:
        return {int(k): s for s, k in enumerate(self.kf_ids)}

    def kf_bindings(self, slot: int) -> np.ndarray:
        o, n = int(self.kp_off[slot]), int(self.kp_n[slot])
        return self.bindings[o:o + n].astype(np.int64)

    def observations(self) -> list[dict]:
        out, w = [], 0
        for i in range(len(self.nobs)):
            n = int(self.nobs[i])
            out.append({int(self.obs_kf[w + k]): int(self.obs_kp[w + k]) for k in range(n)})
            w += n
        return out

    def structural_digest(self) -> str:
        """Same digest as oracle.lm_oracle.structural_digest (everything but positions)."""
        import hashlib

        h = hashlib.sha256()
        live = sorted((int(self.kf_ids[s]), s) for s in range(len(self.kf_ids)) if self.kf_state[s] == 2)
        for k, s in live:
            h.update(f"kf {k} ".encode())
            h.update(self.kf_bindings(s).tobytes())
        obs = self.observations()
        for i in np.flatnonzero(self.alive):
            i = int(i)
            h.update(f"mp {i} {int(self.found[i])} {int(self.visible[i])} ".encode())
            h.update(self.rep[i].tobytes())
            h.update(str(sorted(obs[i].items())).encode())
            h.update(self.counts[i].astype(np.int64).tobytes())
        return h.hexdigest()


def export_snapshot(ctx: Context, map_idx: int, with_covis: bool = True, kf_cap: int = 0) -> MapSnapshot:
    lib = ctx.lib
    sizes = _lib.MapSizes()
    check(lib.lm_map_sizes_get(ctx.h, map_idx, C.byref(sizes)), ctx.h)
    ns = max(sizes.n_kf_slots, 1)
    ids = np.zeros(ns, np.int64)
    st = np.zeros(ns, np.int32)
    off = np.zeros(ns, np.int32)
    kn = np.zeros(ns, np.int32)
    got = C.c_int32()
    check(lib.lm_export_keyframes(ctx.h, map_idx, ptr(ids, C.c_int64), ptr(st, C.c_int32), ptr(off, C.c_int32),
                                  ptr(kn, C.c_int32), ns, C.byref(got)), ctx.h)
    nslot = got.value
    bind = np.zeros(max(sizes.n_keypoints, 1), np.int32)
    check(lib.lm_export_bindings(ctx.h, map_idx, ptr(bind, C.c_int32), len(bind)), ctx.h)
    n = sizes.n_points
    L = None
    pos = np.zeros((max(n, 1), 3))
    rep = np.zeros((max(n, 1), 32), np.uint8)
    alive = np.zeros(max(n, 1), np.uint8)
    found = np.zeros(max(n, 1), np.int32)
    vis = np.zeros(max(n, 1), np.int32)
    nobs = np.zeros(max(n, 1), np.int32)
    # counts width: infer from the map (levels) via a probe of caps kept on the Python side
    L = ctx._levels[map_idx]
    counts = np.zeros((max(n, 1), L), np.int32)
    cap = max(sizes.obs_used, 1)
    okf = np.zeros(cap, np.int64)
    okp = np.zeros(cap, np.int32)
    check(lib.lm_export_points(ctx.h, map_idx, n, ptr(pos, C.c_double), ptr(rep, C.c_uint8), ptr(alive, C.c_uint8),
                               ptr(found, C.c_int32), ptr(vis, C.c_int32), ptr(nobs, C.c_int32),
                               ptr(counts, C.c_int32), ptr(okf, C.c_int64), ptr(okp, C.c_int32), cap), ctx.h)
    cov = None
    if with_covis:
        K = ctx._kf_cap[map_idx]
        cov = np.zeros((K, K), np.int32)
        check(lib.lm_export_covis(ctx.h, map_idx, ptr(cov, C.c_int32), K * K), ctx.h)
    tot = int(nobs[:n].sum())
    return MapSnapshot(ids[:nslot], st[:nslot], off[:nslot], kn[:nslot], bind[:sizes.n_keypoints], pos[:n], rep[:n],
                       alive[:n].astype(bool), found[:n], vis[:n], nobs[:n], counts[:n], okf[:tot], okp[:tot], cov)


def create_map(ctx: Context, num_levels: int, scale_factor: float, store: StoreConfig, cfg: MapConfig) -> int:
    caps = map_caps(num_levels, scale_factor, store, cfg)
    idx = C.c_int32()
    check(ctx.lib.lm_map_create(ctx.h, C.byref(caps), C.byref(idx)), ctx.h)
    if not hasattr(ctx, "_levels"):
        ctx._levels, ctx._kf_cap = {}, {}
    ctx._levels[idx.value] = num_levels
    ctx._kf_cap[idx.value] = store.max_keyframes
    return idx.value


class CovisibilityView:
    """Read view of the device covisibility matrix with CovisibilityGraph's queries
    (mapmodel.py:80-110): one row per call."""

    def __init__(self, model: "MapModel"):
        self._m = model

    def _row(self, kf_id: int) -> list[tuple[int, int]]:
        m = self._m
        if kf_id not in m._kfs:
            return []
        cap = max(16, len(m._kfs))
        ids = np.zeros(cap, np.int64)
        w = np.zeros(cap, np.int32)
        n = C.c_int32()
        m.ctx.call("lm_covis_row", m.map, int(kf_id), ptr(ids, C.c_int64), ptr(w, C.c_int32), cap, C.byref(n))
        return [(int(ids[k]), int(w[k])) for k in range(n.value)]

    def weight(self, a: int, b: int) -> int:
        return dict(self._row(a)).get(b, 0)

    def neighbors(self, kf_id: int, min_weight: int = 1) -> list[tuple[int, int]]:
        items = [(k, w) for k, w in self._row(kf_id) if w >= min_weight]
        items.sort(key=lambda p: (-p[1], p[0]))
        return items


class KeyframeTable(Mapping):
    """``MapModel.keyframes``: the caller's KeyFrame objects, each one's ``mp_bindings``
    brought up to date (one keyframe's slots, D2H) when the map changed since its last read."""

    def __init__(self, model: "MapModel"):
        self._m = model

    def __getitem__(self, kf_id):
        kf = self._m._kfs[kf_id]
        self._m._sync_bindings(kf)
        return kf

    def __iter__(self):
        return iter(self._m._kfs)

    def __len__(self):
        return len(self._m._kfs)

    def __contains__(self, kf_id):
        return kf_id in self._m._kfs


class PointTable(Mapping):
    """``MapModel.points``: id -> MapPoint snapshot (dead points included, like the
    reference's dict). Single lookups export one record; iteration exports the map."""

    def __init__(self, model: "MapModel"):
        self._m = model

    def __getitem__(self, mp_id):
        m = self._m
        if not isinstance(mp_id, (int, np.integer)) or not 0 <= int(mp_id) < m._next_id():
            raise KeyError(mp_id)
        return m._point(int(mp_id))

    def __iter__(self):
        return iter(range(self._m._next_id()))

    def __len__(self):
        return self._m._next_id()

    def __contains__(self, mp_id):
        return isinstance(mp_id, (int, np.integer)) and 0 <= int(mp_id) < self._m._next_id()

    def values(self):
        return self._m._all_points()

    def items(self):
        return [(p.mp_id, p) for p in self._m._all_points()]


class MapModel:
    """Device-resident map; same operations and error behaviour as the reference MapModel."""

    def __init__(self, num_levels: int, config: MapConfig | None = None, *, scale_factor: float = 1.2,
                 store: StoreConfig | None = None, device: int = 0):
        self.config = config or MapConfig()
        self.num_levels = num_levels
        self.scale_factor = scale_factor
        self.store_config = store or StoreConfig()
        self.ctx = Context.get(device)
        self.map = create_map(self.ctx, num_levels, scale_factor, self.store_config, self.config)
        self._kfs: dict[int, KeyFrame] = {}
        self._kf_seen: dict[int, int] = {}  # kf id -> map version its bindings were read at
        self._version = 0
        self._snap = None
        self._snap_version = -1
        self._cache_version = -1
        self._cache: dict[int, MapPoint] = {}
        self._n_points = 0
        self._foreign = False
        self._pending: dict[int, MapPoint] = {}
        self._pose_ref: dict = {}

    def close(self):
        """Free the device map (lm_map_destroy); the model is unusable afterwards."""
        if self.map is not None and self.ctx.h:
            self.ctx.call("lm_map_destroy", self.map)
        self.map = None

    def reset(self):
        """Back to an empty map (device arenas kept, lm_map_reset)."""
        self.ctx.call("lm_map_reset", self.map)
        for kf in self._kfs.values():
            _HOME.pop(id(kf), None)
        self._kfs.clear()
        self._kf_seen.clear()
        self._pose_ref.clear()
        self._pending.clear()
        self._foreign = False
        self._version += 1

    # ------------------------------------------------------------------ plumbing
    def _call(self, name, *args):
        if self._pending:
            self._flush_points()
        self._version += 1  # even a failing call may have changed the map
        self.ctx.call(name, *args)

    def _flush_points(self):
        """Write back attribute assignments on MapPoint snapshots (LBA positions, counters)."""
        pend, self._pending = self._pending, {}
        moved = [p for p in pend.values() if p.alive]
        if moved:
            ids = np.array([p.mp_id for p in moved], np.int64)
            pos = np.array([np.asarray(p.position, np.float64).reshape(3) for p in moved])
            self._version += 1
            self.ctx.call("lm_mp_patch_positions", self.map, len(ids), ptr(ids, C.c_int64), ptr(pos, C.c_double))
        for p in pend.values():
            self._version += 1
            self.ctx.call("lm_mp_set_counts", self.map, int(p.mp_id), int(p.found_count), int(p.visible_count))

    def sync_host_writes(self):
        """Push host-side writes the reference makes directly on its objects (LBA assigns
        ``kf.pose`` and ``mp.position``, localba.py:571-574) to the device. The stage
        functions call this on entry, so a reference pipeline with LBA needs nothing else."""
        if self._pending:
            self._flush_points()
        for k, kf in self._kfs.items():
            if kf.pose is not self._pose_ref.get(k) and kf.alive:
                self.set_pose(k, kf.pose)

    def invalidate(self):
        self._version += 1

    def _fresh(self):
        if self._pending:
            self._flush_points()
        if self._cache_version != self._version:
            self._cache.clear()
            sizes = _lib.MapSizes()
            check(self.ctx.lib.lm_map_sizes_get(self.ctx.h, self.map, C.byref(sizes)), self.ctx.h)
            self._n_points = sizes.n_points
            self._cache_version = self._version

    def _next_id(self) -> int:
        self._fresh()
        return self._n_points

    def _snapshot(self) -> MapSnapshot:
        """Whole-map export (audit, iteration): O(map), cached until the next mutation."""
        if self._pending:
            self._flush_points()
        if self._snap_version != self._version:
            self._snap = export_snapshot(self.ctx, self.map)
            self._snap_version = self._version
        return self._snap

    def _sync_bindings(self, kf):
        if self._kf_seen.get(kf.kf_id) == self._version:
            return
        n = kf.num_keypoints
        buf = np.zeros(max(n, 1), np.int64)
        got = C.c_int32()
        self.ctx.call("lm_kf_bindings", self.map, int(kf.kf_id), ptr(buf, C.c_int64), len(buf), C.byref(got))
        kf.mp_bindings[:] = buf[:n]
        self._kf_seen[kf.kf_id] = self._version

    def _point(self, mp_id: int) -> MapPoint:
        self._fresh()
        p = self._cache.get(mp_id)
        if p is None:
            rec = _lib.PointRecord()
            cap = max(16, len(self._kfs))
            okf = np.zeros(cap, np.int64)
            okp = np.zeros(cap, np.int32)
            self.ctx.call("lm_mp_get", self.map, mp_id, C.byref(rec), ptr(okf, C.c_int64), ptr(okp, C.c_int32), cap)
            n = rec.nobs
            p = MapPoint(mp_id, np.array(rec.pos[:], np.float64), np.frombuffer(bytes(rec.rep), np.uint8).copy(),
                         int(rec.first_kf_id), {int(okf[k]): int(okp[k]) for k in range(n)}, int(rec.found),
                         int(rec.visible), bool(rec.alive), np.array(rec.counts[:self.num_levels], np.int64))
            object.__setattr__(p, "_model", self)
            self._cache[mp_id] = p
        return p

    def _all_points(self) -> list[MapPoint]:
        s = self._snapshot()
        obs = s.observations()
        first = [-1] * len(s.alive)
        out = [MapPoint(i, s.pos[i].copy(), s.rep[i].copy(), first[i], obs[i], int(s.found[i]), int(s.visible[i]),
                        bool(s.alive[i]), s.counts[i].astype(np.int64)) for i in range(len(s.alive))]
        for p in out:
            object.__setattr__(p, "_model", self)
        return out

    # ------------------------------------------------------------------ keyframes
    def insert_keyframe(self, kf) -> int:
        """insert_keyframe (mapmodel.py:185-199): pre-bound slots become observations. Any
        KeyFrame-shaped object works (this package's or the reference's). Residency and the
        upload ledger entry belong to the store (DeviceStore.upload_keyframe)."""
        if kf.kf_id in self._kfs:
            raise InvalidArgumentError(f"duplicate keyframe id {kf.kf_id}")
        k = kf.intrinsics
        if k.num_levels != self.num_levels or k.scale_factor != self.scale_factor:
            raise InvalidArgumentError("keyframe pyramid differs from the map's (num_levels, scale_factor)")
        stage_keyframe(self.ctx, self.map, kf)
        self._call("lm_kf_insert", self.map, int(kf.kf_id))
        self._kfs[kf.kf_id] = kf
        self._pose_ref[kf.kf_id] = kf.pose
        kf.alive = True
        _HOME[id(kf)] = (weakref.ref(self), kf.kf_id)
        return kf.kf_id

    @property
    def keyframes(self) -> KeyframeTable:
        return KeyframeTable(self)

    def kill_keyframe(self, kf_id: int):
        self._require_kf(kf_id)
        self._call("lm_kf_kill", self.map, int(kf_id))
        self._kfs[kf_id].alive = False

    def live_keyframes(self) -> list:
        return [self.keyframes[k] for k, kf in self._kfs.items() if kf.alive]

    def _require_kf(self, kf_id):
        kf = self._kfs.get(kf_id)
        if kf is None:
            raise InvalidArgumentError(f"unknown keyframe {kf_id}")
        if not kf.alive:
            raise InvalidStateError(f"keyframe {kf_id} is dead")
        return kf

    def set_pose(self, kf_id: int, pose: SE3Pose):
        """LBA pose write-back (localba.py:571-574 assigns kf.pose): device tables follow."""
        kf = self._kfs.get(kf_id)
        if kf is None:
            raise InvalidArgumentError(f"unknown keyframe {kf_id}")
        q = np.ascontiguousarray(pose.quat, dtype=np.float64)
        t = np.ascontiguousarray(pose.trans, dtype=np.float64)
        self._call("lm_kf_set_pose", self.map, int(kf_id), ptr(q, C.c_double), ptr(t, C.c_double))
        kf.pose = pose
        self._pose_ref[kf_id] = pose

    def patch_positions(self, ids, positions):
        """LBA position write-back (localba.py:571-574 assigns mp.position), batched."""
        ids = np.ascontiguousarray(ids, dtype=np.int64)
        pos = np.ascontiguousarray(positions, dtype=np.float64).reshape(len(ids), 3)
        self._call("lm_mp_patch_positions", self.map, len(ids), ptr(ids, C.c_int64), ptr(pos, C.c_double))

    # ------------------------------------------------------------------ points
    @property
    def points(self) -> PointTable:
        return PointTable(self)

    def live_points(self) -> list[MapPoint]:
        return [p for p in self._all_points() if p.alive]

    @property
    def counter_matrix(self) -> np.ndarray:
        return self._snapshot().counts.astype(np.int64)

    def new_map_point(self, position, descriptor, first_kf_id: int) -> MapPoint:
        pos = np.ascontiguousarray(position, dtype=np.float64).reshape(3)
        d = np.ascontiguousarray(descriptor, dtype=np.uint8).reshape(32)
        out = C.c_int64()
        self._call("lm_mp_new", self.map, ptr(pos, C.c_double), ptr(d, C.c_uint8), int(first_kf_id), C.byref(out))
        return self.points[out.value]

    def add_observation(self, mp_id: int, kf_id: int, kp_index: int):
        self._require_kf(kf_id)
        self._call("lm_obs_add", self.map, int(mp_id), int(kf_id), int(kp_index))

    def erase_observation(self, mp_id: int, kf_id: int):
        self._call("lm_obs_erase", self.map, int(mp_id), int(kf_id))

    def kill_map_point(self, mp_id: int):
        self._call("lm_mp_kill", self.map, int(mp_id))

    def replace_map_point(self, loser_id: int, winner_id: int) -> int:
        mig = C.c_int32()
        self._call("lm_mp_replace", self.map, int(loser_id), int(winner_id), C.byref(mig))
        return mig.value

    def set_counts(self, mp_id: int, found: int, visible: int):
        self._call("lm_mp_set_counts", self.map, int(mp_id), int(found), int(visible))

    # ------------------------------------------------------------------ queries
    @property
    def graph(self) -> CovisibilityView:
        return CovisibilityView(self)

    def covisible_neighbors(self, kf_id: int, n: int | None = None) -> list[int]:
        self._require_kf(kf_id)
        buf = np.zeros(max(1024, len(self._kfs)), np.int64)
        got = C.c_int32()
        self.ctx.call("lm_covisible_neighbors", self.map, int(kf_id), -1 if n is None else int(n),
                      ptr(buf, C.c_int64), len(buf), C.byref(got))
        return [int(x) for x in buf[:got.value]]

    def bound_points_of(self, kf_id: int) -> list[int]:
        if kf_id not in self._kfs:
            raise KeyError(kf_id)
        n = self._kfs[kf_id].num_keypoints
        buf = np.zeros(max(n, 1), np.int64)
        got = C.c_int32()
        self.ctx.call("lm_bound_points", self.map, int(kf_id), ptr(buf, C.c_int64), len(buf), C.byref(got))
        return [int(x) for x in buf[:got.value]]

    def audit(self) -> list[str]:
        """Brute-force recheck of counters, weights and binding bijectivity (mapmodel.py:304-353),
        run on the device (lm_audit); violations formatted like the reference's."""
        from .audit import device_audit

        return device_audit(self)

    # ------------------------------------------------------------------ store binding
    def _use_store(self, store) -> bool:
        """Bind the store a stage was called with. Returns True when it is this map's
        device store (the kernels do the accounting); a foreign store (e.g. the reference's
        DeviceStore) keeps its own ledger, fed by the facade, and residency is not enforced
        on the device."""
        self.sync_host_writes()
        if isinstance(store, DeviceStore):
            store._attach(self)
            return True
        if not self._foreign:
            self.ctx.call("lm_map_enforce_residency", self.map, 0)
            self._foreign = True
        return False

    # ------------------------------------------------------------------ snapshots
    def import_reference(self, ref_model, ref_store=None, recent=None):
        """Load a reference MapModel's state (plus its DeviceStore residency and ledger, and
        the pipeline's probation list) into this empty device map (lm_import_snapshot)."""
        from .snapshot import import_reference

        import_reference(self, ref_model, ref_store, recent)


# keyframe object -> (model, kf id): lets a DeviceStore find the device map a keyframe was
# inserted into (the reference pipeline creates the model and the store independently)
_HOME: dict[int, tuple] = {}


# ---------------------------------------------------------------------- store (device ledger views)


@dataclass
class StoredKeyFrame:
    kf_id: int
    payload_bytes: int
    resident: bool = True


class TransferLedger:
    """TransferLedger (devicestore.py:25-48) read from the device ledger (lm_ledger,
    lm_ledger_log): the kernels account every upload, neighbour access and small transfer."""

    def __init__(self, store: "DeviceStore"):
        self._s = store

    def _raw(self) -> _lib.Ledger:
        lg = _lib.Ledger()
        m = self._s._model
        if m is not None:
            m.ctx.call("lm_ledger", m.map, C.byref(lg))
        return lg

    @property
    def persistent_bytes_up(self) -> int:
        return int(self._raw().persistent_bytes_up)

    @property
    def naive_bytes_up(self) -> int:
        return int(self._raw().naive_bytes_up)

    @property
    def evictions(self) -> int:
        return int(self._raw().evictions)

    @property
    def per_stage_small_transfers(self) -> list[tuple[str, int]]:
        m = self._s._model
        if m is None:
            return []
        n = int(self._raw().small_transfer_events)
        buf = np.zeros(max(n, 1), np.int64)
        got = C.c_int32()
        m.ctx.call("lm_ledger_log", m.map, 0, ptr(buf, C.c_int64), len(buf), C.byref(got))
        return [("triangulation", -int(b) - 1) if b < 0 else ("fusion", int(b)) for b in buf[:got.value]]

    def as_dict(self) -> dict:
        lg = self._raw()
        small = {}
        if lg.small_bytes_triangulation:
            small["triangulation"] = int(lg.small_bytes_triangulation)
        if lg.small_bytes_fusion or lg.small_transfer_events:
            small["fusion"] = int(lg.small_bytes_fusion)
        p, nv = int(lg.persistent_bytes_up), int(lg.naive_bytes_up)
        return {"persistent_bytes_up": p, "naive_bytes_up": nv, "naive_over_persistent": nv / p if p > 0 else 0.0,
                "small_transfer_bytes_by_stage": small, "small_transfer_events": int(lg.small_transfer_events),
                "evictions": int(lg.evictions)}


class DeviceStore:
    """DeviceStore (devicestore.py:51-109) over the device map that holds the keyframes:
    residency is the map's per-slot flag, the ledger is the one the kernels keep. It binds
    to the MapModel its first uploaded keyframe was inserted into; a keyframe that is in no
    map is staged into a private ledger-only device map."""

    def __init__(self, config: StoreConfig | None = None, model: MapModel | None = None):
        self.config = config or StoreConfig()
        self._model = model
        self.ledger = TransferLedger(self)

    def _bind(self, kf) -> MapModel:
        home = _HOME.get(id(kf))
        m = home[0]() if home and home[1] == kf.kf_id else None
        if m is None:  # not in any map: the store's own device map
            if self._model is None:
                k = kf.intrinsics
                self._model = MapModel(k.num_levels, scale_factor=k.scale_factor, store=StoreConfig(
                    capacity=self.config.capacity, max_keyframes=min(4096, max(16, self.config.capacity + 8)),
                    max_points=16, obs_pool_entries=64, max_keypoints=1 << 22,
                    max_keypoints_per_kf=max(8192, kf.num_keypoints)))
            m = self._model
            if kf.kf_id not in m._kfs:
                m.insert_keyframe(kf)
        if self._model is None:
            self._model = m
        elif self._model is not m:
            raise InvalidArgumentError(f"keyframe {kf.kf_id} belongs to another map than this store's")
        return m

    def _attach(self, model: MapModel):
        if self._model is None:
            self._model = model
        elif self._model is not model:
            raise InvalidArgumentError("this DeviceStore holds the keyframes of another map")

    def payload_bytes(self, num_keypoints: int) -> int:
        return num_keypoints * self.config.keypoint_record_bytes + num_keypoints * self.config.descriptor_bytes

    def _resident(self, kf_id: int) -> tuple[bool, int]:
        if self._model is None:
            return False, 0
        r, n = C.c_int32(), C.c_int32()
        self._model.ctx.call("lm_kf_resident", self._model.map, int(kf_id), C.byref(r), C.byref(n))
        return bool(r.value), int(n.value)

    def is_resident(self, kf_id: int) -> bool:
        return self._resident(kf_id)[0]

    def resident_count(self) -> int:
        return self._resident(-1)[1]

    def upload_keyframe(self, kf) -> StoredKeyFrame:
        m = self._bind(kf)
        res, count = self._resident(kf.kf_id)
        if res:
            raise InvalidStateError(f"keyframe {kf.kf_id} already resident")
        if count >= self.config.capacity:
            raise StoreCapacityError(f"store capacity {self.config.capacity} exceeded; size the pre-allocation")
        m._call("lm_kf_upload", m.map, int(kf.kf_id))
        return StoredKeyFrame(kf.kf_id, self.payload_bytes(kf.num_keypoints))

    def record_neighbor_access(self, stage: str, neighbor_ids) -> int:
        """Explicit access accounting (the device stages account their own accesses)."""
        m = self._model
        delta = 0
        for k in neighbor_ids:
            if m is None or not self.is_resident(k):
                raise InvalidStateError(f"stage {stage!r} accessed non-resident keyframe {k}")
            delta += self.payload_bytes(m._kfs[k].num_keypoints)
        if delta:
            _ledger_add(m, naive=delta)
        return delta

    def record_small_transfer(self, stage: str, nbytes: int):
        if nbytes < 0:
            raise InvalidArgumentError("transfer size must be non-negative")
        if stage not in ("fusion", "triangulation"):
            raise InvalidArgumentError(f"the device ledger keeps stages 'fusion' and 'triangulation', not {stage!r}")
        if self._model is None:
            raise InvalidStateError("store has no device map yet (upload a keyframe first)")
        _ledger_add(self._model, small=(stage, nbytes))

    def evict_keyframe(self, kf_id: int) -> StoredKeyFrame:
        m = self._model
        if m is None or not self.is_resident(kf_id):
            raise InvalidArgumentError(f"keyframe {kf_id} is not resident")
        m._call("lm_kf_evict", m.map, int(kf_id))
        kf = m._kfs.get(kf_id)
        return StoredKeyFrame(kf_id, self.payload_bytes(kf.num_keypoints) if kf is not None else 0, False)


def _ledger_add(m: MapModel, naive: int = 0, small: tuple | None = None):
    """Host-initiated ledger entries (explicit record_* calls): one device ledger update."""
    m.ctx.call("lm_ledger_add", m.map, int(naive), 1 if small and small[0] == "triangulation" else 0,
               int(small[1]) if small else 0, 1 if small else 0)
