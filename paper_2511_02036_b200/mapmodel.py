"""Device-backed map with the reference's MapModel interface.

The state lives on the GPU (csrc/lm_map.cuh); this class is the host handle. Reads
(``keyframes``, ``points``, ``graph``, ``counter_matrix``, ``audit``) come from a state
export that is refreshed lazily after any mutation; mutations are single-op kernels that
run the same device code as the hot-path stages. Mirrors
pkg/src/localmap/mapmodel.py (KeyFrame 24-62, MapPoint 65-77, CovisibilityGraph 80-110,
MapModel 113-353) and devicestore.py (TransferLedger 25-48, DeviceStore 51-109).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from itertools import combinations

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
    """Snapshot of one device map point (read-only view)."""

    mp_id: int
    position: np.ndarray
    rep_descriptor: np.ndarray
    first_kf_id: int
    observations: dict = field(default_factory=dict)
    found_count: int = 1
    visible_count: int = 1
    alive: bool = True
    scale_counts: np.ndarray = None


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
    """Read view of the device covisibility matrix with the reference graph's queries."""

    def __init__(self, model: "MapModel"):
        self._m = model

    def weight(self, a: int, b: int) -> int:
        s = self._m._snapshot()
        so = s.slot_of()
        if a not in so or b not in so:
            return 0
        return int(s.covis[so[a], so[b]])

    def neighbors(self, kf_id: int, min_weight: int = 1) -> list[tuple[int, int]]:
        s = self._m._snapshot()
        so = s.slot_of()
        if kf_id not in so:
            return []
        row = s.covis[so[kf_id]]
        items = [(int(s.kf_ids[t]), int(row[t])) for t in range(len(s.kf_ids)) if row[t] >= min_weight and row[t] > 0]
        items.sort(key=lambda p: (-p[1], p[0]))
        return items


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
        self._version = 0
        self._snap = None
        self._snap_version = -1

    # ------------------------------------------------------------------ plumbing
    def _call(self, name, *args):
        self.ctx.call(name, *args)
        self._version += 1

    def _snapshot(self) -> MapSnapshot:
        if self._snap_version != self._version:
            self._snap = export_snapshot(self.ctx, self.map)
            self._snap_version = self._version
            so = self._snap.slot_of()
            for k, kf in self._kfs.items():
                s = so[k]
                kf.mp_bindings[:] = self._snap.kf_bindings(s)
                kf.alive = int(self._snap.kf_state[s]) == 2
        return self._snap

    def invalidate(self):
        self._version += 1

    # ------------------------------------------------------------------ keyframes
    def insert_keyframe(self, kf: KeyFrame) -> int:
        if kf.kf_id in self._kfs:
            raise InvalidArgumentError(f"duplicate keyframe id {kf.kf_id}")
        k = kf.intrinsics
        if k.num_levels != self.num_levels or k.scale_factor != self.scale_factor:
            raise InvalidArgumentError("keyframe pyramid differs from the map's (num_levels, scale_factor)")
        stage_keyframe(self.ctx, self.map, kf)
        self._call("lm_kf_insert", self.map, int(kf.kf_id))
        self._kfs[kf.kf_id] = kf
        return kf.kf_id

    @property
    def keyframes(self) -> dict:
        self._snapshot()
        return self._kfs

    def kill_keyframe(self, kf_id: int):
        self._require_kf(kf_id)
        self._call("lm_kf_kill", self.map, int(kf_id))

    def live_keyframes(self) -> list[KeyFrame]:
        return [kf for kf in self.keyframes.values() if kf.alive]

    def _require_kf(self, kf_id):
        kf = self.keyframes.get(kf_id)
        if kf is None:
            raise InvalidArgumentError(f"unknown keyframe {kf_id}")
        if not kf.alive:
            raise InvalidStateError(f"keyframe {kf_id} is dead")
        return kf

    # ------------------------------------------------------------------ points
    @property
    def points(self) -> dict:
        s = self._snapshot()
        obs = s.observations()
        out = {}
        for i in range(len(s.alive)):
            out[i] = MapPoint(i, s.pos[i].copy(), s.rep[i].copy(), -1, obs[i], int(s.found[i]), int(s.visible[i]),
                              bool(s.alive[i]), s.counts[i].astype(np.int64))
        return out

    def live_points(self) -> list[MapPoint]:
        return [p for p in self.points.values() if p.alive]

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
        if kf_id not in self._kfs:
            raise InvalidArgumentError(f"unknown keyframe {kf_id}")
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
        buf = np.zeros(1024, np.int64)
        got = C.c_int32()
        self.ctx.call("lm_covisible_neighbors", self.map, int(kf_id), -1 if n is None else int(n),
                      ptr(buf, C.c_int64), len(buf), C.byref(got))
        return [int(x) for x in buf[:got.value]]

    def bound_points_of(self, kf_id: int) -> list[int]:
        s = self._snapshot()
        b = s.kf_bindings(s.slot_of()[kf_id])
        return [int(m) for m in b if m != UNBOUND and s.alive[m]]

    def audit(self) -> list[str]:
        """Brute-force recheck of counters, weights and binding bijectivity (mapmodel.py:304-353)."""
        s = self._snapshot()
        bad = []
        obs = s.observations()
        so = s.slot_of()
        for i in range(len(s.alive)):
            if not s.alive[i]:
                if obs[i]:
                    bad.append(f"dead map point {i} retains observations")
                continue
            exp = np.zeros(self.num_levels, np.int64)
            for k, kp in obs[i].items():
                st = so[k]
                if s.kf_state[st] != 2:
                    bad.append(f"map point {i} observes dead keyframe {k}")
                    continue
                if s.kf_bindings(st)[kp] != i:
                    bad.append(f"binding mismatch: map point {i} vs slot ({k}, {kp})")
                exp[int(self._kfs[k].kp_level[kp])] += 1
            if not np.array_equal(exp, s.counts[i].astype(np.int64)):
                bad.append(f"scale_counts mismatch for map point {i}")
        live = sorted(k for k, st in so.items() if s.kf_state[st] == 2)
        bound = {}
        for k in live:
            b = s.kf_bindings(so[k])
            for kp in np.flatnonzero(b != UNBOUND):
                m = int(b[kp])
                if m >= len(s.alive) or not s.alive[m]:
                    bad.append(f"slot ({k}, {int(kp)}) bound to dead point {m}")
                elif obs[m].get(k) != int(kp):
                    bad.append(f"slot ({k}, {int(kp)}) not in map point {m} observations")
            bound[k] = {int(m) for m in b if m != UNBOUND and m < len(s.alive) and s.alive[m]}
        for a, b in combinations(live, 2):
            if len(bound[a] & bound[b]) != int(s.covis[so[a], so[b]]):
                bad.append(f"covisibility weight mismatch for pair ({a}, {b})")
        return bad


# ---------------------------------------------------------------------- ledger (host model)


@dataclass
class StoredKeyFrame:
    kf_id: int
    payload_bytes: int
    resident: bool = True


@dataclass
class TransferLedger:
    persistent_bytes_up: int = 0
    naive_bytes_up: int = 0
    per_stage_small_transfers: list = field(default_factory=list)
    evictions: int = 0

    def as_dict(self) -> dict:
        small: dict[str, int] = {}
        for stage, nbytes in self.per_stage_small_transfers:
            small[stage] = small.get(stage, 0) + nbytes
        ratio = self.naive_bytes_up / self.persistent_bytes_up if self.persistent_bytes_up > 0 else 0.0
        return {"persistent_bytes_up": self.persistent_bytes_up, "naive_bytes_up": self.naive_bytes_up,
                "naive_over_persistent": ratio, "small_transfer_bytes_by_stage": small,
                "small_transfer_events": len(self.per_stage_small_transfers), "evictions": self.evictions}


class DeviceStore:
    """Transfer ledger of the persistent keyframe store (devicestore.py:51-109 semantics)."""

    def __init__(self, config: StoreConfig | None = None):
        self.config = config or StoreConfig()
        self.ledger = TransferLedger()
        self._stored: dict[int, StoredKeyFrame] = {}

    def payload_bytes(self, n: int) -> int:
        return n * self.config.keypoint_record_bytes + n * self.config.descriptor_bytes

    def is_resident(self, kf_id: int) -> bool:
        e = self._stored.get(kf_id)
        return e is not None and e.resident

    def resident_count(self) -> int:
        return sum(1 for e in self._stored.values() if e.resident)

    def upload_keyframe(self, kf: KeyFrame) -> StoredKeyFrame:
        if self.is_resident(kf.kf_id):
            raise InvalidStateError(f"keyframe {kf.kf_id} already resident")
        if self.resident_count() >= self.config.capacity:
            raise StoreCapacityError(f"store capacity {self.config.capacity} exceeded; size the pre-allocation")
        e = StoredKeyFrame(kf.kf_id, self.payload_bytes(kf.num_keypoints))
        self._stored[kf.kf_id] = e
        self.ledger.persistent_bytes_up += e.payload_bytes
        return e

    def record_neighbor_access(self, stage: str, neighbor_ids) -> int:
        delta = 0
        for k in neighbor_ids:
            e = self._stored.get(k)
            if e is None or not e.resident:
                raise InvalidStateError(f"stage {stage!r} accessed non-resident keyframe {k}")
            delta += e.payload_bytes
        self.ledger.naive_bytes_up += delta
        return delta

    def record_small_transfer(self, stage: str, nbytes: int):
        if nbytes < 0:
            raise InvalidArgumentError("transfer size must be non-negative")
        self.ledger.per_stage_small_transfers.append((stage, nbytes))
        self.ledger.persistent_bytes_up += nbytes
        self.ledger.naive_bytes_up += nbytes

    def evict_keyframe(self, kf_id: int) -> StoredKeyFrame:
        e = self._stored.get(kf_id)
        if e is None or not e.resident:
            raise InvalidArgumentError(f"keyframe {kf_id} is not resident")
        e.resident = False
        self.ledger.evictions += 1
        return e
