"""ctypes binding of include/lm_b200.h (the package's only route to the device).

There is no CPU fallback: if ``liblm_b200.so`` is missing, or no CUDA device can be opened,
every entry point raises ``DeviceError``.
"""

from __future__ import annotations

import atexit
import ctypes as C
import os
import threading

import numpy as np

from .errors import (
    DegenerateGeometryError,
    DeviceError,
    InvalidArgumentError,
    InvalidStateError,
    LocalMapError,
    SlotConflictError,
    StoreCapacityError,
)

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "liblm_b200.so")

MAX_NEIGHBORS = 64
MAX_TARGETS = 320
ACT_ADD, ACT_MERGE = 1, 2

i32, i64, f64, u8 = C.c_int32, C.c_int64, C.c_double, C.c_uint8
P = C.POINTER


class MapCaps(C.Structure):
    _fields_ = [("max_keyframes", i32), ("max_keypoints", i32), ("max_keypoints_per_kf", i32),
                ("max_points", i32), ("obs_pool_entries", i32), ("num_levels", i32), ("scale_factor", f64),
                ("min_covis_weight", i32), ("min_obs_keep", i32), ("keypoint_record_bytes", i32),
                ("descriptor_bytes", i32), ("map_point_record_bytes", i32), ("store_capacity", i32)]


class MatchCfg(C.Structure):
    _fields_ = [("match_max_distance", i32), ("chi2_epi", f64), ("level_window", i32)]


class GateCfg(C.Structure):
    _fields_ = [("cos_parallax_max", f64), ("chi2_mono", f64), ("scale_ratio_slack", f64)]


class FuseCfg(C.Structure):
    _fields_ = [("match_max_distance", i32), ("fuse_radius", f64), ("min_view_cos", f64),
                ("dist_band_slack", f64), ("level_window", i32), ("n1", i32), ("n2", i32)]


class CullCfg(C.Structure):
    _fields_ = [("found_ratio_min", f64), ("probation_kfs", i32), ("min_obs_graduate", i32)]


class StepParams(C.Structure):
    _fields_ = [("neighbor_count", i32), ("do_cull", i32), ("do_create", i32), ("do_fuse", i32),
                ("processed_index", i32), ("match", MatchCfg), ("gate", GateCfg), ("fuse", FuseCfg),
                ("cull", CullCfg)]


class StepStats(C.Structure):
    _fields_ = [("created", i32), ("conflicts", i32), ("degenerate", i32), ("gate_parallax", i32),
                ("gate_depth", i32), ("gate_reprojection", i32), ("gate_scale", i32),
                ("n_degenerate_neighbors", i32), ("degenerate_neighbors", i64 * MAX_NEIGHBORS),
                ("n_neighbors", i32), ("neighbors", i64 * MAX_NEIGHBORS), ("n_targets", i32),
                ("merged", i32), ("observations_added", i32), ("stale", i32), ("culled", i32),
                ("first_new_id", i64), ("error", i32), ("n_candidates", i32), ("match_pairs", i64),
                ("fuse_bytes", i64), ("fuse_passes", i64), ("fuse_points", i64), ("fuse_actions", i64),
                ("apply_rounds", i64), ("fuse_cycles", i64 * 16),
                ("rev_passes_acting", i64), ("rev_passes_redo", i64), ("fuse_bytes_rev", i64), ("rev_mergeable", i64), ("dbg", i64 * 16),
                ("borderline", i64 * 4), ("match_second_half", i64)]


class Candidate(C.Structure):
    _fields_ = [("neighbor_kf_id", i64), ("kp_index_current", i32), ("kp_index_neighbor", i32),
                ("distance", i32), ("pad", i32)]


class FuseActionC(C.Structure):
    _fields_ = [("target_kf_id", i64), ("mp_id_projected", i64), ("kp_index_hit", i32), ("kind", i32),
                ("existing_mp_id", i64)]


class Ledger(C.Structure):
    _fields_ = [("persistent_bytes_up", i64), ("naive_bytes_up", i64), ("small_bytes_triangulation", i64),
                ("small_bytes_fusion", i64), ("small_transfer_events", i64), ("evictions", i64)]


class PointRecord(C.Structure):
    _fields_ = [("pos", f64 * 3), ("rep", u8 * 32), ("first_kf_id", i64), ("alive", i32), ("found", i32),
                ("visible", i32), ("nobs", i32), ("counts", i32 * 16)]


class Snapshot(C.Structure):
    _fields_ = [("n_kf", i32), ("kf_id", P(i64)), ("kf_alive", P(u8)), ("kf_resident", P(u8)), ("quat", P(f64)),
                ("trans", P(f64)), ("cam", P(f64)), ("kp_n", P(i32)), ("u", P(f64)), ("v", P(f64)),
                ("level", P(i64)), ("desc", P(u8)), ("bindings", P(i64)), ("n_points", i32), ("pos", P(f64)),
                ("rep", P(u8)), ("alive", P(u8)), ("found", P(i32)), ("visible", P(i32)), ("first_kf", P(i64)),
                ("n_recent", i32), ("recent_id", P(i64)), ("recent_born", P(i32)), ("ledger", Ledger)]


class AuditRecord(C.Structure):
    _fields_ = [("code", i32), ("kp", i32), ("mp", i64), ("kf_a", i64), ("kf_b", i64)]


class KfCullCfg(C.Structure):
    _fields_ = [("redundancy_ratio", f64), ("min_redundant_observers", i32), ("scale_tolerance_levels", i32)]


class MapSizes(C.Structure):
    _fields_ = [("n_kf_slots", i32), ("n_points", i32), ("n_keypoints", i32), ("obs_used", i32),
                ("recent_n", i32)]


_SIGS = {
    "lm_version": ([], i32),
    "lm_ctx_create": ([i32, P(C.c_void_p)], i32),
    "lm_ctx_destroy": ([C.c_void_p], i32),
    "lm_last_error": ([C.c_void_p], C.c_char_p),
    "lm_map_create": ([C.c_void_p, P(MapCaps), P(i32)], i32),
    "lm_map_reset": ([C.c_void_p, i32], i32),
    "lm_map_destroy": ([C.c_void_p, i32], i32),
    "lm_map_sizes_get": ([C.c_void_p, i32, P(MapSizes)], i32),
    "lm_synchronize": ([C.c_void_p], i32),
    "lm_ctx_set_pdl": ([C.c_void_p, i32], i32),
    "lm_kf_stage": ([C.c_void_p, i32, i64, P(f64), P(f64), P(f64), i32, P(f64), P(f64), P(i64), P(u8), P(i64)], i32),
    "lm_kf_record_bytes": ([i32, C.c_uint32], C.c_uint64),
    "lm_kf_stage_record": ([C.c_void_p, i32, C.c_void_p, C.c_uint64, P(i64)], i32),
    "lm_kf_insert": ([C.c_void_p, i32, i64], i32),
    "lm_kf_kill": ([C.c_void_p, i32, i64], i32),
    "lm_cull_keyframes": ([C.c_void_p, i32, P(i64), i32, P(KfCullCfg), P(i64), P(i32)], i32),
    "lm_step": ([C.c_void_p, i32, i64, P(StepParams), P(StepStats)], i32),
    "lm_step_batch": ([C.c_void_p, i32, P(i32), P(i64), P(StepParams), P(StepStats)], i32),
    "lm_step_stats_fetch": ([C.c_void_p, i32, P(i32), P(StepStats)], i32),
    "lm_create_map_points": ([C.c_void_p, i32, i64, i32, P(MatchCfg), P(GateCfg), P(StepStats)], i32),
    "lm_run_fusion": ([C.c_void_p, i32, i64, P(FuseCfg), P(StepStats)], i32),
    "lm_cull_recent": ([C.c_void_p, i32, i32, P(CullCfg), P(i32)], i32),
    "lm_cull_recent_list": ([C.c_void_p, i32, i32, P(CullCfg), i32, P(i64), P(i32), P(i64), P(i32), P(i64), P(i32),
                             P(i32)], i32),
    "lm_search": ([C.c_void_p, i32, i64, i64, P(MatchCfg), P(u8), P(u8), P(Candidate), i32, P(i32)], i32),
    "lm_fusion_targets": ([C.c_void_p, i32, i64, i32, i32, P(i64), i32, P(i32)], i32),
    "lm_fuse_pass": ([C.c_void_p, i32, P(i64), i32, i64, P(FuseCfg), P(FuseActionC), i32, P(i32), P(i64), P(i32)], i32),
    "lm_apply_fusion": ([C.c_void_p, i32, P(FuseActionC), i32, P(i32)], i32),
    "lm_mp_new": ([C.c_void_p, i32, P(f64), P(u8), i64, P(i64)], i32),
    "lm_obs_add": ([C.c_void_p, i32, i64, i64, i32], i32),
    "lm_obs_erase": ([C.c_void_p, i32, i64, i64], i32),
    "lm_mp_kill": ([C.c_void_p, i32, i64], i32),
    "lm_mp_replace": ([C.c_void_p, i32, i64, i64, P(i32)], i32),
    "lm_mp_set_counts": ([C.c_void_p, i32, i64, i32, i32], i32),
    "lm_covisible_neighbors": ([C.c_void_p, i32, i64, i32, P(i64), i32, P(i32)], i32),
    "lm_ledger": ([C.c_void_p, i32, P(Ledger)], i32),
    "lm_ledger_log": ([C.c_void_p, i32, i64, P(i64), i32, P(i32)], i32),
    "lm_ledger_add": ([C.c_void_p, i32, i64, i32, i64, i32], i32),
    "lm_audit": ([C.c_void_p, i32, P(AuditRecord), i32, P(i32)], i32),
    "lm_debug_corrupt": ([C.c_void_p, i32, i32, i64, i64, i32], i32),
    "lm_kf_upload": ([C.c_void_p, i32, i64], i32),
    "lm_kf_evict": ([C.c_void_p, i32, i64], i32),
    "lm_kf_resident": ([C.c_void_p, i32, i64, P(i32), P(i32)], i32),
    "lm_map_enforce_residency": ([C.c_void_p, i32, i32], i32),
    "lm_kf_set_pose": ([C.c_void_p, i32, i64, P(f64), P(f64)], i32),
    "lm_mp_patch_positions": ([C.c_void_p, i32, i32, P(i64), P(f64)], i32),
    "lm_mp_get": ([C.c_void_p, i32, i64, P(PointRecord), P(i64), P(i32), i32], i32),
    "lm_mp_alive": ([C.c_void_p, i32, i32, P(i64), P(u8)], i32),
    "lm_kf_bindings": ([C.c_void_p, i32, i64, P(i64), i32, P(i32)], i32),
    "lm_bound_points": ([C.c_void_p, i32, i64, P(i64), i32, P(i32)], i32),
    "lm_covis_row": ([C.c_void_p, i32, i64, P(i64), P(i32), i32, P(i32)], i32),
    "lm_import_snapshot": ([C.c_void_p, i32, P(Snapshot)], i32),
    "lm_export_keyframes": ([C.c_void_p, i32, P(i64), P(i32), P(i32), P(i32), i32, P(i32)], i32),
    "lm_export_bindings": ([C.c_void_p, i32, P(i32), i32], i32),
    "lm_export_points": ([C.c_void_p, i32, i32, P(f64), P(u8), P(u8), P(i32), P(i32), P(i32), P(i32), P(i64),
                          P(i32), i32], i32),
    "lm_export_covis": ([C.c_void_p, i32, P(i32), i32], i32),
    "lm_recent_export": ([C.c_void_p, i32, P(i64), P(i32), i32, P(i32)], i32),
    "lm_recent_import": ([C.c_void_p, i32, P(i64), P(i32), i32], i32),
    "lm_map_rewind": ([C.c_void_p, i32], i32),
    "lm_timer_start": ([C.c_void_p], i32),
    "lm_timer_stop": ([C.c_void_p, P(C.c_float)], i32),
    "lm_timer_start_joint": ([C.c_void_p, C.c_void_p], i32),
    "lm_timer_stop_joint": ([C.c_void_p, C.c_void_p, P(C.c_float)], i32),
    "lm_timer_start_multi": ([P(C.c_void_p), i32], i32),
    "lm_timer_stop_multi": ([P(C.c_void_p), i32, P(C.c_float)], i32),
    "lm_flush_l2": ([C.c_void_p, i64], i32),
    "lm_launch_count": ([C.c_void_p], i64),
    "lm_totals_fetch": ([C.c_void_p, i32, P(StepStats)], i32),
    "lm_profile_enable": ([C.c_void_p, i32], i32),
    "lm_profile_read": ([C.c_void_p, P(f64), P(i64)], i32),
    "lm_bench_popc": ([C.c_void_p, P(f64)], i32),
    "lm_host_fundamental": ([P(f64), P(f64), P(f64), P(f64), P(f64), P(f64), P(f64)], i32),
    "lm_host_projection": ([P(f64), P(f64), P(f64), P(f64), P(f64), P(f64)], i32),
    "lm_host_triangulate": ([P(f64), P(f64), P(f64), P(f64), P(f64), P(f64)], i32),
}

EXPORTED = tuple(_SIGS)

_lib = None
_lock = threading.Lock()


def load():
    """Load the native library (raises DeviceError if it was not built)."""
    global _lib
    with _lock:
        if _lib is None:
            path = os.environ.get("LM_B200_LIB", LIB_PATH)  # (experiments: an alternative build)
            if not os.path.exists(path):
                raise DeviceError(f"native library {path} is missing; run __graft_entry__.build()")
            lib = C.CDLL(path)
            for name, (args, res) in _SIGS.items():
                fn = getattr(lib, name)
                fn.argtypes = args
                fn.restype = res
            _lib = lib
        return _lib


_ERRORS = {-1: InvalidArgumentError, -2: InvalidStateError, -3: SlotConflictError, -4: StoreCapacityError,
           -5: DeviceError, -6: DegenerateGeometryError}


def check(rc: int, ctx=None):
    if rc == 0:
        return
    msg = load().lm_last_error(ctx).decode() if ctx else f"status {rc}"
    raise _ERRORS.get(rc, LocalMapError)(msg)


def ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(P(ctype))


class Context:
    """One CUDA device + stream + its maps (a process-wide singleton per device)."""

    _by_device: dict[int, "Context"] = {}

    def __init__(self, device: int = 0):
        lib = load()
        h = C.c_void_p()
        rc = lib.lm_ctx_create(device, C.byref(h))
        if rc != 0:
            msg = lib.lm_last_error(h).decode() if h else "lm_ctx_create failed"
            if h:
                lib.lm_ctx_destroy(h)
            raise DeviceError(msg)
        self.h = h
        self.device = device
        self.lib = lib
        atexit.register(self.close)

    def close(self):
        """Free every device buffer of this context (lm_ctx_destroy); idempotent."""
        if self.h:
            self.lib.lm_ctx_destroy(self.h)
            self.h = None
            Context._by_device.pop(self.device, None)

    @classmethod
    def get(cls, device: int = 0) -> "Context":
        if device not in cls._by_device:
            cls._by_device[device] = Context(device)
        return cls._by_device[device]

    def call(self, name: str, *args):
        check(getattr(self.lib, name)(self.h, *args), self.h)
