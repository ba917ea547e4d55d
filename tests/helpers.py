"""Shared test helpers: workload records -> device keyframes / oracle keyframes, and
device-vs-oracle state comparison. Test infrastructure (may import oracle/)."""

from __future__ import annotations

import numpy as np

from oracle import lm_oracle as O
from paper_2511_02036_b200.mapmodel import KeyFrame


def cam_of(seq):
    c = seq.config
    return O.Cam(c.fx, c.fy, c.cx, c.cy, c.width, c.height, c.num_levels, c.scale_factor)


def device_kf(rec, intr) -> KeyFrame:
    return KeyFrame(int(rec.kf_id), rec.pose_init, intr, rec.kp_u, rec.kp_v, rec.kp_level, rec.descriptors,
                    frame_index=int(rec.frame_index))


def compare_state(snap, omap: O.OracleMap, pos_rtol=1e-4) -> dict:
    """Structural equality (bitwise) + position agreement (relative) of device vs oracle."""
    out = {"structural_equal": snap.structural_digest() == O.structural_digest(omap)}
    n = len(snap.alive)
    live_o = sorted(p.mp_id for p in omap.live_points())
    live_d = [int(i) for i in np.flatnonzero(snap.alive)]
    out["live_equal"] = live_o == live_d
    worst = 0.0
    if out["live_equal"] and live_d:
        a = snap.pos[live_d]
        b = np.stack([omap.pts[i].pos for i in live_d])
        rel = np.abs(a - b) / np.maximum(np.abs(b), 1e-6)
        worst = float(np.max(np.linalg.norm(a - b, axis=1) / np.maximum(np.linalg.norm(b, axis=1), 1e-12)))
    out["pos_worst_rel"] = worst
    out["pos_ok"] = worst <= pos_rtol
    out["n_points"] = n
    return out


def first_difference(snap, omap: O.OracleMap) -> str:
    """Human-readable first structural difference (debug aid)."""
    obs = snap.observations()
    for i in range(max(len(snap.alive), omap.next_id)):
        if i >= len(snap.alive) or i not in omap.pts:
            return f"point id space differs at {i} (device {len(snap.alive)}, oracle {omap.next_id})"
        p = omap.pts[i]
        if bool(snap.alive[i]) != p.alive:
            return f"mp {i} alive device={bool(snap.alive[i])} oracle={p.alive}"
        if not p.alive:
            continue
        if obs[i] != p.obs:
            return f"mp {i} obs device={obs[i]} oracle={p.obs}"
        if (snap.found[i], snap.visible[i]) != (p.found, p.visible):
            return f"mp {i} found/visible device={(snap.found[i], snap.visible[i])} oracle={(p.found, p.visible)}"
        if not np.array_equal(snap.rep[i], p.rep):
            return f"mp {i} rep differs"
        if not np.array_equal(snap.counts[i], omap.counts[i]):
            return f"mp {i} counts device={snap.counts[i]} oracle={omap.counts[i]}"
    so = snap.slot_of()
    for k, kf in omap.kfs.items():
        b = snap.kf_bindings(so[k])
        if not np.array_equal(b, kf.bind):
            j = int(np.flatnonzero(b != kf.bind)[0])
            return f"kf {k} binding[{j}] device={b[j]} oracle={kf.bind[j]}"
    return "no structural difference found"
