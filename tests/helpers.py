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


def rep_descriptor(descs_sorted: np.ndarray) -> np.ndarray:
    """_refresh_rep_descriptor (mapmodel.py:165-181) over descriptors sorted by (kf, kp)."""
    if len(descs_sorted) == 1:
        return descs_sorted[0]
    x = np.bitwise_xor(descs_sorted[:, None, :], descs_sorted[None, :, :])
    dist = np.bitwise_count(x).sum(axis=2, dtype=np.int64).astype(np.float64)
    np.fill_diagonal(dist, np.nan)
    return descs_sorted[int(np.argmin(np.nanmedian(dist, axis=1)))]


def audit_snapshot(snap, kfs=None, sample_rep: int = 0, seed: int = 0) -> list[str]:
    """Vectorised MapModel.audit (mapmodel.py:304-353) over a device snapshot: binding <->
    observation bijection, live keyframes only, per-level counters, covisibility weight ==
    shared bound points for every live pair; with the keyframes (list of KeyFrame) also the
    counters and, on `sample_rep` sampled points, the representative descriptor."""
    import scipy.sparse as sp

    bad = []
    n = len(snap.alive)
    so = snap.slot_of()
    pid = np.repeat(np.arange(n), snap.nobs)
    if np.any(~snap.alive & (snap.nobs > 0)):
        bad.append("dead point keeps observations")
    slot_lut = np.full(int(max(snap.kf_ids.max(initial=0), 0)) + 1, -1, np.int64)
    for k, sl in so.items():
        slot_lut[k] = sl
    slots = slot_lut[snap.obs_kf] if len(pid) else np.zeros(0, np.int64)
    if len(pid):
        if np.any(snap.kf_state[slots] != 2):
            bad.append("observation of a non-live keyframe")
        g = snap.kp_off[slots] + snap.obs_kp
        if np.any(snap.bindings[g] != pid):
            bad.append(f"{int(np.sum(snap.bindings[g] != pid))} observations not mirrored by bindings")
        own = np.full(len(snap.bindings), -1, np.int64)
        own[g] = pid
    else:
        own = np.full(len(snap.bindings), -1, np.int64)
    live_slots = [s for s in range(len(snap.kf_ids)) if snap.kf_state[s] == 2]
    rows, cols = [], []
    for r, s in enumerate(live_slots):
        b = snap.kf_bindings(s)
        idx = np.flatnonzero(b >= 0)
        m = b[idx]
        if np.any(m >= n) or np.any(~snap.alive[np.minimum(m, n - 1)]):
            bad.append(f"slot of keyframe {int(snap.kf_ids[s])} bound to a dead point")
        if np.any(own[snap.kp_off[s] + idx] != m):
            bad.append(f"binding of keyframe {int(snap.kf_ids[s])} missing from the point's observations")
        rows.append(np.full(len(m), r))
        cols.append(m)
    if live_slots and snap.covis is not None:
        B = sp.csr_matrix((np.ones(sum(len(c) for c in cols), np.int64), (np.concatenate(rows), np.concatenate(cols))),
                          shape=(len(live_slots), max(n, 1)))
        Wt = (B @ B.T).toarray()
        np.fill_diagonal(Wt, 0)
        Wd = snap.covis[np.ix_(live_slots, live_slots)].astype(np.int64)
        np.fill_diagonal(Wd, 0)
        if not np.array_equal(Wt, Wd):
            bad.append(f"covisibility differs on {int(np.sum(Wt != Wd)) // 2} keyframe pairs")
    if kfs is not None and len(pid):
        byid = {kf.kf_id: kf for kf in kfs}
        L = snap.counts.shape[1]
        lev_pool = np.zeros(len(snap.bindings), np.int64)
        for s in range(len(snap.kf_ids)):
            k = int(snap.kf_ids[s])
            if k in byid:
                o = int(snap.kp_off[s])
                lv = np.asarray(byid[k].kp_level, np.int64)
                lev_pool[o:o + len(lv)] = lv
        exp = np.zeros((n, L), np.int64)
        np.add.at(exp, (pid, lev_pool[snap.kp_off[slots] + snap.obs_kp]), 1)
        alive = np.flatnonzero(snap.alive)
        if not np.array_equal(exp[alive], snap.counts[alive].astype(np.int64)):
            bad.append("per-level counters differ from the observations")
        if sample_rep:
            rng = np.random.default_rng(seed)
            cand = alive[snap.nobs[alive] > 0]
            pick = rng.choice(cand, size=min(sample_rep, len(cand)), replace=False)
            starts = np.concatenate([[0], np.cumsum(snap.nobs)])
            for i in pick:
                a, b = starts[i], starts[i + 1]
                ent = sorted(zip(snap.obs_kf[a:b].tolist(), snap.obs_kp[a:b].tolist()))
                descs = np.stack([np.asarray(byid[k].descriptors)[kp] for k, kp in ent])
                if not np.array_equal(rep_descriptor(descs), snap.rep[i]):
                    bad.append(f"representative descriptor of point {int(i)}")
    return bad
