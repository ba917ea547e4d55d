"""TEST INFRASTRUCTURE ONLY -- CPU oracle for the triangulate + fuse hot path.

This module is the parity checker, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg
may import it. The CUDA path in ``paper_2511_02036_b200`` must never route through here.

It restates, in NumPy, the reference ``localmap`` package's algorithm for
CreateNewMapPoints + SearchAndFuse (plus the recent-point cull that runs between
keyframes), evaluating every floating-point expression in the reference's order so that
its outputs are bit-identical to the reference on the same inputs. Pinning: the script
``tests/golden/make_golden.py`` runs the real reference (importable only in the build
container) and freezes its outputs; ``tests/test_oracle_golden.py`` checks this module
against those fixtures. Function-by-function provenance (paths relative to
``/root/reference/pkg/src/localmap``):

  pose math ............ geometry.py:33-114, 193-198      fundamental ... geometry.py:287-304
  epipolar ............. geometry.py:307-322              DLT ........... geometry.py:258-284
  gates ................ geometry.py:341-353, 407-459     hamming ....... geometry.py:373-396
  map state ............ mapmodel.py:80-353               search ........ triangulation.py:63-136
  create_map_points .... triangulation.py:195-300         fusion ........ fusion.py:38-347
  recent-point cull .... culling.py:28-59                 per-KF driver . pipeline.py:152-195
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass, field

import numpy as np

UNBOUND = -1
INF_KEY = np.int64(1 << 40)


class OracleError(Exception):
    pass


# ----------------------------------------------------------------------------- pose math


def rot_of(q) -> np.ndarray:
    """Rotation matrix of a canonical unit quaternion (x, y, z, w), elementwise form."""
    x, y, z, w = q
    xx, yy, zz = x * x, y * y, z * z
    xy, xz, yz = x * y, x * z, y * z
    wx, wy, wz = w * x, w * y, w * z
    return np.array([[1 - 2 * (yy + zz), 2 * (xy - wz), 2 * (xz + wy)],
                     [2 * (xy + wz), 1 - 2 * (xx + zz), 2 * (yz - wx)],
                     [2 * (xz - wy), 2 * (yz + wx), 1 - 2 * (xx + yy)]])


def rows_dot(r, x, y, z):
    return (r[0, 0] * x + r[0, 1] * y + r[0, 2] * z,
            r[1, 0] * x + r[1, 1] * y + r[1, 2] * z,
            r[2, 0] * x + r[2, 1] * y + r[2, 2] * z)


def canon_quat(q):
    q = np.array(q, dtype=np.float64)
    n = np.sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3])
    q /= n
    return -q if q[3] < 0 else q


def cam_center(q, t):
    c = rows_dot(rot_of(q).T, t[0], t[1], t[2])
    return np.array([-c[0], -c[1], -c[2]])


def cam_apply(q, t, p):
    r = rows_dot(rot_of(q), p[0], p[1], p[2])
    return np.array([r[0] + t[0], r[1] + t[1], r[2] + t[2]])


def kmat(cam):
    return np.array([[cam.fx, 0.0, cam.cx], [0.0, cam.fy, cam.cy], [0.0, 0.0, 1.0]])


def fundamental(qa, ta, ca, qb, tb, cb):
    """F mapping pixels of view a to lines in view b, or None for zero baseline."""
    x, y, z, w = qa
    ai = rows_dot(rot_of(qa).T, ta[0], ta[1], ta[2])
    qi = canon_quat([-x, -y, -z, w])
    ti = np.array([-ai[0], -ai[1], -ai[2]])
    bx, by, bz, bw = qb
    ix, iy, iz, iw = qi
    qr = canon_quat([bw * ix + bx * iw + by * iz - bz * iy,
                     bw * iy - bx * iz + by * iw + bz * ix,
                     bw * iz + bx * iy - by * ix + bz * iw,
                     bw * iw - bx * ix - by * iy - bz * iz])
    rt = rows_dot(rot_of(qb), ti[0], ti[1], ti[2])
    t = np.array([rt[0] + tb[0], rt[1] + tb[1], rt[2] + tb[2]])
    if float(np.sqrt(t[0] ** 2 + t[1] ** 2 + t[2] ** 2)) < 1e-9:
        return None
    sk = np.array([[0.0, -t[2], t[1]], [t[2], 0.0, -t[0]], [-t[1], t[0], 0.0]])
    e = sk @ rot_of(qr)
    return np.linalg.inv(kmat(cb)).T @ e @ np.linalg.inv(kmat(ca))


def epi_d2(f, ua, va, ub, vb):
    l0 = f[0, 0] * ua + f[0, 1] * va + f[0, 2]
    l1 = f[1, 0] * ua + f[1, 1] * va + f[1, 2]
    l2 = f[2, 0] * ua + f[2, 1] * va + f[2, 2]
    num = l0 * ub + l1 * vb + l2
    num = num * num
    den = l0 * l0 + l1 * l1
    with np.errstate(divide="ignore", invalid="ignore"):
        d2 = num / den
    return np.where(den > 0, d2, np.inf)


def popc_rows(a, b):
    """Hamming distance of paired rows, (..., 32) uint8 -> int64."""
    return np.bitwise_count(np.bitwise_xor(a, b)).sum(axis=-1, dtype=np.int64)


def popc_cross(a, b):
    return np.bitwise_count(np.bitwise_xor(a[:, None, :], b[None, :, :])).sum(axis=2, dtype=np.int64)


# ----------------------------------------------------------------------------- map state


@dataclass
class Cam:
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    num_levels: int = 8
    scale_factor: float = 1.2


@dataclass
class OKF:
    kf_id: int
    quat: np.ndarray
    trans: np.ndarray
    cam: Cam
    u: np.ndarray
    v: np.ndarray
    level: np.ndarray
    desc: np.ndarray
    bind: np.ndarray
    alive: bool = True

    @property
    def n(self):
        return len(self.u)

    def center(self):
        return cam_center(self.quat, self.trans)


@dataclass
class OPoint:
    mp_id: int
    pos: np.ndarray
    rep: np.ndarray
    first_kf: int
    obs: dict = field(default_factory=dict)
    found: int = 1
    visible: int = 1
    alive: bool = True


class OracleMap:
    """Single-writer map: keyframes, points, per-level counters, covisibility weights."""

    def __init__(self, num_levels: int = 8, min_covis_weight: int = 1, min_obs_keep: int = 2):
        self.L = num_levels
        self.min_w = min_covis_weight
        self.min_obs_keep = min_obs_keep
        self.kfs: dict[int, OKF] = {}
        self.pts: dict[int, OPoint] = {}
        self.adj: dict[int, dict[int, int]] = {}
        self.counts: dict[int, np.ndarray] = {}
        self.next_id = 0

    # -- covisibility (mapmodel.py:80-110)
    def _bump(self, a, b, d):
        if a == b:
            return
        for x, y in ((a, b), (b, a)):
            row = self.adj.setdefault(x, {})
            w = row.get(y, 0) + d
            if w <= 0:
                row.pop(y, None)
            else:
                row[y] = w

    def weight(self, a, b):
        return self.adj.get(a, {}).get(b, 0)

    def neighbors(self, kf_id, n=None):
        row = self.adj.get(kf_id, {})
        ranked = sorted(((k, w) for k, w in row.items() if w >= self.min_w), key=lambda p: (-p[1], p[0]))
        ids = [k for k, _ in ranked if self.kfs[k].alive]
        return ids if n is None else ids[:n]

    # -- observation bookkeeping (mapmodel.py:150-181)
    def _link(self, p: OPoint, kf: OKF, kp: int):
        for other in p.obs:
            self._bump(kf.kf_id, other, +1)
        p.obs[kf.kf_id] = kp
        kf.bind[kp] = p.mp_id
        self.counts[p.mp_id][kf.level[kp]] += 1

    def _unlink(self, p: OPoint, kf_id: int):
        kp = p.obs.pop(kf_id)
        kf = self.kfs[kf_id]
        kf.bind[kp] = UNBOUND
        self.counts[p.mp_id][kf.level[kp]] -= 1
        for other in p.obs:
            self._bump(kf_id, other, -1)

    def refresh_rep(self, p: OPoint):
        """Observing descriptor with the smallest median distance to the others; first wins.

        The reference's nanmedian over float distances equals half the sum of the two
        middle order statistics of the n-1 off-diagonal integers, so it is compared as
        that (exact) integer sum here.
        """
        items = sorted(p.obs.items())
        if not items:
            return
        d = np.stack([self.kfs[k].desc[i] for k, i in items])
        if len(items) == 1:
            p.rep = d[0].copy()
            return
        m = popc_cross(d, d)
        np.fill_diagonal(m, 1 << 20)
        s = np.sort(m, axis=1)
        k = len(items) - 1
        med2 = s[:, (k - 1) // 2] + s[:, k // 2]
        p.rep = d[int(np.argmin(med2))].copy()

    # -- public ops (mapmodel.py:185-300)
    def insert_keyframe(self, kf: OKF):
        if kf.kf_id in self.kfs:
            raise OracleError(f"duplicate keyframe {kf.kf_id}")
        self.kfs[kf.kf_id] = kf
        for kp in np.flatnonzero(kf.bind != UNBOUND):
            p = self.pts[int(kf.bind[kp])]
            if not p.alive or kf.kf_id in p.obs:
                raise OracleError("bad pre-bound slot")
            self._link(p, kf, int(kp))
            self.refresh_rep(p)

    def new_point(self, pos, desc, first_kf) -> OPoint:
        p = OPoint(self.next_id, np.asarray(pos, dtype=np.float64).copy(),
                   np.asarray(desc, dtype=np.uint8).copy(), first_kf)
        self.pts[p.mp_id] = p
        self.counts[p.mp_id] = np.zeros(self.L, dtype=np.int64)
        self.next_id += 1
        return p

    def add_obs(self, mp_id, kf_id, kp):
        p = self.pts[mp_id]
        kf = self.kfs[kf_id]
        if not p.alive or not kf.alive:
            raise OracleError("dead entity")
        if kf.bind[kp] != UNBOUND or kf_id in p.obs:
            raise OracleError("slot conflict")
        self._link(p, kf, kp)
        self.refresh_rep(p)

    def erase_obs(self, mp_id, kf_id):
        p = self.pts[mp_id]
        self._unlink(p, kf_id)
        if len(p.obs) < self.min_obs_keep:
            self.kill_point(mp_id)
        else:
            self.refresh_rep(p)

    def kill_point(self, mp_id):
        p = self.pts[mp_id]
        for k in sorted(p.obs):
            self._unlink(p, k)
        p.alive = False

    def replace(self, loser_id, winner_id):
        lo, wi = self.pts[loser_id], self.pts[winner_id]
        for k, kp in sorted(lo.obs.items()):
            self._unlink(lo, k)
            if k not in wi.obs:
                self._link(wi, self.kfs[k], kp)
        wi.found += lo.found
        wi.visible += lo.visible
        lo.alive = False
        self.refresh_rep(wi)

    def kill_keyframe(self, kf_id):
        """mapmodel.py:275-283 (+ CovisibilityGraph.drop_keyframe 107-110)."""
        kf = self.kfs[kf_id]
        for mp_id in sorted(set(int(m) for m in kf.bind if m != UNBOUND)):
            p = self.pts[mp_id]
            if p.alive and kf_id in p.obs:
                self.erase_obs(mp_id, kf_id)
        kf.alive = False
        for other in self.adj.pop(kf_id, {}):
            self.adj.get(other, {}).pop(kf_id, None)

    def bound_points(self, kf_id):
        out = []
        for m in self.kfs[kf_id].bind:
            if m != UNBOUND and self.pts[int(m)].alive:
                out.append(int(m))
        return out

    def live_points(self):
        return [p for p in self.pts.values() if p.alive]

    def audit(self) -> list[str]:
        bad = []
        for p in self.pts.values():
            if not p.alive:
                if p.obs:
                    bad.append(f"dead {p.mp_id} keeps obs")
                continue
            exp = np.zeros(self.L, dtype=np.int64)
            for k, kp in p.obs.items():
                kf = self.kfs[k]
                if not kf.alive or kf.bind[kp] != p.mp_id:
                    bad.append(f"binding {p.mp_id} ({k},{kp})")
                exp[kf.level[kp]] += 1
            if not np.array_equal(exp, self.counts[p.mp_id]):
                bad.append(f"counters {p.mp_id}")
        live = sorted(k for k, kf in self.kfs.items() if kf.alive)
        sets = {k: set(self.bound_points(k)) for k in live}
        for i, a in enumerate(live):
            for b in live[i + 1:]:
                if len(sets[a] & sets[b]) != self.weight(a, b):
                    bad.append(f"covis ({a},{b})")
        return bad


# ----------------------------------------------------------------------------- triangulation


@dataclass
class CreateStats:
    created: int = 0
    conflicts: int = 0
    degenerate: int = 0
    gate_failures: dict = field(default_factory=dict)
    degenerate_neighbors: list = field(default_factory=list)


def search_pairs(cur: OKF, nbr: OKF, f, chi2_epi, max_dist, level_window, unb_cur, unb_nbr):
    """Per unbound current keypoint: lowest (distance, neighbour index) among unbound,
    level-window, distance<=max, epipolar<=thr neighbour keypoints; then one-to-one per
    neighbour keypoint keeping the lowest (distance, current index); sorted by current."""
    sig2 = np.array([nbr.cam.scale_factor ** (2 * lv) for lv in range(nbr.cam.num_levels)])
    thr = chi2_epi * sig2[nbr.level]
    rows = np.flatnonzero(unb_cur)
    picks = []
    for s in range(0, len(rows), 256):
        blk = rows[s:s + 256]
        dist = popc_cross(cur.desc[blk], nbr.desc)
        ok = unb_nbr[None, :] & (np.abs(nbr.level[None, :] - cur.level[blk][:, None]) <= level_window)
        ok &= dist <= max_dist
        ri, ci = np.nonzero(ok)
        if len(ri):
            gi = blk[ri]
            ok[ri, ci] = epi_d2(f, cur.u[gi], cur.v[gi], nbr.u[ci], nbr.v[ci]) <= thr[ci]
        key = np.where(ok, dist * np.int64(nbr.n) + np.arange(nbr.n, dtype=np.int64)[None, :], INF_KEY)
        best = key.min(axis=1) if nbr.n else np.full(len(blk), INF_KEY)
        for r in np.flatnonzero(best < INF_KEY):
            picks.append((int(blk[r]), int(best[r] % nbr.n), int(best[r] // nbr.n)))
    keep: dict[int, tuple[int, int]] = {}
    for i, j, d in picks:
        if j not in keep or (d, i) < keep[j]:
            keep[j] = (d, i)
    return sorted(((i, j, d) for j, (d, i) in keep.items()))


def dlt_point(qa, ta, ca_cam, qb, tb, cb_cam, pa, pb):
    """Homogeneous DLT; returns (point or None for degenerate)."""
    ca, cb = cam_center(qa, ta), cam_center(qb, tb)
    if float(np.sqrt(np.sum((ca - cb) ** 2))) < 1e-9:
        return None
    def pmat(q, t, cam):
        m = np.eye(4)
        m[:3, :3] = rot_of(q)
        m[:3, 3] = t
        return kmat(cam) @ m[:3, :]
    pa_m, pb_m = pmat(qa, ta, ca_cam), pmat(qb, tb, cb_cam)
    a = np.empty((4, 4))
    a[0] = pa[0] * pa_m[2] - pa_m[0]
    a[1] = pa[1] * pa_m[2] - pa_m[1]
    a[2] = pb[0] * pb_m[2] - pb_m[0]
    a[3] = pb[1] * pb_m[2] - pb_m[1]
    h = np.linalg.svd(a)[2][-1]
    if abs(h[3]) < 1e-12:
        return None
    return h[:3] / h[3]


def gate_reason(a: OKF, b: OKF, pa, pb, la, lb, point, cos_max, chi2_mono, slack):
    """None if the candidate passes, else the first failing gate's name."""
    ca, cb = a.center(), b.center()
    ra, rb = point - ca, point - cb
    na = float(np.sqrt(ra[0] ** 2 + ra[1] ** 2 + ra[2] ** 2))
    nb = float(np.sqrt(rb[0] ** 2 + rb[1] ** 2 + rb[2] ** 2))
    if na < 1e-12 or nb < 1e-12:
        return "parallax"
    c = float(ra[0] * rb[0] + ra[1] * rb[1] + ra[2] * rb[2]) / (na * nb)
    if not (min(1.0, max(-1.0, c)) < cos_max):
        return "parallax"
    xa, xb = cam_apply(a.quat, a.trans, point), cam_apply(b.quat, b.trans, point)
    if xa[2] <= 0 or xb[2] <= 0:
        return "positive-depth"
    for kf, x, pix, lv in ((a, xa, pa, la), (b, xb, pb, lb)):
        u = kf.cam.fx * (x[0] / x[2]) + kf.cam.cx
        v = kf.cam.fy * (x[1] / x[2]) + kf.cam.cy
        if (u - pix[0]) ** 2 + (v - pix[1]) ** 2 > chi2_mono * kf.cam.scale_factor ** (2 * lv):
            return "reprojection"
    da = float(np.sqrt(np.sum((point - ca) ** 2)))
    db = float(np.sqrt(np.sum((point - cb) ** 2)))
    if da < 1e-12 or db < 1e-12:
        return "scale"
    rd = da / db
    rs = a.cam.scale_factor ** la / b.cam.scale_factor ** lb
    sl = slack * max(a.cam.scale_factor, b.cam.scale_factor)
    if not (rs / sl <= rd <= rs * sl):
        return "scale"
    return None


@dataclass
class MatchCfg:
    match_max_distance: int = 50
    chi2_epi: float = 3.84
    level_window: int = 1


@dataclass
class GateCfg:
    cos_parallax_max: float = 0.9998
    chi2_mono: float = 5.991
    scale_ratio_slack: float = 1.5


def pick_neighbors(m: OracleMap, cur_id: int, n: int) -> list[int]:
    nb = m.neighbors(cur_id, n)
    if len(nb) < n:
        for k in sorted((k for k, kf in m.kfs.items() if kf.alive and k != cur_id), reverse=True):
            if len(nb) >= n:
                break
            if k not in nb:
                nb.append(k)
    return nb


def create_points(m: OracleMap, cur_id: int, n: int, mc: MatchCfg = None, gc: GateCfg = None,
                  stats: CreateStats = None, log: dict | None = None) -> list[int]:
    mc, gc = mc or MatchCfg(), gc or GateCfg()
    stats = stats if stats is not None else CreateStats()
    cur = m.kfs[cur_id]
    nbrs = pick_neighbors(m, cur_id, n)
    if log is not None:
        log["neighbors"] = list(nbrs)
    if not nbrs:
        return []
    unb_cur = cur.bind == UNBOUND
    snap = {k: m.kfs[k].bind == UNBOUND for k in nbrs}
    cands = []
    for k in nbrs:
        nb = m.kfs[k]
        f = fundamental(cur.quat, cur.trans, cur.cam, nb.quat, nb.trans, nb.cam)
        got = [] if f is None else search_pairs(cur, nb, f, mc.chi2_epi, mc.match_max_distance,
                                                 mc.level_window, unb_cur, snap[k])
        if not got and f is None:
            stats.degenerate_neighbors.append(k)
        cands.extend((k, i, j, d) for i, j, d in got)
    if log is not None:
        log["candidates"] = list(cands)
    out = []
    for k, i, j, d in cands:
        nb = m.kfs[k]
        if cur.bind[i] != UNBOUND or nb.bind[j] != UNBOUND:
            stats.conflicts += 1
            continue
        pa, pb = (cur.u[i], cur.v[i]), (nb.u[j], nb.v[j])
        x = dlt_point(cur.quat, cur.trans, cur.cam, nb.quat, nb.trans, nb.cam, pa, pb)
        if x is None:
            stats.degenerate += 1
            continue
        why = gate_reason(cur, nb, pa, pb, int(cur.level[i]), int(nb.level[j]), x,
                          gc.cos_parallax_max, gc.chi2_mono, gc.scale_ratio_slack)
        if why is not None:
            stats.gate_failures[why] = stats.gate_failures.get(why, 0) + 1
            continue
        p = m.new_point(x, cur.desc[i], cur_id)
        m.add_obs(p.mp_id, cur_id, i)
        m.add_obs(p.mp_id, k, j)
        out.append(p.mp_id)
        stats.created += 1
    return out


# ----------------------------------------------------------------------------- fusion

MERGE = "merge"
ADD = "add-observation"


@dataclass
class FuseCfg:
    match_max_distance: int = 50
    fuse_radius: float = 3.0
    min_view_cos: float = 0.5
    dist_band_slack: float = 1.5
    level_window: int = 1
    n1: int = 20
    n2: int = 5


def fusion_targets(m: OracleMap, cur_id, n1, n2):
    first = m.neighbors(cur_id, n1)
    out, seen = list(first), set(first) | {cur_id}
    for f in first:
        got = 0
        for s in m.neighbors(f):
            if got >= n2:
                break
            if s not in seen:
                out.append(s)
                seen.add(s)
                got += 1
    return out


def point_views(m: OracleMap, ids, slack, L, sf):
    n = len(ids)
    pos, rep = np.zeros((n, 3)), np.zeros((n, 32), dtype=np.uint8)
    lo_a, hi_a, view = np.zeros(n), np.zeros(n), np.zeros((n, 3))
    live = np.zeros(n, dtype=bool)
    for r, pid in enumerate(ids):
        p = m.pts.get(pid)
        if p is None or not p.alive or not p.obs:
            continue
        live[r] = True
        pos[r], rep[r] = p.pos, p.rep
        lo, hi, acc = np.inf, -np.inf, np.zeros(3)
        for k, kp in sorted(p.obs.items()):
            kf = m.kfs[k]
            ray = p.pos - kf.center()
            dd = float(np.sqrt(ray[0] ** 2 + ray[1] ** 2 + ray[2] ** 2))
            if dd <= 0:
                continue
            d0 = dd / sf ** int(kf.level[kp])
            lo, hi = min(lo, d0), max(hi, d0)
            acc += ray / dd
        if not np.isfinite(lo):
            live[r] = False
            continue
        nrm = float(np.sqrt(acc[0] ** 2 + acc[1] ** 2 + acc[2] ** 2))
        view[r] = acc / nrm if nrm > 0 else acc
        lo_a[r], hi_a[r] = lo, hi
    return pos, rep, live, lo_a / slack, hi_a * sf ** (L - 1) * slack, lo_a, view


def fuse_gather(m: OracleMap, ids, tgt_id, fc: FuseCfg = None):
    """(actions, visible ids) of projecting `ids` into keyframe `tgt_id`."""
    fc = fc or FuseCfg()
    t = m.kfs[tgt_id]
    if not ids:
        return [], []
    L, sf = t.cam.num_levels, t.cam.scale_factor
    pos, rep, live, blo, bhi, d0, view = point_views(m, ids, fc.dist_band_slack, L, sf)
    r = rot_of(t.quat)
    tt = t.trans
    c = t.center()
    px, py, pz = pos[:, 0], pos[:, 1], pos[:, 2]
    qx, qy, qz = rows_dot(r, px, py, pz)
    zc = qz + tt[2]
    with np.errstate(divide="ignore", invalid="ignore"):
        u = t.cam.fx * ((qx + tt[0]) / zc) + t.cam.cx
        v = t.cam.fy * ((qy + tt[1]) / zc) + t.cam.cy
    inview = (zc > 0) & (u >= 0) & (u < t.cam.width) & (v >= 0) & (v < t.cam.height)
    dx, dy, dz = px - c[0], py - c[1], pz - c[2]
    d = np.sqrt(dx * dx + dy * dy + dz * dz)
    with np.errstate(divide="ignore", invalid="ignore"):
        cosv = (dx * view[:, 0] + dy * view[:, 1] + dz * view[:, 2]) / d
        lraw = np.log(d / d0) / np.log(sf)
    lraw = np.where(np.isfinite(lraw), lraw, 0.0)
    lp = np.clip(np.rint(lraw), 0, L - 1).astype(np.int64)
    rad = fc.fuse_radius * np.array([sf ** lv for lv in range(L)])[lp]
    ok = live & (zc > 0) & inview & (d >= blo) & (d <= bhi) & (cosv >= fc.min_view_cos)
    visible = [ids[i] for i in np.flatnonzero(ok)]
    acts = []
    for i in np.flatnonzero(ok):
        du, dv = t.u - u[i], t.v - v[i]
        win = np.flatnonzero((du * du + dv * dv <= rad[i] * rad[i]) & (np.abs(t.level - lp[i]) <= fc.level_window))
        if not len(win):
            continue
        dist = popc_rows(t.desc[win], rep[i][None, :])
        good = dist <= fc.match_max_distance
        if not good.any():
            continue
        j = int(win[int(np.argmin(np.where(good, dist, INF_KEY)))])
        pid = ids[i]
        owner = int(t.bind[j])
        if owner == UNBOUND:
            if tgt_id not in m.pts[pid].obs:
                acts.append((tgt_id, pid, j, None, ADD))
        elif owner != pid and m.pts[owner].alive:
            acts.append((tgt_id, pid, j, owner, MERGE))
    return acts, visible


def _merge_pair(m: OracleMap, a: OPoint, b: OPoint):
    if len(a.obs) == len(b.obs):
        lo, wi = (a, b) if a.mp_id > b.mp_id else (b, a)
    elif len(a.obs) < len(b.obs):
        lo, wi = a, b
    else:
        lo, wi = b, a
    m.replace(lo.mp_id, wi.mp_id)
    wi.found += 1


def fuse_apply(m: OracleMap, acts) -> dict:
    cnt = {"merged": 0, "observations_added": 0, "stale": 0}
    for tgt, pid, j, other_id, kind in acts:
        p = m.pts.get(pid)
        t = m.kfs.get(tgt)
        if p is None or not p.alive or t is None or not t.alive:
            cnt["stale"] += 1
            continue
        if kind == MERGE:
            o = m.pts.get(other_id)
            if o is None or not o.alive or o.mp_id == p.mp_id or int(t.bind[j]) != o.mp_id:
                cnt["stale"] += 1
                continue
            _merge_pair(m, p, o)
            cnt["merged"] += 1
            continue
        now = int(t.bind[j])
        if now != UNBOUND:
            o = m.pts.get(now)
            if o is None or not o.alive or o.mp_id == p.mp_id:
                cnt["stale"] += 1
                continue
            _merge_pair(m, p, o)
            cnt["merged"] += 1
            continue
        if tgt in p.obs:
            cnt["stale"] += 1
            continue
        m.add_obs(pid, tgt, j)
        p.found += 1
        cnt["observations_added"] += 1
    return cnt


def fuse_keyframe(m: OracleMap, cur_id, fc: FuseCfg = None, log: dict | None = None) -> dict:
    fc = fc or FuseCfg()
    tot = {"merged": 0, "observations_added": 0, "stale": 0}
    targets = fusion_targets(m, cur_id, fc.n1, fc.n2)
    if log is not None:
        log["targets"] = list(targets)
        log["passes"] = []
    if not targets:
        return tot
    fwd = m.bound_points(cur_id)
    batch = []
    for t in targets:
        acts, vis = fuse_gather(m, fwd, t, fc)
        batch.extend(acts)
        for pid in vis:
            m.pts[pid].visible += 1
        if log is not None:
            log["passes"].append(("fwd", t, acts, vis))
    for k, v in fuse_apply(m, batch).items():
        tot[k] += v
    for t in targets:
        pts = m.bound_points(t)
        acts, vis = fuse_gather(m, pts, cur_id, fc)
        for pid in vis:
            if m.pts[pid].alive:
                m.pts[pid].visible += 1
        if log is not None:
            log["passes"].append(("rev", t, acts, vis))
        for k, v in fuse_apply(m, acts).items():
            tot[k] += v
    return tot


# ----------------------------------------------------------------------------- cull + driver


@dataclass
class CullCfg:
    found_ratio_min: float = 0.25
    probation_kfs: int = 3
    min_obs_graduate: int = 3


def cull_recent(m: OracleMap, recent: list, now: int, cc: CullCfg = None):
    cc = cc or CullCfg()
    removed, keep = [], []
    for mp_id, born in recent:
        p = m.pts.get(mp_id)
        if p is None or not p.alive:
            continue
        if p.found / max(p.visible, 1) < cc.found_ratio_min:
            m.kill_point(mp_id)
            removed.append(mp_id)
        elif now - born >= cc.probation_kfs:
            if len(p.obs) < cc.min_obs_graduate:
                m.kill_point(mp_id)
                removed.append(mp_id)
        else:
            keep.append((mp_id, born))
    return removed, keep


@dataclass
class KfCullCfg:
    redundancy_ratio: float = 0.9
    min_redundant_observers: int = 3
    scale_tolerance_levels: int = 0


def kf_redundant(m: OracleMap, kf_id: int, cc: KfCullCfg) -> bool:
    """is_redundant_baseline culling.py:60-92 (observation-list walk)."""
    kf = m.kfs[kf_id]
    red = considered = 0
    for kp, mp_id in enumerate(kf.bind):
        if mp_id == UNBOUND or not m.pts[int(mp_id)].alive:
            continue
        considered += 1
        limit = int(kf.level[kp]) + cc.scale_tolerance_levels
        others = sum(1 for k2, kp2 in m.pts[int(mp_id)].obs.items() if k2 != kf_id and int(m.kfs[k2].level[kp2]) <= limit)
        red += others >= cc.min_redundant_observers
    return considered > 0 and red >= cc.redundancy_ratio * considered


def cull_keyframes(m: OracleMap, candidates, cc: KfCullCfg = None) -> list[int]:
    """culling.py:127-154 (the store's eviction is the caller's)."""
    cc = cc or KfCullCfg()
    removed = []
    for k in sorted(set(candidates)):
        if k == 0 or k not in m.kfs or not m.kfs[k].alive:
            continue
        if kf_redundant(m, k, cc):
            m.kill_keyframe(k)
            removed.append(k)
    return removed


class OraclePipeline:
    """Per keyframe: insert -> recent-point cull -> create -> fuse (pipeline.py:152-195,
    with LBA and keyframe culling force-skipped as in the throughput benches)."""

    def __init__(self, num_levels=8, neighbor_count=10, mc=None, gc=None, fc=None, cc=None):
        self.map = OracleMap(num_levels)
        self.n = neighbor_count
        self.mc, self.gc, self.fc, self.cc = mc or MatchCfg(), gc or GateCfg(), fc or FuseCfg(), cc or CullCfg()
        self.recent: list = []
        self.processed = 0
        self.stats = CreateStats()
        self.fused = {"merged": 0, "observations_added": 0, "stale": 0}
        self.culled: list = []

    def step(self, kf: OKF):
        self.map.insert_keyframe(kf)
        removed, self.recent = cull_recent(self.map, self.recent, self.processed, self.cc)
        self.culled.extend(removed)
        made = create_points(self.map, kf.kf_id, self.n, self.mc, self.gc, self.stats)
        self.recent.extend((i, self.processed) for i in made)
        for k, v in fuse_keyframe(self.map, kf.kf_id, self.fc).items():
            self.fused[k] += v
        self.processed += 1
        return made


# ----------------------------------------------------------------------------- digests


def structural_digest(m: OracleMap) -> str:
    """Everything but point positions, bitwise (positions are tolerance-checked apart)."""
    h = hashlib.sha256()
    for k in sorted(k for k, kf in m.kfs.items() if kf.alive):
        h.update(f"kf {k} ".encode())
        h.update(np.asarray(m.kfs[k].bind, dtype=np.int64).tobytes())
    for p in sorted(m.live_points(), key=lambda p: p.mp_id):
        h.update(f"mp {p.mp_id} {p.found} {p.visible} ".encode())
        h.update(p.rep.tobytes())
        h.update(str(sorted(p.obs.items())).encode())
        h.update(np.asarray(m.counts[p.mp_id], dtype=np.int64).tobytes())
    return h.hexdigest()


def okf_from_record(rec, cam: Cam) -> OKF:
    """Oracle keyframe from a workload record (fields kp_u, kp_v, kp_level, descriptors)."""
    return OKF(int(rec.kf_id), np.array(rec.pose_init.quat, dtype=np.float64),
               np.array(rec.pose_init.trans, dtype=np.float64), cam,
               np.array(rec.kp_u, dtype=np.float64), np.array(rec.kp_v, dtype=np.float64),
               np.array(rec.kp_level, dtype=np.int64), np.array(rec.descriptors, dtype=np.uint8),
               np.full(len(rec.kp_u), UNBOUND, dtype=np.int64))
