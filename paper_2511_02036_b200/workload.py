"""Seeded synthetic local-mapping workloads (bench and test inputs, not the hot path).

Restates the reference's generator (pkg/src/localmap/synth.py) so that the same
``WorldConfig`` yields the *same* keyframes, bit for bit, without the reference installed
(it is absent on the GPU box). The random stream is consumed in exactly the reference's
order: landmarks (synth.py:190-224), base descriptors, duplicate twins (synth.py:244-263),
then per keyframe a visibility permutation, pixel noise, per-observation bit flips,
spurious features and pose noise (synth.py:277-363). ``tests/test_workload.py`` pins the
output against golden digests produced by the reference itself.

``BENCH_CONFIGS`` names the BASELINE.json configs.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import InvalidArgumentError, LocalMapError
from .geometry import CameraIntrinsics, SE3Pose, exp_so3, flip_descriptor_bits, random_descriptors

LINE, ORBIT, CORRIDOR = "line", "orbit", "corridor-loop"


@dataclass
class WorldConfig:
    seed: int = 0
    landmark_count: int = 400
    extent: float = 20.0
    trajectory: str = LINE
    keyframe_count: int = 30
    features_per_kf: int = 300
    pixel_noise_sigma: float = 0.0
    descriptor_flip_bits: int = 0
    spurious_feature_fraction: float = 0.0
    duplicate_injection_rate: float = 0.0
    twin_flip_bits: int = 45
    pose_noise_trans: float | None = None
    pose_noise_rot_deg: float | None = None
    frames_per_keyframe: int = 10
    min_covisible: int = 20
    retry_budget: int = 5
    width: int = 640
    height: int = 480
    fx: float = 460.0
    fy: float = 460.0
    cx: float = 320.0
    cy: float = 240.0
    num_levels: int = 8
    scale_factor: float = 1.2
    depth_near: float = 2.0
    depth_far: float = 40.0

    def __post_init__(self):
        if self.trajectory not in (LINE, ORBIT, CORRIDOR):
            raise InvalidArgumentError(f"unknown trajectory kind {self.trajectory!r}")
        if self.keyframe_count < 2 or self.landmark_count < 1:
            raise InvalidArgumentError("need at least 2 keyframes and 1 landmark")
        if self.pose_noise_trans is None:
            self.pose_noise_trans = 0.02 * self.pixel_noise_sigma
        if self.pose_noise_rot_deg is None:
            self.pose_noise_rot_deg = 0.2 * self.pixel_noise_sigma

    def intrinsics(self) -> CameraIntrinsics:
        return CameraIntrinsics(self.fx, self.fy, self.cx, self.cy, self.width, self.height,
                                self.num_levels, self.scale_factor)


@dataclass
class FrameRecord:
    kf_id: int
    frame_index: int
    pose_gt: SE3Pose
    pose_init: SE3Pose
    kp_u: np.ndarray
    kp_v: np.ndarray
    kp_level: np.ndarray
    descriptors: np.ndarray
    landmark_ids: np.ndarray


@dataclass
class Sequence:
    config: WorldConfig
    landmarks: np.ndarray
    canonical_ids: np.ndarray
    duplicate_pairs: list
    records: list = field(default_factory=list)

    def intrinsics(self) -> CameraIntrinsics:
        return self.config.intrinsics()


def _aim(center, target, up=(0.0, -1.0, 0.0)) -> SE3Pose:
    """Camera at `center` looking at `target` (synth.py:175-187)."""
    up = np.asarray(up, dtype=np.float64)
    fwd = np.asarray(target, dtype=np.float64) - center
    fwd = fwd / np.linalg.norm(fwd)
    right = np.cross(up, fwd)
    nr = np.linalg.norm(right)
    if nr < 1e-9:
        right = np.cross(np.array([1.0, 0.0, 0.0]), fwd)
        nr = np.linalg.norm(right)
    right /= nr
    down = np.cross(fwd, right)
    rot = np.stack([right, down, fwd])
    return SE3Pose.from_rotation_matrix(rot, -rot @ np.asarray(center, dtype=np.float64))


def _trajectory(cfg: WorldConfig) -> list[SE3Pose]:
    n = cfg.keyframe_count
    if cfg.trajectory == LINE:
        return [_aim(np.array([x, 0.0, 0.0]), np.array([x, 0.0, 10.0]))
                for x in np.linspace(-cfg.extent / 2, cfg.extent / 2, n)]
    zup = np.array([0.0, 0.0, 1.0])
    if cfg.trajectory == ORBIT:
        r = cfg.extent / 2
        out = []
        for i in range(n):
            a = 2 * np.pi * i / n
            out.append(_aim(np.array([r * np.cos(a), r * np.sin(a), 0.0]), np.zeros(3), up=zup))
        return out
    length, wid = cfg.extent, cfg.extent / 2
    corners = np.array([[0.0, 0.0], [length, 0.0], [length, wid], [0.0, wid], [0.0, 0.0]])
    seg = np.array([np.linalg.norm(corners[i + 1] - corners[i]) for i in range(4)])
    perim = float(seg.sum())

    def at(s):
        s = s % perim
        acc = 0.0
        for i in range(4):
            if s <= acc + seg[i] or i == 3:
                f = (s - acc) / seg[i]
                xy = corners[i] + f * (corners[i + 1] - corners[i])
                return np.array([xy[0], xy[1], 0.0])
            acc += seg[i]

    return [_aim(at(s), at(s + 5.0), up=zup) for s in np.linspace(0.0, perim, n, endpoint=False)]


def _landmarks(cfg: WorldConfig, rng) -> np.ndarray:
    n = cfg.landmark_count
    if cfg.trajectory == LINE:
        h = cfg.extent / 2
        return np.column_stack([rng.uniform(-h - 4, h + 4, n), rng.uniform(-4.0, 4.0, n),
                                rng.uniform(4.0, 16.0, n)])
    if cfg.trajectory == ORBIT:
        return rng.normal(0.0, cfg.extent / 8, (n, 3))
    length, wid = cfg.extent, cfg.extent / 2
    side = rng.integers(0, 4, n)
    along = rng.uniform(0.0, 1.0, n)
    lateral = rng.uniform(1.5, 5.0, n) * rng.choice([-1.0, 1.0], n)
    height = rng.uniform(-2.5, 2.5, n)
    pts = np.zeros((n, 3))
    frames = {0: (lambda a: [a * length, 0.0], [0.0, 1.0]),
              1: (lambda a: [length, a * wid], [-1.0, 0.0]),
              2: (lambda a: [length * (1 - a), wid], [0.0, -1.0]),
              3: (lambda a: [0.0, wid * (1 - a)], [1.0, 0.0])}
    for i in range(n):
        base_fn, perp = frames[int(side[i])]
        xy = np.array(base_fn(along[i])) + np.array(perp) * lateral[i]
        pts[i] = [xy[0], xy[1], height[i]]
    return pts


def _levels(depth: np.ndarray, cfg: WorldConfig) -> np.ndarray:
    base = (cfg.depth_far / cfg.depth_near) ** (1.0 / cfg.num_levels)
    d = np.maximum(depth, cfg.depth_near * 1.0001)
    lv = np.floor(np.log(d / cfg.depth_near) / np.log(base)).astype(np.int64)
    return np.clip(lv, 0, cfg.num_levels - 1)


def generate_sequence(cfg: WorldConfig) -> Sequence:
    rng = np.random.default_rng(cfg.seed)
    poses = _trajectory(cfg)
    why = ""
    for _ in range(max(1, cfg.retry_budget)):
        base = _landmarks(cfg, rng)
        base_desc = random_descriptors(rng, cfg.landmark_count)
        n_dup = int(round(cfg.duplicate_injection_rate * cfg.landmark_count))
        sources = rng.choice(cfg.landmark_count, size=n_dup, replace=False) if n_dup else np.zeros(0, int)
        pos, desc = [base], [base_desc]
        canon = list(range(cfg.landmark_count))
        parity = np.zeros(cfg.landmark_count, dtype=np.int64)
        pairs = []
        for src in sorted(int(s) for s in sources):
            twin = len(canon)
            pos.append(base[src:src + 1])
            desc.append(flip_descriptor_bits(rng, base_desc[src], cfg.twin_flip_bits)[None, :])
            canon.append(src)
            parity[src] = 1
            parity = np.append(parity, 2)
            pairs.append((src, twin))
        inst_pos, inst_desc = np.vstack(pos), np.vstack(desc)
        records, why = _observe(cfg, poses, inst_pos, inst_desc, parity, rng)
        if records is not None:
            return Sequence(cfg, inst_pos, np.array(canon, dtype=np.int64), pairs, records)
    raise LocalMapError(f"covisibility constraint unsatisfied after {cfg.retry_budget} attempts: {why}")


def _observe(cfg, poses, inst_pos, inst_desc, parity, rng):
    out = []
    prev: set[int] = set()
    rot_sigma = np.deg2rad(cfg.pose_noise_rot_deg)
    paired = (parity == 1).any()
    for kf_id, pose in enumerate(poses):
        cam_pts = (pose.rotation_matrix() @ inst_pos.T).T + pose.trans
        z = cam_pts[:, 2]
        with np.errstate(divide="ignore", invalid="ignore"):
            u = cfg.fx * (cam_pts[:, 0] / z) + cfg.cx
            v = cfg.fy * (cam_pts[:, 1] / z) + cfg.cy
        vis = ((z > cfg.depth_near * 0.5) & (z < cfg.depth_far * 1.5) & (u >= 0) & (u < cfg.width)
               & (v >= 0) & (v < cfg.height))
        if paired:
            want = 1 if kf_id % 2 == 0 else 2
            vis &= (parity == 0) | (parity == want)
        cand = np.flatnonzero(vis)
        take = np.sort(cand[rng.permutation(len(cand))[: cfg.features_per_kf]])
        us, vs = u[take], v[take]
        if cfg.pixel_noise_sigma > 0:
            us = us + rng.normal(0, cfg.pixel_noise_sigma, len(take))
            vs = vs + rng.normal(0, cfg.pixel_noise_sigma, len(take))
            keep = (us >= 0) & (us < cfg.width) & (vs >= 0) & (vs < cfg.height)
            take, us, vs = take[keep], us[keep], vs[keep]
        levels = _levels(z[take], cfg)
        if cfg.descriptor_flip_bits > 0 and len(take):
            d = np.stack([flip_descriptor_bits(rng, inst_desc[i], cfg.descriptor_flip_bits) for i in take])
        elif cfg.descriptor_flip_bits > 0:
            d = np.zeros((0, 32), dtype=np.uint8)
        else:
            d = inst_desc[take].copy()
        ids = take.astype(np.int64)
        n_spur = int(round(cfg.spurious_feature_fraction * len(take)))
        if n_spur:
            su = rng.uniform(0, cfg.width, n_spur)
            sv = rng.uniform(0, cfg.height, n_spur)
            sl = rng.integers(0, cfg.num_levels, n_spur)
            sd = random_descriptors(rng, n_spur)
            us, vs = np.concatenate([us, su]), np.concatenate([vs, sv])
            levels = np.concatenate([levels, sl])
            d = np.vstack([d, sd]) if len(d) else sd
            ids = np.concatenate([ids, np.full(n_spur, -1, dtype=np.int64)])
        cur = set(int(i) for i in take)
        if kf_id > 0 and len(prev & cur) < cfg.min_covisible:
            return None, f"keyframes {kf_id - 1}->{kf_id} share {len(prev & cur)} < {cfg.min_covisible} landmarks"
        prev = cur
        if kf_id >= 2 and (cfg.pose_noise_trans > 0 or rot_sigma > 0):
            drot = exp_so3(rng.normal(0, max(rot_sigma, 1e-12), 3))
            dt = rng.normal(0, max(cfg.pose_noise_trans, 1e-12), 3)
            pose_init = pose.compose(SE3Pose.from_rotation_matrix(drot, dt))
        else:
            pose_init = pose
        out.append(FrameRecord(kf_id, kf_id * cfg.frames_per_keyframe, pose, pose_init,
                               us, vs, levels, d, ids))
    return out, ""


# BASELINE.json configs. C1..C4 are single sessions; C5 = 64 x C2 shape.
BENCH_CONFIGS = {
    "c1": dict(seed=101, landmark_count=6000, keyframe_count=11, features_per_kf=1000,
               trajectory=LINE, extent=4.0, min_covisible=50, descriptor_flip_bits=3,
               pixel_noise_sigma=0.8),
    "c2": dict(seed=202, landmark_count=8000, keyframe_count=200, features_per_kf=1200,
               trajectory=LINE, extent=40.0, width=752, height=480, fx=458.0, fy=457.0,
               cx=367.0, cy=248.0, min_covisible=50, descriptor_flip_bits=3, pixel_noise_sigma=0.8),
    "c3": dict(seed=303, landmark_count=12000, keyframe_count=500, features_per_kf=1500,
               trajectory=ORBIT, width=512, height=512, fx=190.0, fy=190.0, cx=255.5, cy=255.5,
               min_covisible=50, descriptor_flip_bits=3, pixel_noise_sigma=0.8),
    "c4": dict(seed=404, landmark_count=40000, keyframe_count=60, features_per_kf=5000,
               trajectory=LINE, extent=40.0, width=752, height=480, fx=458.0, fy=457.0,
               cx=367.0, cy=248.0, min_covisible=50, descriptor_flip_bits=3, pixel_noise_sigma=0.8),
}
# neighbour counts / fusion n1 per config
BENCH_STAGE = {"c1": (10, 20, 5), "c2": (20, 20, 5), "c3": (30, 30, 5), "c4": (50, 50, 5)}


def bench_world(name: str, seed: int | None = None) -> WorldConfig:
    kw = dict(BENCH_CONFIGS[name])
    if seed is not None:
        kw["seed"] = seed
    return WorldConfig(**kw)
