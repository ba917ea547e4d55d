"""Host-side pose and camera carriers of the drop-in API.

These are the *input* types a caller hands to the device map (keyframe poses and pinhole
intrinsics); the per-pair math on the hot path (fundamental matrices, epipolar distances,
DLT, gates, projections) runs in CUDA (csrc/lm_math.cuh). The arithmetic here follows the
reference's IEEE evaluation order exactly, because the synthetic workload generator
(workload.py) must reproduce the reference sequences bit for bit:

* SE3Pose            geometry.py:33-114 (quat xyzw, unit, w >= 0; world->camera)
* quat_from_matrix   geometry.py:134-162 (Shepperd)
* exp_so3 / skew     geometry.py:165-190
* CameraIntrinsics   geometry.py:201-234
* descriptors        geometry.py:358-370
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import InvalidArgumentError

DESCRIPTOR_BYTES = 32
DESCRIPTOR_BITS = 256


def _vec(x, n: int) -> np.ndarray:
    a = np.asarray(x, dtype=np.float64)
    if a.shape != (n,):
        raise InvalidArgumentError(f"expected a length-{n} vector, got shape {a.shape}")
    return a


def _rot_apply(r: np.ndarray, x, y, z):
    """Row-wise R @ p as three left-to-right dot products (geometry.py:193-198)."""
    return (
        r[0, 0] * x + r[0, 1] * y + r[0, 2] * z,
        r[1, 0] * x + r[1, 1] * y + r[1, 2] * z,
        r[2, 0] * x + r[2, 1] * y + r[2, 2] * z,
    )


def _quat_mul(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    ax, ay, az, aw = a
    bx, by, bz, bw = b
    return np.array(
        [
            aw * bx + ax * bw + ay * bz - az * by,
            aw * by - ax * bz + ay * bw + az * bx,
            aw * bz + ax * by - ay * bx + az * bw,
            aw * bw - ax * bx - ay * by - az * bz,
        ]
    )


def quat_from_matrix(m: np.ndarray) -> np.ndarray:
    """Shepperd's branch on the largest diagonal term; returns (x, y, z, w)."""
    d0, d1, d2 = m[0, 0], m[1, 1], m[2, 2]
    trace = d0 + d1 + d2
    if trace > 0:
        s = np.sqrt(trace + 1.0) * 2
        return np.array([(m[2, 1] - m[1, 2]) / s, (m[0, 2] - m[2, 0]) / s,
                         (m[1, 0] - m[0, 1]) / s, 0.25 * s])
    if d0 > d1 and d0 > d2:
        s = np.sqrt(1.0 + d0 - d1 - d2) * 2
        return np.array([0.25 * s, (m[0, 1] + m[1, 0]) / s,
                         (m[0, 2] + m[2, 0]) / s, (m[2, 1] - m[1, 2]) / s])
    if d1 > d2:
        s = np.sqrt(1.0 + d1 - d0 - d2) * 2
        return np.array([(m[0, 1] + m[1, 0]) / s, 0.25 * s,
                         (m[1, 2] + m[2, 1]) / s, (m[0, 2] - m[2, 0]) / s])
    s = np.sqrt(1.0 + d2 - d0 - d1) * 2
    return np.array([(m[0, 2] + m[2, 0]) / s, (m[1, 2] + m[2, 1]) / s,
                     0.25 * s, (m[1, 0] - m[0, 1]) / s])


def skew(v) -> np.ndarray:
    x, y, z = _vec(v, 3)
    return np.array([[0.0, -z, y], [z, 0.0, -x], [-y, x, 0.0]])


def exp_so3(phi) -> np.ndarray:
    """Rodrigues' formula."""
    phi = _vec(phi, 3)
    theta = float(np.sqrt(phi[0] ** 2 + phi[1] ** 2 + phi[2] ** 2))
    k = skew(phi)
    kk = k @ k
    if theta < 1e-12:
        return np.eye(3) + k + 0.5 * kk
    a = np.sin(theta) / theta
    b = (1.0 - np.cos(theta)) / (theta * theta)
    return np.eye(3) + a * k + b * kk


@dataclass(frozen=True)
class SE3Pose:
    """World-to-camera transform p_cam = R p_world + t; quat is (x, y, z, w)."""

    quat: np.ndarray
    trans: np.ndarray

    def __post_init__(self):
        q = _vec(self.quat, 4).copy()
        norm = np.sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3])
        if not (norm > 0 and np.isfinite(norm)):
            raise InvalidArgumentError("quaternion norm must be positive and finite")
        q /= norm
        if q[3] < 0:
            q = -q
        t = _vec(self.trans, 3).copy()
        q.flags.writeable = False
        t.flags.writeable = False
        object.__setattr__(self, "quat", q)
        object.__setattr__(self, "trans", t)

    @staticmethod
    def identity() -> "SE3Pose":
        return SE3Pose(np.array([0.0, 0.0, 0.0, 1.0]), np.zeros(3))

    @staticmethod
    def from_rotation_matrix(rot, trans) -> "SE3Pose":
        return SE3Pose(quat_from_matrix(np.asarray(rot, dtype=np.float64)), trans)

    def rotation_matrix(self) -> np.ndarray:
        x, y, z, w = self.quat
        xx, yy, zz = x * x, y * y, z * z
        xy, xz, yz = x * y, x * z, y * z
        wx, wy, wz = w * x, w * y, w * z
        return np.array(
            [
                [1 - 2 * (yy + zz), 2 * (xy - wz), 2 * (xz + wy)],
                [2 * (xy + wz), 1 - 2 * (xx + zz), 2 * (yz - wx)],
                [2 * (xz - wy), 2 * (yz + wx), 1 - 2 * (xx + yy)],
            ]
        )

    def compose(self, other: "SE3Pose") -> "SE3Pose":
        """self @ other (other applied first)."""
        rx, ry, rz = _rot_apply(self.rotation_matrix(), *other.trans)
        t = self.trans
        return SE3Pose(_quat_mul(self.quat, other.quat), np.array([rx + t[0], ry + t[1], rz + t[2]]))

    def inverse(self) -> "SE3Pose":
        x, y, z, w = self.quat
        ix, iy, iz = _rot_apply(self.rotation_matrix().T, *self.trans)
        return SE3Pose(np.array([-x, -y, -z, w]), np.array([-ix, -iy, -iz]))

    def transform(self, point) -> np.ndarray:
        p = _vec(point, 3)
        rx, ry, rz = _rot_apply(self.rotation_matrix(), p[0], p[1], p[2])
        t = self.trans
        return np.array([rx + t[0], ry + t[1], rz + t[2]])

    def center(self) -> np.ndarray:
        cx, cy, cz = _rot_apply(self.rotation_matrix().T, *self.trans)
        return np.array([-cx, -cy, -cz])

    def matrix(self) -> np.ndarray:
        m = np.eye(4)
        m[:3, :3] = self.rotation_matrix()
        m[:3, 3] = self.trans
        return m


@dataclass(frozen=True)
class CameraIntrinsics:
    """Pinhole camera with an ORB-style image pyramid (level 0 = finest)."""

    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    num_levels: int = 8
    scale_factor: float = 1.2

    def __post_init__(self):
        if self.fx <= 0 or self.fy <= 0:
            raise InvalidArgumentError("focal lengths must be positive")
        if not (0 <= self.cx < self.width and 0 <= self.cy < self.height):
            raise InvalidArgumentError("principal point must lie inside the image")
        if self.num_levels < 1:
            raise InvalidArgumentError("num_levels must be >= 1")
        if self.scale_factor <= 1.0:
            raise InvalidArgumentError("scale_factor must be > 1")

    def level_scale(self, level: int) -> float:
        return self.scale_factor ** level

    def level_sigma2(self, level: int) -> float:
        return self.scale_factor ** (2 * level)

    def sigma2_table(self) -> np.ndarray:
        return np.array([self.level_sigma2(lv) for lv in range(self.num_levels)])

    def matrix(self) -> np.ndarray:
        return np.array([[self.fx, 0.0, self.cx], [0.0, self.fy, self.cy], [0.0, 0.0, 1.0]])


def project(k: CameraIntrinsics, p_cam):
    """Single camera-frame point to pixels, or None when out of view (geometry.py:237-255)."""
    x, y, z = _vec(p_cam, 3)
    with np.errstate(divide="ignore", invalid="ignore"):
        u = k.fx * (x / z) + k.cx
        v = k.fy * (y / z) + k.cy
    if not (z > 0 and 0 <= u < k.width and 0 <= v < k.height):
        return None
    return float(u), float(v)


def random_descriptors(rng: np.random.Generator, n: int) -> np.ndarray:
    return rng.integers(0, 256, size=(n, DESCRIPTOR_BYTES), dtype=np.uint8)


def flip_descriptor_bits(rng: np.random.Generator, desc: np.ndarray, nbits: int) -> np.ndarray:
    out = desc.copy()
    if nbits <= 0:
        return out
    for bit in rng.choice(DESCRIPTOR_BITS, size=min(nbits, DESCRIPTOR_BITS), replace=False):
        out[bit >> 3] ^= np.uint8(1 << (int(bit) & 7))
    return out


def hamming(a: np.ndarray, b: np.ndarray) -> int:
    """Popcount distance of two 32-byte descriptors (host convenience; geometry.py:373-379)."""
    return int(np.bitwise_count(np.bitwise_xor(np.asarray(a, np.uint8), np.asarray(b, np.uint8))).sum())
