"""CPU tests of the native library's host-compiled math (the same lm_math.cuh the kernels
use) against the oracle / NumPy: fundamental matrices and projection matrices must be
bit-identical; the DLT null vector within the 1e-4 relative contract."""

from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

from oracle import lm_oracle as O
from paper_2511_02036_b200 import _lib
from paper_2511_02036_b200.geometry import SE3Pose, exp_so3


def _pose(rng, scale=1.0):
    return SE3Pose.from_rotation_matrix(exp_so3(rng.normal(0, 0.3, 3)), rng.normal(0, scale, 3))


def _arr(x):
    return np.ascontiguousarray(x, dtype=np.float64)


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for name in _lib.EXPORTED:
        assert hasattr(lib, name), name
    assert lib.lm_version() == 1


def test_fundamental_bit_exact():
    lib = _lib.load()
    rng = np.random.default_rng(5)
    for _ in range(3000):
        a, b = _pose(rng), _pose(rng)
        ca = np.array([rng.uniform(150, 900), rng.uniform(150, 900), rng.uniform(100, 600), rng.uniform(100, 500)])
        cb = ca if rng.uniform() < 0.5 else np.array([rng.uniform(150, 900), rng.uniform(150, 900),
                                                      rng.uniform(100, 600), rng.uniform(100, 500)])
        cam_a = O.Cam(*ca, 1280, 960)
        cam_b = O.Cam(*cb, 1280, 960)
        want = O.fundamental(a.quat, a.trans, cam_a, b.quat, b.trans, cam_b)
        got = np.zeros(9)
        rc = lib.lm_host_fundamental(_lib.ptr(_arr(a.quat), C.c_double), _lib.ptr(_arr(a.trans), C.c_double),
                                     _lib.ptr(_arr(b.quat), C.c_double), _lib.ptr(_arr(b.trans), C.c_double),
                                     _lib.ptr(_arr(ca), C.c_double), _lib.ptr(_arr(cb), C.c_double),
                                     _lib.ptr(got, C.c_double))
        assert rc == 0
        assert np.array_equal(got.reshape(3, 3), want)


def test_fundamental_zero_baseline_degenerate():
    lib = _lib.load()
    p = SE3Pose.identity()
    cam = _arr([460, 460, 320, 240])
    got = np.zeros(9)
    rc = lib.lm_host_fundamental(_lib.ptr(_arr(p.quat), C.c_double), _lib.ptr(_arr(p.trans), C.c_double),
                                 _lib.ptr(_arr(p.quat), C.c_double), _lib.ptr(_arr(p.trans), C.c_double),
                                 _lib.ptr(cam, C.c_double), _lib.ptr(cam, C.c_double), _lib.ptr(got, C.c_double))
    assert rc == _lib.C.c_int32(-6).value


def test_projection_and_center_bit_exact():
    lib = _lib.load()
    rng = np.random.default_rng(9)
    for _ in range(2000):
        p = _pose(rng, 3.0)
        cam = _arr([rng.uniform(150, 900), rng.uniform(150, 900), rng.uniform(100, 600), rng.uniform(100, 500)])
        R, Cc, Pm = np.zeros(9), np.zeros(3), np.zeros(12)
        lib.lm_host_projection(_lib.ptr(_arr(p.quat), C.c_double), _lib.ptr(_arr(p.trans), C.c_double),
                               _lib.ptr(cam, C.c_double), _lib.ptr(R, C.c_double), _lib.ptr(Cc, C.c_double),
                               _lib.ptr(Pm, C.c_double))
        assert np.array_equal(R.reshape(3, 3), p.rotation_matrix())
        assert np.array_equal(Cc, p.center())
        K = np.array([[cam[0], 0.0, cam[2]], [0.0, cam[1], cam[3]], [0.0, 0.0, 1.0]])
        assert np.array_equal(Pm.reshape(3, 4), K @ p.matrix()[:3, :])


def test_dlt_within_contract():
    lib = _lib.load()
    rng = np.random.default_rng(13)
    cam = O.Cam(460.0, 460.0, 320.0, 240.0, 640, 480)
    worst = 0.0
    n = 0
    while n < 1000:
        a, b = _pose(rng), _pose(rng)
        X = rng.normal(0, 1, 3) + np.array([0, 0, 6.0])
        xa, xb = O.cam_apply(a.quat, a.trans, X), O.cam_apply(b.quat, b.trans, X)
        if xa[2] <= 0.5 or xb[2] <= 0.5:
            continue
        pa = (cam.fx * xa[0] / xa[2] + cam.cx, cam.fy * xa[1] / xa[2] + cam.cy)
        pb = (cam.fx * xb[0] / xb[2] + cam.cx, cam.fy * xb[1] / xb[2] + cam.cy)
        want = O.dlt_point(a.quat, a.trans, cam, b.quat, b.trans, cam, pa, pb)
        Ra, Ca, Pa = np.zeros(9), np.zeros(3), np.zeros(12)
        Rb, Cb, Pb = np.zeros(9), np.zeros(3), np.zeros(12)
        c4 = _arr([cam.fx, cam.fy, cam.cx, cam.cy])
        for p, R, Cc, Pm in ((a, Ra, Ca, Pa), (b, Rb, Cb, Pb)):
            lib.lm_host_projection(_lib.ptr(_arr(p.quat), C.c_double), _lib.ptr(_arr(p.trans), C.c_double),
                                   _lib.ptr(c4, C.c_double), _lib.ptr(R, C.c_double), _lib.ptr(Cc, C.c_double),
                                   _lib.ptr(Pm, C.c_double))
        got = np.zeros(3)
        pix = _arr([pa[0], pa[1], pb[0], pb[1]])
        rc = lib.lm_host_triangulate(_lib.ptr(Pa, C.c_double), _lib.ptr(Pb, C.c_double), _lib.ptr(Ca, C.c_double),
                                     _lib.ptr(Cb, C.c_double), _lib.ptr(pix, C.c_double), _lib.ptr(got, C.c_double))
        assert rc == 0 and want is not None
        worst = max(worst, float(np.linalg.norm(got - want) / np.linalg.norm(want)))
        n += 1
    assert worst < 1e-9, worst
