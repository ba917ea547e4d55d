"""Builds the native library in-tree: paper_2511_02036_b200/liblm_b200.so (sm_100a).

Flags that matter for parity: device code is compiled with --fmad=false (no contraction of
a*b+c into FMA: NumPy never fuses) and IEEE division/sqrt (nvcc defaults); host code with
-ffp-contract=off. Explicit fma() calls remain fused on both sides (lm_math.cuh).
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = os.path.join(HERE, "csrc", "lm_b200.cu")
DEPS = [os.path.join(HERE, "csrc", f) for f in ("lm_b200.cu", "lm_kernels.cuh", "lm_map.cuh", "lm_math.cuh",
                                                          "lm_audit.cuh")] + [
    os.path.join(ROOT, "include", "lm_b200.h")]
LIB = os.path.join(HERE, "liblm_b200.so")


def nvcc_cmd(out: str = LIB) -> list[str]:
    nvcc = os.environ.get("NVCC", "nvcc")
    return [
        nvcc, "-O3", "-std=c++17", "-shared", "-lineinfo",
        "-gencode", "arch=compute_100a,code=sm_100a",
        "--fmad=false", "-prec-div=true", "-prec-sqrt=true",
        "-Xcompiler", "-fPIC,-ffp-contract=off,-O2",
        "-Xptxas", "-v",
        "-I", os.path.join(ROOT, "include"),
        "-o", out, SRC,
    ]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    if force or stale():
        cmd = nvcc_cmd()
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + r.stdout + r.stderr)
        log = os.path.join(HERE, "csrc", "ptxas.log")
        with open(log, "w") as fh:
            fh.write(r.stderr)
        if verbose:
            sys.stderr.write(r.stderr)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
