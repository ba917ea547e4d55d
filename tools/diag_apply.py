"""Diagnostics (a -DLM_DIAG build of the library, selected with LM_B200_LIB): the C2 sequence
once, then per forward-apply phase the sum over rounds of the slowest thread's time in that
phase, against the phase walls the step statistics report.

    LM_B200_LIB=$PWD/ab/F.so python tools/diag_apply.py
"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from helpers import device_kf  # noqa: E402
from paper_2511_02036_b200 import _lib  # noqa: E402
from paper_2511_02036_b200 import workload as W  # noqa: E402
from paper_2511_02036_b200.config import FuseConfig, MatchConfig  # noqa: E402
from paper_2511_02036_b200.session import LocalMapper, store_for  # noqa: E402


def run(seq, intr):
    dev = LocalMapper(intr, neighbor_count=20, match=MatchConfig(neighbor_count=20), fuse=FuseConfig(n1=20, n2=5),
                      store=store_for(200, seq.config.features_per_kf + 64))
    for rec in seq.records:
        dev.process(device_kf(rec, intr))
    return dev


def main():
    lib = _lib.load()
    fn = lib.lm_debug_diag
    fn.argtypes = [C.POINTER(C.c_uint64), C.c_int]
    seq = W.generate_sequence(W.bench_world("c2"))
    intr = seq.intrinsics()
    run(seq, intr)  # warm-up
    buf = (C.c_uint64 * 64)()
    fn(buf, 64)
    dev = run(seq, intr)
    fn(buf, 64)
    tot = dev.totals()
    names = ["reserve", "check", "heads", "members+merges", "group pairs"]
    print("rounds", buf[16])
    for k, nm in enumerate(names):
        print(f"{nm:16s} slowest-thread sum {buf[8 + k] / 1e6:8.3f} ms")
    print("pending at round start (rounds 1..4, 5+):", [buf[17 + r] for r in range(5)])
    modes = ["SLOT", "EX", "SH", "PAIR"]
    print("blocked by (first failing key) for ADD:", {m: buf[24 + k] for k, m in enumerate(modes)},
          "MERGE:", {m: buf[28 + k] for k, m in enumerate(modes)})
    # reverse walk (k_fuse_rev, ns summed over the sequence): select phase, direct passes
    np_ = max(buf[59], 1)
    nd = max(buf[56], 1)
    print(f"rev iterations {buf[59]}  direct passes {buf[56]} ({buf[57]} actions)  items re-evaluated {buf[58]}")
    print(f"rev select: bits loaded {buf[48] / np_ / 1e3:.2f} us  actions extracted {buf[49] / np_ / 1e3:.2f} us  "
          f"warp-0 select {buf[50] / np_ / 1e3:.2f} us  to the barrier {buf[51] / np_ / 1e3:.2f} us (per iteration)")
    print(f"rev direct: walk+command {buf[52] / nd / 1e3:.2f} us  apply wall {buf[53] / nd / 1e3:.2f} us  "
          f"slowest add_direct {buf[54] / nd / 1e3:.2f} us  (CTA 0's {buf[55] / nd / 1e3:.2f} us) per direct pass")
    fc, dbg = list(tot.fuse_cycles), list(tot.dbg)
    print(f"walls: reserve+check {fc[13] / 1e6:.3f} ms  heads {dbg[8] / 1e6:.3f} ms  members {dbg[9] / 1e6:.3f} ms  "
          f"compaction {fc[15] / 1e6:.3f} ms  fwd apply total {fc[3] / 1e6:.3f} ms")


if __name__ == "__main__":
    main()
