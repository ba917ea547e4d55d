"""Driver for compute-sanitizer runs (scripts/sanitize.sh): one workload through the native
session for a few keyframes, checked against the reference golden digests where frozen.

    python tools/sanitize_run.py <golden workload | c2> <keyframes>
"""

from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from helpers import device_kf  # noqa: E402
from paper_2511_02036_b200 import workload as W  # noqa: E402
from paper_2511_02036_b200.config import FuseConfig, MatchConfig  # noqa: E402
from paper_2511_02036_b200.session import LocalMapper, store_for  # noqa: E402


def main():
    name, n_kf = sys.argv[1], int(sys.argv[2])
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))
    if name in gold["workloads"]:
        cfg = W.WorldConfig(**gold["workloads"][name]["config"])
        n_nbr, n1, steps = gold["pipeline"][name]["neighbor_count"], 20, gold["pipeline"][name]["steps"]
    else:
        cfg = W.bench_world(name)
        n_nbr, n1, _ = W.BENCH_STAGE[name]
        path = os.path.join(ROOT, "tests", "golden", f"steady_{name}.json")
        steps = json.load(open(path))["steps"] if os.path.isfile(path) else None
    seq = W.generate_sequence(cfg)
    intr = seq.intrinsics()
    dev = LocalMapper(intr, neighbor_count=n_nbr, match=MatchConfig(neighbor_count=n_nbr), fuse=FuseConfig(n1=n1),
                      store=store_for(len(seq.records), cfg.features_per_kf + 64))
    ok = True
    for k, rec in enumerate(seq.records[:n_kf]):
        dev.process(device_kf(rec, intr))
        if steps is not None and k < len(steps):
            ok &= dev.snapshot(with_covis=False).structural_digest() == steps[k]["digest"]
    print(f"sanitize_run {name}: {min(n_kf, len(seq.records))} keyframes, digests equal to the reference: {ok}")
    sys.exit(0 if ok else 3)


if __name__ == "__main__":
    main()
