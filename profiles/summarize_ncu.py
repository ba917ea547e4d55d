"""Summarise ncu captures into profiles/ (tracked):

    python profiles/summarize_ncu.py <full.ncu-rep> <launches.csv> <tag>

Writes profiles/ncu_summary.json (per kernel: duration, dram bytes per launch, achieved
occupancy, issue activity, pipe utilisation — from the `--set full` capture) and
profiles/<tag>_launches.md (share of device time per kernel from the
`--metrics gpu__time_duration.sum` launch list; cold-cache and serialised, so compare
shares, not absolutes)."""

from __future__ import annotations

import collections
import csv
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "alu_cycles_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_cycles_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_cycles_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pipe_active_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_elapsed": "xu_pipe_elapsed_pct",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__registers_per_thread": "registers",
    "l1tex__t_bytes.sum": "l1_bytes",
    "lts__t_bytes.sum": "l2_bytes",
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
        "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
        "second": 1}


def kname(raw: str) -> str:
    """Kernel name without namespace, arguments or the timer-free instantiation tag
    (k_fuse_rev<false> is the kernel every step launches; <true> is the profile pass's)."""
    n = raw.split("(")[0].replace("lm::", "").replace("void ", "")
    for k in ("k_fuse_rev", "k_fuse_apply", "k_cull"):  # template <bool P>: phase timers
        for tag, lab in (("<false>", ""), ("<0>", ""), ("<true>", " (profile pass)"), ("<1>", " (profile pass)")):
            if n == k + tag:
                return k + lab
    return n


def full_summary(rep: str) -> dict:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    per = collections.defaultdict(list)
    for r in rows[2:]:
        name = kname(r[hdr.index("Kernel Name")])
        d = {}
        for m, key in METRICS.items():
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                d[key] = v * UNIT.get(units[i], 1)
        per[name].append(d)
    summ = {}
    for k, lst in per.items():
        avg = {key: sum(x.get(key, 0) for x in lst) / len(lst) for key in lst[0]}
        avg["launches_captured"] = len(lst)
        avg["dram_bytes_per_launch"] = avg.get("dram_read", 0) + avg.get("dram_write", 0)
        summ[k] = avg
    return summ


def launch_shares(path: str) -> list[tuple[str, int, float, float]]:
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        agg[kname(r[ki])].append(float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1e-9))
    tot = sum(sum(v) for v in agg.values())
    return sorted(((k, len(v), sum(v) / len(v), sum(v) / tot) for k, v in agg.items()), key=lambda t: -t[3])


def main():
    rep, launches, tag = sys.argv[1], sys.argv[2], sys.argv[3]
    summ = full_summary(rep)
    with open(os.path.join(HERE, "ncu_summary.json"), "w") as fh:
        json.dump({"source": os.path.basename(rep), "tag": tag, **summ}, fh, indent=1, sort_keys=True)
    lines = [f"# {tag}: device-time share per kernel (ncu launch list, cold-cache, serialised)", "",
             "| kernel | launches | mean us | share |", "|---|---|---|---|"]
    for k, n, mean, share in launch_shares(launches):
        lines.append(f"| {k} | {n} | {mean * 1e6:.1f} | {100 * share:.1f}% |")
    lines += ["", f"# {tag}: `ncu --set full` per-launch averages", "",
              "| kernel | us | dram B/launch | occupancy % | issue active % | alu % | xu (POPC) % active / elapsed | fp64 % |",
              "|---|---|---|---|---|---|---|---|"]
    for k, d in sorted(summ.items()):
        if not isinstance(d, dict):
            continue
        lines.append(f"| {k} | {d.get('duration', 0) * 1e6:.1f} | {d.get('dram_bytes_per_launch', 0):.0f} | "
                     f"{d.get('achieved_occupancy_pct', 0):.1f} | {d.get('issue_active_pct', 0):.1f} | "
                     f"{d.get('alu_cycles_pct', 0):.1f} | {d.get('xu_pipe_active_pct', 0):.1f} / "
                     f"{d.get('xu_pipe_elapsed_pct', 0):.1f} | {d.get('fp64_cycles_pct', 0):.1f} |")
    with open(os.path.join(HERE, f"{tag}_summary.md"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
