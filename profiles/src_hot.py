"""Stall samples aggregated per CUDA source line for one kernel of an ncu report:
    python profiles/src_hot.py report.ncu-rep <kernel-regex> [n]"""
import collections
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--launch-count", "1", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
agg = collections.Counter()
text = {}
fname = None
line = None
hdr = None
for r in csv.reader(out.splitlines()):
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        si = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if not hdr or len(r) < len(hdr):
        continue
    if r[0]:
        line = (fname, r[0])
        text[line] = r[1].strip()[:80]
    try:
        v = float(r[si] or 0)
    except ValueError:
        continue
    agg[line] += v
tot = sum(agg.values()) or 1
for (f, l), v in agg.most_common(n):
    print(f"{100 * v / tot:5.1f}%  {f}:{l}  {text.get((f, l), '')}")
