"""Top stall-sampled SASS instructions of a kernel in an ncu report:
    python profiles/sass_hot.py report.ncu-rep <kernel-regex> [n]"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]
si = h.index("Warp Stall Sampling (All Samples)")
body = [r for r in rows[hi + 1:] if len(r) > si and r[si].replace(".", "").isdigit()]
tot = sum(float(r[si]) for r in body) or 1.0
for idx, r in sorted(enumerate(body), key=lambda t: -float(t[1][si]))[:n]:
    print(f"{100 * float(r[si]) / tot:5.1f}%  #{idx:5d}  {r[1].strip()[:90]}")
