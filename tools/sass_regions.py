#!/usr/bin/env python
"""Warp-instructions executed per SASS line of one kernel, printed as runs of
lines with equal execution counts (basic blocks) -- shows where the
instruction budget goes.  python tools/sass_regions.py rep.ncu-rep regex"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
minfrac = float(sys.argv[3]) if len(sys.argv) > 3 else 0.005
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kre,
                      "--print-source", "sass"], capture_output=True, text=True).stdout
lines = txt.splitlines()
i = next(j for j, l in enumerate(lines) if l.startswith('"Address"'))
end = next((j for j in range(i + 1, len(lines)) if lines[j].startswith('"Kernel Name"')),
           len(lines))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[i:end]))))
tot = sum(int(r["Instructions Executed"] or 0) for r in rows)
blocks = []
for idx, r in enumerate(rows):
    ex = int(r["Instructions Executed"] or 0)
    if blocks and blocks[-1][2] == ex:
        blocks[-1][1] = idx
        blocks[-1][3] += ex
        blocks[-1][4].append(r["Source"].strip().split()[0] if r["Source"].strip() else "")
    else:
        blocks.append([idx, idx, ex, ex, [r["Source"].strip().split()[0] if r["Source"].strip() else ""]])
print(f"total {tot} warp-instructions")
for b0, b1, ex, s, ops in blocks:
    if s / tot >= minfrac:
        print(f"lines {b0:5d}-{b1:5d} x{ex:10d}  n={b1 - b0 + 1:3d}  {100 * s / tot:5.1f}%  "
              f"{' '.join(o for o in ops[:14])}")
