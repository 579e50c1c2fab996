#!/usr/bin/env python
"""Hottest SASS instructions (warp-stall samples) of one kernel from an
ncu report:  python tools/sass_hot.py report.ncu-rep kernel_regex [top]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kre,
                      "--print-source", "sass"], capture_output=True, text=True).stdout
lines = txt.splitlines()
i = next(j for j, l in enumerate(lines) if l.startswith('"Address"'))
end = next((j for j in range(i + 1, len(lines)) if lines[j].startswith('"Kernel Name"')),
           len(lines))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[i:end]))))
tot = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows)
inst = sum(int(r["Instructions Executed"] or 0) for r in rows)
print(f"{len(rows)} SASS lines, {tot} samples, {inst} warp-instructions executed")
stall_cols = [c for c in rows[0] if c.startswith("stall_") and "Not Issued" not in c]
for idx, r in enumerate(rows):
    r["_i"] = idx
hot = sorted(rows, key=lambda r: -int(r["Warp Stall Sampling (All Samples)"] or 0))[:top]
for r in sorted(hot, key=lambda r: r["_i"]):
    s = int(r["Warp Stall Sampling (All Samples)"] or 0)
    st = sorted(((int(r[c] or 0), c[6:]) for c in stall_cols), reverse=True)[:2]
    print(f"{r['_i']:5d} {100.0 * s / tot:5.1f}% ex={int(r['Instructions Executed'] or 0):9d} "
          f"{r['Source'].strip()[:60]:60s} {st}")
