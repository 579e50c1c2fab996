#!/usr/bin/env python
"""Shared-memory wavefronts per SASS line of one kernel (actual vs ideal):
where a kernel's shared-memory traffic and bank conflicts come from.
    python tools/smem_lines.py rep.ncu-rep kernel_regex [top]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kre,
                      "--print-source", "sass"], capture_output=True, text=True).stdout
lines = txt.splitlines()
i = next(j for j, l in enumerate(lines) if l.startswith('"Address"'))
end = next((j for j in range(i + 1, len(lines)) if lines[j].startswith('"Kernel Name"')),
           len(lines))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[i:end]))))


def num(r, k):
    try:
        return float(r.get(k) or 0)
    except ValueError:
        return 0.0


tot = sum(num(r, "L1 Wavefronts Shared") for r in rows)
ideal = sum(num(r, "L1 Wavefronts Shared Ideal") for r in rows)
print(f"shared wavefronts {tot:.0f} (ideal {ideal:.0f}, excess {tot - ideal:.0f})")
rs = sorted(rows, key=lambda r: -num(r, "L1 Wavefronts Shared"))[:top]
for r in rs:
    w, wi = num(r, "L1 Wavefronts Shared"), num(r, "L1 Wavefronts Shared Ideal")
    print(f"{rows.index(r):5d} {100 * w / tot:5.1f}% wf={w:10.0f} ideal={wi:10.0f} "
          f"ex={int(num(r, 'Instructions Executed')):9d} {r['Source'][:60]}")
