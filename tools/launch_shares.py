#!/usr/bin/env python
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
per-kernel time and share of the captured region.

    python tools/launch_shares.py gpurun_out/launches.csv [--steps 2] [--json out.json]
"""
import argparse
import csv
import io
import json
import re
from collections import OrderedDict


def parse(path):
    text = open(path).read()
    start = text.index('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    out = OrderedDict()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        m = re.search(r"(\w+?)(<[^(]*>)?\(", name)
        short = m.group(1) if m else name
        if m and m.group(2):
            short += m.group(2)
        ns = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        scale = {"ns": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(unit, 1.0)
        d = out.setdefault(short, {"launches": 0, "ns": 0.0})
        d["launches"] += 1
        d["ns"] += ns * scale
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--json")
    a = ap.parse_args()
    k = parse(a.csv)
    tot = sum(d["ns"] for d in k.values())
    res = []
    for name, d in sorted(k.items(), key=lambda kv: -kv[1]["ns"]):
        res.append({"kernel": name, "launches_per_step": d["launches"] / a.steps,
                    "us_per_step": d["ns"] / a.steps / 1e3, "share": d["ns"] / tot})
        print(f"{name:40s} {d['launches'] / a.steps:6.1f} {d['ns'] / a.steps / 1e3:10.1f} us "
              f"{100 * d['ns'] / tot:6.1f} %")
    print(f"{'total':40s} {'':6s} {tot / a.steps / 1e3:10.1f} us")
    if a.json:
        json.dump({"source": a.csv, "steps": a.steps, "total_us_per_step": tot / a.steps / 1e3,
                   "kernels": res}, open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()
