#!/usr/bin/env python
"""Per-kernel key counters from `ncu -i X.ncu-rep --page raw --csv` output.

    python tools/ncu_summary.py gpurun_out/full_tag_raw.csv [--json out.json]
"""
import argparse
import csv
import json
import re

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.per_cycle_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "smsp__inst_executed.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
]
STALL = re.compile(r"smsp__average_warps_issue_stalled_(\w+)_per_issue_active\.ratio")


def load(path):
    text = open(path).read()
    rows = list(csv.reader(text[text.index('"ID"'):].splitlines()))
    head, units, data = rows[0], rows[1], rows[2:]
    out = []
    for r in data:
        d = dict(zip(head, r))
        name = d.get("Kernel Name", "?")
        m = re.search(r"(\w+?)(<[^(]*>)?\(", name)
        short = (m.group(1) + (m.group(2) or "")) if m else name
        ent = {"kernel": short}
        for k in KEYS:
            if k in d and d[k] not in ("", "n/a"):
                ent[k] = d[k] + (" " + units[head.index(k)] if units[head.index(k)] else "")
        stalls = {}
        for k, v in d.items():
            mm = STALL.fullmatch(k)
            if mm and v not in ("", "n/a"):
                try:
                    stalls[mm.group(1)] = float(v.replace(",", ""))
                except ValueError:
                    pass
        ent["top_stalls"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:5])
        out.append(ent)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("raw_csv")
    ap.add_argument("--json")
    ap.add_argument("-k", default=None)
    a = ap.parse_args()
    res = load(a.raw_csv)
    if a.k:
        res = [r for r in res if re.search(a.k, r["kernel"])]
    for r in res:
        print(json.dumps(r, indent=1))
    if a.json:
        json.dump(res, open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()
