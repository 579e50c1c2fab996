#!/usr/bin/env python
"""Copy one tools/gpu_final.sh run from gpurun_out/ into profiles/ (the
round's judged evidence) and print the numbers the docs quote.

    python tools/refresh_profiles.py <tag> [--round 01]
"""
import argparse
import json
import os
import shutil

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")


def json_line(path):
    lines = [x for x in open(path) if x.startswith("{")]
    return json.loads(lines[-1]) if lines else None


def mbytes(v):
    x, unit = v.split()
    return float(x) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("tag")
    ap.add_argument("--round", default="01")
    a = ap.parse_args()
    t, r = a.tag, a.round
    bench = json_line(os.path.join(OUT, f"bench_{t}.log"))
    ref = json_line(os.path.join(OUT, f"bench_ref_{t}.log"))
    json.dump(bench, open(os.path.join(PROF, f"bench_r{r}.json"), "w"), indent=1)
    if ref:
        json.dump(ref, open(os.path.join(PROF, f"bench_ref_r{r}.json"), "w"), indent=1)
    for src, dst in ((f"launches_{t}.csv", f"launches_r{r}.csv"),
                     (f"launch_shares_{t}.json", f"launch_shares_r{r}.json"),
                     (f"timeline_{t}.json", f"timeline_r{r}.json"),
                     (f"render_sweep_{t}.json", f"render_sweep_r{r}.json")):
        if os.path.exists(os.path.join(OUT, src)):
            shutil.copy(os.path.join(OUT, src), os.path.join(PROF, dst))
    kernels = json.load(open(os.path.join(OUT, f"ncu_full_{t}.json")))
    src = ("ncu --set full --clock-control none --nvtx-include timed/, bench.py --steps 1 "
           "--warmup 3 (C3: 1M Gaussians, 16 slices of 256x256 per launch), one launch per kernel")
    json.dump({"source": src, "kernels": kernels},
              open(os.path.join(PROF, f"ncu_full_r{r}.json"), "w"), indent=1)
    traffic = {"source": src, "note": "dram bytes per launch (one launch covers the 16-slice batch)"}
    for k in kernels:
        traffic[k["kernel"].split("(")[0] + "_dram_bytes"] = (
            mbytes(k["dram__bytes_read.sum"]) + mbytes(k["dram__bytes_write.sum"]))
    json.dump(traffic, open(os.path.join(PROF, "ncu_traffic.json"), "w"), indent=1)
    print("value", round(bench["value"], 1), "ms/step", round(bench["ms_per_step"], 4),
          "e2e", round(bench["e2e"]["value"], 1), "cpu", bench["cpu_baseline"]["value"])
    print("roofline", json.dumps(bench["roofline"])[:300])
    print("stages", {k: round(v, 4) for k, v in bench["stage_ms_per_step"].items()})
    print("tts", bench.get("time_to_ssim"))
    print("clocks", bench.get("clocks"))
    if ref:
        print("reference", ref["value"], ref.get("cpu_baseline"))
    for k in kernels:
        print(k["kernel"][:28], k["gpu__time_duration.sum"], k["smsp__inst_executed.sum"],
              k["smsp__issue_active.avg.pct_of_peak_sustained_active"],
              k["launch__registers_per_thread"])


if __name__ == "__main__":
    main()
