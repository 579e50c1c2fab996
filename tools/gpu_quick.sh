#!/bin/bash
# GPU tests + a 30-step bench + the ncu launch list (shares), for one change.
tag=${1:-cur}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -n 4 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench_${tag}.log 2>&1
python - "$tag" <<'PY'
import json, sys
l = [x for x in open(f"gpurun_out/bench_{sys.argv[1]}.log") if x.startswith("{")]
if l:
    d = json.loads(l[-1])
    print("value", round(d["value"], 1), "ms/step", round(d["ms_per_step"], 4), "e2e", round(d.get("e2e", {}).get("value", 0), 1), "clocks", d.get("clocks"))
    print({k: round(v, 4) for k, v in d["stage_ms_per_step"].items()})
else:
    print(open(f"gpurun_out/bench_{sys.argv[1]}.log").read()[-3000:])
PY
ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none \
    --csv --log-file gpurun_out/launches_${tag}.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_${tag}.log 2>&1
python tools/launch_shares.py gpurun_out/launches_${tag}.csv --steps 2 --json gpurun_out/launch_shares_${tag}.json > gpurun_out/launch_shares_${tag}.txt; head -12 gpurun_out/launch_shares_${tag}.txt
