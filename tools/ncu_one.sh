#!/bin/bash
# One `ncu --set full` capture of one kernel of a timed bench step (run under
# gpurun from the repo root): tools/ncu_one.sh <tag> <kernel-regex> [count]
tag=$1; regex=$2; cnt=${3:-1}
mkdir -p gpurun_out
ncu --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on \
    -k regex:"${regex}" -c ${cnt} -f -o gpurun_out/one_${tag} \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_one_${tag}.log 2>&1
ncu -i gpurun_out/one_${tag}.ncu-rep --page raw --csv > gpurun_out/one_${tag}_raw.csv 2>/dev/null
ncu -i gpurun_out/one_${tag}.ncu-rep --page source --csv > gpurun_out/one_${tag}_src.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/one_${tag}_raw.csv
