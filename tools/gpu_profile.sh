#!/bin/bash
# One profiling pass on the GPU box (run under gpurun from the repo root):
#   tools/gpu_profile.sh <tag> [kernel-regex]
# 1) ncu launch list of 2 timed bench steps (cold-cache, serialised: compare
#    shares), 2) one `ncu --set full` capture of each matched kernel in the
#    timed region.  Outputs land in gpurun_out/.
tag=${1:-cur}
regex=${2:-"forward_kernel|backward_kernel|update_gather|prepare_count|prepare_emit|finalize_records|loss_tile|build_records"}
mkdir -p gpurun_out
ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none \
    --csv --log-file gpurun_out/launches_${tag}.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_${tag}.log 2>&1
python tools/launch_shares.py gpurun_out/launches_${tag}.csv --steps 2 \
    --json gpurun_out/launch_shares_${tag}.json > gpurun_out/launch_shares_${tag}.txt
ncu --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on \
    -k regex:"${regex}" -c 12 -f -o gpurun_out/full_${tag} \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_${tag}.log 2>&1
ncu -i gpurun_out/full_${tag}.ncu-rep --page raw --csv > gpurun_out/full_${tag}_raw.csv 2>/dev/null
cat gpurun_out/launch_shares_${tag}.txt
