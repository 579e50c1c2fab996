#!/bin/bash
# The round's measurement set on one B200 (run under gpurun from the repo
# root):  tools/gpu_final.sh <tag>
#   GPU tests + smoke, the default bench line (e2e, roofline, CPU arm, time to
#   SSIM), the reference arm, the ncu launch list + --set full summaries of
#   the step's kernels, the CUPTI timeline and the C5 render sweep.  Outputs
#   land in gpurun_out/; copy what is judged into profiles/.
tag=${1:-final}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_${tag}.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_${tag}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${tag}.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke_${tag}.log
timeout 600 python bench.py > gpurun_out/bench_${tag}.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_${tag}.log 2>&1
bash tools/gpu_profile.sh ${tag} > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/full_${tag}_raw.csv --json gpurun_out/ncu_full_${tag}.json > /dev/null 2>&1
timeout 300 python tools/gpu_timeline.py --out gpurun_out/timeline_${tag}.json > gpurun_out/timeline_${tag}.log 2>&1
timeout 600 python tools/render_sweep.py --out gpurun_out/render_sweep_${tag}.json > gpurun_out/render_sweep_${tag}.log 2>&1
tail -n 2 gpurun_out/pytest_gpu_${tag}.log gpurun_out/smoke_${tag}.log
grep -h '^{' gpurun_out/bench_${tag}.log gpurun_out/bench_ref_${tag}.log | cut -c1-400
cat gpurun_out/launch_shares_${tag}.txt | head -14
