#!/bin/bash
# PDL-off sweep: one bench per kernel name launched without the attribute
run() {
  tag=$1; off=$2
  UGS_PDL_OFF=$off python bench.py --steps 20 --warmup 5 --no-tts --no-cpu-baseline --no-e2e > gpurun_out/pdl_$tag.log 2>&1
  python - "$tag" <<'PY'
import json, sys
tag = sys.argv[1]
l = [x for x in open(f"gpurun_out/pdl_{tag}.log") if x.startswith("{")]
print(f"{tag:24s}", "FAILED" if not l else f"{json.loads(l[-1])['ms_per_step']:.4f}")
PY
}
for rep in 1 2; do
run base ""
for k in prepare_count_kernel plan_slices_kernel prepare_scan_kernel warp_offsets_kernel build_records_kernel scan_reduce_kernel slice_hist_kernel "slice_scatter_kernel<8>" slice_ranges_kernel forward_kernel loss_tile_kernel loss_reduce_kernel backward_kernel bg_slice_kernel update_gather_kernel; do
  run "$k" "$k"
done
done
