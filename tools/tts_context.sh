#!/bin/bash
# time-to-SSIM inside bench.py under different preceding legs
run() {
  tag=$1; shift
  python bench.py "$@" > gpurun_out/ttsctx_$tag.log 2>&1
  python - "$tag" <<'PY'
import json, sys
t = sys.argv[1]
l = [x for x in open(f"gpurun_out/ttsctx_{t}.log") if x.startswith("{")]
print(t, json.loads(l[-1]).get("time_to_ssim", {}).get("reached_s") if l else "FAILED")
PY
}
run default
run noe2e --no-e2e
run nocpu --no-cpu-baseline
run noe2e_nocpu --no-e2e --no-cpu-baseline
run default2
