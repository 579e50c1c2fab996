#!/bin/bash
# time to 0.99 held-out SSIM (C2, batch 48) for library variants, alternating:
#   tools/tts_ab.sh tag1 tag2 ...   ("base" = the default build)
for rep in 1 2 3; do
for v in "$@"; do
  if [ $v = base ]; then lib=""; else lib=paper_2505_05643_b200/variants/libugs_$v.so; fi
  UGS_LIB=$lib python tools/time_to_ssim.py --batch 48 --eval-every 10 --budget 60 --out gpurun_out/tts_$v.json > gpurun_out/tts_$v.log 2>&1
  echo "$v $(tail -1 gpurun_out/tts_$v.log)"
done
done
