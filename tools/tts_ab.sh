#!/bin/bash
for rep in 1 2; do
for v in base noorder; do
  if [ $v = base ]; then lib=""; else lib=paper_2505_05643_b200/variants/libugs_$v.so; fi
  UGS_LIB=$lib python tools/time_to_ssim.py --batch 48 --eval-every 10 --budget 60 --out gpurun_out/tts_$v.json > gpurun_out/tts_$v.log 2>&1
  echo "$v $(tail -1 gpurun_out/tts_$v.log)"
done
done
