#!/bin/bash
# Bench stage times for each in-tree libugs variant (tools/build_variant.py):
#   tools/variant_sweep.sh tag1 tag2 ...   ("base" = the default build)
for tag in "$@"; do
  if [ "$tag" = base ]; then lib=""; else lib=paper_2505_05643_b200/variants/libugs_${tag}.so; fi
  UGS_LIB=$lib python bench.py --steps 20 --warmup 5 --no-tts --no-cpu-baseline --no-e2e \
      > gpurun_out/var_${tag}.log 2>&1
  python - "$tag" <<'PY'
import json, sys
tag = sys.argv[1]
l = [x for x in open(f"gpurun_out/var_{tag}.log") if x.startswith("{")]
if not l:
    print(tag, "FAILED"); sys.exit()
d = json.loads(l[-1]); st = d["stage_ms_per_step"]
print(f"{tag:10s} step {d['ms_per_step']:.4f} ms  fwd {st['forward']*1e3:.1f}  bwd {st['backward']*1e3:.1f}  "
      f"count {st['prepare_count']*1e3:.1f} emit {st['prepare_emit']*1e3:.1f} sort {st['sort']*1e3:.1f} "
      f"fin {st['finalize']*1e3:.1f} upd {st['update']*1e3:.1f} loss {st['loss']*1e3:.1f} us")
PY
done
