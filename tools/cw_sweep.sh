#!/bin/bash
# Consumer-warp count of the TMA step kernel: default vs the wide CTA
# (RBFFD_TMA_CW), per benchmark width.  Output: one bench line per run in
# gpurun_out/cw_<workload>_<cw>.json
set -u
run() {  # workload steps cw
  local w=$1 k=$2 cw=$3
  RBFFD_TMA_CW=$cw python bench.py --workload "$w" --gpu-setup --quick --steps "$k" --warmup 5 \
    > "gpurun_out/cw_${w}_${cw}.json" 2> "gpurun_out/cw_${w}_${cw}.err"
  python - "$w" "$cw" <<'PY'
import json, sys
w, cw = sys.argv[1], sys.argv[2]
d = json.loads(open(f"gpurun_out/cw_{w}_{cw}.json").read().strip().splitlines()[-1])
print(f"{w:6s} cw={cw:3s} {d['value']:.4e} upd/s  {d['ms_per_step']*1e3:8.2f} us/step  stream frac {d['roofline']['frac']:.3f}")
PY
}
for rep in 1 2; do
  run c2 200 0; run c2 200 23
  run c2x10 100 0; run c2x10 100 23
  run c3 100 0; run c3 100 18
  run c4 40 0; run c4 40 11
done
