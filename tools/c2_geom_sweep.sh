#!/bin/bash
# C2 ring geometry re-sweep on the round-2 kernel: slices per stage and
# L2-resident ring-fill chunks (RBFFD_TMA_SPS, RBFFD_L2_RES_CHUNKS).
run() {
  echo -n "$* "
  env "$@" python bench.py --workload c2 --gpu-setup --quick --steps 400 --warmup 10 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(f\"{d['ms_per_step']*1e3:7.2f} us/step  {d['value']:.4e}\")"
}
for rep in 1 2; do
  run RBFFD_TMA_SPS=4
  run RBFFD_TMA_SPS=3
  run RBFFD_TMA_SPS=5
  run RBFFD_TMA_SPS=6
  run RBFFD_L2_RES_CHUNKS=0
  run RBFFD_L2_RES_CHUNKS=8
  run RBFFD_L2_RES_CHUNKS=24
  run RBFFD_L2_RES_CHUNKS=40
  run RBFFD_TMA_STAGES=9
done
