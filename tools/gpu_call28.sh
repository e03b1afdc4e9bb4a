# Chunk-contiguous packed stream for the persistent loop: A/B and parity.
set -x
run() {
  echo -n "$W $* "
  env "$@" timeout 300 python bench.py --workload $W --gpu-setup --quick --steps $K --warmup 10 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(f\"{d['ms_per_step']*1e3:8.2f} us/step  {d['value']:.4e}  frac {d['roofline']['frac']:.3f}\")"
}
for rep in 1 2; do
  W=c2; K=400
  run RBFFD_LOOP_PACKED=1
  run RBFFD_LOOP_PACKED=0
  W=c2x10; K=60
  run RBFFD_LOOP_PACKED=1
  run RBFFD_LOOP_PACKED=0
  W=c3; K=60
  run RBFFD_LOOP_PACKED=1
  run RBFFD_LOOP_PACKED=0
done
W=c4; K=30
run RBFFD_LOOP_PACKED=1
run RBFFD_LOOP_PACKED=0
RBFFD_LOOP_PACKED=1 timeout 1500 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_packed28.log 2>&1; tail -3 gpurun_out/pytest_packed28.log
echo done
