set -x
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_steady_gpu.py tests/test_perf_gpu.py -q -x -p no:cacheprovider -k "not config5 and not configs_3_4" > gpurun_out/pytest_loop.log 2>&1; tail -3 gpurun_out/pytest_loop.log
run() {
  echo -n "$* "
  env "$@" timeout 300 python bench.py --workload $W --gpu-setup --quick --steps $K --warmup 10 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(f\"{d['ms_per_step']*1e3:8.2f} us/step  {d['value']:.4e}\")"
}
for rep in 1 2; do
  W=c2; K=400
  run RBFFD_PERSIST=1
  run RBFFD_PERSIST=0
  run RBFFD_PERSIST=0 RBFFD_L2_RES_CHUNKS=4
  run RBFFD_PERSIST=0 RBFFD_L2_RES_CHUNKS=6
  run RBFFD_PERSIST=0 RBFFD_L2_RES_CHUNKS=8
  run RBFFD_PERSIST=0 RBFFD_L2_RES_CHUNKS=10
  run RBFFD_PERSIST=0 RBFFD_L2_RES_CHUNKS=12
  run RBFFD_PERSIST=0 RBFFD_L2_RES_CHUNKS=8 RBFFD_TMA_SPS=5
  run RBFFD_PERSIST=1 RBFFD_TMA_SPS=5
  W=c2x10; K=100
  run RBFFD_PERSIST=1
  run RBFFD_PERSIST=0
  run RBFFD_PERSIST=0 RBFFD_L2_RES_CHUNKS=8
  W=c3; K=100
  run RBFFD_PERSIST=1
  run RBFFD_PERSIST=0
  run RBFFD_PERSIST=0 RBFFD_L2_RES_CHUNKS=8
done
echo done
