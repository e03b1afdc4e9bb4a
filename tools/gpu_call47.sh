set -x
run() {
  echo -n "$W default "
  timeout 300 python bench.py --workload $W --gpu-setup --quick --steps $K --warmup 10 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(f\"{d['ms_per_step']*1e3:8.2f} us/step  {d['value']:.4e}\")"
}
W=c2; K=400; run
W=c2x10; K=60; run
W=c3; K=60; run
W=c4; K=24; run
timeout 1500 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_par47.log 2>&1; tail -3 gpurun_out/pytest_par47.log
echo done
