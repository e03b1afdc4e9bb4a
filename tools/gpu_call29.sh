# Loop without the final publish copy: parity suite, short/long runs.
set -x
run() {
  echo -n "$W K=$K $* "
  env "$@" timeout 300 python bench.py --workload $W --gpu-setup --quick --steps $K --warmup 5 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(f\"{d['ms_per_step']*1e3:8.2f} us/step  {d['value']:.4e}  median5 {d['timing_repeats']['median_ms_per_step']*1e3:8.2f}\")"
}
W=c2
for rep in 1 2; do K=20; run X=1; K=400; run X=1; done
timeout 1500 python -m pytest tests/test_parity_gpu.py tests/test_weights_gpu.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_pub29.log 2>&1; tail -3 gpurun_out/pytest_pub29.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -8
echo done
