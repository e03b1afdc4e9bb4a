set -x
run() {
  echo -n "$W $* "
  env "$@" timeout 300 python bench.py --workload $W --gpu-setup --quick --steps $K --warmup 10 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(f\"{d['ms_per_step']*1e3:8.2f} us/step  {d['value']:.4e}  frac {d['roofline']['frac']:.3f}\")"
}
for rep in 1 2; do
  W=c2; K=400
  run RBFFD_LOOP_SPS=5
  run RBFFD_LOOP_SPS=4
  run RBFFD_LOOP_SPS=6
  run RBFFD_LOOP_SPS=8
  run RBFFD_LOOP_SPS=5 RBFFD_LOOP_STAGES=8
  W=c3; K=100
  run RBFFD_LOOP_SPS=3
  run RBFFD_LOOP_SPS=2
  run RBFFD_LOOP_SPS=4
  W=c4; K=40
  run RBFFD_LOOP_SPS=1
  run RBFFD_LOOP_SPS=2
  run RBFFD_PERSIST=0
done
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_all4.log 2>&1; tail -3 gpurun_out/pytest_all4.log
echo done
