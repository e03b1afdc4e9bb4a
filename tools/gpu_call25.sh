# Slot barrier vs arrival counter in the persistent loop: A/B, trace, parity.
set -x
run() {
  echo -n "$W $* "
  env "$@" timeout 300 python bench.py --workload $W --gpu-setup --quick --steps $K --warmup 10 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(f\"{d['ms_per_step']*1e3:8.2f} us/step  {d['value']:.4e}  frac {d['roofline']['frac']:.3f}\")"
}
for rep in 1 2; do
  W=c2; K=400
  run RBFFD_LOOP_BARRIER=slots
  run RBFFD_LOOP_BARRIER=counter
  W=c2x10; K=60
  run RBFFD_LOOP_BARRIER=slots
  run RBFFD_LOOP_BARRIER=counter
done
W=c3; K=60
run RBFFD_LOOP_BARRIER=slots
run RBFFD_LOOP_BARRIER=counter
for b in slots counter; do
  rm -f /tmp/t.bin; RBFFD_LOOP_BARRIER=$b RBFFD_LIB=$PWD/exp/lib_trace.so RBFFD_TRACE=/tmp/t.bin timeout 300 python bench.py --workload c2 --gpu-setup --quick --steps 200 --warmup 5 > /dev/null 2>&1
  echo "trace $b"; python tools/trace_summary.py /tmp/t.bin 2>&1 | tail -9
done
timeout 1500 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_parity25.log 2>&1; tail -3 gpurun_out/pytest_parity25.log
echo done
