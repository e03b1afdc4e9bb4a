# L2 policy of the persistent loop's stream (RBFFD_LOOP_POLICY 0 first / 1 normal / 2 unchanged).
set -x
run() {
  echo -n "$W $* "
  env "$@" timeout 300 python bench.py --workload $W --gpu-setup --quick --steps $K --warmup 10 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(f\"{d['ms_per_step']*1e3:8.2f} us/step  {d['value']:.4e}\")"
}
for rep in 1 2; do
  W=c2; K=400
  for pp in 0 1 2; do run RBFFD_LOOP_POLICY=$pp; done
  W=c3; K=60
  for pp in 0 1 2; do run RBFFD_LOOP_POLICY=$pp; done
done
echo done
