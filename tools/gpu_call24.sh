# Persistent loop: L2-resident share of the stream (RBFFD_LOOP_RES = chunks per
# CTA and step streamed with evict_last), C2 and m=2 N=1e7.
set -x
run() {
  echo -n "$W $* "
  env "$@" timeout 300 python bench.py --workload $W --gpu-setup --quick --steps $K --warmup 10 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(f\"{d['ms_per_step']*1e3:8.2f} us/step  {d['value']:.4e}  frac {d['roofline']['frac']:.3f}\")"
}
for rep in 1 2; do
  W=c2; K=400
  for r in 0 4 8 12 16 20 24 32; do run RBFFD_LOOP_RES=$r; done
done
W=c2x10; K=60
for r in 0 8 16; do run RBFFD_LOOP_RES=$r; done
echo done
