# Slices-per-stage sweep of the TMA ring across workloads (bench.py --quick).
run() { w=$1; shift; echo "== $w $*"; env "$@" timeout 300 python bench.py --workload $w --steps $STEPS --warmup 10 --quick 2>&1 | grep -E "^device" | sed 's/(0.*//;s/(1.*//'; }
STEPS=3000; for s in 0 5 6 8; do run c2 RBFFD_TMA_SPS=$s; done
STEPS=400; run c2x10 RBFFD_X=0; run c2x10 RBFFD_TMA_SPS=6; run c2x10 RBFFD_TMA_SPS=8
STEPS=400; run c3 RBFFD_TMA_SPS=3
STEPS=100; run c4 RBFFD_X=0; run c4 RBFFD_TMA_SPS=2
