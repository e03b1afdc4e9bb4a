# A/B of slices per stage at n=15 (C2 and N=1e7), alternating, bench.py --quick.
run() { w=$1; shift; echo "== $w $*"; env "$@" timeout 300 python bench.py --workload $w --steps $STEPS --warmup 20 --quick 2>&1 | grep -E "^device" | sed 's/(0.*//;s/(1.*//'; }
STEPS=5000; for i in 1 2; do run c2 RBFFD_TMA_SPS=4; run c2 RBFFD_TMA_SPS=3; run c2 RBFFD_TMA_SPS=2; done
STEPS=800; run c2x10 RBFFD_TMA_SPS=4; run c2x10 RBFFD_TMA_SPS=3
