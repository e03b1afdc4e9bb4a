# A/B of slices per stage at m=2 n=15 N=1e7 (alternating, bench.py --quick).
run() { echo "== $*"; env "$@" timeout 300 python bench.py --workload c2x10 --steps 1000 --warmup 20 --quick 2>&1 | grep -E "^device" | sed 's/(0.*//;s/(1.*//'; }
for i in 1 2 3; do run RBFFD_TMA_SPS=4; run RBFFD_TMA_SPS=5; done
