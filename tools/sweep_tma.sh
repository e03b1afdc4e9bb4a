# TMA-ring geometry / variant sweep on the C2 workload (bench.py --quick).
run() { echo "== $*"; env "$@" timeout 300 python bench.py --steps 4000 --warmup 50 --quick $BENCH_ARGS 2>&1 | grep -E "^device" | sed 's/(0.*//'; }
BENCH_ARGS=--native run RBFFD_TMA_RPL=1
BENCH_ARGS=--native run RBFFD_TMA_RPL=2
run RBFFD_TMA_RPL=0
run RBFFD_TMA_RPL=1
BENCH_ARGS="--ldg" run RBFFD_TMA_RPL=0
