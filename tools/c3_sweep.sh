run() { echo "== $*"; env "$@" timeout 300 python bench.py --workload c3 --steps 400 --warmup 10 --quick 2>&1 | grep -E "^device" | sed 's/(0.*//;s/(1.*//'; }
run RBFFD_X=0
run RBFFD_TMA_SPS=1
run RBFFD_TMA_SPS=3
run RBFFD_TMA_SPS=4
run RBFFD_IDX16=0
run RBFFD_X=0
