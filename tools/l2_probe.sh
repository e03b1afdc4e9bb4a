# L2-resident ring-fill chunks (RBFFD_L2_RES_CHUNKS = per-CTA leading chunks streamed with
# L2::evict_last; default = 1.5 x ring stages), quick bench; optional workload as $1.
W=${1:-c2}
run() { echo "== $*"; env "$@" timeout 300 python bench.py --workload $W --steps ${STEPS:-4000} --warmup 20 --quick 2>&1 >/dev/null | grep -E "^device"; }
for r in 0 8 11 16 22 30 0 16 22; do run RBFFD_L2_RES_CHUNKS=$r; done
