# L2-resident ring-fill chunks (RBFFD_L2_RES_CHUNKS = per-CTA leading chunks streamed with
# L2::evict_last; default = ring stages), quick bench; optional workload as $1.
W=${1:-c2}
run() { echo "== $*"; env "$@" timeout 300 python bench.py --workload $W --steps ${STEPS:-4000} --warmup 20 --quick 2>&1 >/dev/null | grep -E "^device"; }
for r in 0 4 8 12 16 0 4 8 12 16; do run RBFFD_L2_RES_CHUNKS=$r; done
