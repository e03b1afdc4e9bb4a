# A/B of alternative builds placed in exp/ (RBFFD_LIB) against the default library, quick bench lines
for lib in default "$@" default "$@"; do
  for w in c2 c2x10; do
    st=4000; [ $w != c2 ] && st=300
    echo "== $lib $w"
    if [ $lib = default ]; then timeout 300 python bench.py --workload $w --steps $st --warmup 10 --quick 2>&1 >/dev/null | grep -E "^device" | sed 's/ algorithmic.*//';
    else RBFFD_LIB=$PWD/$lib timeout 300 python bench.py --workload $w --steps $st --warmup 10 --quick 2>&1 >/dev/null | grep -E "^device" | sed 's/ algorithmic.*//'; fi
  done
done
