# TMA ring depth sweep (RBFFD_TMA_STAGES; "def" = the library's default), quick bench lines
for w in ${@:-c2}; do
  st=4000; [ $w != c2 ] && st=200
  for e in def 8 11 def 8 11; do
    echo "== $w stages=$e"
    if [ $e = def ]; then timeout 300 python bench.py --workload $w --steps $st --warmup 10 --quick 2>&1 >/dev/null | grep -E "^device" | sed 's/ algorithmic.*//';
    else RBFFD_TMA_STAGES=$e timeout 300 python bench.py --workload $w --steps $st --warmup 10 --quick 2>&1 >/dev/null | grep -E "^device" | sed 's/ algorithmic.*//'; fi
  done
done
