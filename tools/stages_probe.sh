# TMA ring depth sweep (RBFFD_TMA_STAGES), quick bench lines; args: workloads
for w in ${@:-c3 c4}; do
  st=4000; [ $w != c2 ] && st=200
  for e in 8 10 11 8 10 11; do echo "== $w stages=$e"; RBFFD_TMA_STAGES=$e timeout 300 python bench.py --workload $w --steps $st --warmup 10 --quick 2>&1 >/dev/null | grep -E "^device" | sed 's/ algorithmic.*//'; done
done
