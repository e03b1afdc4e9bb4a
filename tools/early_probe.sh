# early stage release A/B (RBFFD_EARLY), single-step kernel (pair off), quick bench lines
for w in c2 c2x10 c3; do
  st=4000; [ $w != c2 ] && st=400
  for e in 0 1 0 1; do echo "== $w early=$e"; RBFFD_PAIR=0 RBFFD_EARLY=$e timeout 300 python bench.py --workload $w --steps $st --warmup 20 --quick 2>&1 >/dev/null | grep -E "^device" | sed 's/ algorithmic.*//'; done
done
