#!/bin/bash
# A/B of the step kernel: round-1 tree (exp_old/, its own bench), alternative
# builds of the current tree (exp/*.so via RBFFD_LIB, same ABI) and the current
# library, on the benchmark widths (device setup).  Usage: ab_old_new.sh [lib.so ...]
set -u
line() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(f\"{d['value']:.4e} upd/s {d['ms_per_step']*1e3:9.2f} us/step\")"; }
WS=${WS:-"c4 c3 c2"}
for rep in 1 2; do
  for w in $WS; do
    k=200; [ $w = c3 ] && k=100; [ $w = c4 ] && k=40
    if [ -d exp_old ]; then echo -n "$w old  "; (cd exp_old && python bench.py --workload $w --quick --steps $k --warmup 5 2>/dev/null | line); fi
    for lib in "$@"; do
      echo -n "$w $(basename $lib) "; RBFFD_LIB=$PWD/$lib python bench.py --workload $w --gpu-setup --quick --steps $k --warmup 5 2>/dev/null | line
    done
    echo -n "$w cur  "; python bench.py --workload $w --gpu-setup --quick --steps $k --warmup 5 2>/dev/null | line
  done
done
