set -x
python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "not config5" > gpurun_out/pytest_chain.log 2>&1; tail -3 gpurun_out/pytest_chain.log
for c in 1 0; do
  rm -f /tmp/t.bin; RBFFD_CHAIN=$c RBFFD_LIB=$PWD/exp/lib_trace.so RBFFD_TRACE=/tmp/t.bin python bench.py --workload c2 --gpu-setup --quick --steps 200 --warmup 5 > gpurun_out/trace_chain$c.json 2>&1; python tools/trace_summary.py /tmp/t.bin > gpurun_out/trace_chain$c.txt 2>&1
done
for rep in 1 2; do for w in c2 c2x10 c3 c4; do for c in 1 0; do
  k=300; [ $w = c2x10 ] && k=100; [ $w = c3 ] && k=100; [ $w = c4 ] && k=40
  echo -n "$w chain=$c "; RBFFD_CHAIN=$c python bench.py --workload $w --gpu-setup --quick --steps $k --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(f\"{d['value']:.4e} upd/s {d['ms_per_step']*1e3:9.2f} us/step frac {d['roofline']['frac']:.3f}\")"
done; done; done
echo done
