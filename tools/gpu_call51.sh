set -x
OUT=gpurun_out
for W in c3 c2x10; do
  C="python bench.py --workload $W --gpu-setup --quick --steps 8 --warmup 3"
  timeout 600 $C > $OUT/r51_plain_$W.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none -k regex:stream_loop -s 1 -c 1 -o /tmp/r51_$W $C > $OUT/r51_ncu_$W.log 2>&1; echo full_$W=$?
  python tools/ncu_summary.py /tmp/r51_$W.ncu-rep $OUT/r51_loop_${W}_ncu_full.json; echo sum_$W=$?
  rm -f /tmp/r51_$W.ncu-rep
done
echo done
