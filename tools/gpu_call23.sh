# Round-2 final measurement pass: official bench lines, reference arm, the
# in-process group probe, ncu launch list and --set full of stream_loop_kernel
# (reports summarised on the box and deleted: gpurun brings back <= 64 MiB).
set -x
OUT=gpurun_out
timeout 300 python bench.py --workload c4 --gpu-setup --quick --steps 40 --warmup 10 > $OUT/r2_c4_default.json 2>/dev/null; echo c4=$?
timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/r2_bench.json 2> $OUT/r2_bench.err; echo bench=$?
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $OUT/r2_ref.json 2> $OUT/r2_ref.err; echo ref=$?
timeout 600 python tools/group_probe.py 2e6 > $OUT/r2_group_probe.log 2>&1; echo group=$?
if [ -f exp/lib_trace.so ]; then
  rm -f /tmp/t.bin; RBFFD_LIB=$PWD/exp/lib_trace.so RBFFD_TRACE=/tmp/t.bin timeout 300 python bench.py --workload c2 --gpu-setup --quick --steps 200 --warmup 5 > $OUT/r2_trace_c2.json 2>&1
  python tools/trace_summary.py /tmp/t.bin > $OUT/r2_trace_c2_loop.txt 2>&1; echo trace=$?
fi
CMD="python bench.py --steps 20 --warmup 5 --quick"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/r2_launches.csv $CMD > $OUT/r2_ncu_launch.log 2>&1; echo launches=$?
for W in c2 c3 c4; do
  C="python bench.py --workload $W --gpu-setup --quick --steps 8 --warmup 3"
  timeout 600 $C > $OUT/r2_plain_$W.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:stream_loop -s 1 -c 1 -o /tmp/r2_loop_$W $C > $OUT/r2_ncu_full_$W.log 2>&1; echo full_$W=$?
  python tools/ncu_summary.py /tmp/r2_loop_$W.ncu-rep $OUT/r2_loop_${W}_ncu_full.json; echo sum_$W=$?
  ncu -i /tmp/r2_loop_$W.ncu-rep --page raw --csv 2>/dev/null | gzip > $OUT/r2_loop_${W}_raw.csv.gz
  ncu -i /tmp/r2_loop_$W.ncu-rep --page details --csv 2>/dev/null | gzip > $OUT/r2_loop_${W}_details.csv.gz
  [ $W = c2 ] && ncu -i /tmp/r2_loop_$W.ncu-rep --page source --csv 2>/dev/null | gzip > $OUT/r2_loop_${W}_source.csv.gz
  rm -f /tmp/r2_loop_$W.ncu-rep
done
du -sh $OUT
echo done
