# Round-2 final measurement pass: official bench lines, reference arm, the
# in-process group probe, ncu launch list and --set full of stream_loop_kernel.
set -x
OUT=gpurun_out
timeout 300 python bench.py --workload c4 --gpu-setup --quick --steps 40 --warmup 10 > $OUT/r2_c4_default.json 2>/dev/null; echo c4=$?
timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/r2_bench.json 2> $OUT/r2_bench.err; echo bench=$?
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $OUT/r2_ref.json 2> $OUT/r2_ref.err; echo ref=$?
timeout 600 python tools/group_probe.py 2e6 > $OUT/r2_group_probe.log 2>&1; echo group=$?
CMD="python bench.py --steps 20 --warmup 5 --quick"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/r2_launches.csv $CMD > $OUT/r2_ncu_launch.log 2>&1; echo launches=$?
for W in c2 c3 c4; do
  C="python bench.py --workload $W --gpu-setup --quick --steps 8 --warmup 3"
  timeout 600 $C > $OUT/r2_plain_$W.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:stream_loop -s 1 -c 1 -o $OUT/r2_loop_$W $C > $OUT/r2_ncu_full_$W.log 2>&1; echo full_$W=$?
done
echo done
