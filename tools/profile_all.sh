# Round profiling pass (profiles/): full C2 bench line, ncu launch list, ncu --set full of
# the default step kernel at C2 / C3 / C4 and of the two-step kernel where it is the default.
OUT=gpurun_out
timeout 600 python bench.py > $OUT/bench_c2.json 2> $OUT/bench_c2.err; echo bench=$?
CMD="python bench.py --steps 300 --warmup 10 --quick"
$CMD > $OUT/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launch.log 2>&1; echo launches=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_tma -s 150 -c 1 -o $OUT/prof_c2 $CMD > $OUT/ncu_c2.log 2>&1; echo c2=$?
for w in c3 c4; do
  C="python bench.py --workload $w --steps 40 --warmup 5 --quick"
  $C > $OUT/plain_$w.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:step_tma -s 20 -c 1 -o $OUT/prof_$w $C > $OUT/ncu_$w.log 2>&1; echo $w=$?
done
P="python tools/pair_run.py 20000 200"
$P > $OUT/plain_pair.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pair_tma -s 40 -c 1 -o $OUT/prof_pair20k $P > $OUT/ncu_pair.log 2>&1; echo pair=$?
# summaries (the .ncu-rep files are too large to bring back all at once)
for t in c2 c3 c4 pair20k; do
  [ -f $OUT/prof_$t.ncu-rep ] && python tools/ncu_summary.py $OUT/prof_$t.ncu-rep $OUT/ncu_$t.json > /dev/null
done
ncu -i $OUT/prof_c2.ncu-rep --page source --csv --print-source sass > $OUT/prof_c2_sass.csv 2>/dev/null
rm -f $OUT/prof_c3.ncu-rep $OUT/prof_c4.ncu-rep $OUT/prof_pair20k.ncu-rep
du -sh $OUT
