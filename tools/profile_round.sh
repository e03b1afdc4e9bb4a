# One profiling pass for profiles/: full bench line, ncu launch list, ncu --set full of the step kernel.
set -x
OUT=gpurun_out
timeout 600 python bench.py > $OUT/bench_full.json 2> $OUT/bench_full.err; echo bench=$?
CMD="python bench.py --steps 300 --warmup 10 --quick"
$CMD > $OUT/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launch.log 2>&1; echo launches=$?
$CMD > $OUT/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:step_tma -s 150 -c 1 -o $OUT/prof_step $CMD > $OUT/ncu_full.log 2>&1; echo full=$?
