# ncu --set full of one default C2 step launch (after a plain run exits 0).
OUT=gpurun_out
CMD="python bench.py --steps 300 --warmup 10 --quick $BENCH_ARGS"
$CMD > $OUT/plain_step.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:step_ -s 150 -c 1 -o $OUT/prof_${TAG:-step} $CMD > $OUT/ncu_${TAG:-step}.log 2>&1; echo ncu=$?
