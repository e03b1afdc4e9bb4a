# Full bench.py lines for every BASELINE config that fits one GPU (profiles/r01_*_bench.json).
OUT=gpurun_out
timeout 600 python bench.py --workload c1 --steps 100000 --warmup 100 --cpu-budget 10 > $OUT/bench_c1.json 2> $OUT/bench_c1.err; echo c1=$?
timeout 1200 python bench.py --workload c2x10 --steps 1000 --warmup 20 --cpu-budget 15 > $OUT/bench_c2x10.json 2> $OUT/bench_c2x10.err; echo c2x10=$?
timeout 1200 python bench.py --workload c3 --steps 500 --warmup 10 --cpu-budget 20 > $OUT/bench_c3.json 2> $OUT/bench_c3.err; echo c3=$?
timeout 1800 python bench.py --workload c4 --steps 200 --warmup 5 --cpu-budget 20 > $OUT/bench_c4.json 2> $OUT/bench_c4.err; echo c4=$?
