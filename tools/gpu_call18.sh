set -x
python bench.py --workload c1 --steps 2000 --warmup 10 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 1200 python bench.py --workload c5 --gpu-setup --quick --steps 30 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
for w in c3 c4; do
  python bench.py --workload $w --gpu-setup --quick --steps 10 --warmup 3 > gpurun_out/plain_$w.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:step_tma_kernel -s 6 -c 1 -o gpurun_out/prof_${w}_r02 python bench.py --workload $w --gpu-setup --quick --steps 10 --warmup 3 > gpurun_out/ncu_$w.log 2>&1
done
echo done
