set -x
timeout 1500 python bench.py --workload c5 --gpu-setup --quick --steps 10 --warmup 3 > gpurun_out/r50_c5.json 2> gpurun_out/r50_c5.err; echo c5=$?
tail -5 gpurun_out/r50_c5.err
echo done
