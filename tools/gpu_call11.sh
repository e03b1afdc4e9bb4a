set -x
WS="c4" ./tools/ab_old_new.sh > gpurun_out/ab4.log 2>&1
rm -f /tmp/t.bin; RBFFD_LIB=$PWD/exp/lib_trace.so RBFFD_TRACE=/tmp/t.bin python bench.py --workload c2 --gpu-setup --quick --steps 200 --warmup 5 > gpurun_out/trace_c2b.json 2>&1; python tools/trace_summary.py /tmp/t.bin > gpurun_out/trace_c2b.txt 2>&1
rm -f /tmp/t.bin; RBFFD_LIB=$PWD/exp/lib_trace.so RBFFD_TRACE=/tmp/t.bin python bench.py --workload c2x10 --gpu-setup --quick --steps 100 --warmup 5 > gpurun_out/trace_c2x10.json 2>&1; python tools/trace_summary.py /tmp/t.bin > gpurun_out/trace_c2x10.txt 2>&1
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02b.json 2> gpurun_out/bench_r02b.err
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ref_r02b.json 2> gpurun_out/ref_r02b.err
python bench.py --workload c2 --quick --steps 20 --warmup 5 > gpurun_out/plain_q.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_r02.csv python bench.py --workload c2 --quick --steps 20 --warmup 5 > gpurun_out/ncu_launch.log 2>&1
echo done
