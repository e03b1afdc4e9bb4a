set -x
WS="c4 c2" ./tools/ab_old_new.sh exp/lib_loop2.so exp/lib_q642.so > gpurun_out/ab3.log 2>&1
rm -f /tmp/t.bin; RBFFD_TRACE=/tmp/t.bin python bench.py --workload c2 --gpu-setup --quick --steps 200 --warmup 5 > gpurun_out/trace_c2.json 2>&1; python tools/trace_summary.py /tmp/t.bin > gpurun_out/trace_c2.txt 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --force-dist --steps 20 --warmup 5 > gpurun_out/dist1.json 2> gpurun_out/dist1.err
python bench.py --workload c2 --gpu-setup --quick --steps 20 --warmup 5 > gpurun_out/plain_c2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:step_tma_kernel -s 10 -c 1 -o gpurun_out/prof_c2_r02 python bench.py --workload c2 --gpu-setup --quick --steps 20 --warmup 5 > gpurun_out/ncu_c2.log 2>&1
echo done
