set -x
free -g > gpurun_out/c5d_free0.txt
(while true; do free -g | sed -n 2p >> gpurun_out/c5d_mem.txt; sleep 10; done) & M=$!
timeout 2400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --force-dist --workload c5 --steps 20 --warmup 3 > gpurun_out/dist_c5.json 2> gpurun_out/dist_c5.err
echo rc=$?
kill $M
echo done
