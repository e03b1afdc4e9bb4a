set -x
timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 1 --force-dist --workload c5 --steps 10 --warmup 3 > gpurun_out/dist52.json 2> gpurun_out/dist52.err; echo dist=$?
tail -4 gpurun_out/dist52.err
echo done
