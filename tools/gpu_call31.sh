set -x
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --force-dist --steps 20 --warmup 5 > gpurun_out/dist31.json 2> gpurun_out/dist31.err; echo dist=$?; tail -c 1500 gpurun_out/dist31.json; tail -5 gpurun_out/dist31.err
echo done
