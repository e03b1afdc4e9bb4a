set -x
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --force-dist --steps 20 --warmup 5 > gpurun_out/dist32.json 2> gpurun_out/dist32.err; echo dist=$?; tail -c 2000 gpurun_out/dist32.json; tail -3 gpurun_out/dist32.err
timeout 1500 python -m pytest tests/test_parity_gpu.py tests/test_dsetup_gpu.py tests/test_multiprocess_gpu.py -m gpu -q -x -p no:cacheprovider -k "partitioned or dsetup or rank or process or group" > gpurun_out/pytest_grp32.log 2>&1; tail -3 gpurun_out/pytest_grp32.log
echo done
