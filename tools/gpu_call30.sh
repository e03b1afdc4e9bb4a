set -x
timeout 1200 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -p no:cacheprovider -k "partitioned" > gpurun_out/pytest_part30.log 2>&1; tail -3 gpurun_out/pytest_part30.log
timeout 600 python tools/group_probe.py 2e6 > gpurun_out/group_probe30.log 2>&1; cat gpurun_out/group_probe30.log
echo done
