# Fused partitioned persistent loop: parity tests of the partitioned paths, group probe.
set -x
timeout 1200 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -p no:cacheprovider -k "partitioned" > gpurun_out/pytest_part26.log 2>&1; tail -15 gpurun_out/pytest_part26.log
timeout 900 python -m pytest tests/test_dsetup_gpu.py tests/test_multiprocess_gpu.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_dset26.log 2>&1; tail -5 gpurun_out/pytest_dset26.log
timeout 600 python tools/group_probe.py 2e6 > gpurun_out/group_probe26.log 2>&1; cat gpurun_out/group_probe26.log
echo done
