set -x
timeout 1500 python -m pytest tests/test_parity_gpu.py tests/test_dsetup_gpu.py tests/test_multiprocess_gpu.py -m gpu -q -x -p no:cacheprovider -k "partitioned or dsetup or rank or process or group" > gpurun_out/pytest_grp38.log 2>&1; tail -3 gpurun_out/pytest_grp38.log
timeout 600 python tools/group_probe.py 2e6 > gpurun_out/group_probe38.log 2>&1; cat gpurun_out/group_probe38.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
echo done
