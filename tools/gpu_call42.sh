set -x
timeout 1500 python -m pytest tests/test_parity_gpu.py tests/test_dsetup_gpu.py tests/test_multiprocess_gpu.py -m gpu -q -x -p no:cacheprovider -k "partitioned or dsetup or rank or process or group" > gpurun_out/pytest_grp42.log 2>&1; tail -3 gpurun_out/pytest_grp42.log
timeout 600 python tools/group_probe.py 1e6 2>&1 | grep -v "copy\|push kernels"
timeout 600 python tools/group_probe.py 2e6 2>&1 | grep -v "copy\|push kernels"
rm -f /tmp/g.bin; RBFFD_LIB=$PWD/exp/lib_trace.so RBFFD_TRACE=/tmp/g.bin timeout 600 python tools/group_trace.py 1e6 2 2>&1 | tail -3
python tools/trace_summary.py /tmp/g.bin 2>&1 | tail -10
echo done
