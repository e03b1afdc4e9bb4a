set -x
timeout 600 python tools/group_probe.py 1e6 > gpurun_out/group_probe34.log 2>&1; cat gpurun_out/group_probe34.log
rm -f /tmp/g.bin; RBFFD_LIB=$PWD/exp/lib_trace.so RBFFD_TRACE=/tmp/g.bin timeout 600 python tools/group_trace.py 1e6 2 2>&1 | tail -5
python tools/trace_summary.py /tmp/g.bin 2>&1 | tail -20
echo done
