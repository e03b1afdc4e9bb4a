set -x
timeout 600 python tools/group_probe.py 1e6 > gpurun_out/group_probe33.log 2>&1; cat gpurun_out/group_probe33.log
echo done
