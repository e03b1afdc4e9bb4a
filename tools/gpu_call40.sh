set -x
timeout 300 python tools/e2e_phases.py 20 > gpurun_out/e2e40.log 2>&1; tail -32 gpurun_out/e2e40.log
echo done
