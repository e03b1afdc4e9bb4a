# Final HEAD check: smoke and the whole GPU suite.
set -x
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke44.log 2>&1; echo smoke=$?; cat gpurun_out/smoke44.log
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_all44.log 2>&1; tail -3 gpurun_out/pytest_all44.log
echo done
