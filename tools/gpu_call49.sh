# Final HEAD check: smoke, the whole GPU suite, the driver's bench commands, e2e phases.
set -x
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke49.log 2>&1; echo smoke=$?; cat gpurun_out/smoke49.log
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_all49.log 2>&1; tail -3 gpurun_out/pytest_all49.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r49_bench.json 2> gpurun_out/r49_bench.err; echo bench=$?
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r49_ref.json 2> gpurun_out/r49_ref.err; echo ref=$?
timeout 300 python tools/e2e_phases.py 20 > gpurun_out/e2e49.log 2>&1; tail -14 gpurun_out/e2e49.log
echo done
