# Full check of HEAD: smoke, the whole GPU suite, the driver's bench commands.
set -x
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke27.log 2>&1; echo smoke=$?; cat gpurun_out/smoke27.log
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_all27.log 2>&1; tail -3 gpurun_out/pytest_all27.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r27_bench.json 2> gpurun_out/r27_bench.err; echo bench=$?
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r27_ref.json 2> gpurun_out/r27_ref.err; echo ref=$?
echo done
