set -x
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r48_bench.json 2> gpurun_out/r48_bench.err; echo bench=$?
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r48_ref.json 2> gpurun_out/r48_ref.err; echo ref=$?
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke48.log 2>&1; echo smoke=$?
echo done
