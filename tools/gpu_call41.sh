# HEAD check: smoke, the whole GPU suite, the driver's bench commands, launch list.
set -x
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke41.log 2>&1; echo smoke=$?; cat gpurun_out/smoke41.log
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_all41.log 2>&1; tail -3 gpurun_out/pytest_all41.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r41_bench.json 2> gpurun_out/r41_bench.err; echo bench=$?
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r41_ref.json 2> gpurun_out/r41_ref.err; echo ref=$?
CMD="python bench.py --steps 20 --warmup 5 --quick"
$CMD > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r41_launches.csv $CMD > gpurun_out/r41_ncu_launch.log 2>&1; echo launches=$?
echo done
