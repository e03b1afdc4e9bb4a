set -x
python tools/e2e_phases.py 20 > gpurun_out/e2e_phases5.log 2>&1; tail -16 gpurun_out/e2e_phases5.log
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider --durations=10 > gpurun_out/pytest_all3.log 2>&1; tail -14 gpurun_out/pytest_all3.log
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ref_r02c.json 2> gpurun_out/ref_r02c.err
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02c.json 2> gpurun_out/bench_r02c.err; tail -8 gpurun_out/bench_r02c.err
echo done
