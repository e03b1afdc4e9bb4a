set -x
RBFFD_SEG=1 timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -p no:cacheprovider -k "segment or synthetic_fixed or tma or full_size_config2 or streaming or every_width or idx16" > gpurun_out/pytest_seg.log 2>&1; tail -3 gpurun_out/pytest_seg.log
for rep in 1 2; do for w in c2 c2x10 c3 c4; do for sg in 1 0; do
  k=300; [ $w = c2x10 ] && k=100; [ $w = c3 ] && k=100; [ $w = c4 ] && k=40
  echo -n "$w seg=$sg "; RBFFD_SEG=$sg timeout 400 python bench.py --workload $w --gpu-setup --quick --steps $k --warmup 5 2>gpurun_out/seg_$w_$sg.err | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(f\"{d['value']:.4e} upd/s {d['ms_per_step']*1e3:9.2f} us/step frac {d['roofline']['frac']:.3f}\")"
done; done; done
echo done
