# e2e thread split: host-prep pool vs OpenMP staging threads (run_time_loop at C2, 20 steps).
set -x
for cfg in "X=1" "OMP_NUM_THREADS=12 RBFFD_HOST_THREADS=4" "OMP_NUM_THREADS=10 RBFFD_HOST_THREADS=6" "OMP_NUM_THREADS=8 RBFFD_HOST_THREADS=8" "OMP_NUM_THREADS=16 RBFFD_HOST_THREADS=4" "OMP_NUM_THREADS=14 RBFFD_HOST_THREADS=2"; do
  echo "== $cfg"
  env $cfg RBFFD_VERBOSE=0 timeout 300 python tools/e2e_phases.py 20 2>&1 | grep "^call" | tail -3
done
echo done
