# ncu --set full of the fused partitioned loop (two in-process parts, 2e6 nodes, 200 steps).
set -x
timeout 600 python tools/group_trace.py 2e6 2 > gpurun_out/plain43.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:part_loop -c 1 -o /tmp/r2_part $(echo python tools/group_trace.py 2e6 2) > gpurun_out/ncu43.log 2>&1; echo ncu=$?
python tools/ncu_summary.py /tmp/r2_part.ncu-rep gpurun_out/r2_part_loop_ncu_full.json; echo sum=$?
ncu -i /tmp/r2_part.ncu-rep --page details --csv 2>/dev/null | gzip > gpurun_out/r2_part_loop_details.csv.gz
rm -f /tmp/r2_part.ncu-rep
cat gpurun_out/plain43.log
echo done
