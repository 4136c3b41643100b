#!/bin/bash
# Round-2 profiling on the GPU box (outputs in gpurun_out/): the per-shape
# table (C1..C5, limiter comparison, sheath refinement sweep), the C5 and C3
# launch lists with DRAM bytes per launch (ncu, 3 metrics: one pass), and one
# --set full capture of the x and v sweeps at C3.
set -u
python scripts/shape_table.py --out gpurun_out/r02_shapes > gpurun_out/r2_shapes.log 2>&1
echo "shapes rc=$?"
B="python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --exact-steps 0"
$B > gpurun_out/r2_plain_c5.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/r2_c5_launches.csv $B > gpurun_out/r2_ncu_c5.log 2>&1
echo "ncu c5 rc=$?"
B3="python bench.py --config C3 --steps 2 --warmup 3 --no-cpu --no-e2e --exact-steps 0"
$B3 > gpurun_out/r2_plain_c3.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/r2_c3_launches.csv $B3 > gpurun_out/r2_ncu_c3ll.log 2>&1
echo "ncu c3 ll rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"xsweep|vsweep" -s 6 -c 3 \
    -o gpurun_out/r2_prof_c3 $B3 > gpurun_out/r2_ncu_c3full.log 2>&1
echo "ncu c3 full rc=$?"
