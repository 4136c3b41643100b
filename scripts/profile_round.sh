#!/bin/bash
# Run on the GPU box: bench line, ncu launch list of the same command, one
# --set full capture of the dominant kernel. Outputs land in gpurun_out/.
set -u
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu"
python bench.py --steps 20 --warmup 3 > gpurun_out/bench_full.log 2>&1
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_ll.log 2>&1
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"xsweep|vsweep" -s 6 -c 3 \
    -o gpurun_out/prof_top $CMD > gpurun_out/ncu_full.log 2>&1
echo done
