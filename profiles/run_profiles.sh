#!/bin/bash
# Profiling recipe used for profiles/ (run under gpurun, 1 GPU).  Each ncu run
# follows the identical plain command, which must exit 0 first.
set -x
CMD="python bench.py --steps 2 --warmup 1 --no-cpu --no-secondary"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
CMD1="python bench.py --steps 1 --warmup 0 --no-cpu --no-secondary"
$CMD1 > gpurun_out/plain1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"rollout_tc_kernel" -c 1 -o gpurun_out/prof_full $CMD1 > gpurun_out/ncu_full.log 2>&1
echo done
