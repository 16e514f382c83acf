#!/bin/bash
# Full ncu capture (with source) of the first K1 launch of the default bench
# workload; the plain command must exit 0 first.
W=${1:-manipulator3}
CMD1="python bench.py --steps 1 --warmup 0 --no-cpu --no-secondary --workload $W"
$CMD1 > gpurun_out/plain_k1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"rollout_tc_kernel" -c 1 -o gpurun_out/k1_$W $CMD1 > gpurun_out/ncu_k1.log 2>&1
tail -2 gpurun_out/ncu_k1.log
