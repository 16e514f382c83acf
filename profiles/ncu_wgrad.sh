#!/bin/bash
# ncu --set full of the critic update's wgrad_kernel and critic_tc_kernel (H=64, B=65,536)
CMD="python profiles/critic_sweep.py --hidden 64 --batch 65536 --no-torch --steps 2"
$CMD > gpurun_out/wg_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"wgrad_kernel" -c 1 -o /tmp/wg $CMD > gpurun_out/ncu_wg.log 2>&1
ncu -i /tmp/wg.ncu-rep --page source --csv --print-source sass > gpurun_out/wg_src.csv 2>/dev/null
ncu -i /tmp/wg.ncu-rep --page raw --csv > gpurun_out/wg_raw.csv 2>/dev/null
ncu -i /tmp/wg.ncu-rep --page details --csv > gpurun_out/wg_details.csv 2>/dev/null
tail -2 gpurun_out/ncu_wg.log
