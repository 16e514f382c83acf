#!/bin/bash
# ncu --set full of the B=128 update-cycle critic kernel; summaries exported on the box
python profiles/cycle_small.py > gpurun_out/cyc_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"critic_kernel|vp_kernel" -c 3 -o /tmp/cycle_critic python profiles/cycle_small.py > gpurun_out/ncu_cycle.log 2>&1
ncu -i /tmp/cycle_critic.ncu-rep --page source --csv --print-source sass > gpurun_out/cycle_critic_src.csv 2>/dev/null
ncu -i /tmp/cycle_critic.ncu-rep --page raw --csv > gpurun_out/cycle_critic_raw.csv 2>/dev/null
ncu -i /tmp/cycle_critic.ncu-rep --page details --csv > gpurun_out/cycle_critic_details.csv 2>/dev/null
ls -la gpurun_out
