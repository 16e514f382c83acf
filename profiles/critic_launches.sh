#!/bin/bash
# launch list of the H=64 B=65,536 critic update (and the full capture of its per-sample kernel)
CMD="python profiles/critic_sweep.py --hidden 64 --batch 65536 --no-torch"
$CMD > gpurun_out/crit_plain.log 2>&1 && cat gpurun_out/crit_plain.log && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/crit_launches.csv $CMD > gpurun_out/crit_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:critic_tc_kernel -c 1 -o /tmp/crit $CMD > gpurun_out/crit_full.log 2>&1
ncu -i /tmp/crit.ncu-rep --page source --csv --print-source sass > gpurun_out/crit_src.csv 2>/dev/null
ncu -i /tmp/crit.ncu-rep --page raw --csv > gpurun_out/crit_raw.csv 2>/dev/null
ncu -i /tmp/crit.ncu-rep --page details --csv > gpurun_out/crit_details.csv 2>/dev/null
echo done
