#!/bin/bash
# per-kernel device times of the B=128 update cycle (pointmass shapes), plus the wall time per cycle
python profiles/engine_cycle.py > gpurun_out/cycle_plain.log 2>&1 && cat gpurun_out/cycle_plain.log && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cycle_launches.csv python -c "
import sys; sys.path.insert(0,'profiles'); import engine_cycle; engine_cycle.main(M=8)" > gpurun_out/cycle_ncu.log 2>&1
echo done
