#!/bin/bash
# ncu --set full of the B=128 update-cycle kernels (critic_kernel, the actor's vp_kernel)
CMD='python -c "import sys; sys.path.insert(0,\"profiles\"); import engine_cycle; engine_cycle.main(M=4)"'
eval $CMD > gpurun_out/cyc_plain.log 2>&1 && \
eval ncu --set full --clock-control none --import-source on -k regex:"critic_kernel|vp_kernel" -c 3 -o gpurun_out/cycle_full $CMD > gpurun_out/ncu_cycle.log 2>&1
tail -2 gpurun_out/ncu_cycle.log
