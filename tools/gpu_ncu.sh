#!/bin/bash
# ncu evidence for one round: launch lists of both scheduling modes + full captures of the persistent
# kernel and of the two assembly kernels (level path).  Numbers printed under ncu are not bench values.
set -x
mkdir -p gpurun_out
W=${1:-pegase9241_k16}
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_persistent_$W.csv python tools/profile_solve.py $W 4 > gpurun_out/profile_p1.log 2>&1
GSE_PERSISTENT=0 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/launches_levels_$W.csv python tools/profile_solve.py $W 2 > gpurun_out/profile_p0.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gn_solve_kernel -s 2 -c 1 -f -o gpurun_out/solve_full_$W python tools/profile_solve.py $W 4 > gpurun_out/ncu_solve.log 2>&1
GSE_PERSISTENT=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"accumulate_staged_kernel|eval_templates_kernel" -s 10 -c 2 -f -o gpurun_out/assembly_full_$W python tools/profile_solve.py $W 3 > gpurun_out/ncu_asm.log 2>&1
ls -la gpurun_out/*.ncu-rep; tail -3 gpurun_out/ncu_solve.log
