#!/bin/bash
# ncu launch list (per-kernel device time) for one warm solve of the bench workload.
set -x
mkdir -p gpurun_out
W=${1:-pegase9241_k16}
# solve = 5 iterations x 56 launches = 280 launches; skip the first (cold) solve
ncu --metrics gpu__time_duration.sum --clock-control none -s 281 -c 280 --csv --log-file gpurun_out/launches_$W.csv python tools/profile_solve.py $W 2 > gpurun_out/profile_$W.log 2>&1
python tools/summarize_launches.py gpurun_out/launches_$W.csv > gpurun_out/launches_$W.txt
cat gpurun_out/launches_$W.txt
