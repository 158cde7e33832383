#!/bin/bash
# ncu launch list (per-kernel device time) for one warm solve of the bench workload.
set -x
mkdir -p gpurun_out
W=${1:-pegase9241_k16}
# two solves are captured; the summary keeps the second (warm) one
ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/launches_$W.csv python tools/profile_solve.py $W 2 > gpurun_out/profile_$W.log 2>&1
python tools/summarize_launches.py gpurun_out/launches_$W.csv second-half > gpurun_out/launches_$W.txt
cat gpurun_out/launches_$W.txt
