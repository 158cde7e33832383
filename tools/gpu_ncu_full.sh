#!/bin/bash
# ncu --set full capture of a few launches of one kernel (regex $1), skipping $2 matching launches.
set -x
mkdir -p gpurun_out
K=${1:-front_task_kernel}; S=${2:-44}; C=${3:-3}; W=${4:-pegase9241_k16}; O=${5:-prof}
ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c $C -f -o gpurun_out/$O python tools/profile_solve.py $W 1 > gpurun_out/$O.log 2>&1
ls -la gpurun_out/$O.ncu-rep
