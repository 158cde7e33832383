#!/bin/bash
# compute-sanitizer memcheck + racecheck of one persistent-kernel solve and one level-path solve per case
mkdir -p gpurun_out
OUT=gpurun_out/sanitizer.txt
echo "compute-sanitizer (CUDA 12.9) on B200, tools/sanitize_solve.py: one persistent-kernel solve + one level-path solve per case" > $OUT
for CASE in ieee118_k6 pegase2869_k8; do
  for TOOL in memcheck racecheck; do
    echo "== $TOOL $CASE" >> $OUT
    timeout 900 compute-sanitizer --tool $TOOL python tools/sanitize_solve.py $CASE 2>&1 | grep -v "^$" | tail -12 >> $OUT
  done
done
cat $OUT
