#!/bin/bash
# A/B builds on the GPU box: each argument is one GSE_NVCC_DEFINES string ("" = defaults); per build the parity
# tests that cover the panel (test_gpu_linalg, test_gpu_parity) and the bench at the latency-bound shapes.
# usage: tools/gpu_ab.sh "" "-DGSE_TILE_SOLVE32=0"
mkdir -p gpurun_out
OUT=gpurun_out/ab.txt
: > $OUT
for D in "$@"; do
  GSE_NVCC_DEFINES="$D" python -c "from paper_2604_23175_b200 import build; build.build(force=True)" > gpurun_out/ab_build.log 2>&1 || { echo "BUILD FAILED [$D]" >> $OUT; continue; }
  timeout 900 python -m pytest tests/test_gpu_linalg.py tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -1 | sed "s/^/[$D] pytest: /" >> $OUT
  for rep in 1 2; do
    for W in ${AB_WORKLOADS:-pegase9241_k16 pegase2869_k8 activsg10k_k32}; do
      timeout 300 python bench.py --steps 30 --no-cpu --no-profile --workload $W 2>/dev/null > gpurun_out/sw.json
      python -c "import json; d=json.load(open('gpurun_out/sw.json')); print('[$D] $W', round(d['ms_per_step'],4), 'e2e', round(d['time_to_converge_ms']['warm_e2e'],4))" >> $OUT
    done
  done
done
# leave the default build behind
python -c "from paper_2604_23175_b200 import build; build.build(force=True)" >> gpurun_out/ab_build.log 2>&1
cat $OUT
