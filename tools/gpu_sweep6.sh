#!/bin/bash
# tile height of the boundary-tree fronts alone (GSE_GAMMA_TILE_ROWS), latency-bound shapes
for W in pegase9241_k16 activsg10k_k32 pegase2869_k8; do
  for T in 0 16 24 40 48; do
    GSE_GAMMA_TILE_ROWS=$T timeout 300 python bench.py --steps 20 --no-cpu --workload $W 2>/dev/null > gpurun_out/sw.json
    python -c "import json; d=json.load(open('gpurun_out/sw.json')); print('$W gamma_tile=$T', round(d['ms_per_step'],4), int(d['plan']['tasks']))"
  done
done
