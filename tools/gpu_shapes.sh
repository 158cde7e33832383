#!/bin/bash
# GPU parity suites under build-option overrides: other tile heights, pivot caps, leaf sizes, the panel / update
# task split and the level-launch scheduler exercise panel shapes the defaults do not produce.
for E in "GSE_TILE_ROWS=48" "GSE_TILE_ROWS=96" "GSE_MAX_PIVOTS=32" "GSE_LEAF_BUSES=8 GSE_TILE_ROWS=16" "GSE_SPLIT_MIN=16" "GSE_PERSISTENT=0" "GSE_FUSED_UPDATE=0"; do
  echo "== $E"; env $E timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_linalg.py -x -q 2>&1 | tail -2
done
