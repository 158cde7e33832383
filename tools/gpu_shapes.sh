#!/bin/bash
# GPU parity suites under build-option overrides: other tile heights, pivot caps, leaf sizes, the panel / update
# task split, the level-launch scheduler, the counter hand-off in the back-substitution exercise panel shapes and
# code paths the defaults do not produce.  (The scale suite asserts the persistent plan and runs four rank plans
# side by side: it is skipped for the level-launch scheduler and for 96-row tiles, which do not fit two CTAs per SM.)
for E in "GSE_TILE_ROWS=48" "GSE_TILE_ROWS=96" "GSE_MAX_PIVOTS=32" "GSE_LEAF_BUSES=8 GSE_TILE_ROWS=16" "GSE_SPLIT_MIN=16" "GSE_PERSISTENT=0" "GSE_FUSED_UPDATE=0" "GSE_BWD_POLL=0" "GSE_GAMMA_TILE_ROWS=16" "GSE_FUSED_UPDATE=0 GSE_TILE_ROWS=24"; do
  SUITES="tests/test_gpu_parity.py tests/test_gpu_linalg.py tests/test_gpu_scale.py"
  case "$E" in "GSE_TILE_ROWS=96"|"GSE_PERSISTENT=0") SUITES="tests/test_gpu_parity.py tests/test_gpu_linalg.py";; esac
  echo "== $E"; env $E timeout 900 python -m pytest $SUITES -x -q 2>&1 | tail -2
done
