#!/bin/bash
# parameter sweep of the persistent scheduler (env overrides read by gse_plan_create)
mkdir -p gpurun_out
run() { env "$@" timeout 300 python bench.py --steps 20 --no-cpu --no-profile 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', round(d['ms_per_step'],4), round(d['e2e']['value'],1))"; }
run GSE_SPLIT_MIN=1000
run GSE_SPLIT_MIN=32
run GSE_SPLIT_MIN=48
run GSE_SPLIT_MIN=16
run GSE_SPLIT_MIN=48 GSE_TILE_ROWS=32
run GSE_SPLIT_MIN=48 GSE_TILE_ROWS=64
run GSE_SPLIT_MIN=1000 GSE_TILE_ROWS=32
run GSE_SPLIT_MIN=1000 GSE_TILE_ROWS=64
run GSE_SPLIT_MIN=32 GSE_LEAF_BUSES=32
run GSE_SPLIT_MIN=32 GSE_LEAF_BUSES=64
run GSE_SPLIT_MIN=32 GSE_LEAF_BUSES=24
run GSE_SPLIT_MIN=32 GSE_GAMMA_LEAF=8
run GSE_SPLIT_MIN=32 GSE_GAMMA_LEAF=32
run GSE_SPLIT_MIN=32 GSE_MAX_PIVOTS=32
