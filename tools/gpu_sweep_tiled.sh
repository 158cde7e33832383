#!/bin/bash
# throughput-regime sweep (~100k buses / 128 areas): build options through the GSE_* overrides
W=${1:-tiled101k_k128}
run() { env "$@" timeout 400 python bench.py --workload $W --steps 8 --no-cpu --no-profile 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', round(d['ms_per_step'],4), round(d['e2e']['value'],1))"; }
run GSE_NOP=1
run GSE_TILE_ROWS=32
run GSE_TILE_ROWS=64
run GSE_TILE_ROWS=96
run GSE_SPLIT_MIN=16
run GSE_SPLIT_MIN=32
run GSE_SPLIT_MIN=32 GSE_TILE_ROWS=64
run GSE_SPLIT_MIN=32 GSE_TILE_ROWS=96
run GSE_MAX_PIVOTS=32
run GSE_FUSED_UPDATE=1
run GSE_LEAF_BUSES=64
run GSE_GAMMA_LEAF=32
