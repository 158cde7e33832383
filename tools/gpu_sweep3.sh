#!/bin/bash
# build-option sweep after the pipelined panel (env overrides read by gse_plan_create)
W=${1:-pegase9241_k16}
run() { env "$@" timeout 300 python bench.py --workload $W --steps 20 --no-cpu --no-profile 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', round(d['ms_per_step'],4), round(d['e2e']['value'],1))"; }
run GSE_NOP=1
run GSE_TILE_ROWS=32
run GSE_TILE_ROWS=40
run GSE_TILE_ROWS=56
run GSE_TILE_ROWS=64
run GSE_TILE_ROWS=72
run GSE_TILE_ROWS=96
run GSE_LEAF_BUSES=32
run GSE_LEAF_BUSES=40
run GSE_LEAF_BUSES=64
run GSE_LEAF_BUSES=64 GSE_TILE_ROWS=64
run GSE_GAMMA_LEAF=8
run GSE_GAMMA_LEAF=32
run GSE_SEPW=1.0
run GSE_SEPW=3.0
run GSE_GAMMA_SEPW=1.0
run GSE_GAMMA_SEPW=3.0
