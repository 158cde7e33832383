#!/bin/bash
# build-option sweep after the round-2 scheduling changes (env overrides read by gse_plan_create)
W=${1:-pegase9241_k16}
run() { env "$@" timeout 300 python bench.py --workload $W --steps 30 --no-cpu --no-profile 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', round(d['ms_per_step'],4), d['plan']['fronts'], d['plan']['levels'])"; }
run GSE_NOP=1
run GSE_LEAF_BUSES=32
run GSE_LEAF_BUSES=40
run GSE_LEAF_BUSES=56
run GSE_LEAF_BUSES=64
run GSE_LEAF_BUSES=80
run GSE_GAMMA_LEAF=8
run GSE_GAMMA_LEAF=12
run GSE_GAMMA_LEAF=24
run GSE_GAMMA_LEAF=32
run GSE_SEPW=1.0
run GSE_SEPW=3.0
run GSE_SEPW=4.0
run GSE_GAMMA_SEPW=1.0
run GSE_GAMMA_SEPW=3.0
run GSE_GAMMA_SEPW=4.0
run GSE_TILE_ROWS=24
run GSE_TILE_ROWS=40
run GSE_TILE_ROWS=48
