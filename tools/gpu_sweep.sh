#!/bin/bash
run() { echo "=== $*"; env "$@" python bench.py --steps 10 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', round(d['value'],1), round(d['ms_per_step'],3), {k: round(v*1e6,1) for k,v in d['phase_s_per_iteration'].items()}, d['plan'])"; }
run GSE_GAMMA_LEAF=8
run GSE_GAMMA_LEAF=32
run GSE_GAMMA_LEAF=64
run GSE_TILE_ROWS=32
run GSE_TILE_ROWS=64
run GSE_TILE_ROWS=96
run GSE_MAX_PIVOTS=32
run GSE_MAX_PIVOTS=32 GSE_LEAF_BUSES=24
run GSE_LEAF_BUSES=32
run GSE_LEAF_BUSES=64
