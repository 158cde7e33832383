#!/bin/bash
# throughput-regime sweep after the relaxed interior amalgamation
W=${1:-tiled101k_k128}
run() { env "$@" timeout 400 python bench.py --workload $W --steps 8 --no-cpu --no-profile 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', round(d['ms_per_step'],4), d['plan']['fronts'], d['plan']['levels'], d['plan']['tasks'])"; }
run GSE_NOP=1
run GSE_LEAF_BUSES=32
run GSE_LEAF_BUSES=64
run GSE_LEAF_BUSES=96
run GSE_LEAF_BUSES=24
run GSE_TILE_ROWS=40
run GSE_TILE_ROWS=56
run GSE_TILE_ROWS=64
run GSE_SEPW=1.0
run GSE_SEPW=3.0
run GSE_FUSED_UPDATE=1
run GSE_CHAIN_MODE=2
