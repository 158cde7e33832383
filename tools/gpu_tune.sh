#!/bin/bash
# correctness + per-level timing under a few tile sizes
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for T in 96 64 48; do
  echo "=== GSE_TILE_ROWS=$T"
  GSE_TILE_ROWS=$T python tools/profile_levels.py pegase9241_k16 2>&1 | grep -E "launches, sum|^front |^backward |^eval|^accum|launch (3|8|16|17|20|26) " 
  GSE_TILE_ROWS=$T python bench.py --steps 10 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value'], d['ms_per_step'], d['phase_s_per_iteration'])"
done
