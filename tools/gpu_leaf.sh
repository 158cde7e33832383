#!/bin/bash
for LB in 64 96 128 192; do
  echo "=== GSE_LEAF_BUSES=$LB"
  GSE_LEAF_BUSES=$LB python bench.py --steps 10 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value'], d['ms_per_step'], d['phase_s_per_iteration'], d['plan'])"
done
