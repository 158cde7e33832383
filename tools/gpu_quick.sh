#!/bin/bash
# correctness (GPU tests) + per-level timing + a short bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python tools/profile_levels.py pegase9241_k16 2>&1 | grep -E "launches, sum|^front |^backward |^eval|^accum|launch (2|3|8|14|15|16|17|20|26|28) "
python bench.py --steps 20 --no-cpu 2>/dev/null > gpurun_out/bench_quick.json; python -c "import json; d=json.load(open('gpurun_out/bench_quick.json')); print('bench', d['value'], d['ms_per_step'], d['e2e']['value'], d['phase_s_per_iteration'])"
