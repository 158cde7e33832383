#!/bin/bash
# development loop: GPU parity tests (bounded), persistent-kernel timeline, short bench in both scheduling modes
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -8
timeout 300 python tools/persist_trace.py ${1:-pegase9241_k16} > gpurun_out/trace.txt 2>&1; head -${2:-14} gpurun_out/trace.txt
for P in 1 0; do
  GSE_PERSISTENT=$P timeout 300 python bench.py --steps 20 --no-cpu 2>gpurun_out/bench_p$P.err > gpurun_out/bench_p$P.json
  python -c "import json; d=json.load(open('gpurun_out/bench_p$P.json')); print('persistent=$P', d['value'], d['ms_per_step'], d['e2e']['value'], d['phase_s_per_iteration'])" || tail -5 gpurun_out/bench_p$P.err
done
