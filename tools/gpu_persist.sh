#!/bin/bash
# persistent dataflow kernel: smoke, parity tests (bounded), bench in both scheduling modes
mkdir -p gpurun_out
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -8
for P in 1 0; do
  GSE_PERSISTENT=$P timeout 300 python bench.py --steps 20 --no-cpu 2>gpurun_out/bench_p$P.err > gpurun_out/bench_p$P.json
  python -c "import json; d=json.load(open('gpurun_out/bench_p$P.json')); print('persistent=$P', d['value'], d['ms_per_step'], d['e2e']['value'], d['phase_s_per_iteration'], d['plan'])" || tail -5 gpurun_out/bench_p$P.err
done
GSE_STAMPS=0 timeout 300 python bench.py --steps 20 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nostamps', d['value'], d['ms_per_step'], d['e2e']['value'])"
