#!/bin/bash
# Round evidence in one gpurun call: smoke + GPU tests + bench lines of every workload + reference arm +
# persistent-kernel timeline + sanitizer + ncu launch lists / full captures.  Outputs in gpurun_out/.
mkdir -p gpurun_out
bash tools/gpu_check.sh > gpurun_out/check.log 2>&1
for W in pegase2869_k8 activsg10k_k32 tiled101k_k176 tiled101k_k128; do
  timeout 900 python bench.py --workload $W --steps 20 > gpurun_out/bench_$W.json 2> gpurun_out/bench_$W.err
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
timeout 300 python tools/persist_trace.py pegase9241_k16 > gpurun_out/trace.txt 2>&1
timeout 300 python tools/persist_trace.py tiled101k_k176 > gpurun_out/trace_tiled.txt 2>&1
bash tools/gpu_sanitize.sh > /dev/null 2>&1
bash tools/gpu_ncu.sh pegase9241_k16 > gpurun_out/ncu.log 2>&1
for f in gpurun_out/launches_persistent_pegase9241_k16.csv gpurun_out/launches_levels_pegase9241_k16.csv; do python tools/summarize_launches.py $f second-half > ${f%.csv}.txt 2>&1; done
tail -4 gpurun_out/check.log | cut -c1-300; head -3 gpurun_out/trace.txt; tail -3 gpurun_out/sanitizer.txt; ls -la gpurun_out/*.ncu-rep
for W in pegase2869_k8 activsg10k_k32 tiled101k_k176 tiled101k_k128 reference; do cut -c1-220 gpurun_out/bench_$W.json; done
