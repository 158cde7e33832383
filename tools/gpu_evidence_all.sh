#!/bin/bash
# one gpurun call for everything tools/collect_evidence.sh reads (round evidence: ~15 GPU-minutes)
bash tools/gpu_evidence.sh > gpurun_out/evidence.log 2>&1
bash tools/gpu_ncu.sh tiled101k_k128 > gpurun_out/ncu_tiled.log 2>&1
GSE_TRACE_HIST=1 timeout 300 python tools/persist_trace.py tiled101k_k128 > gpurun_out/trace_tiled128.txt 2>&1
timeout 600 python tools/linked_bench.py pegase9241_k16 1 2 4 > gpurun_out/linked_bench.txt 2>&1
timeout 600 python tools/ipc_two_process.py pegase9241_k16 2 > gpurun_out/ipc.txt 2>&1
timeout 600 python tools/ipc_two_process.py pegase2869_k8 3 >> gpurun_out/ipc.txt 2>&1
tail -12 gpurun_out/evidence.log | cut -c1-250
tail -3 gpurun_out/linked_bench.txt; tail -3 gpurun_out/ipc.txt
