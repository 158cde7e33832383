#!/bin/bash
# Copies what tools/gpu_evidence.sh (+ gpu_ncu.sh tiled101k_k128, the traces, linked_bench, ipc) left in gpurun_out/
# into profiles/ under round-prefixed names, and regenerates the summaries that are read here (ncu reports, SASS counts).
#   bash tools/collect_evidence.sh r02
R=${1:-r02}; P=profiles; G=gpurun_out
cp $G/bench.json $P/${R}_bench.json
for W in pegase2869_k8 activsg10k_k32 tiled101k_k176 tiled101k_k128; do cp $G/bench_$W.json $P/${R}_bench_$W.json; done
cp $G/bench_reference.json $P/${R}_bench_reference.json
cp $G/trace.txt $P/${R}_persistent_timeline_pegase9241_k16.txt
cp $G/trace_tiled128.txt $P/${R}_persistent_timeline_tiled101k_k128.txt
cp $G/sanitizer.txt $P/${R}_compute_sanitizer.txt
cp $G/launches_persistent_pegase9241_k16.txt $P/${R}_launches_persistent_pegase9241_k16.txt
cp $G/launches_levels_pegase9241_k16.txt $P/${R}_launches_levels_pegase9241_k16.txt
cp $G/linked_bench.txt $P/${R}_linked_rank_plans_one_gpu.txt
cp $G/ipc.txt $P/${R}_ipc_rank_processes_one_gpu.txt
[ -f $G/sweep_tiled.txt ] && cp $G/sweep_tiled.txt $P/${R}_sweep_tiled101k_k128.txt
python tools/ncu_summary.py $G/solve_full_pegase9241_k16.ncu-rep > $P/${R}_ncu_full_gn_solve_kernel.txt 2>&1
python tools/ncu_summary.py $G/solve_full_tiled101k_k128.ncu-rep > $P/${R}_ncu_full_gn_solve_kernel_tiled101k_k128.txt 2>&1
python tools/ncu_summary.py $G/assembly_full_pegase9241_k16.ncu-rep > $P/${R}_ncu_full_assembly_kernels.txt 2>&1
python tools/ncu_summary.py $G/assembly_full_tiled101k_k128.ncu-rep > $P/${R}_ncu_full_assembly_kernels_tiled101k_k128.txt 2>&1
python tools/sass_counts.py > $P/${R}_sass_counts.txt
for f in $G/launches_persistent_tiled101k_k128.csv $G/launches_levels_tiled101k_k128.csv; do python tools/summarize_launches.py $f second-half > $P/${R}_$(basename ${f%.csv}).txt 2>&1; done
grep -h "dram__bytes\|gpu__time_duration" $P/${R}_ncu_full_gn_solve_kernel.txt $P/${R}_ncu_full_gn_solve_kernel_tiled101k_k128.txt
