"""Summarise an `ncu --set full` report (read here with `ncu -i REP --page raw --csv`) into the few
numbers DESIGN.md / bench.py quote: duration, DRAM traffic, pipe activity, occupancy, stall reasons."""
import csv
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]
KEYS = [
    "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "launch__shared_mem_per_block_static", "launch__occupancy_limit_shared_mem",
    "launch__occupancy_limit_registers", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum", "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed.sum.per_cycle_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "sm__ops_path_tensor_src_fp64.sum", "sm__ops_path_tensor_src_fp64.sum.pct_of_peak_sustained_elapsed",
    "smsp__inst_executed.sum", "smsp__cycles_active.avg",
]
for r in rows[2:]:
    d = dict(zip(hdr, r))
    u = dict(zip(hdr, units))
    print("kernel:", d.get("Kernel Name", "?"))
    for k in KEYS:
        if k in d:
            print(f"  {k:84s} {d[k]:>16s} {u[k]}")
    stalls = sorted(((float(v.replace(',', '')), k) for k, v in d.items()
                     if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio") and v not in ("", "n/a")),
                    reverse=True)
    print("  warp stall reasons (warps stalled per issue-active cycle):")
    for v, k in stalls[:8]:
        print(f"    {k[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]:28s} {v:8.3f}")
    rd = float(d.get("dram__bytes_read.sum", "0").replace(',', '')); wr = float(d.get("dram__bytes_write.sum", "0").replace(',', ''))
    print(f"  dram traffic read+write: {rd + wr:.3f} {u.get('dram__bytes_read.sum','')}")
