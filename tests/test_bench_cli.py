"""bench.py launch plumbing that needs no GPU: `--gpus N` outside a launcher re-executes itself under
torch.distributed.run with N ranks (the driver starts its scaling runs the same way)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_gpus_n_spawns_n_ranks():
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--spawn-check"],
                         capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["spawn_check"] and line["n_gpus"] == 2 and line["rank_sum"] == 3.0
    assert "spawning 2 ranks" in out.stderr


def test_reference_arm_prints_the_contract_line():
    """`bench.py --impl reference` (the CPU arm the driver runs beside the B200 arm): one JSON line with the
    B200 arm's metric / unit / config keys, `impl: reference`, a `cpu_baseline` describing the run and an `e2e`
    that repeats the line's own value with zero copies.  Smallest workload, one solve (a few seconds)."""
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload", "pegase2869_k8",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=600, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["unit"] == "GN iterations/s" and line["higher_is_better"] is True
    assert line["dtype"] == "f64" and line["vs_baseline"] is None and line["steps"] == 1 and line["warmup"] == 0
    cfg = line["config"]
    assert cfg["workload"] == "pegase2869_k8" and cfg["areas"] == 8 and cfg["n_bus"] == 2869 and cfg["iterations_per_solve"] == 5
    assert set(cfg) == {"workload", "areas", "n_bus", "rows", "n_gamma", "iterations_per_solve", "l2"}
    cb = line["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["value"] == line["value"] and cb["sample"]
    assert line["e2e"] == {"value": line["value"], "unit": line["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert line["value"] > 0 and abs(line["value"] - cfg["iterations_per_solve"] / (line["ms_per_step"] * 1e-3)) < 1e-6 * line["value"]
