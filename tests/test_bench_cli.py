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
