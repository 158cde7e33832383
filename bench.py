#!/usr/bin/env python
"""bench.py -- GN iterations/s and time-to-converge of the multi-area state estimator.

    python bench.py --gpus N --steps K --warmup W            # B200 arm (this repo's CUDA path)
    python bench.py --impl reference --gpus N --steps K ...  # the reference algorithm on host cores

A "step" is one full flat-start Gauss-Newton solve (to convergence) of the workload
BASELINE.json's metric is quoted on: the PEGASE-9241-shaped grid split into 16 areas
(configs[2]; 91,919 measurement rows, n_Gamma = 716), synthetic measurements.

One JSON line on stdout (rank 0).  `value` = GN iterations per second with inputs resident in
HBM (device-timed solve loop); `e2e` = the same metric through the public API with HOST
buffers (measurement values + weights host->device, flat start host->device, estimate
device->host inside the timed region); `roofline` = the dominant kernel group against the
measured peaks; `cpu_baseline` = the C oracle port (oracle/) on this box's host cores.
"""

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

WORKLOADS = {"pegase2869_k8": "pegase2869", "pegase9241_k16": "pegase9241", "activsg10k_k32": "activsg10k",
             "tiled101k_k176": "tiled", "tiled101k_k128": "tiled"}


def build_workload(name):
    import paper_2604_23175_b200 as G
    from paper_2604_23175_b200 import synth
    shape = WORKLOADS[name]
    if shape == "tiled":
        # BASELINE.json configs[4]: ~100k buses tiled from PEGASE areas (11 tiles of the 9241-bus shape with
        # its committed 16-area partition each: 101,651 buses, 176 areas, n_Gamma = 7996)
        net, _ = synth.tiled_network(synth.shaped_network("pegase9241"), 11)
        ms = G.generate_measurements(net, G.MeasurementConfig(seed=0))
        if name == "tiled101k_k128":
            # the 128 areas BASELINE.json names: partition_network of this package on the tiled grid (committed; 34 s)
            part = G.load_partition(net, synth.golden_partition("tiled101k_k128"))
        else:
            part = G.load_partition(net, synth.tile_partition(synth.golden_partition("pegase9241"), 11))
        return net, ms, part
    net = synth.shaped_network(shape)
    ms = G.generate_measurements(net, G.MeasurementConfig(seed=0))
    part = G.load_partition(net, synth.golden_partition(shape))
    return net, ms, part


METRIC_NAMES = {"pegase9241_k16": "GN iterations/s (PEGASE-9241-shape MASE, 16 areas)"}


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            return json.load(fh), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region (NVML every ~2 ms; nvidia-smi as the fallback)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index, self.samples, self._stop = index, [], threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _setup(self):
        # NVML (nvidia_ml_py, the library nvidia-smi itself reads) answers in well under a millisecond, so the short
        # timed region of a latency-bound solve (tens of ms) still gets tens of samples; the nvidia-smi process
        # (~50 ms per call) is the fallback when NVML cannot be loaded.  Loaded BEFORE the timed region starts (import +
        # nvmlInit + handle lookup take tens of ms: done inside the sampling thread they left one sample per run).
        try:
            import pynvml
            pynvml.nvmlInit()
            uuid = None
            try:
                import torch
                uuid = str(torch.cuda.get_device_properties(self.index).uuid)
            except Exception:
                pass
            h = None
            if uuid:
                for cand in (uuid, "GPU-" + uuid):
                    try:
                        h = pynvml.nvmlDeviceGetHandleByUUID(cand.encode() if isinstance(cand, str) else cand)
                        break
                    except Exception:
                        h = None
            self._nv = (pynvml, h if h is not None else pynvml.nvmlDeviceGetHandleByIndex(self.index))
        except Exception:
            self._nv = None

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                if nv:
                    P, h = nv
                    r = P.nvmlDeviceGetCurrentClocksEventReasons(h) if hasattr(P, "nvmlDeviceGetCurrentClocksEventReasons") \
                        else P.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                    flag = lambda bit: "Active" if r & bit else "Not Active"
                    self.samples.append([str(P.nvmlDeviceGetClockInfo(h, P.NVML_CLOCK_SM)), str(P.nvmlDeviceGetMaxClockInfo(h, P.NVML_CLOCK_SM)),
                                         flag(0x8), flag(0x40), flag(0x20), flag(0x4)])
                    self._stop.wait(0.002)
                    continue
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                nv = None
            self._stop.wait(0.2 if not nv else 0.002)

    def __enter__(self):
        self._setup()
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self):
        sm = [float(s[0]) for s in self.samples if s and s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if len(s) > 1 and s[1].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({n for s in self.samples for n, v in zip(names, s[2:6]) if v.lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def cpu_solve_is_unbounded(net, part):
    """True when one CPU solve of the workload cannot fit the bench's time bound (~100k-bus grid)."""
    return net.n_bus > 50000


def cpu_reference(net, ms, part, threads, budget_s=20.0, min_runs=2, exact_steps=None, warmup=1):
    """Time the C oracle port (the reference's algorithm) on this host: solves/s, iterations."""
    from oracle.mase_oracle import Oracle
    t0 = time.perf_counter()
    orc = Oracle(net, ms, part.area_of_bus)
    setup = time.perf_counter() - t0
    if cpu_solve_is_unbounded(net, part):
        # the dense boundary Cholesky alone is > 100 GFLOP per iteration in the scalar port: the bounded
        # sample is ONE GN iteration from the flat start (no warm-up), not a solve to convergence
        t0 = time.perf_counter()
        res = orc.solve(max_iter=1, threads=threads)
        return res, time.perf_counter() - t0, setup, 1
    for _ in range(max(1, warmup)):
        res = orc.solve(threads=threads)    # warm-up
    times = []
    while (len(times) < exact_steps) if exact_steps else (len(times) < min_runs or (sum(times) < budget_s and len(times) < 50)):
        t0 = time.perf_counter()
        res = orc.solve(threads=threads)
        times.append(time.perf_counter() - t0)
    return res, float(np.mean(times)), setup, len(times)


REF_DIR = os.path.join(ROOT, "oracle", "_ref")


def workload_config(workload, net, ms, part, n_gamma, iterations):
    """`config` of the JSON line: a function of the workload only, identical in both arms."""
    return {"workload": workload, "areas": int(part.k), "n_bus": int(net.n_bus), "rows": int(ms.m), "n_gamma": int(n_gamma),
            "iterations_per_solve": int(iterations),
            "l2": "B200 arm: flushed between steps (256 MB write); reference arm: host caches, nothing flushed"}


def time_python_reference(net, ms, part, max_bus=20000):
    """ONE flat-start solve of the UNMODIFIED reference package (installed by __graft_entry__.build() into the
    git-ignored oracle/_ref with `pip install --target`; it travels to the GPU box with the snapshot), through its
    own public API: gridse.solve_multiarea on the same network / measurement set / partition, single BLAS thread
    (the reference is single-threaded Python; un-pinned OpenBLAS only adds noise).  Returns a dict or None."""
    if not os.path.isdir(os.path.join(REF_DIR, "gridse")) or net.n_bus > max_bus:
        return None
    import dataclasses
    sys.path.insert(0, REF_DIR)
    try:
        import gridse as R
        from threadpoolctl import threadpool_limits
        rnet = R.BusBranchNetwork.from_components([R.Bus(**dataclasses.asdict(b)) for b in net.buses],
                                                  [R.Branch(**dataclasses.asdict(b)) for b in net.branches])
        rms = R.generate_measurements(rnet, R.MeasurementConfig(seed=0))
        same_inputs = bool(np.array_equal(rms.z, ms.z) and np.array_equal(rms.weight, ms.weight))
        rpart = R.load_partition(rnet, part.area_of_bus)
        with threadpool_limits(limits=1):
            t0 = time.perf_counter()
            est, rep = R.solve_multiarea(rnet, rms, rpart)
            sec = time.perf_counter() - t0
        return {"kind": "reference", "what": "gridse.solve_multiarea (unmodified reference, oracle/_ref), one flat-start solve "
                "incl. its per-call symbolic setup, 1 thread", "solve_s": sec, "iterations": int(rep.iterations),
                "converged": bool(rep.converged), "it_per_s": rep.iterations / sec, "objective": float(rep.objective),
                "same_inputs_as_gpu_arm": same_inputs, "va": est.va, "vm": est.vm}
    finally:
        sys.path.remove(REF_DIR)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import mase_oracle
    from oracle.mase_oracle import Oracle
    net, ms, part = build_workload(args.workload)
    threads = min(mase_oracle.max_threads(), part.k, os.cpu_count() or 1)
    res, sec, setup, runs = cpu_reference(net, ms, part, threads, exact_steps=args.steps, warmup=args.warmup)
    value = res["iterations"] / sec
    pyref = time_python_reference(net, ms, part)
    if pyref:
        pyref["state_max_abs_diff_vs_port"] = float(max(np.max(np.abs(pyref.pop("va") - res["va"])), np.max(np.abs(pyref.pop("vm") - res["vm"]))))
    line = {
        "impl": "reference", "metric": METRIC_NAMES.get(args.workload, f"GN iterations/s ({args.workload} MASE)"), "value": value,
        "unit": "GN iterations/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": workload_config(args.workload, net, ms, part, Oracle(net, ms, part.area_of_bus).n_gamma, res["iterations"]),
        "cpu_baseline": {"value": value, "unit": "GN iterations/s", "cores": threads, "kind": "port",
                         "reference_python_s": pyref["solve_s"] if pyref else None, "reference_python": pyref,
                         "sample": (f"{runs} full flat-start solves" if not cpu_solve_is_unbounded(net, part) else
                                    "ONE GN iteration from the flat start (a solve to convergence does not fit the time bound)")
                                   + f" of {args.workload} (C restatement of the reference "
                                   f"algorithm, oracle/mase_oracle.c; analysis {setup:.2f}s excluded)"},
        "e2e": {"value": value, "unit": "GN iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "time_to_converge_ms": sec * 1e3, "objective": res["objective"],
    }
    print(json.dumps(line), flush=True)


def dgemm_peak(torch, dev):
    """Measured FP64 GEMM throughput on this box (MEASURED_PEAKS.json has no FP64 figure)."""
    n = 4096
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    torch.matmul(a, b)
    torch.cuda.synchronize(dev)
    best = 1e9
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        torch.cuda.synchronize(dev)
        best = min(best, e0.elapsed_time(e1))
    return 2.0 * n ** 3 / (best * 1e-3) / 1e12


def spawn_ranks(args):
    """`python bench.py --gpus N` (N > 1) outside a launcher: re-execute this command under
    torch.distributed.run with one rank per GPU (what the driver does itself for its scaling runs)."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    print(f"[bench] spawning {args.gpus} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    sys.exit(subprocess.call(cmd))


def run_spawn_check(args):
    """Rendezvous + one collective per rank without touching a GPU (`--spawn-check`, gloo): proves that the
    N-rank launch path of this file works on a box without N GPUs (tests/test_bench_cli.py)."""
    import torch
    import torch.distributed as dist
    rank, world = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        dist.init_process_group("gloo")
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t)
        dist.barrier()
    if rank == 0:
        print(json.dumps({"spawn_check": True, "n_gpus": world, "requested": args.gpus, "rank_sum": float(t[0]),
                          "backend": "gloo"}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_gpu(args):
    import torch
    import paper_2604_23175_b200 as G
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but the launcher started {world} rank(s)")
    if torch.cuda.device_count() < world:
        if rank == 0:
            print(json.dumps({"error": f"--gpus {world} needs {world} CUDA devices, this box has {torch.cuda.device_count()}",
                              "n_gpus": world}), flush=True)
        raise SystemExit(2)
    if world > 1:
        import torch.distributed as dist
        from paper_2604_23175_b200.distributed import DistributedEstimator
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        # communicator line per rank (NCCL_DEBUG=INFO adds NCCL's own transport / NVLS lines)
        probe = torch.ones(1, device=torch.device("cuda", local))
        dist.all_reduce(probe)
        print(f"[bench] rank {rank}/{world} cuda:{local} {torch.cuda.get_device_name(local)} NCCL "
              f"{'.'.join(str(v) for v in torch.cuda.nccl.version())} all_reduce ok ({int(probe[0])})", file=sys.stderr, flush=True)
    dev = torch.device("cuda", local)
    net, ms, part = build_workload(args.workload)
    torch.zeros(1, device=dev)                       # CUDA context creation is not part of the plan build
    torch.cuda.synchronize(dev)

    # cold path, step 0: the partitioner itself (C++ passes; the reference takes 24 s / 182 s / 79 s at the three
    # named shapes).  The bench then uses the committed partition, which this must reproduce bus for bus.
    partition_s = None
    if rank == 0 and WORKLOADS[args.workload] != "tiled":
        t0 = time.perf_counter()
        again = G.partition_network(net, part.k, seed=0)
        partition_s = time.perf_counter() - t0
        assert np.array_equal(again.area_of_bus, part.area_of_bus), "partition_network does not reproduce the committed partition"

    t0 = time.perf_counter()
    if world > 1:
        # (GSE_BENCH_EXCHANGE=collective keeps the ranks on the level-launch path with torch.distributed collectives)
        est = DistributedEstimator(net, ms, part, device=local, exchange=os.environ.get("GSE_BENCH_EXCHANGE", "auto"))
    else:
        est = G.MultiAreaEstimator(net, ms, part, device=local)
    plan_s = time.perf_counter() - t0

    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)   # > 126 MB L2

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def one_step(e2e=False):
        """One flat-start solve; returns (device seconds, wall seconds, iterations)."""
        flush.zero_()
        torch.cuda.synchronize(dev)
        t = time.perf_counter()
        if e2e:
            if world == 1:
                est.update_from_pinned()              # this step's z, w: pinned host memory -> device (async, plan stream)
            else:
                est.update_measurements(ms)
        state, rep = est.estimate()               # flat start h2d, GN loop, state d2h
        wall = time.perf_counter() - t
        return est.last_gpu_s, wall, rep

    if world == 1:
        zv, wv = est.pinned_inputs()                  # the scan's inputs live in pinned host memory
        zv[:] = ms.z
        wv[:] = ms.weight
    for _ in range(max(args.warmup, 3)):
        one_step()
    barrier()
    dev_s, e2e_s, iters = [], [], 0
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            g, w, rep = one_step()
            dev_s.append(g)
            iters += rep.iterations
        barrier()
        for _ in range(args.steps):
            g, w, rep_e = one_step(e2e=True)
            e2e_s.append(w)
    barrier()
    tot_dev, tot_e2e = float(np.sum(dev_s)), float(np.sum(e2e_s))
    if world > 1:
        t = torch.tensor([tot_dev, tot_e2e], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_dev, tot_e2e = float(t[0]), float(t[1])
    if rank != 0:
        return
    it_per_solve = rep.iterations
    value = iters / tot_dev
    e2e_value = it_per_solve * args.steps / tot_e2e

    # ---- roofline of the dominant kernel -------------------------------------------------------------
    # One solve = ONE launch of gn_solve_kernel (the persistent dataflow kernel: every GN iteration
    # and the objective).  Its duration is measured live above (CUDA events on the plan's stream
    # around the launch).  Algorithmic work per launch = per-iteration figures x
    # iterations; the FP64 tensor bound is the larger of the two lower bounds, so it is the primary.
    peaks, peak_src = measured_peaks()
    roof, phases, stats, level_phases = None, None, est.plan.stats() if world == 1 else {}, None
    if world == 1:
        t_launch = tot_dev / args.steps
        fp64_peak = dgemm_peak(torch, dev)
        flops = stats["dense_flops"] * it_per_solve
        abytes = stats["alg_bytes"] * it_per_solve
        traffic = None
        tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tpath):
            traffic = json.load(open(tpath)).get(args.workload, {}).get("gn_solve_kernel")
        phases = {p: float(rep.timings[p]) / it_per_solve for p in G.solver.PHASES}   # in-kernel globaltimer stamps
        t_asm = max(phases["assembly"], 1e-9)
        roof = {"kernel": "gn_solve_kernel", "bound": "tensor", "achieved": flops / t_launch / 1e12, "peak": fp64_peak,
                "unit": "TFLOP/s", "frac": flops / t_launch / 1e12 / fp64_peak, "traffic": traffic,
                "traffic_unit": "bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum, ncu --set full, profiles/)",
                "peak_source": "cuBLAS FP64 DGEMM 4096^3 measured in this run (MEASURED_PEAKS.json has no FP64 figure)",
                "flops_per_launch": flops, "launch_s": t_launch,
                "other": {"bound": "hbm", "achieved": abytes / t_launch / 1e9, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                          "frac": abytes / t_launch / 1e9 / peaks["hbm_gbs"], "bytes_per_launch": abytes,
                          "peak_source": f"MEASURED_PEAKS.json ({peak_src})",
                          "assembly_phase": {"what": "template evaluation + fused accumulation items inside the kernel "
                                                     "(phase time from in-kernel globaltimer stamps)",
                                             "achieved": stats["alg_bytes"] / t_asm / 1e9,
                                             "frac": stats["alg_bytes"] / t_asm / 1e9 / peaks["hbm_gbs"],
                                             "bytes_per_iteration": stats["alg_bytes"], "s_per_iteration": t_asm}}}
        if not args.no_profile:
            # the same solve on the level-launch path (one kernel per tree level, CUDA events between phases)
            prof = G.MultiAreaEstimator(net, ms, part, config=G.SolverConfig(profile_phases=True), device=local)
            for _ in range(3):
                prof.estimate()
            acc = np.zeros(5)
            reps = 5
            for _ in range(reps):
                flush.zero_()
                torch.cuda.synchronize(dev)
                _, r = prof.estimate()
                acc += np.array([r.timings[p] for p in G.solver.PHASES])
            level_phases = dict(zip(G.solver.PHASES, (float(x) for x in acc / (reps * it_per_solve))))
            prof.close()


    # ---- CPU baseline: the oracle port, bounded sample ---------------------------------------------
    cpu = None
    if world == 1 and not args.no_cpu and cpu_solve_is_unbounded(net, part):
        cpu = {"value": None, "unit": "GN iterations/s", "cores": 1, "kind": "port",
               "sample": f"skipped at {args.workload}: one GN iteration of the scalar port takes minutes here (dense Cholesky of the "
                         f"n_gamma = {est.n_gamma} boundary system, the reference's algorithm); `--impl reference` times that one iteration"}
    elif world == 1 and not args.no_cpu:
        res1, sec1, setup1, runs1 = cpu_reference(net, ms, part, 1, budget_s=10.0)
        pyref = time_python_reference(net, ms, part)
        if pyref:
            va_r, vm_r = pyref.pop("va"), pyref.pop("vm")
            state_now, _ = est.estimate()
            pyref["gpu_state_max_rel_diff"] = float(max(np.max(np.abs(state_now.va - va_r) / np.maximum(np.abs(va_r), 1.0)),
                                                        np.max(np.abs(state_now.vm - vm_r) / np.abs(vm_r))))
            pyref["gpu_objective_rel_diff"] = abs(pyref["objective"] - rep.objective) / pyref["objective"]
        cpu = {"value": res1["iterations"] / sec1, "unit": "GN iterations/s", "cores": 1, "kind": "port",
               "reference_python_s": pyref["solve_s"] if pyref else None, "reference_python": pyref,
               "sample": f"{runs1} full flat-start solves of {args.workload}, oracle/mase_oracle.c single thread; "
                         f"host has {os.cpu_count()} cores; analysis {setup1:.2f}s excluded",
               "time_to_converge_ms": sec1 * 1e3, "iterations": res1["iterations"],
               "objective_rel_diff": abs(res1["objective"] - rep.objective) / res1["objective"]}

    # the reference's own entry point (solve_multiarea(net, ms, part), reference solver.py:204-205; what its harness
    # calls 11 times per cell, harness.py:115-158): first call = analysis + upload + solve, later calls hit the plan cache
    drop_in = None
    if world == 1 and not args.no_profile:
        G.solver.clear_plan_cache()
        t0 = time.perf_counter()
        st_d, rep_d = G.solve_multiarea(net, ms, part)
        cold = time.perf_counter() - t0
        warm = []
        for _ in range(10):
            t0 = time.perf_counter()
            st_d, rep_d = G.solve_multiarea(net, ms, part)
            warm.append(time.perf_counter() - t0)
        drop_in = {"call": "solve_multiarea(net, ms, part)", "cold_s": cold, "warm_ms": float(np.median(warm)) * 1e3,
                   "iterations": rep_d.iterations, "plan_cache": dict(G.solver.plan_cache_stats)}
        G.solver.clear_plan_cache()

    m, nb = ms.m, net.n_bus
    line = {
        "metric": METRIC_NAMES.get(args.workload, f"GN iterations/s ({args.workload} MASE)"), "value": value, "unit": "GN iterations/s",
        "n_gpus": world, "steps": args.steps, "warmup": max(args.warmup, 3),
        "ms_per_step": tot_dev / args.steps * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args.workload, net, ms, part, est.n_gamma, it_per_solve),
        "converged": bool(rep.converged), "parallelism": f"areas sharded over {world} GPU(s), one process per GPU",
        "exchange": ("none (single rank)" if world == 1 else
                     "in-kernel over peer memory (CUDA IPC / NVLink): one persistent launch per rank and solve" if getattr(est, "linked", False)
                     else "torch.distributed collectives between level launches"),
        "time_to_converge_ms": {"warm_device": tot_dev / args.steps * 1e3, "warm_e2e": tot_e2e / args.steps * 1e3,
                                "plan_build_s": plan_s, "partition_s": partition_s},
        "objective": rep.objective,
        "drop_in": drop_in,
        "e2e": {"value": e2e_value, "unit": "GN iterations/s", "h2d_bytes_per_step": 16 * m,
                "d2h_bytes_per_step": 16 * nb + 16 * it_per_solve},
        "gpu_launches": int(est.launches_per_solve * args.steps * 2),
        "clocks": clocks.summary(),
    }
    if roof:
        line["roofline"] = roof
        line["phase_s_per_iteration"] = phases
        if level_phases:
            line["level_path_phase_s_per_iteration"] = level_phases
        line["plan"] = {k: stats[k] for k in ("fronts", "levels", "tasks", "max_front", "persistent", "solve_ctas",
                                             "solve_smem_bytes", "items_per_iteration")}
    if cpu:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)
    est.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="pegase9241_k16", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-profile", action="store_true", help="skip the per-phase profile pass (development sweeps)")
    ap.add_argument("--spawn-check", action="store_true", help="N-rank launch + one gloo collective, no GPU work")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and (args.impl == "b200" or args.spawn_check):
        spawn_ranks(args)
    if args.spawn_check:
        run_spawn_check(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
