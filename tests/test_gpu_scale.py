"""Size-independent properties at the largest BASELINE.json configuration (~100k buses: 11 tiles of
the PEGASE-9241 shape, 176 areas, n_Gamma = 7996) and equivalence of the two schedulers.

The CPU oracle needs minutes per iteration at this size (dense n_Gamma^3 / 3 boundary Cholesky), so
parity is checked through properties the domain offers: a noiseless measurement set must return the
generating state (reference test_solver.py:80-102), repeated solves must be bit-identical
(test_solver.py:314-322), and the persistent dataflow kernel must reproduce the level-launch path
bit for bit (same arithmetic, different scheduling).  Needs a B200: ``pytest -m gpu``.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G():
    import paper_2604_23175_b200 as G
    return G


@pytest.fixture(scope="module")
def tiled(G):
    from paper_2604_23175_b200 import synth
    base = synth.shaped_network("pegase9241")
    net, _ = synth.tiled_network(base, 11)
    part = G.load_partition(net, synth.tile_partition(synth.golden_partition("pegase9241"), 11))
    noisy = G.generate_measurements(net, G.MeasurementConfig(seed=0))
    exact = G.generate_measurements(net, G.MeasurementConfig(sigma_vm=0.0, sigma_power=0.0))
    est = G.MultiAreaEstimator(net, noisy, part)
    yield net, part, noisy, exact, est
    est.close()


def test_tiled_100k_shape(tiled):
    net, part, noisy, exact, est = tiled
    assert net.n_bus == 11 * 9241 and part.k == 176
    assert noisy.m == 3 * net.n_bus + 4 * net.n_branch
    assert est.n_gamma == 7996
    st = est.plan.stats()
    assert st["persistent"] == 1.0 and st["solve_ctas"] >= 148


def test_tiled_100k_noiseless_returns_truth(tiled):
    net, part, noisy, exact, est = tiled
    est.update_measurements(exact)
    state, rep = est.estimate()
    assert rep.converged and rep.iterations <= 6
    va_true = np.array([b.va_true for b in net.buses]); vm_true = np.array([b.vm_true for b in net.buses])
    assert np.max(np.abs(state.va - va_true)) < 1e-8
    assert np.max(np.abs(state.vm - vm_true) / vm_true) < 1e-8
    assert rep.objective < 1e-16 * exact.m


def test_tiled_100k_bitwise_repeatable_and_scheduler_independent(G, tiled):
    net, part, noisy, exact, est = tiled
    est.update_measurements(noisy)
    s1, r1 = est.estimate()
    s2, r2 = est.estimate()
    assert r1.converged and r1.iterations == r2.iterations
    assert np.array_equal(s1.va, s2.va) and np.array_equal(s1.vm, s2.vm) and r1.objective == r2.objective
    assert est.last_deltas[-1] < 1e-6
    # per-phase timings of the persistent kernel (device stamps): all present, sum within the total
    assert sum(r1.timings[p] for p in G.solver.PHASES) <= r1.timings["total"]
    lvl = G.MultiAreaEstimator(net, noisy, part, config=G.SolverConfig(profile_phases=True))
    try:
        s3, r3 = lvl.estimate()
    finally:
        lvl.close()
    assert r3.iterations == r1.iterations
    assert np.array_equal(s1.va, s3.va) and np.array_equal(s1.vm, s3.vm)
    assert r3.objective == r1.objective
    # the tiles are weakly coupled copies of one grid: J is close to 11 x the single-grid optimum
    assert 10.5 * 73721.5 < r1.objective < 11.5 * 73721.5


def test_tiled_100k_in_128_areas_gives_the_same_estimate(G, tiled):
    """BASELINE.json's ~100k-bus configuration names 128 areas: the committed partition_network result of
    this package on the tiled grid (cases/part_tiled101k_k128.json).  The WLS optimum does not depend on
    the partition: same iteration count, same state (to solver accuracy) and objective as with 176 areas;
    noiseless measurements return the truth."""
    from paper_2604_23175_b200 import synth
    net, part176, noisy, exact, est176 = tiled
    part = G.load_partition(net, synth.golden_partition("tiled101k_k128"))
    assert part.k == 128
    est = G.MultiAreaEstimator(net, noisy, part)
    try:
        est176.update_measurements(noisy)
        s176, r176 = est176.estimate()
        s128, r128 = est.estimate()
        assert r128.converged and r128.iterations == r176.iterations
        assert np.max(np.abs(s128.va - s176.va)) < 1e-9 and np.max(np.abs(s128.vm - s176.vm)) < 1e-9
        assert abs(r128.objective - r176.objective) <= 1e-10 * r176.objective
        again, r2 = est.estimate()
        assert np.array_equal(again.va, s128.va) and np.array_equal(again.vm, s128.vm)
        est.update_measurements(exact)
        st, rep = est.estimate()
        va_true = np.array([b.va_true for b in net.buses]); vm_true = np.array([b.vm_true for b in net.buses])
        assert rep.converged and np.max(np.abs(st.va - va_true)) < 1e-8 and np.max(np.abs(st.vm - vm_true) / vm_true) < 1e-8
    finally:
        est.close()


def test_tiled_100k_in_128_areas_matches_the_reference_run(G, tiled):
    """BASELINE.json configs[4] against the UNMODIFIED reference: tests/golden/tiled101k_k128.npz holds the
    reference's own solve_multiarea run of this configuration (make_golden.py tiled101k: 197 s of CPU, LAPACK
    Cholesky of the n_Gamma = 5692 boundary system).  Same GN iteration count, per-iteration stacked norms,
    final va / vm within 1e-8 relative, J within 1e-10 relative (north_star tolerances) -- on the
    persistent kernel and on the level-launch path."""
    from conftest import load_golden
    from paper_2604_23175_b200 import synth
    g = load_golden("tiled101k_k128")
    net, _, noisy, _, _ = tiled
    assert np.array_equal(synth.golden_partition("tiled101k_k128"), g["area_of_bus"])
    zs = g["z_sum"]
    assert abs(noisy.z.sum() - zs[0]) <= 1e-12 * zs[1] and abs(noisy.weight.sum() - zs[2]) <= 1e-12 * zs[2]
    part = G.load_partition(net, g["area_of_bus"])
    for cfg in (G.SolverConfig(), G.SolverConfig(profile_phases=True)):
        est = G.MultiAreaEstimator(net, noisy, part, config=cfg)
        try:
            state, rep = est.estimate()
            assert est.n_gamma == int(g["n_gamma"]) == 5692
            assert rep.iterations == int(g["iterations"]) == 5 and rep.converged == bool(g["converged"])
            # (the intermediate iterates of this ill-conditioned ~100k-bus system differ by ~1e-8 between two
            # elimination orders -- the reference factors S_Gamma densely in natural order -- and the norms with
            # them; the fixed point they converge to is compared at the north_star tolerances below)
            assert np.allclose(est.last_deltas, g["deltas"], rtol=1e-6, atol=1e-7)
            assert np.max(np.abs(state.va - g["va"]) / np.maximum(np.abs(g["va"]), 1.0)) < 1e-8
            assert np.max(np.abs(state.vm - g["vm"]) / np.abs(g["vm"])) < 1e-8
            jref = float(g["objective"])
            assert abs(rep.objective - jref) <= 1e-10 * jref
        finally:
            est.close()


@pytest.mark.parametrize("name", ["ieee14_k2", "ieee118_k6", "pegase2869_k8", "pegase9241_k16", "activsg10k_k32"])
def test_persistent_kernel_matches_level_path_bitwise(G, name):
    from conftest import build_case
    net, ms, part, g = build_case(name)
    a, ra = G.solve_multiarea(net, ms, part)
    b, rb = G.solve_multiarea(net, ms, part, config=G.SolverConfig(profile_phases=True))
    assert ra.iterations == rb.iterations == int(g["iterations"])
    assert np.array_equal(a.va, b.va) and np.array_equal(a.vm, b.vm)
    assert ra.objective == rb.objective


@pytest.mark.parametrize("name", ["ieee118_k6", "pegase2869_k8", "pegase9241_k16"])
def test_backsubstitution_handoff_through_the_data_matches_the_counter_handoff_bitwise(G, name, monkeypatch):
    """The persistent kernel hands the solution entries of the back-substitution over through the entries themselves
    (armed by the forward pass, polled by the descendants; ``GSE_BWD_POLL=0`` keeps the completion counters).  Same
    arithmetic either way: identical bits, also on the third solve of one plan and after a level-launch solve
    (which does not arm anything) in between."""
    from conftest import build_case
    net, ms, part, g = build_case(name)
    est = G.MultiAreaEstimator(net, ms, part)                      # (plans read the override when they are built)
    monkeypatch.setenv("GSE_BWD_POLL", "0")
    ctr = G.MultiAreaEstimator(net, ms, part)
    monkeypatch.delenv("GSE_BWD_POLL")
    try:
        a, ra = est.estimate()
        b, rb = ctr.estimate()
        assert ra.iterations == rb.iterations == int(g["iterations"])
        assert np.array_equal(a.va, b.va) and np.array_equal(a.vm, b.vm) and ra.objective == rb.objective
        lv, rl = G.solve_multiarea(net, ms, part, config=G.SolverConfig(profile_phases=True))      # level path, same cached plan family
        for _ in range(2):
            c, rc = est.estimate()
            assert rc.iterations == ra.iterations and np.array_equal(c.va, a.va) and np.array_equal(c.vm, a.vm)
        assert np.array_equal(lv.va, a.va) and np.array_equal(lv.vm, a.vm)
    finally:
        est.close(); ctr.close()


def test_persistent_kernel_iteration_cap_and_failure(G):
    """max_outer_iterations is honoured inside the kernel (converged=False, last iterate returned --
    reference test_solver.py:271-276) and a non-SPD area still raises (test_solver.py:335-342)."""
    from conftest import build_case
    net, ms, part, g = build_case("ieee118_k6")
    est, rep = G.solve_multiarea(net, ms, part, config=G.SolverConfig(max_outer_iterations=2))
    assert rep.iterations == 2 and not rep.converged
    ref, rref = G.solve_multiarea(net, ms, part, config=G.SolverConfig(max_outer_iterations=2, profile_phases=True))
    assert np.array_equal(est.va, ref.va) and np.array_equal(est.vm, ref.vm)
    only_vm = G.generate_measurements(net, G.MeasurementConfig(types=(G.MeasurementType.VM,)))
    with pytest.raises(G.SolverError, match="area"):
        G.solve_multiarea(net, only_vm, part)


def test_pinned_input_refresh_matches_staged_refresh(G):
    """update_from_pinned (async copies from caller-visible pinned buffers) == update_measurements."""
    from conftest import build_case
    net, ms, part, g = build_case("ieee118_k6")
    est = G.MultiAreaEstimator(net, ms, part)
    try:
        masked = G.apply_mask(ms, G.MeasurementType.QF)
        est.update_measurements(masked)
        a, ra = est.estimate()
        est.update_measurements(ms)
        zv, wv = est.pinned_inputs()
        zv[:] = masked.z
        wv[:] = masked.weight
        est.update_from_pinned()
        b, rb = est.estimate()
        assert ra.iterations == rb.iterations and np.array_equal(a.va, b.va) and np.array_equal(a.vm, b.vm)
        assert ra.objective == rb.objective
    finally:
        est.close()


@pytest.mark.parametrize("name,world", [("ieee118_k6", 2), ("pegase2869_k8", 3)])
def test_rank_sharded_plans_on_one_device_match_single_plan_bitwise(G, name, world):
    """The multi-rank device path without a cluster: ``world`` rank plans (each owning a block of
    areas) live on the one GPU and exchange their packed (S_b | b_hat) segments and delta_x_Gamma
    with device copies -- exactly what the NCCL send/recv + broadcast of distributed.py move.  The
    result must equal the single-plan solve bit for bit (blocks are summed on the coordinator in
    area order)."""
    import torch
    from conftest import build_case
    from paper_2604_23175_b200.distributed import CudaEngine, area_work_estimate, assign_areas
    net, ms, part, g = build_case(name)
    bord, maps = G.build_variable_maps(net, part)
    cfg = G.SolverConfig()
    ref, rref = G.solve_multiarea(net, ms, part, maps=(bord, maps), config=cfg)
    area_rank = assign_areas(area_work_estimate(maps), world)
    assert len(set(area_rank.tolist())) == world
    engines = [CudaEngine(net, ms, part, bord, maps, cfg, r, world, area_rank, 0) for r in range(world)]
    try:
        flat = G.StateVector.flat_start(net)
        for e in engines:
            e.load_state(flat.va, flat.vm)
        off = engines[0].offsets
        iterations = 0
        for it in range(1, cfg.max_outer_iterations + 1):
            for e in engines:
                e.phase_local()
                e.sync()
            for r in range(1, world):                       # the variable-size gather to the coordinator
                mine = np.flatnonzero(area_rank == r)
                lo, hi = int(off[mine[0]]), int(off[mine[-1] + 1])
                engines[0].exchange[lo:hi].copy_(engines[r].exchange[lo:hi])
            torch.cuda.synchronize()
            engines[0].phase_boundary()
            engines[0].sync()
            for r in range(1, world):                       # the broadcast of delta_x_Gamma
                engines[r].delta.copy_(engines[0].delta)
            torch.cuda.synchronize()
            delta = max(e.phase_recover() for e in engines)
            iterations = it
            if delta < cfg.convergence_tol:
                break
        assert iterations == rref.iterations
        state = engines[0].state.clone()
        for r in range(1, world):                           # interiors of the other ranks' areas
            m = engines[r].owned_mask
            state[:, m] = engines[r].state[:, m]
        out = state.cpu().numpy()
        assert np.array_equal(out[0], ref.va) and np.array_equal(out[1], ref.vm)
    finally:
        for e in engines:
            e.close()


@pytest.mark.parametrize("name,world", [("ieee118_k6", 2), ("pegase2869_k8", 3)])
def test_rank_sharded_plans_enqueue_only_pipeline_matches_single_plan_bitwise(G, name, world):
    """The pipelined multi-rank iteration (gse_phase_*_async on one shared stream): no host
    synchronisation between the phases and the exchanges, one status read per iteration.  Device
    copies on that stream stand in for the NCCL send/recv, broadcast and MAX all-reduce."""
    import torch
    from conftest import build_case
    from paper_2604_23175_b200.distributed import CudaEngine, area_work_estimate, assign_areas
    net, ms, part, g = build_case(name)
    bord, maps = G.build_variable_maps(net, part)
    cfg = G.SolverConfig()
    ref, rref = G.solve_multiarea(net, ms, part, maps=(bord, maps), config=cfg)
    area_rank = assign_areas(area_work_estimate(maps), world)
    stream = torch.cuda.Stream(torch.device("cuda", 0))
    engines = [CudaEngine(net, ms, part, bord, maps, cfg, r, world, area_rank, 0, stream=stream) for r in range(world)]
    try:
        flat = G.StateVector.flat_start(net)
        for e in engines:
            e.load_state(flat.va, flat.vm)
        off = engines[0].offsets
        iterations, deltas = 0, []
        with torch.cuda.stream(stream):
            for it in range(1, cfg.max_outer_iterations + 1):
                for e in engines:
                    e.phase_local_async()
                for r in range(1, world):
                    mine = np.flatnonzero(area_rank == r)
                    lo, hi = int(off[mine[0]]), int(off[mine[-1] + 1])
                    engines[0].exchange[lo:hi].copy_(engines[r].exchange[lo:hi], non_blocking=True)
                engines[0].phase_boundary_async()
                for r in range(1, world):
                    engines[r].delta.copy_(engines[0].delta, non_blocking=True)
                for e in engines:
                    e.phase_recover_async()
                status = torch.stack([e.status for e in engines]).amax(dim=0)      # the MAX all-reduce
                delta, failed = (float(v) for v in status.cpu())                    # the one host wait
                assert failed == 0.0
                iterations = it
                deltas.append(delta)
                if delta < cfg.convergence_tol:
                    break
        assert iterations == rref.iterations
        state = engines[0].state.clone()
        for r in range(1, world):
            m = engines[r].owned_mask
            state[:, m] = engines[r].state[:, m]
        out = state.cpu().numpy()
        assert np.array_equal(out[0], ref.va) and np.array_equal(out[1], ref.vm)
    finally:
        for e in engines:
            e.close()


def test_distributed_estimator_reports_unobservable_area_through_status(G):
    """Enqueue-only phases cannot raise: the failure flag rides in status[1] and the owning rank's
    gse_check names the area (reference solver.py:250-251)."""
    from conftest import build_case
    from paper_2604_23175_b200.distributed import DistributedEstimator
    net, ms, part, g = build_case("ieee14_k2")
    vm_only = G.apply_mask(ms, lambda t, tg: t != G.MeasurementType.VM)   # reference test_solver.py:335-342
    est = DistributedEstimator(net, vm_only, part)
    try:
        with pytest.raises(G.SolverError, match="likely locally unobservable"):
            est.estimate()
    finally:
        est.close()


def test_distributed_estimator_single_rank_on_device(G):
    """DistributedEstimator with its product engine (CudaEngine) on one rank == MultiAreaEstimator."""
    from conftest import build_case
    from paper_2604_23175_b200.distributed import DistributedEstimator
    net, ms, part, g = build_case("ieee118_k6")
    est = DistributedEstimator(net, ms, part)
    try:
        st, rep = est.estimate()
    finally:
        est.close()
    ref, rref = G.solve_multiarea(net, ms, part)
    assert rep.iterations == rref.iterations and rep.converged
    assert np.array_equal(st.va, ref.va) and np.array_equal(st.vm, ref.vm) and rep.objective == rref.objective


def _run_tool(script, *args, timeout=300):
    """A tool script in a process of its own: kernels that wait for one another stay isolated from this session's
    CUDA context (a watchdog abort is sticky for the process it happens in)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    return subprocess.run([sys.executable, os.path.join(root, "tools", script), *[str(a) for a in args]],
                          capture_output=True, text=True, timeout=timeout)


@pytest.mark.parametrize("name,world", [("ieee118_k6", 2), ("pegase2869_k8", 3), ("pegase9241_k16", 4)])
def test_peer_linked_rank_plans_match_single_plan_bitwise(name, world):
    """The exchanges INSIDE the persistent kernels (gse_peer_link): every rank plan runs the whole GN loop in one
    launch; area roots store (S_b | b_hat) into the coordinator's buffer, the coordinator's back-substitution
    tasks store delta_x_Gamma into every rank's solution vector, the norm is max-merged with atomics.  Same
    iteration count, per-iteration norms, state bits and J as the single-plan solve, twice in a row
    (tools/linked_check.py: ``world`` rank plans side by side on the one GPU)."""
    out = _run_tool("linked_check.py", name, world)
    assert out.returncode == 0 and "linked ok" in out.stdout, out.stdout[-2000:] + out.stderr[-2000:]


def test_peer_linked_solve_reports_unobservable_area_on_every_rank():
    """A factorisation that fails on one rank stops ALL ranks at the end of that iteration with the same error
    (the failure code is max-merged into every rank's copy; reference solver.py:250-251)."""
    out = _run_tool("linked_check.py", "--unobservable")
    assert out.returncode == 0 and "linked ok" in out.stdout, out.stdout[-2000:] + out.stderr[-2000:]


def test_peer_linked_ranks_in_separate_processes_over_cuda_ipc():
    """The multi-process form of the in-kernel exchange: two rank PROCESSES (gloo for the host plumbing) map each
    other's buffers with CUDA IPC handles and solve with one persistent launch each -- here time-sharing the one
    GPU, on a node one process per GPU.  tools/ipc_two_process.py asserts bit-equality with the single-plan solve,
    twice in a row, through DistributedEstimator(exchange="peer")."""
    out = _run_tool("ipc_two_process.py", "ieee118_k6", 2, timeout=240)
    assert out.returncode == 0 and "ipc ok" in out.stdout, out.stdout[-2000:] + out.stderr[-2000:]
