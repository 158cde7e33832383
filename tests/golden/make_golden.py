"""Generate the golden fixtures in this directory from the UNMODIFIED reference.

Run once in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports ``gridse`` from /root/reference/pkg/src and the reference's own
synthetic-grid generator from /root/reference/pkg/tests/conftest.py, runs
``solve_multiarea`` / ``fused_accumulate`` / ``schur_condense`` /
``assemble_boundary`` on the BASELINE.json configurations (and a few edge
cases), and stores inputs + outputs as ``.npz``.  Nothing at test time reads
/root/reference: the tests load these files only.

``tiled101k`` runs the reference once on the ~100k-bus / 128-area configuration (BASELINE.json configs[4];
minutes of CPU) and stores the end state, J and the per-iteration norms.

Also writes the reference partitioner's ``area_of_bus`` for the three named
shapes to ``paper_2604_23175_b200/cases/part_<shape>.json`` (the reference
partitioner takes 23 s / 141 s / 79 s there).
"""

import json
import os
import sys
import time

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")

import numpy as np  # noqa: E402
import gridse as R  # noqa: E402
from conftest import make_path4, random_network  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = os.path.join(HERE, "..", "..", "paper_2604_23175_b200", "cases")
SHAPES = {"pegase2869": (2869, 4582, 8), "pegase9241": (9241, 16049, 16),
          "activsg10k": (10000, 12706, 32)}


def solve_and_record(name, net, ms, part, detail, cfg=None, recipe=None):
    cfg = cfg or R.SolverConfig()
    bord, maps = R.build_variable_maps(net, part)
    out = {
        "recipe": json.dumps(recipe or {}),
        "area_of_bus": part.area_of_bus.astype(np.int32),
        "n_gamma": bord.n_gamma,
        "z_sum": np.array([ms.z.sum(), np.abs(ms.z).sum(), ms.weight.sum()]),
    }
    if detail:
        out.update(z=ms.z, weight=ms.weight, mtype=ms.mtype.astype(np.int32),
                   target=ms.target.astype(np.int32))
    # flat-start blocks, Schur blocks and the boundary system (first iteration)
    st = R.StateVector.flat_start(net)
    xg = bord.gather(st.va, st.vm)
    schurs = []
    for a, m in enumerate(maps):
        blk = R.fused_accumulate(m, ms, m.gather_interior(st.va, st.vm), xg[m.boundary_selector])
        cache = R.symbolic_analyze(blk.g_ii)
        R.numeric_refactor(cache, blk.g_ii.data)
        sch = R.schur_condense(cache, blk.g_ib, blk.g_bb, blk.b_i, blk.b_b)
        schurs.append(sch)
        out[f"a{a}_dims"] = np.array([m.n_interior, m.n_boundary, blk.g_ii.nnz, blk.g_ib.nnz])
        out[f"a{a}_sel"] = m.boundary_selector.astype(np.int32)
        if detail:
            out[f"a{a}_ii_ptr"] = blk.g_ii.indptr.astype(np.int32)
            out[f"a{a}_ii_idx"] = blk.g_ii.indices.astype(np.int32)
            out[f"a{a}_ib_ptr"] = blk.g_ib.indptr.astype(np.int32)
            out[f"a{a}_ib_idx"] = blk.g_ib.indices.astype(np.int32)
            out[f"a{a}_data_ii"] = blk.g_ii.data
            out[f"a{a}_data_ib"] = blk.g_ib.data
            out[f"a{a}_g_bb"] = blk.g_bb
            out[f"a{a}_s_b"] = sch.s_b
        else:  # fingerprints only (sums are order-sensitive at 1e-16, compared at 1e-12)
            out[f"a{a}_sum_ii"] = np.array([blk.g_ii.data.sum(), np.abs(blk.g_ii.data).sum()])
            out[f"a{a}_sb_diag"] = np.diag(sch.s_b).copy()
        out[f"a{a}_b_i"] = blk.b_i
        out[f"a{a}_b_b"] = blk.b_b
        out[f"a{a}_b_hat"] = sch.b_hat
    if bord.n_gamma:
        bs = R.assemble_boundary(schurs, [m.boundary_selector for m in maps], bord.n_gamma)
        dxg = R.dense_cholesky_solve(bs.s_gamma, bs.b_gamma)
        if detail:
            out["s_gamma"] = bs.s_gamma
        out["s_gamma_diag"] = np.diag(bs.s_gamma).copy()
        out["b_gamma"] = bs.b_gamma
        out["dx_gamma"] = dxg
    # the solve itself
    trace = []
    t0 = time.perf_counter()
    est, rep = R.solve_multiarea(net, ms, part, maps=(bord, maps), config=cfg,
                                 on_iteration=lambda it, s, d: trace.append((s, d)))
    wall = time.perf_counter() - t0
    out.update(iterations=rep.iterations, converged=rep.converged, objective=rep.objective,
               deltas=np.array([d for _, d in trace]), va=est.va, vm=est.vm,
               ref_wall_s=wall, ref_timings=json.dumps(rep.timings))
    if detail:
        out["trace_va"] = np.array([s.va for s, _ in trace])
        out["trace_vm"] = np.array([s.vm for s, _ in trace])
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    print(f"{name}: iters {rep.iterations} conv {rep.converged} J {rep.objective!r} "
          f"n_gamma {bord.n_gamma} wall {wall:.2f}s", flush=True)


def main(which):
    if "small" in which:
        net = R.load_case("/root/reference/pkg/cases/ieee14.m")
        ms = R.generate_measurements(net, R.MeasurementConfig(seed=0))
        for k in (1, 2, 3, 14):
            solve_and_record(f"ieee14_k{k}", net, ms, R.partition_network(net, k, seed=0), True,
                             recipe={"case": "ieee14.m", "meas_seed": 0, "k": k, "part_seed": 0})
        net = R.load_case("/root/reference/pkg/cases/ieee118.m")
        ms = R.generate_measurements(net, R.MeasurementConfig(seed=0))
        for k in (3, 6):
            solve_and_record(f"ieee118_k{k}", net, ms, R.partition_network(net, k, seed=0), True,
                             recipe={"case": "ieee118.m", "meas_seed": 0, "k": k, "part_seed": 0})
        # slack on the boundary, noiseless (reference test_solver.py:95-102)
        net = make_path4(slack_pos=1)
        ms = R.generate_measurements(net, R.MeasurementConfig(sigma_vm=0.0, sigma_power=0.0))
        solve_and_record("path4_slack_boundary", net, ms, R.load_partition(net, [0, 0, 1, 1]), True,
                         cfg=R.SolverConfig(convergence_tol=1e-10),
                         recipe={"gen": "make_path4(slack_pos=1)", "sigma": 0.0,
                                 "area_of_bus": [0, 0, 1, 1], "tol": 1e-10})
        # random grids, one with a masked family (reference test_assembly.py:200-216)
        net = random_network(300, 11)
        ms = R.generate_measurements(net, R.MeasurementConfig(seed=4))
        solve_and_record("rand300_k3_maskpf", net, R.apply_mask(ms, R.MeasurementType.PF),
                         R.partition_network(net, 3, seed=0), True,
                         recipe={"gen": "random_network(300, 11)", "meas_seed": 4, "k": 3,
                                 "mask": "PF"})
        net = random_network(120, 3, 0.3)
        ms = R.generate_measurements(net, R.MeasurementConfig(seed=2))
        solve_and_record("rand120_k4", net, ms, R.partition_network(net, 4, seed=1), True,
                         recipe={"gen": "random_network(120, 3, 0.3)", "meas_seed": 2, "k": 4,
                                 "part_seed": 1})
    if "inner" in which:
        # inner_gn_steps > 1 (reference solver.py:253-260): extra interior-only GN steps per outer round
        net = R.load_case("/root/reference/pkg/cases/ieee118.m")
        ms = R.generate_measurements(net, R.MeasurementConfig(seed=0))
        solve_and_record("ieee118_k6_inner2", net, ms, R.partition_network(net, 6, seed=0), True,
                         cfg=R.SolverConfig(inner_gn_steps=2),
                         recipe={"case": "ieee118.m", "meas_seed": 0, "k": 6, "part_seed": 0, "inner": 2})
        net = random_network(120, 3, 0.3)
        ms = R.generate_measurements(net, R.MeasurementConfig(seed=2))
        solve_and_record("rand120_k4_inner3", net, ms, R.partition_network(net, 4, seed=1), True,
                         cfg=R.SolverConfig(inner_gn_steps=3),
                         recipe={"gen": "random_network(120, 3, 0.3)", "meas_seed": 2, "k": 4,
                                 "part_seed": 1, "inner": 3})
    if "refined" in which:
        # solve_centralized with iterative_refinement=True (reference solver.py:181-183, linalg.py:385-392)
        for case, tag in (("ieee14.m", "ieee14"), ("ieee118.m", "ieee118")):
            net = R.load_case(f"/root/reference/pkg/cases/{case}")
            ms = R.generate_measurements(net, R.MeasurementConfig(seed=0))
            trace = []
            est, rep = R.solve_centralized(net, ms, config=R.SolverConfig(iterative_refinement=True),
                                           on_iteration=lambda it, s, d: trace.append((s, d)))
            np.savez_compressed(
                os.path.join(HERE, f"{tag}_centralized_refined.npz"),
                recipe=json.dumps({"case": case, "meas_seed": 0, "refined": True}),
                area_of_bus=np.zeros(net.n_bus, dtype=np.int32), n_gamma=0,
                iterations=rep.iterations, converged=rep.converged, objective=rep.objective,
                deltas=np.array([d for _, d in trace]), va=est.va, vm=est.vm,
                trace_va=np.array([s.va for s, _ in trace]), trace_vm=np.array([s.vm for s, _ in trace]))
            print(f"{tag}_centralized_refined: iters {rep.iterations} J {rep.objective!r}", flush=True)
    for shape in ("pegase2869", "pegase9241", "activsg10k"):
        if shape not in which:
            continue
        n, nbr, k = SHAPES[shape]
        net = random_network(n, seed=n, extra_frac=(nbr - (n - 1)) / n)
        path = os.path.join(CASES, f"part_{shape}.json")
        if os.path.exists(path):
            part = R.load_partition(net, json.load(open(path))["area_of_bus"])
        else:
            part = R.partition_network(net, k, seed=0)
            with open(path, "w") as fh:
                json.dump({"k": k, "area_of_bus": [int(a) for a in part.area_of_bus]}, fh)
        ms = R.generate_measurements(net, R.MeasurementConfig(seed=0))
        solve_and_record(f"{shape}_k{k}", net, ms, part, detail=(shape == "pegase2869"),
                         recipe={"gen": f"random_network({n}, seed={n}, extra_frac=({nbr}-{n - 1})/{n})",
                                 "meas_seed": 0, "k": k, "part_seed": 0})


def tiled_reference_network(base, copies, ties_per_seam=3):
    """The ~100k-bus grid of BASELINE.json configs[4] built from the REFERENCE's own classes: ``copies``
    relabelled copies of ``base`` chained by tie branches (same construction as the product's
    ``synth.tiled_network``; tests/test_host_api.py pins the two to the same Ybus fingerprint)."""
    n = base.n_bus
    buses, branches = [], []
    for c in range(copies):
        for i, b in enumerate(base.buses):
            buses.append(R.Bus(id=c * n + i + 1, base_kv=b.base_kv, gs=b.gs, bs=b.bs,
                               is_slack=(b.is_slack and c == 0), vm_true=b.vm_true, va_true=b.va_true))
        for br in base.branches:
            branches.append(R.Branch(from_bus=c * n + br.from_bus, to_bus=c * n + br.to_bus, r=br.r, x=br.x,
                                     b_charging=br.b_charging, tap=br.tap, shift=br.shift))
        if c:
            for j in range(ties_per_seam):
                branches.append(R.Branch(from_bus=c * n - 1 - 2 * j, to_bus=c * n + 2 * j,
                                         r=0.01 + 0.002 * j, x=0.08 + 0.01 * j, b_charging=0.02))
    return R.BusBranchNetwork.from_components(buses, branches)


def tiled101k():
    """BASELINE.json configs[4]: 11 tiles of the PEGASE-9241 shape (101,651 buses, 1,011,229 rows) in the
    128 areas of cases/part_tiled101k_k128.json, solved ONCE by the unmodified reference
    (solve_multiarea, LAPACK boundary Cholesky of the n_Gamma = 5692 system).  Stores the end state, J,
    the per-iteration norms and first-iteration fingerprints; no per-area detail (the file stays small)."""
    n, nbr, _ = SHAPES["pegase9241"]
    base = random_network(n, seed=n, extra_frac=(nbr - (n - 1)) / n)
    net = tiled_reference_network(base, 11)
    part = R.load_partition(net, json.load(open(os.path.join(CASES, "part_tiled101k_k128.json")))["area_of_bus"])
    ms = R.generate_measurements(net, R.MeasurementConfig(seed=0))
    bord, maps = R.build_variable_maps(net, part)
    trace = []
    t0 = time.perf_counter()
    est, rep = R.solve_multiarea(net, ms, part, maps=(bord, maps),
                                 on_iteration=lambda it, s, d: (trace.append(d), print("  it", it, d, flush=True)))
    wall = time.perf_counter() - t0
    y = net.ybus
    np.savez_compressed(
        os.path.join(HERE, "tiled101k_k128.npz"),
        recipe=json.dumps({"gen": "tiled_network(shaped_network('pegase9241'), 11)", "meas_seed": 0,
                           "partition": "cases/part_tiled101k_k128.json"}),
        area_of_bus=part.area_of_bus.astype(np.int32), n_gamma=bord.n_gamma,
        z_sum=np.array([ms.z.sum(), np.abs(ms.z).sum(), ms.weight.sum()]),
        ybus_sum=np.array([y.data.real.sum(), y.data.imag.sum(), np.abs(y.data).sum(), y.nnz]),
        iterations=rep.iterations, converged=rep.converged, objective=rep.objective,
        deltas=np.array(trace), va=est.va, vm=est.vm, ref_wall_s=wall, ref_timings=json.dumps(rep.timings))
    print(f"tiled101k_k128: iters {rep.iterations} conv {rep.converged} J {rep.objective!r} "
          f"n_gamma {bord.n_gamma} wall {wall:.1f}s", flush=True)


if __name__ == "__main__":
    which = sys.argv[1:] or ["small", "inner", "refined", "pegase2869", "pegase9241", "activsg10k", "tiled101k"]
    main(which)
    if "tiled101k" in which:
        tiled101k()
