"""The C-ABI library loads and exports every symbol include/gridse_b200.h declares (no compute
without a GPU), the product refuses to run without a device, and the plan-time analysis
(csrc/symbolic.cpp) is validated on the CPU through the test-only host interpreter."""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_2604_23175_b200 as G
from paper_2604_23175_b200 import _native, build as native_build
from conftest import SMALL_CASES, build_case, ROOT


def test_library_builds_and_exports_every_declared_symbol():
    path = native_build.build()
    lib = ctypes.CDLL(path)
    header = open(os.path.join(ROOT, "include", "gridse_b200.h")).read()
    declared = set(re.findall(r"\b(gse_[a-z_]+)\s*\(", header))
    assert declared, "no declarations found"
    for sym in sorted(declared):
        assert hasattr(lib, sym), f"{sym} declared in gridse_b200.h but not exported"
    assert set(_native.EXPORTED) <= declared
    lib.gse_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.gse_version()


def test_no_cpu_fallback_without_a_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    net, ms, part, _ = build_case("ieee14_k2")
    with pytest.raises(_native.NativeError) as exc:
        G.solve_multiarea(net, ms, part)
    assert exc.value.code == _native.GSE_E_NO_DEVICE
    bord, maps = G.build_variable_maps(net, part)
    with pytest.raises(_native.NativeError):
        _native.Plan(net, ms, part, bord, maps)


def test_config_validation_matches_reference():
    with pytest.raises(ValueError):
        G.SolverConfig(max_outer_iterations=0)
    with pytest.raises(ValueError):
        G.SolverConfig(convergence_tol=0.0)
    with pytest.raises(ValueError):
        G.SolverConfig(backend="magic")
    assert G.SolverConfig(backend="dense").effective_dense_threshold == 10 ** 9


@pytest.mark.parametrize("name", SMALL_CASES)
@pytest.mark.parametrize("opts", [{}, {"dense": True}, {"leaf": 4, "pmax": 32}])
def test_device_program_on_host_interpreter(name, opts):
    from hostsim import HostSim
    net, ms, part, g = build_case(name)
    bord, maps = G.build_variable_maps(net, part)
    sim = HostSim(net, ms, part, bord, maps, **opts)
    tol = 1e-10 if name == "path4_slack_boundary" else 1e-6
    va, vm, it, conv, deltas = sim.solve(tol=tol)
    assert it == int(g["iterations"]) and conv == bool(g["converged"])
    assert max(np.max(np.abs(va - g["va"])), np.max(np.abs(vm - g["vm"]))) < 1e-9
    # Schur blocks of the last iteration are symmetric-by-construction and finite
    for a in range(part.k):
        s_b, b_hat = sim.area_schur(a)
        assert np.all(np.isfinite(s_b)) and np.array_equal(s_b, s_b.T)


def test_device_program_big_shape_and_sharded_plans():
    from hostsim import HostSim
    net, ms, part, g = build_case("pegase2869_k8")
    bord, maps = G.build_variable_maps(net, part)
    va, vm, it, conv, _ = HostSim(net, ms, part, bord, maps).solve()
    assert it == int(g["iterations"]) and np.max(np.abs(vm - g["vm"])) < 1e-9
    # a rank that owns a subset of the areas still analyses consistently
    area_rank = np.array([0, 0, 0, 1, 1, 1, 1, 1], dtype=np.int32)
    for rank in (0, 1):
        st = HostSim(net, ms, part, bord, maps, rank=rank, world=2, area_rank=area_rank).stats()
        assert st["fronts"] > 0 and st["tasks"] > 0


def test_reference_layout_program_reproduces_oracle_blocks():
    """The accumulation program in the reference's CSR layout (used by fused_accumulate)."""
    from hostsim import HostSim
    from oracle.mase_oracle import Oracle
    net, ms, part, g = build_case("rand120_k4")
    bord, maps = G.build_variable_maps(net, part)
    sim = HostSim(net, ms, part, bord, maps)
    va = np.zeros(net.n_bus)
    va[net.slack] = net.buses[net.slack].va_true
    vm = np.ones(net.n_bus)
    sim.iterate(va.copy(), vm.copy())
    vals, off = sim.ref_blocks()
    orc = Oracle(net, ms, part.area_of_bus)
    orc.assemble(va, vm)
    for a in range(part.k):
        b = orc.blocks(a)
        flat = np.concatenate([b["data_ii"], b["data_ib"], b["g_bb"].ravel(), b["b_i"], b["b_b"]])
        mine = vals[off[a]:off[a + 1]]
        assert np.max(np.abs(mine - flat) / (1 + np.abs(flat))) < 5e-13


def test_plan_build_does_not_depend_on_the_host_thread_count(monkeypatch):
    """symbolic.cpp runs the per-area / per-segment parts of the analysis on a few host threads;
    the program (and hence every bit of the solve) must be the same for any thread count."""
    from hostsim import HostSim
    net, ms, part, g = build_case("pegase2869_k8")
    bord, maps = G.build_variable_maps(net, part)
    outs = []
    for threads in ("1", "3", "16"):
        monkeypatch.setenv("GSE_BUILD_THREADS", threads)
        sim = HostSim(net, ms, part, bord, maps)
        va, vm, it, conv, deltas = sim.solve()
        vals, off = sim.ref_blocks()
        outs.append((sim.stats(), va, vm, it, np.array(deltas), vals))
    for st, va, vm, it, deltas, vals in outs[1:]:
        assert st == outs[0][0] and it == outs[0][3]
        assert np.array_equal(va, outs[0][1]) and np.array_equal(vm, outs[0][2])
        assert np.array_equal(deltas, outs[0][4]) and np.array_equal(vals, outs[0][5])


@pytest.mark.parametrize("name", ["ieee118_k3", "rand300_k3_maskpf", "pegase2869_k8"])
def test_amalgamated_trees_solve_the_same_system(name, monkeypatch):
    """The plan-time tree shaping of round 2 -- relaxed amalgamation of the area interiors (the default of plans above
    30k buses), relaxed boundary amalgamation, fine leaves, 8-aligned supernode pieces -- only changes WHICH front
    eliminates a variable: the host interpreter of the device program must reach the reference's iteration count and
    state with every variant, and the merges must really reduce the number of fronts."""
    from hostsim import HostSim
    net, ms, part, g = build_case(name)
    bord, maps = G.build_variable_maps(net, part)
    base = HostSim(net, ms, part, bord, maps, leaf=8).stats()["fronts"]
    for env in ({"GSE_INTERIOR_MERGE": "1.0"}, {"GSE_INTERIOR_MERGE": "0.3", "GSE_GAMMA_MERGE": "1.0"},
                {"GSE_INTERIOR_MERGE": "1.0", "GSE_NO_GAMMA_MERGE": "1"}):
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        sim = HostSim(net, ms, part, bord, maps, leaf=8, pmax=32 if name == "ieee118_k3" else 0)
        tol = 1e-6
        va, vm, it, conv, deltas = sim.solve(tol=tol)
        assert it == int(g["iterations"]) and conv == bool(g["converged"]), env
        assert max(np.max(np.abs(va - g["va"])), np.max(np.abs(vm - g["vm"]))) < 1e-9, env
        if name != "ieee118_k3":
            assert sim.stats()["fronts"] < base, env
        for k in env:
            monkeypatch.delenv(k)
