"""Peer-linked rank plans side by side on the one GPU, checked against the single-plan solve (run by
tests/test_gpu_scale.py in a process of its own: the rank kernels wait for one another, and a watchdog abort --
should they ever not be resident together -- must not take the CUDA context of the test session with it).
    python tools/linked_check.py <case> <world>            bit-equality with the single plan, twice in a row
    python tools/linked_check.py --unobservable            failure reported on every rank"""
import os
import sys
import threading

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2604_23175_b200 as G
from paper_2604_23175_b200.distributed import CudaEngine, area_work_estimate, assign_areas
from conftest import build_case


def linked_engines(net, ms, part, bord, maps, cfg, world, max_ctas):
    """``world`` rank plans of one problem on the one GPU, peer-linked through their device addresses (the same
    records a multi-process run exchanges through torch.distributed and maps with CUDA IPC)."""
    area_rank = assign_areas(area_work_estimate(maps), world)
    assert len(set(area_rank.tolist())) == world
    engines = [CudaEngine(net, ms, part, bord, maps, cfg, r, world, area_rank, 0, max_ctas=max_ctas) for r in range(world)]
    infos = [e.peer_info() for e in engines]
    for e in engines:
        e.peer_link(infos)
    return engines


def run_linked(engines, cfg, flat):
    """One peer-linked solve: every rank's kernel is launched from its own host thread (the kernels of all ranks
    must be resident together: they wait for each other's area roots, delta_x_Gamma pieces and norms)."""
    for e in engines:
        e.load_state(flat.va, flat.vm)
        e.solve_prepare()
    out = [None] * len(engines)

    def work(k):
        try:
            out[k] = engines[k].solve_linked(cfg)
        except Exception as exc:           # noqa: BLE001 -- handed to the asserting thread
            out[k] = exc
    threads = [threading.Thread(target=work, args=(k,)) for k in range(len(engines))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    return out


def check_case(name, world):
    net, ms, part, g = build_case(name)
    bord, maps = G.build_variable_maps(net, part)
    cfg = G.SolverConfig()
    single = G.MultiAreaEstimator(net, ms, part, maps=(bord, maps), config=cfg)
    ref, rref = single.estimate()
    ref_deltas = list(single.last_deltas)
    single.close()
    engines = linked_engines(net, ms, part, bord, maps, cfg, world, max_ctas=64)
    flat = G.StateVector.flat_start(net)
    for _ in range(2):                                             # (the counters are re-armed per solve)
        reps = run_linked(engines, cfg, flat)
        for r in reps:
            assert not isinstance(r, Exception), r
            assert r.iterations == rref.iterations == int(g["iterations"]) and r.converged
            assert [float(r.delta_inf[k]) for k in range(r.iterations)] == ref_deltas
        state = engines[0].state.clone()
        for r in range(1, world):
            m = engines[r].owned_mask
            state[:, m] = engines[r].state[:, m]
        out = state.cpu().numpy()
        assert np.array_equal(out[0], ref.va) and np.array_equal(out[1], ref.vm), "state differs from the single-plan solve"
        assert engines[0].plan.objective(state[0].data_ptr(), state[1].data_ptr()) == rref.objective
    for e in engines:
        e.close()
    print(f"linked ok: {name} world={world} iterations={rref.iterations} J={rref.objective!r}", flush=True)


def check_unobservable():
    net, ms, part, g = build_case("ieee14_k2")
    vm_only = G.apply_mask(ms, lambda t, tg: t != G.MeasurementType.VM)       # reference test_solver.py:335-342
    bord, maps = G.build_variable_maps(net, part)
    cfg = G.SolverConfig()
    engines = linked_engines(net, vm_only, part, bord, maps, cfg, 2, max_ctas=32)
    reps = run_linked(engines, cfg, G.StateVector.flat_start(net))
    for r in reps:
        assert isinstance(r, G.SolverError) and "likely locally unobservable" in str(r), r
    for e in engines:
        e.close()
    print("linked ok: unobservable area reported on every rank", flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "--unobservable":
        check_unobservable()
    else:
        check_case(sys.argv[1], int(sys.argv[2]))
