"""The multi-rank driver (paper_2604_23175_b200/distributed.py) under ``gloo`` on CPU.

World size 2 and 3, an oracle-backed phase engine injected in place of the CUDA engine (the
driver is engine-agnostic; tests may use the oracle, the product never does).  Checks the
area assignment, the variable-size gather of condensed blocks, the broadcast of the boundary
increment, the MAX all-reduce of the convergence scalar and the state merge -- and that the
result is bit-identical to the single-process oracle solve regardless of the sharding
(blocks are summed on the coordinator in area order).
"""

import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


class OracleEngine:
    """Phase engine over the CPU oracle with the CudaEngine interface."""

    def __init__(self, net, ms, part, bord, maps, cfg, rank, world, area_rank, device):
        import torch
        from oracle.mase_oracle import Oracle
        self.orc = Oracle(net, ms, part.area_of_bus)
        self.rank, self.maps = rank, maps
        self.mine = (np.asarray(area_rank) == rank).astype(np.int32)
        sizes = [m.n_boundary * m.n_boundary + m.n_boundary for m in maps]
        self.offsets = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        self.exchange = torch.zeros(int(self.offsets[-1]), dtype=torch.float64)
        self.delta = torch.zeros(bord.n_gamma, dtype=torch.float64)
        self.state = torch.zeros((2, net.n_bus), dtype=torch.float64)
        owned = np.zeros(net.n_bus, dtype=bool)
        for a, m in enumerate(maps):
            if self.mine[a]:
                owned[m.internal_buses] = True
        self.owned_mask = torch.from_numpy(owned)
        self.n_gamma = bord.n_gamma

    def load_state(self, va, vm):
        self.state[0] = self.state.new_tensor(va)
        self.state[1] = self.state.new_tensor(vm)

    def phase_local(self):
        st = self.state.numpy()
        self.orc.local_masked(st[0].copy(), st[1].copy(), self.mine)
        buf = self.exchange.numpy()
        for a, m in enumerate(self.maps):
            if self.mine[a]:
                s_b, b_hat = self.orc.schur(a)
                lo = int(self.offsets[a])
                nb = m.n_boundary
                buf[lo:lo + nb * nb] = s_b.ravel()
                buf[lo + nb * nb:lo + nb * nb + nb] = b_hat

    def phase_boundary(self):
        buf = self.exchange.numpy()
        for a, m in enumerate(self.maps):
            lo, nb = int(self.offsets[a]), m.n_boundary
            self.orc.set_schur(a, buf[lo:lo + nb * nb].reshape(nb, nb), buf[lo + nb * nb:lo + nb * nb + nb])
        self.orc.boundary()
        self.delta.copy_(self.delta.new_tensor(self.orc.boundary_system()[2]))

    def phase_recover(self):
        self.orc.set_dx_gamma(self.delta.numpy())
        st = self.state.numpy()
        va, vm = st[0].copy(), st[1].copy()
        d = self.orc.recover_masked(va, vm, self.mine)
        self.state[0] = self.state.new_tensor(va)
        self.state[1] = self.state.new_tensor(vm)
        return d

    def inner_step(self):
        st = self.state.numpy()
        va, vm = st[0].copy(), st[1].copy()
        d = self.orc.inner_step_masked(va, vm, self.mine)
        self.state[0] = self.state.new_tensor(va)
        self.state[1] = self.state.new_tensor(vm)
        return d

    def sync(self):
        pass

    def objective(self):
        st = self.state.numpy()
        return self.orc.objective(st[0].copy(), st[1].copy())

    def close(self):
        pass


class AsyncOracleEngine(OracleEngine):
    """The same engine behind the enqueue-only phase interface (CudaEngine.async_phases): exercises the
    pipelined driver path -- failures and the norm travel in ``status`` through one MAX all-reduce."""

    async_phases = True

    def __init__(self, *a, **k):
        import torch
        super().__init__(*a, **k)
        self.status = torch.zeros(2, dtype=torch.float64)
        self.failed = None

    def phase_local_async(self):
        try:
            self.phase_local()
        except Exception as exc:              # a device plan records the failure and keeps going
            self.failed = exc

    def phase_boundary_async(self):
        try:
            self.phase_boundary()
        except Exception as exc:
            self.failed = exc

    def phase_recover_async(self):
        d = 0.0
        if self.failed is None:
            try:
                d = self.phase_recover()
            except Exception as exc:
                self.failed = exc
        self.status[0], self.status[1] = d, 1.0 if self.failed is not None else 0.0

    def check(self):
        if self.failed is not None:
            raise self.failed

    def launches_last(self):
        return 0


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, name, out_dir, async_phases=False, inner=1):
    import torch.distributed as dist
    from conftest import build_case
    from paper_2604_23175_b200.distributed import DistributedEstimator
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        net, ms, part, g = build_case(name)
        from paper_2604_23175_b200 import SolverConfig
        est = DistributedEstimator(net, ms, part, config=SolverConfig(inner_gn_steps=inner),
                                   engine_factory=AsyncOracleEngine if async_phases else OracleEngine)
        trace = []
        state, rep = est.estimate(on_iteration=lambda it, s, d: trace.append(d))
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), va=state.va, vm=state.vm,
                 iterations=rep.iterations, converged=rep.converged, objective=rep.objective,
                 deltas=np.array(trace), area_rank=est.area_rank)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,world,async_phases", [("ieee118_k6", 2, False), ("rand120_k4", 3, False), ("ieee14_k2", 2, False),
                                                     ("ieee118_k6", 2, True), ("rand120_k4", 3, True)])
def test_sharded_solve_is_bit_identical_to_single_process(tmp_path, name, world, async_phases):
    import torch.multiprocessing as mp
    from conftest import build_case
    from oracle.mase_oracle import Oracle
    port = _free_port()
    mp.spawn(_worker, args=(world, port, name, str(tmp_path), async_phases), nprocs=world, join=True)
    net, ms, part, g = build_case(name)
    ref = Oracle(net, ms, part.area_of_bus).solve()
    outs = [np.load(os.path.join(tmp_path, f"rank{r}.npz")) for r in range(world)]
    for r, o in enumerate(outs):
        assert int(o["iterations"]) == ref["iterations"] == int(g["iterations"])
        assert bool(o["converged"]) == ref["converged"]
        # every rank returns the merged state; sharding does not change a single bit
        assert np.array_equal(o["va"], ref["va"]), r
        assert np.array_equal(o["vm"], ref["vm"]), r
        assert float(o["objective"]) == ref["objective"]
        assert np.array_equal(o["deltas"], ref["deltas"])
    ar = outs[0]["area_rank"]
    assert len(np.unique(ar)) == min(world, part.k) and np.all(np.diff(ar) >= 0)   # contiguous, all ranks busy


@pytest.mark.parametrize("name,world,inner,async_phases", [("ieee118_k6_inner2", 2, 2, False), ("rand120_k4_inner3", 3, 3, True)])
def test_sharded_inner_gn_steps_match_single_process_and_reference(tmp_path, name, world, inner, async_phases):
    """SolverConfig.inner_gn_steps > 1 across ranks (reference solver.py:253-260): every rank runs the
    interior-only steps of its own areas, their norm joins the stacked norm of the iteration -- same
    iterates / iteration count as one process and as the reference's stored run."""
    import torch.multiprocessing as mp
    from conftest import build_case
    from oracle.mase_oracle import Oracle
    port = _free_port()
    mp.spawn(_worker, args=(world, port, name, str(tmp_path), async_phases, inner), nprocs=world, join=True)
    net, ms, part, g = build_case(name)
    ref = Oracle(net, ms, part.area_of_bus).solve(inner=inner)
    for r in range(world):
        o = np.load(os.path.join(tmp_path, f"rank{r}.npz"))
        assert int(o["iterations"]) == ref["iterations"] == int(g["iterations"])
        assert np.array_equal(o["va"], ref["va"]) and np.array_equal(o["vm"], ref["vm"]), r
        assert np.array_equal(o["deltas"], ref["deltas"])
        assert np.allclose(o["deltas"], g["deltas"], rtol=1e-6, atol=1e-12)
        assert np.max(np.abs(o["va"] - g["va"])) < 1e-9 and np.max(np.abs(o["vm"] - g["vm"])) < 1e-9


def test_assign_areas_properties():
    from paper_2604_23175_b200.distributed import assign_areas
    rng = np.random.default_rng(0)
    for k in (1, 2, 5, 16, 33, 128):
        work = rng.uniform(1.0, 10.0, k)
        for world in (1, 2, 4, 8):
            ar = assign_areas(work, world)
            assert ar.shape == (k,) and np.all(np.diff(ar) >= 0) and ar[0] == 0
            assert len(np.unique(ar)) == min(world, k)
            loads = np.bincount(ar, weights=work, minlength=min(world, k))
            assert loads.max() <= 2.5 * work.sum() / min(world, k) + work.max()
