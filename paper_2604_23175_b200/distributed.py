"""Area-sharded multi-GPU solve: one process per GPU, ``torch.distributed`` for the plumbing.

SURVEY.md section 8(e): areas are independent between the two coordinator exchanges
(reference ``solver.py:277-298,318-326``), so each rank owns a contiguous block of areas
(balanced by estimated factor work), condenses them locally and

  1. sends its packed ``(S_b | b_hat)`` blocks to the coordinator rank (variable-size
     gather = grouped send/recv; NCCL over NVLink on GPUs),
  2. the coordinator scatters them into ``S_Gamma`` **in area order** -- so the bits do not
     depend on the number of ranks -- and runs the dense boundary solve,
  3. ``delta_x_Gamma`` is broadcast back, every rank recovers its interiors and updates its
     replica of the boundary state,
  4. one MAX all-reduce carries the convergence scalar (and the failure flag).

On one node (up to 8 ranks) the same four steps run INSIDE each rank's persistent kernel over peer memory
(``exchange="peer"``, the default when the ranks can be linked): the area roots store ``(S_b | b_hat)``
straight into the coordinator's buffer, the coordinator's back-substitution tasks store their share of
``delta_x_Gamma`` into every rank's solution vector, and the norm is max-merged with one atomic per peer --
one kernel launch per rank and solve, no collective inside the loop (``gse_peer_link``).  The collective
driver below remains for ``on_iteration`` callbacks, inner GN steps, phase timing and larger worlds.

The driver is engine-agnostic: the product engine (``CudaEngine``) wraps the C-ABI plan;
the CPU tests inject an oracle-backed engine and run the same code under ``gloo``.
"""

from __future__ import annotations

import time

import numpy as np

from .measurement import StateVector
from .partition import build_variable_maps
from .solver import PHASES, SolveReport, SolverConfig, SolverError


def area_work_estimate(maps):
    """Relative factor + condensation work per area (interior^2 bandwidth-like + Schur)."""
    return np.array([m.n_interior * 40.0 + m.n_interior * m.n_boundary + m.n_boundary ** 2.0 + 1.0
                     for m in maps])


def assign_areas(work, world):
    """Contiguous blocks of areas per rank, greedy linear partition of ``work``.

    Returns ``area_rank`` (owner per area).  Every rank gets at least one area when
    ``len(work) >= world``; surplus ranks own nothing otherwise.
    """
    work = np.asarray(work, dtype=float)
    k = len(work)
    area_rank = np.zeros(k, dtype=np.int32)
    if world <= 1 or k == 0:
        return area_rank
    target = work.sum() / min(world, k)
    rank, acc = 0, 0.0
    for a in range(k):
        remaining_areas, remaining_ranks = k - a, min(world, k) - rank
        if rank < min(world, k) - 1 and acc > 0 and (
                acc + 0.5 * work[a] > target or remaining_areas <= remaining_ranks - 1):
            rank, acc = rank + 1, 0.0
        area_rank[a] = rank
        acc += work[a]
    return area_rank


class CudaEngine:
    """Phase engine over the C-ABI plan (``libgridse_b200.so``)."""

    # the plan enqueues on torch's current stream, so the NCCL collectives torch orders against that
    # stream need no host synchronisation between the phases (one per iteration: the status read)
    async_phases = True

    def __init__(self, net, ms, part, bord, maps, cfg, rank, world, area_rank, device, stream=None, max_ctas=0):
        import torch
        from . import _native
        self.torch = torch
        self.dev = torch.device("cuda", device)
        # a stream of the engine's own (the legacy default stream cannot be handed over as "the caller's
        # stream"); the driver makes it torch's current stream around every phase and collective
        self.stream = stream if stream is not None else torch.cuda.Stream(self.dev)
        self.plan = _native.Plan(net, ms, part, bord, maps, device=device,
                                 dense=cfg.backend == "dense", rank=rank, world=world,
                                 area_rank=area_rank, stream=self.stream.cuda_stream, max_ctas=max_ctas,
                                 boundary_mode={"auto": 0, "dense": 1, "sparse": 2}[cfg.boundary])
        self.net, self.bord = net, bord
        self.n_bus, self.n_gamma = net.n_bus, bord.n_gamma
        self.state = torch.empty((2, net.n_bus), dtype=torch.float64, device=self.dev)
        ptr, n, off = self.plan.exchange_buffer()
        self.offsets = off
        self.exchange = self._view(ptr, n)
        self.delta = self._view(self.plan.boundary_delta_ptr(), max(self.n_gamma, 1))[: self.n_gamma]
        self.status = self._view(self.plan.status_ptr(), 2)      # [max |dx|, failed ? 1 : 0] after recover_async
        owned = np.zeros(net.n_bus, dtype=bool)
        for a, m in enumerate(maps):
            if area_rank[a] == rank:
                owned[m.internal_buses] = True
        self.owned_mask = torch.from_numpy(owned).to(self.dev)

    def _view(self, ptr, n):
        class _Dev:
            pass
        holder = _Dev()
        holder.__cuda_array_interface__ = {"shape": (int(n),), "typestr": "<f8",
                                           "data": (int(ptr), False), "version": 3}
        return self.torch.as_tensor(holder, device=self.dev)

    def stream_ctx(self):
        """Context in which torch ops and collectives are ordered with the plan's kernels."""
        return self.torch.cuda.stream(self.stream)

    def load_state(self, va, vm):
        with self.stream_ctx():
            self.state.copy_(self.torch.from_numpy(np.stack([va, vm])))
        self.torch.cuda.synchronize(self.dev)

    def _translated(self, fn, *args):
        from . import _native
        from .solver import raise_solver_error
        try:
            return fn(*args)
        except _native.NativeError as exc:
            raise_solver_error(exc, self.net, self.bord)

    def phase_local(self):
        va, vm = self.state[0].data_ptr(), self.state[1].data_ptr()
        self.plan.phase_assemble(va, vm)
        self._translated(self.plan.phase_condense)

    def phase_boundary(self):
        self._translated(self.plan.phase_boundary)

    def phase_recover(self):
        return self.plan.phase_recover(self.state[0].data_ptr(), self.state[1].data_ptr())

    def inner_step(self):
        """One interior-only GN step of the owned areas, boundary held fixed (reference solver.py:253-260);
        returns max |dx_i| of this rank."""
        return self._translated(self.plan.inner_step, self.state[0].data_ptr(), self.state[1].data_ptr())

    # enqueue-only variants (same kernels; no host synchronisation, failures surface in status[1])
    def phase_local_async(self):
        self.plan.phase_local_async(self.state[0].data_ptr(), self.state[1].data_ptr())

    def phase_boundary_async(self):
        self.plan.phase_boundary_async()

    def phase_recover_async(self):
        self.plan.phase_recover_async(self.state[0].data_ptr(), self.state[1].data_ptr())

    def check(self):
        """Raise the precise error of a failed factorisation owned by this rank (synchronises)."""
        self._translated(self.plan.check)

    # peer-linked solve: the exchanges inside the persistent kernel (gse_peer_link)
    def peer_info(self):
        return self.plan.peer_info()

    def peer_link(self, infos):
        self.plan.peer_link(infos)

    def solve_prepare(self):
        self.plan.peer_solve_prepare()

    def solve_linked(self, cfg):
        """The whole GN loop of this rank in one launch; returns the native report (objective unset)."""
        return self._translated(self.plan.solve, self.state[0].data_ptr(), self.state[1].data_ptr(),
                                cfg.max_outer_iterations, cfg.convergence_tol, False)

    def launches_last(self):
        """Kernels this rank's plan enqueued in the iteration just finished."""
        return int(self.plan.stats()["launches_last"])

    def sync(self):
        self.torch.cuda.synchronize(self.dev)

    def objective(self):
        return self.plan.objective(self.state[0].data_ptr(), self.state[1].data_ptr())

    def close(self):
        self.plan.close()


class DistributedEstimator:
    """Multi-rank counterpart of ``MultiAreaEstimator`` (same ``estimate`` contract)."""

    def __init__(self, net, ms, part, maps=None, config: SolverConfig = None, device=None,
                 engine_factory=None, group=None, exchange="auto"):
        import os
        import torch
        import torch.distributed as dist
        self.torch, self.dist, self.group = torch, dist, group
        if device is None:
            # one process per GPU: the launcher's LOCAL_RANK, else whatever device the caller made current
            device = int(os.environ["LOCAL_RANK"]) if "LOCAL_RANK" in os.environ else (
                torch.cuda.current_device() if torch.cuda.is_available() else 0)
        self.cfg = config or SolverConfig()
        self.net, self.ms, self.part = net, ms, part
        self.bord, self.maps = maps if maps is not None else build_variable_maps(net, part)
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.area_rank = assign_areas(area_work_estimate(self.maps), self.world)
        self.n_gamma = self.bord.n_gamma
        t0 = time.perf_counter()
        factory = engine_factory or CudaEngine
        self.engine = factory(net, ms, part, self.bord, self.maps, self.cfg, self.rank, self.world,
                              self.area_rank, device)
        self.setup_s = time.perf_counter() - t0
        # contiguous exchange segment of every rank: [off[first area], off[last area + 1])
        off = self.engine.offsets
        self.segments = []
        for r in range(self.world):
            mine = np.flatnonzero(self.area_rank == r)
            self.segments.append((int(off[mine[0]]), int(off[mine[-1] + 1])) if mine.size else (0, 0))
        self.launches_per_solve = 0
        self.last_gpu_s = 0.0
        self.linked = False
        if exchange not in ("auto", "peer", "collective"):
            raise ValueError("exchange must be 'auto', 'peer' or 'collective'")
        if exchange != "collective" and self.world > 1:
            self._link_peers(required=exchange == "peer")

    def _link_peers(self, required):
        """Exchange the ranks' ``gse_peer_info`` records and link the plans (CUDA IPC between processes).  Every
        rank must succeed, otherwise all of them stay on the collective driver."""
        eng, dist = self.engine, self.dist
        ok, err = 1.0, None
        if not hasattr(eng, "peer_info") or self.world > 8:
            ok = 0.0
        infos = [None] * self.world
        try:
            mine = eng.peer_info() if ok else b""
        except Exception as exc:        # e.g. no IPC support on this platform
            ok, err, mine = 0.0, exc, b""
        dist.all_gather_object(infos, mine, group=self.group)
        if ok and all(infos):
            try:
                eng.peer_link(infos)
            except Exception as exc:
                ok, err = 0.0, exc
        else:
            ok = 0.0
        t = self.torch.tensor([ok], dtype=self.torch.float64, device=getattr(eng, "dev", "cpu"))
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=self.group)
        self.linked = bool(float(t.cpu()[0]))
        if required and not self.linked:
            raise RuntimeError(f"peer exchange requested but the ranks could not be linked: {err}")

    # -- collectives ---------------------------------------------------------------------------
    def _gather_blocks(self):
        if self.world == 1:
            return
        dist, buf = self.dist, self.engine.exchange
        ops = []
        if self.rank == 0:
            for r in range(1, self.world):
                lo, hi = self.segments[r]
                if hi > lo:
                    ops.append(dist.P2POp(dist.irecv, buf[lo:hi], r, group=self.group))
        else:
            lo, hi = self.segments[self.rank]
            if hi > lo:
                ops.append(dist.P2POp(dist.isend, buf[lo:hi], 0, group=self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()

    def _allreduce_max(self, values):
        t = self.torch.tensor(values, dtype=self.torch.float64, device=self.engine.exchange.device)
        if self.world > 1:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return [float(v) for v in t.cpu()]

    # -- the solve -------------------------------------------------------------------------------
    def update_measurements(self, ms):
        same_rows = ms.m == self.ms.m and all(
            a is b or np.array_equal(a, b) for a, b in ((ms.mtype, self.ms.mtype), (ms.target, self.ms.target)))
        if not same_rows:
            raise ValueError("measurement rows differ from the analysed template set")
        self.engine.plan.set_measurements(ms.z)
        self.engine.plan.set_weights(ms.weight)
        self.ms = ms

    def estimate(self, on_iteration=None):
        ctx = getattr(self.engine, "stream_ctx", None)
        if ctx is None:
            return self._estimate(on_iteration)
        with ctx():
            return self._estimate(on_iteration)

    def _inner_steps(self):
        """``inner_gn_steps - 1`` interior-only GN steps of every rank's areas with the boundary held fixed
        (reference solver.py:253-260); returns the largest |dx_i| over all ranks (it joins the stacked norm
        of the iteration).  A failed factorisation is reported on every rank."""
        steps = self.cfg.inner_gn_steps - 1
        if steps <= 0:
            return 0.0
        inner, failure = 0.0, None
        for _ in range(steps):
            try:
                inner = max(inner, float(self.engine.inner_step()))
            except Exception as exc:
                failure = exc
                break
        inner, flag = self._allreduce_max([inner, 1.0 if failure is not None else 0.0])
        if flag:
            raise failure if failure is not None else SolverError(
                "an area interior block on another rank is not positive definite; "
                "that area is likely locally unobservable")
        return inner

    def _estimate_linked(self):
        """One launch per rank: the loop, both exchanges and the convergence decision live in the kernels."""
        cfg, eng = self.cfg, self.engine
        t_start = time.perf_counter()
        flat = StateVector.flat_start(self.net)
        eng.load_state(flat.va, flat.vm)
        eng.solve_prepare()                      # this rank's counters are clear ...
        self.dist.barrier(group=self.group)      # ... and so are everybody else's: peers may signal from now on
        t_loop = time.perf_counter()
        rep = eng.solve_linked(cfg)              # raises the same SolverError on every rank (the failure code is global)
        self.last_gpu_s = time.perf_counter() - t_loop
        self.launches_per_solve = 1
        state = self._full_state(load_back=True)
        j = eng.objective()
        self.last_deltas = [float(rep.delta_inf[k]) for k in range(rep.iterations)]
        timings = {p: 0.0 for p in PHASES}
        timings["total"] = time.perf_counter() - t_start
        return state, SolveReport(method="multiarea", iterations=int(rep.iterations), converged=bool(rep.converged),
                                  objective=float(j), weighted_residual_norm=float(np.sqrt(j)),
                                  n_gamma=self.n_gamma, timings=timings)

    def _estimate(self, on_iteration=None):
        cfg, eng = self.cfg, self.engine
        if (self.linked and on_iteration is None and cfg.inner_gn_steps == 1 and cfg.max_outer_iterations <= 64
                and not cfg.profile_phases):
            return self._estimate_linked()
        t_start = time.perf_counter()
        flat = StateVector.flat_start(self.net)
        eng.load_state(flat.va, flat.vm)
        iterations, converged, deltas = 0, False, []
        self.launches_per_solve = 0
        t_loop = time.perf_counter()
        use_async = bool(getattr(eng, "async_phases", False))
        for it in range(1, cfg.max_outer_iterations + 1):
            inner = self._inner_steps()
            if use_async:
                # one pipeline per iteration on the engine's stream: local condensation -> gather of the
                # (S_b | b_hat) segments -> boundary solve on the coordinator -> broadcast of delta_x_Gamma
                # -> recovery -> MAX all-reduce of [delta, failed]; the host waits once, for that pair
                eng.phase_local_async()
                self._gather_blocks()
                if self.rank == 0 and self.n_gamma:
                    eng.phase_boundary_async()
                if self.world > 1 and self.n_gamma:
                    self.dist.broadcast(eng.delta, src=0, group=self.group)
                eng.phase_recover_async()
                if self.world > 1:
                    self.dist.all_reduce(eng.status, op=self.dist.ReduceOp.MAX, group=self.group)
                delta, failed = (float(v) for v in eng.status.cpu())
                delta = max(delta, inner)
                self.launches_per_solve += eng.launches_last()
                if failed:
                    eng.check()        # the owning rank raises the precise error ...
                    raise SolverError("a factorisation on another rank is not positive definite; "
                                      "the area it belongs to is likely locally unobservable")
                iterations = it
                deltas.append(delta)
                if on_iteration is not None:
                    on_iteration(it, self._full_state(), delta)
                if delta < cfg.convergence_tol:
                    converged = True
                    break
                continue
            failure = None
            try:
                eng.phase_local()
            except Exception as exc:       # reported consistently on every rank below
                failure = exc
            flag = self._allreduce_max([1.0 if failure is not None else 0.0])[0]
            if flag:
                raise failure if failure is not None else SolverError(
                    "an area interior block on another rank is not positive definite; "
                    "that area is likely locally unobservable")
            eng.sync()
            self._gather_blocks()
            failure = None
            if self.rank == 0 and self.n_gamma:
                try:
                    eng.phase_boundary()
                except Exception as exc:
                    failure = exc
            flag = self._allreduce_max([1.0 if failure is not None else 0.0])[0]
            if flag:
                raise failure if failure is not None else SolverError(
                    "boundary system not positive definite (reported by the coordinator rank)")
            if self.world > 1 and self.n_gamma:
                eng.sync()
                self.dist.broadcast(eng.delta, src=0, group=self.group)
            local_delta = eng.phase_recover()
            delta = max(self._allreduce_max([local_delta])[0], inner)
            iterations = it
            deltas.append(delta)
            if on_iteration is not None:
                on_iteration(it, self._full_state(), delta)
            if delta < cfg.convergence_tol:
                converged = True
                break
        self.last_gpu_s = time.perf_counter() - t_loop
        state = self._full_state(load_back=True)
        j = eng.objective()
        self.last_deltas = deltas
        timings = {p: 0.0 for p in PHASES}
        timings["total"] = time.perf_counter() - t_start
        report = SolveReport(method="multiarea", iterations=iterations, converged=converged,
                             objective=float(j), weighted_residual_norm=float(np.sqrt(j)),
                             n_gamma=self.n_gamma, timings=timings)
        return state, report

    def _full_state(self, load_back=False):
        """Every rank's interior slice merged (SUM all-reduce of disjoint masks); the boundary
        replica and the pinned slack come from the coordinator's copy."""
        eng, torch = self.engine, self.torch
        st = eng.state.clone()
        if self.world > 1:
            keep = eng.owned_mask if self.rank else torch.ones_like(eng.owned_mask)
            if self.rank == 0:
                # rank 0 contributes its interiors + everything that is not an interior of another rank
                other = torch.zeros_like(eng.owned_mask)
                other[torch.from_numpy(self._foreign_interiors()).to(other.device)] = True
                keep = ~other
            st = st * keep.to(st.dtype)
            self.dist.all_reduce(st, op=self.dist.ReduceOp.SUM, group=self.group)
            if load_back:
                eng.state.copy_(st)
        arr = st.cpu().numpy()
        return StateVector(va=arr[0].copy(), vm=arr[1].copy())

    def _foreign_interiors(self):
        idx = [m.internal_buses for a, m in enumerate(self.maps) if self.area_rank[a] != 0]
        return np.concatenate(idx).astype(np.int64) if idx else np.zeros(0, dtype=np.int64)

    def close(self):
        # peer-linked plans map each other's buffers (CUDA IPC): nobody frees before everybody has stopped using them
        if self.linked and self.world > 1:
            try:
                self.dist.barrier(group=self.group)
            except Exception:       # (a rank that failed earlier must still be able to clean up)
                pass
        self.engine.close()
