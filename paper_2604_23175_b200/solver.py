"""WLS Gauss-Newton solvers on the device.

API mirror of the reference's ``gridse.solver`` (reference
``pkg/src/gridse/solver.py:36-346``): ``SolverConfig``, ``SolveReport``,
``BoundarySystem``, ``SolverError``, ``objective``, ``assemble_boundary``,
``solve_multiarea``, ``solve_centralized`` keep their signatures, defaults,
result fields and error texts; the work happens in ``libgridse_b200.so``.

``MultiAreaEstimator`` is the warm path the reference lacks: the plan
(templates, slot map, ordering, fronts, CUDA graph) is built once and reused
across solves -- new measurement values or masks are weight / value refreshes
(reference ``PAPER.md:203,226``: "template indices, mapping arrays, working
buffers allocated once").  PyTorch only owns the device state vectors.
"""

from __future__ import annotations

import json
import os
import threading
import time
from collections import OrderedDict
from dataclasses import dataclass

import numpy as np

from . import _native
from .linalg import NotPositiveDefiniteError
from .measurement import MeasurementSet, StateVector
from .partition import build_variable_maps, partition_network

PHASES = ("assembly", "local_condense", "boundary_assemble", "boundary_solve", "recovery")


class SolverError(RuntimeError):
    pass


@dataclass
class SolverConfig:
    max_outer_iterations: int = 10
    inner_gn_steps: int = 1
    convergence_tol: float = 1e-6
    deterministic: bool = True      # the device path is always bit-stable; kept for API parity
    backend: str = "sparse"         # "dense": chain of dense fronts per area instead of nested dissection
    dense_threshold: int = 64       # kept for API parity (fronts are dense blocks at every size)
    iterative_refinement: bool = False
    # extension: run the level-launch path (one kernel per tree level, no CUDA graph) with CUDA events
    # between the phases instead of the single persistent kernel (which stamps its phases itself)
    profile_phases: bool = False
    # extension: how the reduced boundary system is factored.  "dense" = the reference's dense
    # Cholesky (a chain of dense fronts); "sparse" = the same factorisation with the structural
    # zeros between non-adjacent areas skipped (nested dissection on the area-clique graph);
    # "auto" = dense up to n_Gamma = 192, sparse above.
    boundary: str = "auto"

    def __post_init__(self):
        if self.max_outer_iterations < 1:
            raise ValueError("max_outer_iterations must be >= 1")
        if self.convergence_tol <= 0:
            raise ValueError("convergence_tol must be positive")
        if self.backend not in ("dense", "sparse"):
            raise ValueError(f"unknown backend {self.backend!r}")
        if self.boundary not in ("auto", "dense", "sparse"):
            raise ValueError(f"unknown boundary mode {self.boundary!r}")
        if self.inner_gn_steps < 1:
            raise ValueError("inner_gn_steps must be >= 1")

    @property
    def effective_dense_threshold(self):
        return 10**9 if self.backend == "dense" else self.dense_threshold


@dataclass
class SolveReport:
    method: str
    iterations: int
    converged: bool
    objective: float
    weighted_residual_norm: float
    n_gamma: int
    timings: dict

    def to_dict(self):
        return {
            "method": self.method, "iterations": self.iterations, "converged": self.converged,
            "objective": self.objective, "weighted_residual_norm": self.weighted_residual_norm,
            "n_gamma": self.n_gamma, "timings": dict(self.timings),
        }

    def to_json(self):
        return json.dumps(self.to_dict(), indent=1)


@dataclass
class BoundarySystem:
    s_gamma: np.ndarray
    b_gamma: np.ndarray
    delta_x_gamma: np.ndarray = None


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise _native.NoDeviceError(
            _native.GSE_E_NO_DEVICE, -1, -1,
            "no CUDA device visible: gridse-b200 has no CPU fallback")
    return torch


def raise_solver_error(exc, net, bord, method="multiarea"):
    """Re-raise a ``NativeError`` of the C ABI with the reference's texts (solver.py:250-251,304-309)."""
    if exc.code == _native.GSE_E_NOT_SPD_AREA:
        ctx = f"area {exc.area} interior block"
        inner = NotPositiveDefiniteError(exc.pivot, ctx)
        if method == "centralized":
            raise SolverError(
                f"gain matrix {inner}: system unobservable or ill-conditioned") from inner
        raise SolverError(f"{inner}; area {exc.area} is likely locally unobservable") from inner
    if exc.code == _native.GSE_E_NOT_SPD_BOUNDARY:
        inner = NotPositiveDefiniteError(exc.pivot, "boundary system")
        bus, quant = bord.entries[exc.pivot]
        raise SolverError(
            f"boundary system not positive definite at pivot {exc.pivot} "
            f"(bus {net.buses[bus].id}, {quant})") from inner
    raise exc


class MultiAreaEstimator:
    """Plan once, estimate many times (device-resident Gauss-Newton loop)."""

    def __init__(self, net, ms: MeasurementSet, part, maps=None, config: SolverConfig = None,
                 device=0, method="multiarea", rank=0, world=1, area_rank=None):
        self.cfg = config or SolverConfig()
        self.net, self.part, self.method = net, part, method
        self.bord, self.maps = maps if maps is not None else build_variable_maps(net, part)
        t0 = time.perf_counter()
        torch = _torch()
        self.torch = torch
        self.device = torch.device("cuda", device)
        self.plan = _native.Plan(net, ms, part, self.bord, self.maps, device=device,
                                 dense=self.cfg.backend == "dense", rank=rank, world=world,
                                 area_rank=area_rank,
                                 boundary_mode={"auto": 0, "dense": 1, "sparse": 2}[self.cfg.boundary])
        self.ms = ms
        self.n_gamma = self.bord.n_gamma
        self._flat = np.stack([StateVector.flat_start(net).va, np.ones(net.n_bus)])
        self._host = torch.empty((2, net.n_bus), dtype=torch.float64).pin_memory()
        self._state = torch.empty((2, net.n_bus), dtype=torch.float64, device=self.device)
        self._flat_dev = torch.from_numpy(self._flat).to(self.device)      # the flat start is a constant of the plan
        torch.cuda.current_stream(self.device).synchronize()              # (the plan's stream reads it from now on)
        self._persistent = bool(self.plan.stats()["persistent"])
        self.setup_s = time.perf_counter() - t0

    # -- inputs ----------------------------------------------------------------------
    def update_measurements(self, ms: MeasurementSet):
        """New values / masks on the same rows: refresh z and w, no re-analysis."""
        same_rows = ms.m == self.ms.m and all(
            a is b or np.array_equal(a, b) for a, b in ((ms.mtype, self.ms.mtype), (ms.target, self.ms.target)))
        if not same_rows:
            raise ValueError("measurement rows differ from the analysed template set")
        self.plan.set_measurements(ms.z)
        self.plan.set_weights(ms.weight)
        self.ms = ms
        if getattr(self, "_pin", None) is not None:      # keep the pinned mirror current (update_from_pinned
            self._pin[0].numpy()[:] = ms.z               # would otherwise copy the previous scan back)
            self._pin[1].numpy()[:] = ms.weight

    def pinned_inputs(self):
        """(z, w) numpy views of pinned host buffers owned by the estimator.  A data front end writes
        the next scan's values / weights there in place; ``update_from_pinned`` then moves them to the
        device with one asynchronous copy of the contiguous block (no staging, no host synchronisation)."""
        if getattr(self, "_pin", None) is None:
            self._pin = self.torch.empty((2, self.ms.m), dtype=self.torch.float64).pin_memory()
            self._pin[0].numpy()[:] = self.ms.z
            self._pin[1].numpy()[:] = self.ms.weight
        return self._pin[0].numpy(), self._pin[1].numpy()

    def update_from_pinned(self):
        """Refresh z and w on the device from ``pinned_inputs()`` (same rows, no re-analysis)."""
        if getattr(self, "_pin", None) is None:
            raise RuntimeError("pinned_inputs() must be called (and filled) first")
        self.plan.set_rows_pinned(self._pin[0].data_ptr(), self._pin[1].data_ptr())

    def _ptrs(self):
        return self._state[0].data_ptr(), self._state[1].data_ptr()

    def _load_flat_start(self):
        self._state.copy_(self._flat_dev, non_blocking=True)

    def _read_state(self):
        self._host.copy_(self._state)
        arr = self._host.numpy()
        return StateVector(va=arr[0].copy(), vm=arr[1].copy())

    def _raise(self, exc):
        raise_solver_error(exc, self.net, self.bord, self.method)

    # -- the solve -----------------------------------------------------------------------
    def estimate(self, on_iteration=None, t_start=None):
        """Flat-start GN solve; returns (StateVector, SolveReport)."""
        cfg = self.cfg
        t_start = time.perf_counter() if t_start is None else t_start
        timings = {p: 0.0 for p in PHASES}
        va_ptr, vm_ptr = self._ptrs()
        fused_io = on_iteration is None and cfg.inner_gn_steps == 1 and cfg.max_outer_iterations <= 64
        if not fused_io:
            self._load_flat_start()
            self.torch.cuda.current_stream(self.device).synchronize()
        try:
            # (gse_solve reports at most 64 iterations; longer loops are sequenced here like the callback path)
            if fused_io:
                # flat start (resident on the device) in, final state out to pinned host memory: both ride the
                # plan's stream with the launch -- one host synchronisation per solve
                rep = self.plan.solve_io(self._flat_dev.data_ptr(), va_ptr, vm_ptr, self._host.data_ptr(),
                                         cfg.max_outer_iterations, cfg.convergence_tol, cfg.profile_phases)
                iterations, converged, j = rep.iterations, bool(rep.converged), rep.objective
                self.last_deltas = [rep.delta_inf[i] for i in range(iterations)]
                self.last_loop_s, self.last_gpu_s = rep.loop_s, rep.gpu_s
                # (one launch per solve on the persistent path: no need to ask the plan after every solve)
                self.launches_per_solve = 1 if (self._persistent and not cfg.profile_phases) else int(self.plan.stats()["launches_last"])
                # persistent path: device globaltimer stamps per phase; profile_phases: CUDA events
                # between the phases of the level-launch path
                for p, v in zip(PHASES, rep.phase_s):
                    timings[p] = float(v)
            else:
                iterations, converged = 0, False
                self.last_deltas = []
                t0 = time.perf_counter()
                for it in range(1, cfg.max_outer_iterations + 1):
                    # inner GN steps on the interiors with the boundary held fixed (all but the last,
                    # whose blocks feed the condensation -- reference solver.py:253-260)
                    inner = 0.0
                    for _ in range(cfg.inner_gn_steps - 1):
                        inner = max(inner, self.plan.inner_step(va_ptr, vm_ptr))
                    delta = max(inner, self.plan.iterate(va_ptr, vm_ptr))
                    iterations = it
                    self.last_deltas.append(delta)
                    if on_iteration is not None:
                        on_iteration(it, self._read_state(), delta)
                    if delta < cfg.convergence_tol:
                        converged = True
                        break
                self.last_loop_s = time.perf_counter() - t0
                j = self.plan.objective(va_ptr, vm_ptr)
        except _native.NativeError as exc:
            self._raise(exc)
        if fused_io:
            arr = self._host.numpy()
            state = StateVector(va=arr[0].copy(), vm=arr[1].copy())
        else:
            state = self._read_state()
        timings["total"] = time.perf_counter() - t_start
        report = SolveReport(
            method=self.method, iterations=iterations, converged=converged, objective=float(j),
            weighted_residual_norm=float(np.sqrt(j)), n_gamma=self.n_gamma if self.method == "multiarea" else 0,
            timings=timings)
        return state, report

    def objective(self, state: StateVector) -> float:
        self._host.copy_(self.torch.from_numpy(np.stack([state.va, state.vm])))
        self._state.copy_(self._host)
        return self.plan.objective(*self._ptrs())

    def close(self):
        self.plan.close()


def objective(ms: MeasurementSet, state: StateVector) -> float:
    """WLS objective sum w (z - h(x))^2 on the device (reference solver.py:100-103)."""
    net = ms.net
    est, cached = _cached_estimator(net, ms, _single_area_partition(net), None, None, "centralized")
    try:
        return est.objective(state)
    finally:
        if not cached:
            est.close()


def assemble_boundary(schur_results, selectors, n_gamma) -> BoundarySystem:
    """S_Gamma[sel, sel] += S_b, b_Gamma[sel] += b_hat, areas in ascending order (reference
    solver.py:106-119), summed on the device (``gse_assemble_boundary``)."""
    s_gamma, b_gamma = _native.assemble_boundary_device(
        [r.s_b for r in schur_results], [r.b_hat for r in schur_results], selectors, int(n_gamma))
    return BoundarySystem(s_gamma=s_gamma, b_gamma=b_gamma)


# ---- plan cache of the drop-in entry points ------------------------------------------------------
# The reference re-runs its symbolic setup inside every solve_multiarea call (solver.py:221-229); its
# harness protocol calls it 11 times on the same (net, ms, part) and drops the first (harness.py:135-158).
# Here a repeated call with the same network / partition objects and the same measurement rows reuses
# the analysed plan (z / w are refreshed when the measurement set changed), so the kept signature gets
# the warm path.  Inputs are frozen dataclasses in both packages (never mutated), so object identity of
# net / part plus the row signature of ms identifies the plan.  Entries hold device memory: the cache is
# a small LRU (GSE_PLAN_CACHE entries, default 4; 0 disables it) and clear_plan_cache() frees it.
_PLAN_CACHE: "OrderedDict[tuple, MultiAreaEstimator]" = OrderedDict()
_PLAN_CACHE_LOCK = threading.Lock()
plan_cache_stats = {"hits": 0, "misses": 0}


def _plan_cache_size():
    try:
        return max(0, int(os.environ.get("GSE_PLAN_CACHE", "4")))
    except ValueError:
        return 4


def clear_plan_cache():
    """Destroy every cached plan of ``solve_multiarea`` / ``solve_centralized`` (frees device memory)."""
    with _PLAN_CACHE_LOCK:
        while _PLAN_CACHE:
            _PLAN_CACHE.popitem()[1].close()


def _cached_estimator(net, ms, part, maps, cfg, method):
    """(estimator, cached?) -- a plan analysed for the same objects / rows / plan-shaping options, or a new one."""
    cap = _plan_cache_size()
    cfg = cfg or SolverConfig()
    key = (id(net), id(part), ms.m, cfg.backend, cfg.boundary, method)
    if cap:
        with _PLAN_CACHE_LOCK:
            est = _PLAN_CACHE.get(key)
            if est is not None and est.net is net and est.part is part:
                try:
                    if ms is not est.ms:
                        est.update_measurements(ms)       # raises ValueError when the rows differ
                    _PLAN_CACHE.move_to_end(key)
                    est.cfg = cfg
                    plan_cache_stats["hits"] += 1
                    return est, True
                except ValueError:
                    _PLAN_CACHE.pop(key).close()
    plan_cache_stats["misses"] += 1
    est = MultiAreaEstimator(net, ms, part, maps=maps, config=cfg, method=method)
    if cap:
        with _PLAN_CACHE_LOCK:
            _PLAN_CACHE[key] = est
            while len(_PLAN_CACHE) > cap:
                _PLAN_CACHE.popitem(last=False)[1].close()
    return est, bool(cap)


def _solve_cached(net, ms, part, maps, config, on_iteration, method, t_start):
    est, cached = _cached_estimator(net, ms, part, maps, config, method)
    try:
        return est.estimate(on_iteration=on_iteration, t_start=t_start)
    except BaseException:
        # a failed solve (unobservable area, ...) leaves nothing worth keeping
        with _PLAN_CACHE_LOCK:
            for k, v in list(_PLAN_CACHE.items()):
                if v is est:
                    del _PLAN_CACHE[k]
        est.close()
        cached = False
        raise
    finally:
        if not cached:
            est.close()


def solve_multiarea(net, ms: MeasurementSet, part, maps=None, config: SolverConfig = None,
                    on_iteration=None):
    """Boundary-condensed multi-area WLS-GN; returns (estimate, report).

    Same contract as the reference (solver.py:204-346).  Setup (plan build) is inside
    ``timings['total']`` as it is there -- on the first call for a given (net, part, measurement rows);
    later calls reuse the cached plan (see ``clear_plan_cache``).  ``MultiAreaEstimator`` is the
    explicit form of the warm path.
    """
    t_start = time.perf_counter()
    return _solve_cached(net, ms, part, maps, config, on_iteration, "multiarea", t_start)


def solve_centralized(net, ms: MeasurementSet, config: SolverConfig = None, on_iteration=None):
    """Single-area GN on the device: the k = 1 path of the same plan (one area,
    empty boundary), i.e. the paper's "centralized GPU" baseline."""
    t_start = time.perf_counter()
    if config is not None and config.iterative_refinement:
        return _solve_centralized_refined(net, ms, config, on_iteration, t_start)
    return _solve_cached(net, ms, _single_area_partition(net), None, config, on_iteration, "centralized", t_start)


_K1_PARTS: "OrderedDict[int, tuple]" = OrderedDict()


def _single_area_partition(net):
    """The k = 1 partition of a network, one object per network object (so the plan cache can key on it)."""
    hit = _K1_PARTS.get(id(net))
    if hit is not None and hit[0] is net:
        _K1_PARTS.move_to_end(id(net))
        return hit[1]
    part = partition_network(net, 1)
    _K1_PARTS[id(net)] = (net, part)
    while len(_K1_PARTS) > 8:
        _K1_PARTS.popitem(last=False)
    return part


def _solve_centralized_refined(net, ms, cfg, on_iteration, t_start):
    """``iterative_refinement=True`` (read only by ``solve_centralized`` in the reference,
    solver.py:181-183): the reference's own loop on the device components -- ``fused_accumulate``
    for the gain matrix and right-hand side, ``numeric_refactor`` and ``cache.solve(b,
    refine_with=G)`` (one residual correction, linalg.py:385-392) on the device factorisation."""
    from .assembly import build_patterns, fused_accumulate
    from .linalg import numeric_refactor, symbolic_analyze
    timings = {p: 0.0 for p in PHASES}
    part = partition_network(net, 1)
    _, maps = build_variable_maps(net, part)
    vmap = maps[0]
    pattern = build_patterns(vmap, ms)
    cache = symbolic_analyze(pattern.gii_pattern(), dense_threshold=cfg.effective_dense_threshold,
                             context="gain matrix")
    try:
        state = StateVector.flat_start(net)
        empty = np.zeros(0)
        iterations, converged = 0, False
        for it in range(1, cfg.max_outer_iterations + 1):
            t0 = time.perf_counter()
            x_i = vmap.gather_interior(state.va, state.vm)
            blocks = fused_accumulate(vmap, ms, x_i, empty, pattern=pattern)
            t1 = time.perf_counter()
            try:
                numeric_refactor(cache, blocks.g_ii)
            except NotPositiveDefiniteError as exc:
                raise SolverError(
                    f"gain matrix {exc}: system unobservable or ill-conditioned") from exc
            t2 = time.perf_counter()
            delta = cache.solve(blocks.b_i, refine_with=blocks.g_ii)
            vmap.apply_interior_delta(state.va, state.vm, delta)
            t3 = time.perf_counter()
            timings["assembly"] += t1 - t0
            timings["local_condense"] += t2 - t1
            timings["recovery"] += t3 - t2
            iterations = it
            delta_inf = float(np.max(np.abs(delta))) if delta.size else 0.0
            if on_iteration is not None:
                on_iteration(it, state.copy(), delta_inf)
            if delta_inf < cfg.convergence_tol:
                converged = True
                break
        j = objective(ms, state)
    finally:
        cache.close()
        pattern.plan.close()
    timings["total"] = time.perf_counter() - t_start
    report = SolveReport(method="centralized", iterations=iterations, converged=converged,
                         objective=float(j), weighted_residual_norm=float(np.sqrt(j)), n_gamma=0,
                         timings=timings)
    return state, report
