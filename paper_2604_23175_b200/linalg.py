"""Linear algebra of the solve path on the device.

API mirror of the reference's ``gridse.linalg`` (reference ``pkg/src/gridse/linalg.py:29-434``):
``NotPositiveDefiniteError``, ``SchurResult``, ``SparseCholeskyCache``, ``symbolic_analyze``,
``numeric_refactor``, ``schur_condense``, ``interior_recover``, ``dense_cholesky_solve`` keep their
signatures and error behaviour.  Inside ``solve_multiarea`` these computations are phases of one
device plan (``csrc/symbolic.cpp``: ordering, fronts, Schur-mode tree); the standalone functions
here run the same multifrontal kernels on caller-supplied matrices through *matrix plans*
(``gse_matrix_*``): a one-area Schur-mode tree whose interior block is the cache's matrix and whose
boundary rows are the columns of ``g_ib``.

Differences a caller can observe: the ordering is nested dissection instead of the reference's
greedy minimum degree (the reference allows any ordering, ``SPEC.md:362``), so the intermediate
vector of ``forward`` / ``backward`` lives in THIS factor's coordinates (``cache.perm``, as in the
reference: ``y = L^-1 P b``); ``backward(forward(b))`` equals ``solve(b)`` bit for bit and
``y @ y == b @ G^-1 b`` whatever the ordering.  There is no CPU fallback: every call needs a CUDA device.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from . import _native

DENSE_FALLBACK_DIM = 64


class NotPositiveDefiniteError(ValueError):
    """Cholesky hit a non-positive pivot (unobservable or indefinite system)."""

    def __init__(self, pivot, context="matrix"):
        super().__init__(f"{context} not positive definite at pivot {pivot}")
        self.pivot = int(pivot)
        self.context = context


@dataclass
class SchurResult:
    """Condensed boundary block S_b and right-hand side b_hat of one area."""

    s_b: np.ndarray
    b_hat: np.ndarray


class SparseCholeskyCache:
    """Analyze once, refactor many times (reference linalg.py:132-392), device-resident.

    The symbolic structure (ordering, fronts, extend-add maps) is built per coupling pattern: the
    plain cache (``refactor`` / ``solve``) uses a plan without boundary rows; ``schur_condense``
    with a given ``g_ib`` builds -- once per distinct ``g_ib`` pattern -- the Schur-mode plan whose
    area root delivers ``S_b`` and ``b_hat``.
    """

    def __init__(self, pattern, dense_threshold=DENSE_FALLBACK_DIM, ordering="amd", context="matrix"):
        pattern = sp.csr_matrix(pattern)
        pattern.sort_indices()
        if pattern.shape[0] != pattern.shape[1]:
            raise ValueError("pattern must be square")
        self.n = pattern.shape[0]
        self.context = context
        self.ordering = ordering
        self.pattern_indptr = pattern.indptr.astype(np.int32)
        self.pattern_indices = pattern.indices.astype(np.int32)
        self.mode = "dense" if self.n < dense_threshold else "sparse"
        self._values = None
        self._plans = {}
        self._factorized = False

    # -- plans -----------------------------------------------------------------------
    def _plan(self, g_ib=None):
        if g_ib is None or g_ib.shape[1] == 0:
            key, n_b, ib_ptr, ib_idx = None, 0, None, None
        else:
            g_ib = sp.csr_matrix(g_ib)
            g_ib.sort_indices()
            ib_ptr, ib_idx = g_ib.indptr.astype(np.int32), g_ib.indices.astype(np.int32)
            n_b = g_ib.shape[1]
            key = (n_b, ib_ptr.tobytes(), ib_idx.tobytes())
        if key not in self._plans:
            self._plans[key] = _native.MatrixPlan(self.n, n_b, self.pattern_indptr, self.pattern_indices,
                                                  ib_ptr, ib_idx, dense=self.mode == "dense")
        return self._plans[key]

    def _raise(self, exc):
        if exc.code == _native.GSE_E_NOT_SPD_AREA:
            raise NotPositiveDefiniteError(exc.pivot, self.context) from exc
        raise exc

    def _values_from(self, values):
        """Value array aligned with the pattern, or any sparse matrix with a sub-pattern
        (reference linalg.py:262-290)."""
        if sp.issparse(values):
            m = sp.csr_matrix(values)
            m.sort_indices()
            if m.shape != (self.n, self.n):
                raise ValueError("matrix shape does not match the analyzed pattern")
            if np.array_equal(m.indptr, self.pattern_indptr) and np.array_equal(m.indices, self.pattern_indices):
                return np.asarray(m.data, dtype=float)
            out = np.zeros(self.pattern_indices.size)
            for r in range(self.n):
                lo, hi = self.pattern_indptr[r], self.pattern_indptr[r + 1]
                cols = m.indices[m.indptr[r]:m.indptr[r + 1]]
                pos = np.searchsorted(self.pattern_indices[lo:hi], cols)
                if np.any(pos >= hi - lo) or np.any(self.pattern_indices[lo:hi][pos] != cols):
                    raise ValueError("matrix has entries outside the analyzed pattern")
                out[lo + pos] = m.data[m.indptr[r]:m.indptr[r + 1]]
            return out
        values = np.asarray(values, dtype=float)
        if values.shape != (self.pattern_indices.size,):
            raise ValueError("value array does not match the analyzed pattern")
        return values

    # -- numeric phase -------------------------------------------------------------------
    def refactor(self, values):
        """Value-only refactorisation; raises ``NotPositiveDefiniteError`` with the original index of
        the first non-positive pivot met in elimination order."""
        self._values = self._values_from(values).copy()
        self._factorized = False
        if self.n:
            plan = self._plan()
            try:
                plan.set_values(data_ii=self._values)
                plan.condense()
            except _native.NativeError as exc:
                self._raise(exc)
        self._factorized = True
        return self

    def solve(self, b, refine_with=None):
        """G x = b with the current values; optional single refinement pass against ``refine_with``."""
        if not self._factorized:
            raise RuntimeError("refactor() must run before solve()")
        b = np.asarray(b, dtype=float)
        if b.ndim == 2:
            return np.stack([self.solve(b[:, j], refine_with) for j in range(b.shape[1])], axis=1) if b.shape[1] else b.copy()
        if self.n == 0:
            return np.zeros(0)
        plan = self._plan()
        try:
            plan.set_values(data_ii=self._values, b_i=b)
            plan.condense()
            x = plan.recover()
            if refine_with is not None:
                r = b - refine_with @ x
                plan.set_values(data_ii=self._values, b_i=r)
                plan.condense()
                x = x + plan.recover()
        except _native.NativeError as exc:
            self._raise(exc)
        return x

    @property
    def perm(self):
        """Elimination order of this factor: ``perm[e]`` = original index eliminated at position ``e``
        (reference ``SparseCholeskyCache.perm``; a nested-dissection order here)."""
        return self._plan().perm() if self.n else np.zeros(0, dtype=np.int32)

    def forward(self, b):
        """``y = L^-1 P b`` (reference linalg.py:340-364); ``b`` is a vector or a matrix of columns.  On the device
        the right-hand side rides through the factorisation as one extra row of every front, so this is a
        refactorisation with ``b`` attached."""
        if not self._factorized:
            raise RuntimeError("numeric factorization has not been run")
        b = np.asarray(b, dtype=float)
        if b.ndim == 2:
            return np.stack([self.forward(b[:, j]) for j in range(b.shape[1])], axis=1) if b.shape[1] else b.copy()
        if self.n == 0:
            return b.copy()
        plan = self._plan()
        try:
            plan.set_values(data_ii=self._values, b_i=b)
            plan.condense()
            return plan.forward_get()
        except _native.NativeError as exc:
            self._raise(exc)

    def backward(self, y):
        """``x = P^T L^-T y`` (reference linalg.py:366-383) with the current factor."""
        if not self._factorized:
            raise RuntimeError("numeric factorization has not been run")
        y = np.asarray(y, dtype=float)
        if y.ndim == 2:
            return np.stack([self.backward(y[:, j]) for j in range(y.shape[1])], axis=1) if y.shape[1] else y.copy()
        if self.n == 0:
            return y.copy()
        try:
            return self._plan().backward(y)
        except _native.NativeError as exc:
            self._raise(exc)

    def stats(self):
        """Pattern statistics (the factor is a tree of dense fronts on the device)."""
        return {"n": self.n, "mode": self.mode, "pattern_nnz": int(self.pattern_indices.size)}

    def close(self):
        for p in self._plans.values():
            p.close()
        self._plans = {}


def symbolic_analyze(pattern, dense_threshold=DENSE_FALLBACK_DIM, ordering="amd", context="matrix") -> SparseCholeskyCache:
    """One-time symbolic analysis of a structurally symmetric CSR pattern (reference linalg.py:395-398)."""
    return SparseCholeskyCache(pattern, dense_threshold, ordering, context)


def numeric_refactor(cache: SparseCholeskyCache, values) -> SparseCholeskyCache:
    """Value-only refactorisation (reference linalg.py:401-403)."""
    return cache.refactor(values)


def schur_condense(cache: SparseCholeskyCache, g_ib, g_bb, b_i, b_b) -> SchurResult:
    """S_b = g_bb - g_ib^T g_ii^-1 g_ib, b_hat = b_b - g_ib^T g_ii^-1 b_i (reference linalg.py:410-424)
    with the values of the last ``numeric_refactor``: one forward pass of the Schur-mode tree."""
    g_bb = np.asarray(g_bb, dtype=float)
    b_b = np.asarray(b_b, dtype=float)
    if cache.n == 0:
        return SchurResult(s_b=g_bb.copy(), b_hat=b_b.copy())
    g_ib = sp.csr_matrix(g_ib)
    if g_ib.shape[1] == 0:
        return SchurResult(s_b=g_bb.copy(), b_hat=b_b.copy())
    if not cache._factorized:
        raise RuntimeError("numeric_refactor must run before schur_condense")
    g_ib.sort_indices()
    plan = cache._plan(g_ib)
    try:
        plan.set_values(data_ii=cache._values, data_ib=g_ib.data, g_bb=g_bb, b_i=b_i, b_b=b_b)
        plan.condense()
    except _native.NativeError as exc:
        cache._raise(exc)
    s_b, b_hat = plan.schur()
    return SchurResult(s_b=s_b, b_hat=b_hat)


def interior_recover(cache: SparseCholeskyCache, g_ib, b_i, delta_xb) -> np.ndarray:
    """Interior update after the boundary solve: g_ii^-1 (b_i - g_ib dx_b) (reference linalg.py:427-434)."""
    b_i = np.asarray(b_i, dtype=float)
    if cache.n == 0:
        return np.zeros(0)
    delta_xb = np.asarray(delta_xb, dtype=float)
    if delta_xb.size == 0:
        return cache.solve(b_i)
    g_ib = sp.csr_matrix(g_ib)
    g_ib.sort_indices()
    plan = cache._plan(g_ib)
    try:
        plan.set_values(data_ii=cache._values, data_ib=g_ib.data, b_i=b_i)
        plan.condense()
        return plan.recover(delta_xb)
    except _native.NativeError as exc:
        cache._raise(exc)


def dense_cholesky_solve(a, b, context="matrix"):
    """Dense SPD solve (reference linalg.py:46-61: dpotrf + dpotrs): a chain of dense fronts in natural
    order on the device.  A non-positive pivot raises ``NotPositiveDefiniteError(pivot)``."""
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    n = a.shape[0]
    if a.shape != (n, n) or b.shape[0] != n:
        raise ValueError("shape mismatch")
    if n == 0:
        return np.zeros_like(b)
    cache = SparseCholeskyCache(sp.csr_matrix(np.ones((n, n))), dense_threshold=10**9, context=context)
    try:
        cache.refactor(a.ravel())
        return cache.solve(b)
    finally:
        cache.close()
