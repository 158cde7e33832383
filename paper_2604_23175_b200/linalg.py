"""Linear-algebra result types of the solve path.

Mirrors the public types of the reference's ``gridse.linalg`` (reference
``pkg/src/gridse/linalg.py:29-43``).  The factorisation itself is not a Python
object here: ordering, fronts and the Schur-mode tree are part of the device plan
(``csrc/symbolic.cpp``), ``numeric_refactor`` + ``schur_condense`` are the
``local_condense`` phase and ``interior_recover`` the ``recovery`` phase of that
plan (``AreaCondenser`` below exposes them per area for component parity).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

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
