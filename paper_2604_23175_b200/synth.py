"""Synthetic grids of the BASELINE.json shapes.

The reference ships no PEGASE / ACTIVSg case files; its tests build
PEGASE-*shaped* grids with ``random_network`` (reference
``pkg/tests/conftest.py:52-107``, used for 2869 bus / 4582 branch at
``pkg/tests/test_measurement.py:183-194``).  ``random_network`` here draws
from ``numpy.random.default_rng(seed)`` in the same sequence, so a
``(n_bus, seed, extra_frac)`` triple names the same grid in both packages
(checked by ``tests/test_host_api.py`` against a golden fingerprint).

``tiled_network`` builds the ~100k-bus configuration of SURVEY.md section 8(d):
relabelled copies of one grid chained by tie branches, with an explicit
``area_of_bus`` (the reference partitioner is O(n^2) and unusable there).
"""

from __future__ import annotations

import json
import os

import numpy as np

from .network import Branch, Bus, BusBranchNetwork

SHAPES = {
    # name: (n_bus, n_branch, areas)
    "pegase2869": (2869, 4582, 8),
    "pegase9241": (9241, 16049, 16),
    "activsg10k": (10000, 12706, 32),
}


def random_network(n_bus, seed, extra_frac=0.45):
    """Random connected near-banded grid; bus 0 is the slack with angle 0."""
    rng = np.random.default_rng(seed)
    edges, taken = [], set()
    for i in range(1, n_bus):
        parent = max(0, i - 1 - int(rng.integers(0, 4)))
        edges.append((parent, i))
        taken.add((parent, i))
    target_edges = n_bus - 1 + int(extra_frac * n_bus)
    while len(edges) < target_edges:
        a = int(rng.integers(n_bus))
        b = a + int(rng.integers(2, 12))
        if b >= n_bus or (a, b) in taken:
            continue
        taken.add((a, b))
        edges.append((a, b))

    va = rng.uniform(-0.12, 0.12, size=n_bus)
    va[0] = 0.0
    vm = rng.uniform(0.96, 1.05, size=n_bus)
    buses = []
    for i in range(n_bus):
        gs = float(rng.uniform(0, 0.02)) if rng.random() < 0.1 else 0.0
        bs = float(rng.uniform(-0.1, 0.15)) if rng.random() < 0.1 else 0.0
        buses.append(Bus(id=i + 1, is_slack=(i == 0), gs=gs, bs=bs,
                         vm_true=float(vm[i]), va_true=float(va[i])))
    branches = []
    for f, t in edges:
        x = float(rng.uniform(0.02, 0.2))
        r = float(x * rng.uniform(0.1, 0.4))
        bc = float(rng.uniform(0.0, 0.04))
        tap = float(rng.uniform(0.95, 1.05)) if rng.random() < 0.1 else 1.0
        shift = float(rng.uniform(-0.05, 0.05)) if rng.random() < 0.05 else 0.0
        branches.append(Branch(from_bus=f, to_bus=t, r=r, x=x, b_charging=bc, tap=tap,
                               shift=shift))
    return BusBranchNetwork.from_components(buses, branches)


def shaped_network(name):
    """One of the named PEGASE / ACTIVSg shapes."""
    n_bus, n_branch, _ = SHAPES[name]
    return random_network(n_bus, seed=n_bus, extra_frac=(n_branch - (n_bus - 1)) / n_bus)


def tiled_network(base: BusBranchNetwork, copies: int, ties_per_seam: int = 3):
    """``copies`` relabelled copies of ``base`` chained end to end.

    Copy c's bus i becomes bus ``c*n + i``; only copy 0 keeps the slack.
    Consecutive copies are joined by ``ties_per_seam`` tie branches between
    the tail of one copy and the head of the next (deterministic parameters).
    Returns (network, copy_of_bus).
    """
    n = base.n_bus
    buses, branches = [], []
    for c in range(copies):
        for i, b in enumerate(base.buses):
            buses.append(Bus(id=c * n + i + 1, base_kv=b.base_kv, gs=b.gs, bs=b.bs,
                             is_slack=(b.is_slack and c == 0), vm_true=b.vm_true,
                             va_true=b.va_true))
        for br in base.branches:
            branches.append(Branch(from_bus=c * n + br.from_bus, to_bus=c * n + br.to_bus,
                                   r=br.r, x=br.x, b_charging=br.b_charging, tap=br.tap,
                                   shift=br.shift))
        if c:
            for j in range(ties_per_seam):
                branches.append(Branch(from_bus=c * n - 1 - 2 * j, to_bus=c * n + 2 * j,
                                       r=0.01 + 0.002 * j, x=0.08 + 0.01 * j,
                                       b_charging=0.02))
    net = BusBranchNetwork.from_components(buses, branches)
    return net, np.repeat(np.arange(copies), n)


def tile_partition(base_area_of_bus, copies):
    """Area assignment of a tiled grid: copy c's areas are offset by c*k."""
    base = np.asarray(base_area_of_bus, dtype=int)
    k = int(base.max()) + 1
    return np.concatenate([base + c * k for c in range(copies)])


def golden_partition(name):
    """Committed ``area_of_bus`` produced once by the reference partitioner
    (``tests/golden/make_golden.py``); None when no fixture exists."""
    here = os.path.dirname(os.path.abspath(__file__))
    path = os.path.join(here, "cases", f"part_{name}.json")
    if not os.path.exists(path):
        return None
    with open(path) as fh:
        return np.asarray(json.load(fh)["area_of_bus"], dtype=int)
