"""Area partitioning and boundary / per-area variable maps (host side, once).

API mirror of the reference's ``gridse.partition`` (reference
``pkg/src/gridse/partition.py:23-559``).  ``build_variable_maps`` defines every
index layout the device plan consumes:

* x_Gamma = boundary-bus angles sorted by bus (slack angle absent), then
  magnitudes (reference ``partition.py:489-492``);
* area-local variables = interior ``[theta(internal \\ slack) | V(internal)]``
  followed by boundary ``[theta(lb \\ slack) | V(lb)]`` where ``lb`` is the
  area's own boundary buses plus tie-line far ends (reference
  ``partition.py:494-537``).

``partition_network`` reproduces the reference partitioner's decisions
(seeded farthest-point seeds, smallest-first growth, Lloyd re-centering,
balance / cut refinement, k+1 merge candidates and the (balanced, cuts)
selection key; reference ``partition.py:128-424``) so the same seed yields
the same ``area_of_bus``; it is not accelerated (feed the same ``Partition`` to
oracle and GPU).
"""

from __future__ import annotations

import json
from collections import deque
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp
from scipy.sparse import csgraph

from .network import BusBranchNetwork


class PartitionError(ValueError):
    pass


@dataclass(frozen=True)
class Partition:
    k: int
    area_of_bus: np.ndarray
    cut_branches: np.ndarray
    boundary_buses: np.ndarray
    area_pairs: dict

    def buses_of_area(self, a):
        return np.flatnonzero(self.area_of_bus == a)


@dataclass(frozen=True)
class BoundaryOrdering:
    """Global boundary vector layout: angle block, then magnitude block."""

    entries: tuple
    angle_slot: dict
    mag_slot: dict

    @property
    def n_gamma(self):
        return len(self.entries)

    @property
    def angle_buses(self):
        return np.array([b for b, q in self.entries if q == "va"], dtype=int)

    @property
    def mag_buses(self):
        return np.array([b for b, q in self.entries if q == "vm"], dtype=int)

    def gather(self, va, vm):
        return np.concatenate([va[self.angle_buses], vm[self.mag_buses]])

    def apply_delta(self, va, vm, delta):
        ab, mb = self.angle_buses, self.mag_buses
        va[ab] += delta[: len(ab)]
        vm[mb] += delta[len(ab):]


@dataclass(frozen=True)
class AreaVariableMap:
    """Local variable layout of one area: interior block then boundary block."""

    area: int
    internal_buses: np.ndarray
    local_boundary_buses: np.ndarray
    owned_buses: frozenset
    interior_angle_buses: np.ndarray
    interior_mag_buses: np.ndarray
    interior_angle_slot: dict
    interior_mag_slot: dict
    boundary_angle_slot: dict
    boundary_mag_slot: dict
    boundary_selector: np.ndarray
    slack: int

    @property
    def n_interior(self):
        return len(self.interior_angle_buses) + len(self.interior_mag_buses)

    @property
    def n_boundary(self):
        return len(self.boundary_selector)

    def local_index(self, bus, quant):
        if quant == "va":
            inner, outer = self.interior_angle_slot, self.boundary_angle_slot
        else:
            inner, outer = self.interior_mag_slot, self.boundary_mag_slot
        hit = inner.get(bus)
        return hit if hit is not None else self.n_interior + outer[bus]

    def gather_interior(self, va, vm):
        return np.concatenate([va[self.interior_angle_buses], vm[self.interior_mag_buses]])

    def apply_interior_delta(self, va, vm, delta):
        na = len(self.interior_angle_buses)
        va[self.interior_angle_buses] += delta[:na]
        vm[self.interior_mag_buses] += delta[na:]

    def local_boundary_angle_buses(self):
        return np.array([b for b in self.local_boundary_buses if b != self.slack], dtype=int)


# ---------------------------------------------------------------------------
# Partitioner
# ---------------------------------------------------------------------------

class _Grid:
    """Adjacency lists + branch end arrays shared by the partitioner passes."""

    def __init__(self, net):
        self.n = net.n_bus
        self.nbrs = [net.neighbors(u) for u in range(self.n)]
        self.f = np.array([br.from_bus for br in net.branches], dtype=int)
        self.t = np.array([br.to_bus for br in net.branches], dtype=int)
        if len(self.f):
            ones = np.ones(2 * len(self.f))
            self.csr = sp.csr_matrix(
                (ones, (np.concatenate([self.f, self.t]), np.concatenate([self.t, self.f]))),
                shape=(self.n, self.n))
        else:
            self.csr = sp.csr_matrix((self.n, self.n))
        self._flat = None

    def flat(self):
        """int32 CSR of ``nbrs`` (same neighbor order) + branch ends, for the native passes."""
        if self._flat is None:
            ptr = np.zeros(self.n + 1, dtype=np.int32)
            ptr[1:] = np.cumsum([len(x) for x in self.nbrs])
            idx = np.fromiter((v for x in self.nbrs for v in x), dtype=np.int32, count=int(ptr[-1]))
            self._flat = (ptr, idx, np.ascontiguousarray(self.f, dtype=np.int32),
                          np.ascontiguousarray(self.t, dtype=np.int32))
        return self._flat

    def hop_distance(self, sources):
        dist = np.full(self.n, -1, dtype=int)
        q = deque(sources)
        for s in sources:
            dist[s] = 0
        while q:
            u = q.popleft()
            for v in self.nbrs[u]:
                if dist[v] < 0:
                    dist[v] = dist[u] + 1
                    q.append(v)
        return dist

    def stays_connected(self, area, a, without=None):
        """Is area ``a`` minus bus ``without`` non-empty and connected?"""
        members = np.flatnonzero(area == a)
        if without is not None:
            members = members[members != without]
        if members.size == 0:
            return False
        start = int(members[0])
        seen = {start}
        todo = [start]
        nbrs = self.nbrs
        while todo:
            u = todo.pop()
            for v in nbrs[u]:
                if v != without and area[v] == a and v not in seen:
                    seen.add(v)
                    todo.append(v)
        return len(seen) == members.size

    def components(self, area, a):
        left = {int(u) for u in np.flatnonzero(area == a)}
        out = []
        while left:
            start = min(left)
            seen = {start}
            todo = [start]
            while todo:
                u = todo.pop()
                for v in self.nbrs[u]:
                    if v not in seen and area[v] == a:
                        seen.add(v)
                        todo.append(v)
            out.append(seen)
            left -= seen
        return out

    def cut_count(self, area):
        return int(np.count_nonzero(area[self.f] != area[self.t])) if len(self.f) else 0


def _seed_buses(g, k, seed):
    rng = np.random.default_rng(seed)
    seeds = [int(rng.integers(g.n))]
    while len(seeds) < k:
        dist = g.hop_distance(seeds)
        seeds.append(int(np.flatnonzero(dist == dist.max())[0]))
    return seeds


def _grow(g, seeds):
    """Multi-source growth: the currently smallest area claims one bus per turn."""
    k = len(seeds)
    area = np.full(g.n, -1, dtype=int)
    size = [1] * k
    for a, s in enumerate(seeds):
        area[s] = a
    fronts = [deque(v for v in g.nbrs[s] if area[v] == -1) for s in seeds]
    unclaimed = g.n - k
    live = set(range(k))
    while unclaimed and live:
        a = min(live, key=lambda i: (size[i], i))
        q = fronts[a]
        claimed = False
        while q:
            u = q.popleft()
            if area[u] != -1:
                continue
            area[u] = a
            size[a] += 1
            unclaimed -= 1
            q.extend(v for v in g.nbrs[u] if area[v] == -1)
            claimed = True
            break
        if not claimed:
            live.discard(a)
    if unclaimed:
        starved = min(range(k), key=lambda i: size[i])
        raise PartitionError(
            f"partition infeasible: area {starved} starved with {size[starved]} bus(es) "
            f"while {unclaimed} remain unassigned")
    return area


def _center_of(g, area, a):
    """Minimum-eccentricity bus of the induced subgraph (ties: lowest index)."""
    members = np.flatnonzero(area == a)
    if members.size == 1:
        return int(members[0])
    sub = g.csr[members][:, members]
    dist = csgraph.shortest_path(sub, method="D", unweighted=True)
    dist[~np.isfinite(dist)] = -1.0
    ecc = dist.max(axis=1)
    return int(members[int(np.argmin(ecc))])


def _balance_pass(g, area, k, max_passes=12):
    size = np.bincount(area, minlength=k).astype(int)
    for _ in range(max_passes):
        moved = False
        for u in range(g.n):
            a = int(area[u])
            if size[a] <= 1:
                continue
            options = [b for b in sorted({int(area[v]) for v in g.nbrs[u]} - {a})
                       if size[a] > size[b] + 1]
            if not options:
                continue
            b = min(options, key=lambda i: (size[i], i))
            if not g.stays_connected(area, a, without=u):
                continue
            area[u] = b
            size[a] -= 1
            size[b] += 1
            moved = True
        if not moved:
            break
    return area


def _push_one(g, area, a, b, size):
    for u in range(g.n):
        if area[u] != a or size[a] <= 1:
            continue
        if not any(area[v] == b for v in g.nbrs[u]):
            continue
        if g.stays_connected(area, a, without=u):
            area[u] = b
            size[a] -= 1
            size[b] += 1
            return True
    return False


def _cascade(g, area, k, target_ratio=2.0):
    """Drain the largest area toward the smallest along the area graph."""
    size = np.bincount(area, minlength=k).astype(int)
    for _ in range(2 * g.n):
        if size.max() <= target_ratio * size.min() and \
                size.max() - size.min() <= max(2, size.min()):
            break
        big, small = int(np.argmax(size)), int(np.argmin(size))
        link = {i: set() for i in range(k)}
        for x, y in zip(area[g.f], area[g.t]):
            if x != y:
                link[int(x)].add(int(y))
                link[int(y)].add(int(x))
        came_from = {big: None}
        q = deque([big])
        while q and small not in came_from:
            u = q.popleft()
            for v in sorted(link[u]):
                if v not in came_from:
                    came_from[v] = u
                    q.append(v)
        if small not in came_from:
            break
        route = []
        node = small
        while node is not None:
            route.append(node)
            node = came_from[node]
        route.reverse()
        if not all(_push_one(g, area, x, y, size) for x, y in zip(route, route[1:])):
            break
    return area


def _thin_cuts_py(g, area, k, max_passes=6):
    size = np.bincount(area, minlength=k).astype(int)
    cap = 2 * int(size.min())
    for _ in range(max_passes):
        moved = False
        for u in range(g.n):
            a = int(area[u])
            if size[a] <= 1:
                continue
            nb_area = [int(area[v]) for v in g.nbrs[u]]
            here = nb_area.count(a)
            pick, pick_gain = None, 0
            for b in sorted(set(nb_area) - {a}):
                gain = nb_area.count(b) - here
                if gain > pick_gain and size[b] + 1 <= cap and size[a] - 1 >= 1:
                    pick, pick_gain = b, gain
            if pick is None or not g.stays_connected(area, a, without=u):
                continue
            area[u] = pick
            size[a] -= 1
            size[pick] += 1
            cap = 2 * int(size.min())
            moved = True
        if not moved:
            break
    return area


def _attempt_py(g, k, seed):
    seeds = _seed_buses(g, k, seed)
    area = _grow(g, seeds)
    for _ in range(3):
        centers = [_center_of(g, area, a) for a in range(k)]
        if centers == seeds:
            break
        seeds = centers
        area = _grow(g, seeds)
    area = _balance_pass(g, area, k)
    area = _cascade(g, area, k)
    area = _balance_pass(g, area, k)
    return _thin_cuts_py(g, area, k)


def _native_passes():
    """The C++ restatement of the passes (csrc/partition.cpp) when the library is built; the Python
    passes above are the executable specification it is tested against and the fallback without it."""
    try:
        from . import _native
        return _native.lib()
    except Exception:
        return None


def _i32p(a):
    import ctypes as C
    return a.ctypes.data_as(C.POINTER(C.c_int32))


def _attempt(g, k, seed):
    L = _native_passes()
    if L is None:
        return _attempt_py(g, k, seed)
    ptr, idx, f, t = g.flat()
    first = int(np.random.default_rng(seed).integers(g.n))       # the one random draw (as in _seed_buses)
    area = np.zeros(g.n, dtype=np.int32)
    info = np.zeros(3, dtype=np.int32)
    rc = L.gse_partition_attempt(g.n, _i32p(ptr), _i32p(idx), len(f), _i32p(f), _i32p(t), int(k), first,
                                 _i32p(area), _i32p(info))
    if rc:
        raise PartitionError(
            f"partition infeasible: area {int(info[0])} starved with {int(info[1])} bus(es) "
            f"while {int(info[2])} remain unassigned")
    return area.astype(int)


def _thin_cuts(g, area, k, max_passes=6):
    L = _native_passes()
    if L is None or max_passes != 6:
        return _thin_cuts_py(g, area, k, max_passes)
    ptr, idx, f, t = g.flat()
    out = np.ascontiguousarray(area, dtype=np.int32)
    L.gse_partition_thin_cuts(g.n, _i32p(ptr), _i32p(idx), len(f), _i32p(f), _i32p(t), int(k), _i32p(out))
    return out.astype(int)


def _merged_variants(g, area, k_fine):
    out = []
    touching = sorted({(min(int(x), int(y)), max(int(x), int(y)))
                       for x, y in zip(area[g.f], area[g.t]) if x != y})
    for a, b in touching:
        merged = area.copy()
        merged[merged == b] = a
        _, merged = np.unique(merged, return_inverse=True)
        merged = merged.astype(int)
        size = np.bincount(merged, minlength=k_fine - 1)
        if size.max() / size.min() > 2.0:
            continue
        out.append(_thin_cuts(g, merged, k_fine - 1))
    return out


def _describe(net, area_of_bus, k):
    area = np.asarray(area_of_bus, dtype=int)
    cut, pairs = [], {}
    for e, br in enumerate(net.branches):
        af, at = int(area[br.from_bus]), int(area[br.to_bus])
        if af != at:
            cut.append(e)
            key = (min(af, at), max(af, at))
            pairs[key] = pairs.get(key, 0) + 1
    ends = {net.branches[e].from_bus for e in cut} | {net.branches[e].to_bus for e in cut}
    return Partition(k=k, area_of_bus=area, cut_branches=np.asarray(cut, dtype=int),
                     boundary_buses=np.asarray(sorted(ends), dtype=int), area_pairs=pairs)


def partition_network(net: BusBranchNetwork, k: int, seed: int = 0) -> Partition:
    """Split into k connected areas; deterministic per seed."""
    if not 1 <= k <= net.n_bus:
        raise PartitionError(f"k={k} outside 1..{net.n_bus}")
    if k == 1:
        return _describe(net, np.zeros(net.n_bus, dtype=int), 1)
    g = _Grid(net)
    pool = [_attempt(g, k, seed + 7919 * a) for a in range(3)]
    if k + 1 <= net.n_bus:
        for a in range(2):
            pool.extend(_merged_variants(g, _attempt(g, k + 1, seed + 7919 * a), k + 1))
    best, best_key = None, None
    for area in pool:
        size = np.bincount(area, minlength=k)
        if len(size) != k or size.min() == 0:
            continue
        key = (size.max() / size.min() > 2.0, g.cut_count(area))
        if best_key is None or key < best_key:
            best, best_key = area, key
    part = _describe(net, best, k)
    validate_partition(net, part)
    return part


def load_partition(net: BusBranchNetwork, area_of_bus) -> Partition:
    area = np.asarray(area_of_bus, dtype=int)
    if area.shape != (net.n_bus,):
        raise PartitionError(
            f"assignment covers {area.shape[0] if area.ndim else 0} buses, "
            f"network has {net.n_bus}")
    if area.min() < 0:
        raise PartitionError("negative area index")
    part = _describe(net, area, int(area.max()) + 1)
    validate_partition(net, part)
    return part


def validate_partition(net, part):
    size = np.bincount(part.area_of_bus, minlength=part.k)
    # one labelled component sweep over the intra-area graph covers all areas
    arr = net.branch_arrays() if net.n_branch else None
    if arr is not None:
        keep = part.area_of_bus[arr["from"]] == part.area_of_bus[arr["to"]]
        f, t = arr["from"][keep], arr["to"][keep]
        graph = sp.csr_matrix((np.ones(len(f)), (f, t)), shape=(net.n_bus, net.n_bus))
    else:
        graph = sp.csr_matrix((net.n_bus, net.n_bus))
    n_comp, label = csgraph.connected_components(graph, directed=False)
    if n_comp == part.k and size.min() > 0:
        return
    for a in range(part.k):
        if size[a] == 0:
            raise PartitionError(f"area {a} is empty")
        if len(np.unique(label[part.area_of_bus == a])) > 1:
            comps = _Grid(net).components(part.area_of_bus, a)
            raise PartitionError(
                f"area {a} is disconnected: components "
                + ", ".join(str(sorted(net.buses[u].id for u in c)) for c in comps))


# ---------------------------------------------------------------------------
# Variable maps
# ---------------------------------------------------------------------------

def build_variable_maps(net: BusBranchNetwork, part: Partition):
    """(BoundaryOrdering, [AreaVariableMap per area])."""
    slack = net.slack
    area_of = part.area_of_bus
    boundary = [int(b) for b in part.boundary_buses]
    on_boundary = np.zeros(net.n_bus, dtype=bool)
    on_boundary[boundary] = True

    entries = [(b, "va") for b in boundary if b != slack] + [(b, "vm") for b in boundary]
    angle_slot = {b: i for i, (b, q) in enumerate(entries) if q == "va"}
    mag_slot = {b: i for i, (b, q) in enumerate(entries) if q == "vm"}
    bord = BoundaryOrdering(entries=tuple(entries), angle_slot=angle_slot, mag_slot=mag_slot)

    touched = [set() for _ in range(part.k)]
    for b in boundary:
        touched[int(area_of[b])].add(b)
    for e in part.cut_branches:
        br = net.branches[int(e)]
        touched[int(area_of[br.from_bus])].add(br.to_bus)
        touched[int(area_of[br.to_bus])].add(br.from_bus)

    maps = []
    for a in range(part.k):
        owned = np.flatnonzero(area_of == a)
        internal = owned[~on_boundary[owned]].astype(int)
        lb = np.array(sorted(touched[a]), dtype=int)
        ang_in = internal[internal != slack]
        lb_ang = [int(u) for u in lb if u != slack]
        lb_mag = [int(u) for u in lb]
        maps.append(AreaVariableMap(
            area=a,
            internal_buses=internal,
            local_boundary_buses=lb,
            owned_buses=frozenset(int(u) for u in owned),
            interior_angle_buses=ang_in,
            interior_mag_buses=internal,
            interior_angle_slot={int(u): i for i, u in enumerate(ang_in)},
            interior_mag_slot={int(u): len(ang_in) + i for i, u in enumerate(internal)},
            boundary_angle_slot={u: i for i, u in enumerate(lb_ang)},
            boundary_mag_slot={u: len(lb_ang) + i for i, u in enumerate(lb_mag)},
            boundary_selector=np.array(
                [angle_slot[u] for u in lb_ang] + [mag_slot[u] for u in lb_mag], dtype=int),
            slack=slack,
        ))
    return bord, maps


# ---------------------------------------------------------------------------
# Partition files
# ---------------------------------------------------------------------------

def write_partition_file(part: Partition, path):
    with open(path, "w") as fh:
        json.dump({"k": part.k, "area_of_bus": [int(a) for a in part.area_of_bus]}, fh)
        fh.write("\n")


def read_partition_file(net: BusBranchNetwork, path) -> Partition:
    with open(path) as fh:
        doc = json.load(fh)
    part = load_partition(net, doc["area_of_bus"])
    if "k" in doc and int(doc["k"]) != part.k:
        raise PartitionError(
            f"partition file declares k={doc['k']} but assignment uses {part.k} areas")
    return part
