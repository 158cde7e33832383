"""Host-side API mirror (network / measurement / partition / maps): the reference's own known
answers (tests/test_network.py, test_partition.py, test_measurement.py of the reference) plus
fingerprints of the synthetic BASELINE shapes.  CPU only."""

import hashlib
import json
import os

import numpy as np
import pytest

import paper_2604_23175_b200 as G
from paper_2604_23175_b200 import synth
from conftest import load_golden, make_path4

MIN_CASE = """function mpc = min2
mpc.version = '2';
mpc.baseMVA = 100;
mpc.bus = [
1 3 0 0 0 0 1 1.0 0 138 1 1.06 0.94;
2 1 0 0 0 0 1 0.9 0 138 1 1.06 0.94;
];
mpc.gen = [
1 0 0 10 -10 1.0 100 1 50 0;
];
mpc.branch = [
1 2 0 0.1 0 9900 0 0 0 0 1 -360 360;
];
"""


def test_matpower_subset_and_errors():
    net = G.parse_case(MIN_CASE, "matpower-m")
    assert (net.n_bus, net.n_branch, net.slack, net.buses[1].vm_true) == (2, 1, 0, 0.9)
    assert np.allclose(G.build_ybus(net).toarray(), np.array([[-10j, 10j], [10j, -10j]]), atol=1e-12)
    with pytest.raises(G.CaseError, match="unknown bus reference"):
        G.parse_case(MIN_CASE.replace("1 2 0 0.1", "1 99 0 0.1"), "matpower-m")
    with pytest.raises(G.CaseError, match="line"):
        G.parse_case(MIN_CASE.replace("2 1 0 0", "2 oops 0 0"), "matpower-m")
    with pytest.raises(G.CaseError, match="zero slack"):
        G.parse_case(MIN_CASE.replace("1 3 0", "1 1 0"), "matpower-m")
    with pytest.raises(G.CaseError, match="multiple slack"):
        G.parse_case(MIN_CASE.replace("2 1 0 0 0 0", "2 3 0 0 0 0"), "matpower-m")


def test_ybus_tap_and_shunt():
    buses = [G.Bus(id=1, is_slack=True), G.Bus(id=2)]
    net = G.BusBranchNetwork.from_components(buses, [G.Branch(from_bus=0, to_bus=1, r=0.0, x=0.1, tap=2.0)])
    y = G.build_ybus(net).toarray()
    assert y[0, 0] == pytest.approx(-2.5j, rel=1e-12) and y[1, 1] == pytest.approx(-10j, rel=1e-12)
    assert y[0, 1] == pytest.approx(5j, rel=1e-12)
    net = G.BusBranchNetwork.from_components([G.Bus(id=1, is_slack=True, gs=0.5), G.Bus(id=2)], [])
    assert np.allclose(G.build_ybus(net).toarray(), np.diag([0.5, 0.0]), atol=0)


def test_cases_and_json_round_trip(cases_dir):
    net14 = G.load_case(os.path.join(cases_dir, "ieee14.m"))
    assert (net14.n_bus, net14.n_branch, net14.buses[net14.slack].id) == (14, 20, 1)
    again = G.parse_case(G.to_native_json(net14), "native-json")
    assert np.array_equal(again.ybus.toarray(), net14.ybus.toarray())
    p4 = G.load_case(os.path.join(cases_dir, "path4.json"))
    assert p4.n_bus == 4 and p4.n_branch == 3


def test_partition_goldens(cases_dir):
    # reference tests/test_partition.py:19-25,47
    p4 = make_path4()
    for seed in range(4):
        part = G.partition_network(p4, 2, seed=seed)
        assert sorted(part.cut_branches) == [1] and list(part.boundary_buses) == [1, 2]
    net14 = G.load_case(os.path.join(cases_dir, "ieee14.m"))
    part = G.partition_network(net14, 3, seed=0)
    assert list(part.area_of_bus) == [2, 2, 2, 2, 2, 0, 1, 1, 1, 1, 0, 0, 0, 0]
    net118 = G.load_case(os.path.join(cases_dir, "ieee118.m"))
    a, b = G.partition_network(net118, 6, seed=3), G.partition_network(net118, 6, seed=3)
    assert np.array_equal(a.area_of_bus, b.area_of_bus)
    # the partitions stored in the golden fixtures were produced by the reference partitioner
    for name, k, seed in (("ieee118_k6", 6, 0), ("ieee118_k3", 3, 0)):
        assert np.array_equal(G.partition_network(net118, k, seed=seed).area_of_bus, load_golden(name)["area_of_bus"])
    with pytest.raises(G.PartitionError):
        G.partition_network(p4, 5)
    with pytest.raises(G.PartitionError, match="disconnected"):
        G.load_partition(p4, [0, 1, 0, 1])


def test_native_partition_passes_equal_the_python_passes():
    """csrc/partition.cpp restates the passes of one attempt; the Python passes are its executable
    specification: same areas bus for bus (or the same PartitionError) on random grids, and the big
    shapes reproduce the partitions the reference partitioner itself produced (hundreds of seconds there)."""
    from paper_2604_23175_b200 import partition as P, synth
    assert P._native_passes() is not None, "libgridse_b200.so must be built (python -c 'import __graft_entry__ as g; g.build()')"
    for n, seed, k in [(30, 1, 3), (60, 2, 4), (120, 3, 5), (200, 4, 7), (333, 5, 6), (50, 6, 10), (90, 7, 2), (40, 9, 39)]:
        net = synth.random_network(n, seed, 0.3)
        g = P._Grid(net)
        for s in (0, 1, 7919):
            outs = []
            for fn in (P._attempt, P._attempt_py):
                try:
                    outs.append(fn(g, k, s).tolist())
                except P.PartitionError as exc:
                    outs.append(str(exc))
            assert outs[0] == outs[1], (n, seed, k, s)
            if not isinstance(outs[0], str) and k > 2:
                merged = np.array(outs[0])
                merged[merged == k - 1] = k - 2          # not necessarily connected: the pass only needs sizes >= 1
                assert np.array_equal(P._thin_cuts(g, merged.copy(), k - 1), P._thin_cuts_py(g, merged.copy(), k - 1))
    net = synth.shaped_network("pegase2869")
    assert np.array_equal(G.partition_network(net, 8, seed=0).area_of_bus, synth.golden_partition("pegase2869"))


def test_variable_map_layouts():
    # reference tests/test_partition.py:98-121
    p4 = make_path4()
    bord, maps = G.build_variable_maps(p4, G.load_partition(p4, [0, 0, 1, 1]))
    assert bord.entries == ((1, "va"), (2, "va"), (1, "vm"), (2, "vm")) and bord.n_gamma == 4
    for m in maps:
        assert list(m.local_boundary_buses) == [1, 2] and list(m.boundary_selector) == [0, 1, 2, 3]
    assert list(maps[0].internal_buses) == [0] and list(maps[1].internal_buses) == [3]
    assert 0 not in maps[0].interior_angle_slot
    net = make_path4(slack_pos=1)
    bord, maps = G.build_variable_maps(net, G.load_partition(net, [0, 0, 1, 1]))
    assert bord.n_gamma == 3 and (1, "va") not in bord.entries
    part = G.partition_network(p4, 1)
    bord, maps = G.build_variable_maps(p4, part)
    assert bord.n_gamma == 0 and maps[0].n_boundary == 0 and maps[0].n_interior == 2 * p4.n_bus - 1


def test_measurement_model(cases_dir):
    # reference tests/test_measurement.py:64-77,146-150 and masking semantics
    net14 = G.load_case(os.path.join(cases_dir, "ieee14.m"))
    ms = G.generate_measurements(net14)
    assert ms.m == 3 * 14 + 4 * 20 == 122
    buses = [G.Bus(id=1, is_slack=True), G.Bus(id=2)]
    net = G.BusBranchNetwork.from_components(buses, [G.Branch(from_bus=0, to_bus=1, r=0.0, x=0.1)])
    st = G.StateVector(va=np.array([0.0, 0.0]), vm=np.array([1.0, 0.9]))
    assert G.eval_h(net, G.MeasurementType.QF, 0, st) == pytest.approx(1.0)
    assert G.eval_h(net, G.MeasurementType.PF, 0, st) + G.eval_h(net, G.MeasurementType.PT, 0, st) == pytest.approx(0.0, abs=1e-12)
    masked = G.apply_mask(ms, G.MeasurementType.PF)
    assert masked.m == ms.m and np.all(masked.weight[masked.mtype == 3] == 0.0)
    assert np.array_equal(G.clear_mask(masked).weight, ms.weight)
    w = G.make_measurement_set(net14, [0], [0], [1.0], [0.0]).weight
    assert w[0] == 1.0      # sigma == 0 -> unit weight
    # analytic gradient vs central differences for every type
    rng = np.random.default_rng(0)
    state = G.StateVector(va=rng.uniform(-0.1, 0.1, 14), vm=rng.uniform(0.95, 1.05, 14))
    for r in rng.choice(ms.m, 25, replace=False):
        for (bus, quant), val in G.eval_row_gradient(net14, ms.mtype[r], ms.target[r], state):
            hi, lo = state.copy(), state.copy()
            arr_hi, arr_lo = (hi.va, lo.va) if quant == "va" else (hi.vm, lo.vm)
            arr_hi[bus] += 1e-6
            arr_lo[bus] -= 1e-6
            fd = (G.eval_h(net14, ms.mtype[r], ms.target[r], hi) - G.eval_h(net14, ms.mtype[r], ms.target[r], lo)) / 2e-6
            assert val == pytest.approx(fd, abs=1e-6)


def test_synthetic_shapes_match_the_golden_recipes():
    # PEGASE-2869 shape: 2869 bus / 4582 branch / 26,935 rows (reference test_measurement.py:183-194)
    net = synth.shaped_network("pegase2869")
    ms = G.generate_measurements(net, G.MeasurementConfig(seed=0))
    assert (net.n_bus, net.n_branch, ms.m) == (2869, 4582, 26935)
    g = load_golden("pegase2869_k8")
    assert np.array_equal(ms.z, g["z"])          # same RNG stream, same h(x_true): bit-identical inputs
    assert np.array_equal(synth.golden_partition("pegase2869"), g["area_of_bus"])
    part = G.load_partition(net, g["area_of_bus"])
    bord, _ = G.build_variable_maps(net, part)
    assert bord.n_gamma == int(g["n_gamma"]) == 126


def test_tiled_100k_inputs_match_the_reference_fixture():
    """The ~100k-bus / 128-area fixture (reference run, make_golden.py tiled101k) was generated from the
    reference's own classes: the product's tiled_network / generate_measurements must name the same grid
    and the same measurement set (Ybus and z / w fingerprints), and the committed partition the same areas."""
    g = load_golden("tiled101k_k128")
    net, _ = synth.tiled_network(synth.shaped_network("pegase9241"), 11)
    y = net.ybus
    ys = g["ybus_sum"]
    assert y.nnz == int(ys[3])
    assert abs(y.data.real.sum() - ys[0]) <= 1e-12 * ys[2] and abs(y.data.imag.sum() - ys[1]) <= 1e-12 * ys[2]
    assert abs(np.abs(y.data).sum() - ys[2]) <= 1e-12 * ys[2]
    ms = G.generate_measurements(net, G.MeasurementConfig(seed=0))
    zs = g["z_sum"]
    assert ms.m == 1011229
    assert abs(ms.z.sum() - zs[0]) <= 1e-12 * zs[1] and abs(np.abs(ms.z).sum() - zs[1]) <= 1e-12 * zs[1]
    assert np.array_equal(synth.golden_partition("tiled101k_k128"), g["area_of_bus"])
    part = G.load_partition(net, g["area_of_bus"])
    bord, _ = G.build_variable_maps(net, part)
    assert part.k == 128 and bord.n_gamma == int(g["n_gamma"]) == 5692
    assert int(g["iterations"]) == 5 and bool(g["converged"])


def test_tiled_network_for_the_100k_config():
    base = synth.random_network(60, 5)
    net, copy_of = synth.tiled_network(base, 3)
    assert net.n_bus == 180 and net.n_branch == 3 * base.n_branch + 2 * 3
    area = synth.tile_partition(G.partition_network(base, 2, seed=0).area_of_bus, 3)
    part = G.load_partition(net, area)
    assert part.k == 6 and len(part.cut_branches) > 0
