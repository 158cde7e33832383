"""Shared test plumbing: markers, golden loader, case builders."""

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run with -m gpu on the B200 box)")


def load_golden(name):
    with np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def build_case(name):
    """(net, ms, part, golden) for a golden fixture, rebuilt from its recipe with the
    product's own host API (bit-identical to the reference's; tests/test_host_api.py)."""
    import paper_2604_23175_b200 as G
    from paper_2604_23175_b200 import synth

    g = load_golden(name)
    rec = json.loads(str(g["recipe"]))
    cases = os.path.join(ROOT, "paper_2604_23175_b200", "cases")
    if "case" in rec:
        net = G.load_case(os.path.join(cases, rec["case"]))
    elif rec["gen"].startswith("make_path4"):
        net = make_path4(slack_pos=1)
    else:
        # "random_network(n, seed[, extra_frac])" evaluated against the product's generator
        net = eval(rec["gen"], {"random_network": synth.random_network})
    if "sigma" in rec:
        cfg = G.MeasurementConfig(sigma_vm=rec["sigma"], sigma_power=rec["sigma"])
    else:
        cfg = G.MeasurementConfig(seed=rec["meas_seed"])
    ms = G.generate_measurements(net, cfg)
    if rec.get("mask"):
        ms = G.apply_mask(ms, G.MeasurementType[rec["mask"]])
    part = G.load_partition(net, g["area_of_bus"])
    return net, ms, part, g


def make_path4(slack_pos=0):
    import paper_2604_23175_b200 as G
    buses = [G.Bus(id=i + 1, is_slack=(i == slack_pos), vm_true=1.0 + 0.01 * i, va_true=-0.02 * i)
             for i in range(4)]
    branches = [G.Branch(from_bus=i, to_bus=i + 1, r=0.01, x=0.1, b_charging=0.02)
                for i in range(3)]
    return G.BusBranchNetwork.from_components(buses, branches)


SMALL_CASES = ["ieee14_k1", "ieee14_k2", "ieee14_k3", "ieee14_k14", "ieee118_k3", "ieee118_k6",
               "path4_slack_boundary", "rand300_k3_maskpf", "rand120_k4"]
BIG_CASES = ["pegase2869_k8", "pegase9241_k16", "activsg10k_k32"]


@pytest.fixture(scope="session")
def cases_dir():
    return os.path.join(ROOT, "paper_2604_23175_b200", "cases")
