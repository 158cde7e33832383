"""Command-line front end on the device solvers: the subcommands, flags and exit codes of the
reference's ``gridse`` console script (reference ``pkg/src/gridse/cli.py:30-198``).

    python -m paper_2604_23175_b200.cli run|sweep-k|mask|gen-measurements|partition|compare --case ...

Exit code 0 only when every requested run converged, 1 otherwise, 2 on a solver failure or bad
input.  ``--reuse-plan`` (extension) times warm solves on one device plan instead of rebuilding the
plan inside every solve.
"""

from __future__ import annotations

import argparse
import json
import sys

from . import harness as H
from .measurement import MeasurementConfig, generate_measurements, write_measurements
from .network import load_case
from .partition import build_variable_maps, partition_network, write_partition_file
from .solver import SolverError

COMMANDS = {}


def command(name, help_text, default_k=None, extra=None):
    def register(fn):
        COMMANDS[name] = (fn, help_text, default_k, extra)
        return fn
    return register


def _spec(args, method=None, default_k=None):
    k = int(args.k) if args.k not in (None, "") else None
    spec = H.ExperimentSpec(
        case_path=args.case, case_format=args.format, measurements_path=args.measurements,
        sigma_vm=args.sigma_vm, sigma_power=args.sigma_power, seed=args.seed, partition_path=args.partition,
        k=k, method=method or args.method, repeats=args.repeats, inner_gn_steps=args.inner_steps, tol=args.tol,
        max_iters=args.max_iters, deterministic=args.deterministic, reuse_plan=args.reuse_plan)
    if default_k and spec.method == "multiarea" and not (spec.partition_path or spec.k):
        spec.k = default_k
    return spec


def _emit(text, out):
    if out is None:
        sys.stdout.write(text)


@command("run", "repeated timed solve of one method", default_k=1)
def cmd_run(args):
    doc = H.run_experiment(_spec(args, default_k=1))
    _emit(H.write_run_report(doc, args.out, args.output_format), args.out)
    return 0 if doc["all_converged"] else 1


@command("sweep-k", "partition-count sweep (multi-area)")
def cmd_sweep_k(args):
    ks = [int(v) for v in str(args.k or "2,3,4,6").split(",")]
    args.k = None
    rows = H.sweep_k(_spec(args, method="multiarea"), ks)
    _emit(H.write_rows(rows, H.SWEEP_COLUMNS, args.out, args.output_format), args.out)
    return 0 if all(r["feasible"] and r["converged"] for r in rows) else 1


@command("mask", "flow-family masking study", default_k=1,
         extra=lambda p: p.add_argument("--families", default=None, help="comma list from {none,pf,pt,qf,qt}; default all"))
def cmd_mask(args):
    families = [f.strip() for f in args.families.split(",")] if args.families else None
    rows = H.mask_experiment(_spec(args, default_k=1), families)
    _emit(H.write_rows(rows, H.MASK_COLUMNS, args.out, args.output_format), args.out)
    return 0 if all(r["converged"] is True for r in rows) else 1


@command("gen-measurements", "write a synthetic measurement file")
def cmd_gen_measurements(args):
    if args.out is None:
        raise SystemExit("gen-measurements requires --out")
    ms = generate_measurements(load_case(args.case),
                               MeasurementConfig(sigma_vm=args.sigma_vm, sigma_power=args.sigma_power, seed=args.seed))
    write_measurements(ms, args.out)
    print(f"wrote {ms.m} rows to {args.out}")
    return 0


@command("partition", "partition a case and write the assignment")
def cmd_partition(args):
    net = load_case(args.case)
    part = partition_network(net, int(args.k or 2), seed=args.seed)
    bord, _ = build_variable_maps(net, part)
    if args.out:
        write_partition_file(part, args.out)
    print(json.dumps({"k": part.k, "cut_branches": len(part.cut_branches),
                      "boundary_buses": len(part.boundary_buses), "boundary_dim": bord.n_gamma}))
    return 0


@command("compare", "run both methods and diff the estimates")
def cmd_compare(args):
    spec = _spec(args)
    if not (spec.partition_path or spec.k):
        spec.k = 2
    doc = H.compare_methods(spec)
    text = json.dumps(doc, indent=1) + "\n"
    if args.out:
        with open(args.out, "w") as fh:
            fh.write(text)
    else:
        sys.stdout.write(text)
    return 0 if doc["all_converged"] else 1


def build_parser():
    ap = argparse.ArgumentParser(prog="gridse-b200",
                                 description="Multi-area WLS state estimation on B200: solvers and experiment tables.")
    sub = ap.add_subparsers(dest="command", required=True)
    for name, (fn, help_text, _, extra) in COMMANDS.items():
        p = sub.add_parser(name, help=help_text)
        p.add_argument("--case", required=True, help="case file (.m MATPOWER subset or .json)")
        p.add_argument("--format", choices=["matpower-m", "native-json"], default=None,
                       help="case format override (default: inferred from suffix)")
        p.add_argument("--measurements", default=None, help="measurement file (.json/.csv)")
        p.add_argument("--partition", default=None, help="partition file (JSON)")
        p.add_argument("--k", default=None, help="area count (sweep-k: comma list)")
        p.add_argument("--seed", type=int, default=0, help="noise and partitioner seed")
        p.add_argument("--repeats", type=int, default=11, help="solve repetitions; the first is excluded from means")
        p.add_argument("--method", choices=["centralized", "multiarea"], default="multiarea")
        p.add_argument("--inner-steps", type=int, default=1, dest="inner_steps")
        p.add_argument("--tol", type=float, default=1e-6)
        p.add_argument("--max-iters", type=int, default=10, dest="max_iters")
        p.add_argument("--deterministic", action=argparse.BooleanOptionalAction, default=True)
        p.add_argument("--reuse-plan", action=argparse.BooleanOptionalAction, default=False, dest="reuse_plan",
                       help="extension: build the device plan once and time warm solves")
        p.add_argument("--out", default=None, help="output path (default: stdout)")
        p.add_argument("--output-format", choices=["json", "csv"], default="json", dest="output_format")
        p.add_argument("--sigma-vm", type=float, default=0.01, dest="sigma_vm")
        p.add_argument("--sigma-power", type=float, default=0.02, dest="sigma_power")
        if extra:
            extra(p)
        p.set_defaults(fn=fn)
    return ap


def main(argv=None):
    args = build_parser().parse_args(argv)
    try:
        return args.fn(args)
    except SolverError as exc:
        print(f"solver failure: {exc}", file=sys.stderr)
        return 2
    except (OSError, ValueError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    raise SystemExit(main())
