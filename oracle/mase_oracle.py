"""ctypes front end of the CPU oracle (``oracle/mase_oracle.c``).

TEST INFRASTRUCTURE ONLY -- imported by ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs, never by the
product package.  The C file restates the reference's algorithm
(reference ``pkg/src/gridse/{assembly,linalg,solver,partition}.py``, citations
in the C header); parity is pinned by ``tests/test_oracle_golden.py`` against
fixtures generated from the unmodified reference (``tests/golden/make_golden.py``).

The wrapper is duck-typed: ``net`` needs ``ybus`` (scipy CSR complex),
``branches`` (objects with ``from_bus``, ``to_bus``, ``two_port()``), ``slack``,
``buses[slack].va_true``; ``ms`` needs ``mtype``, ``target``, ``z``, ``weight``.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

_i32p = C.POINTER(C.c_int32)
_f64p = C.POINTER(C.c_double)


class _Desc(C.Structure):
    _fields_ = [
        ("n_bus", C.c_int32), ("n_branch", C.c_int32), ("n_rows", C.c_int32),
        ("n_areas", C.c_int32), ("slack", C.c_int32), ("dense_threshold", C.c_int32),
        ("slack_va", C.c_double),
        ("y_ptr", _i32p), ("y_idx", _i32p), ("y_g", _f64p), ("y_b", _f64p),
        ("br_from", _i32p), ("br_to", _i32p), ("br_y", _f64p),
        ("m_type", _i32p), ("m_target", _i32p), ("m_z", _f64p), ("m_w", _f64p),
        ("area_of_bus", _i32p),
    ]


def build(force=False):
    """Compile the oracle with gcc (recipe: oracle/Makefile)."""
    so = os.path.join(_HERE, "libmase_oracle.so")
    src = os.path.join(_HERE, "mase_oracle.c")
    if force or not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
        subprocess.run(["make", "-C", _HERE, "-s"], check=True)
    return so


def _lib():
    global _LIB
    if _LIB is None:
        lib = C.CDLL(build())
        lib.orc_create.restype = C.c_void_p
        lib.orc_create.argtypes = [C.POINTER(_Desc)]
        lib.orc_n_gamma.argtypes = [C.c_void_p]
        lib.orc_area_dims.argtypes = [C.c_void_p, C.c_int, _i32p]
        lib.orc_area_int.restype = _i32p
        lib.orc_area_int.argtypes = [C.c_void_p, C.c_int, C.c_int]
        lib.orc_area_f64.restype = _f64p
        lib.orc_area_f64.argtypes = [C.c_void_p, C.c_int, C.c_int]
        lib.orc_gamma_f64.restype = _f64p
        lib.orc_gamma_f64.argtypes = [C.c_void_p, C.c_int]
        lib.orc_last_error.argtypes = [C.c_void_p, _i32p]
        lib.orc_local.argtypes = [C.c_void_p, _f64p, _f64p, C.c_int]
        lib.orc_assemble_only.argtypes = [C.c_void_p, _f64p, _f64p]
        lib.orc_boundary.argtypes = [C.c_void_p]
        lib.orc_recover.restype = C.c_double
        lib.orc_recover.argtypes = [C.c_void_p, _f64p, _f64p, C.c_int]
        lib.orc_objective.restype = C.c_double
        lib.orc_objective.argtypes = [C.c_void_p, _f64p, _f64p]
        lib.orc_solve.argtypes = [C.c_void_p, C.c_int, C.c_double, _f64p, _f64p, C.c_int,
                                  _f64p, _f64p, _f64p, _i32p]
        lib.orc_solve_inner.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double, _f64p, _f64p, C.c_int,
                                        _f64p, _f64p, _f64p, _i32p]
        lib.orc_dense_cholesky_solve.argtypes = [_f64p, _f64p, C.c_int, _f64p]
        _LIB = lib
    return _LIB


def _p(a, t):
    return a.ctypes.data_as(t)


class OracleError(RuntimeError):
    def __init__(self, kind, area, pivot):
        self.kind, self.area, self.pivot = kind, area, pivot
        what = f"area {area} interior block" if kind == 1 else "boundary system"
        super().__init__(f"{what} not positive definite at pivot {pivot}")


def two_port_table(net):
    """[n_branch, 8] array ff.re ff.im ft.re ft.im tf.re tf.im tt.re tt.im."""
    out = np.zeros((len(net.branches), 8))
    for e, br in enumerate(net.branches):
        y_ff, y_ft, y_tf, y_tt = br.two_port()
        out[e] = (y_ff.real, y_ff.imag, y_ft.real, y_ft.imag,
                  y_tf.real, y_tf.imag, y_tt.real, y_tt.imag)
    return out


class Oracle:
    """One analysed (network, measurement set, partition) triple."""

    def __init__(self, net, ms, area_of_bus, dense_threshold=64):
        lib = _lib()
        y = net.ybus
        self._keep = k = {}
        k["y_ptr"] = np.ascontiguousarray(y.indptr, dtype=np.int32)
        k["y_idx"] = np.ascontiguousarray(y.indices, dtype=np.int32)
        k["y_g"] = np.ascontiguousarray(y.data.real, dtype=np.float64)
        k["y_b"] = np.ascontiguousarray(y.data.imag, dtype=np.float64)
        k["br_from"] = np.array([b.from_bus for b in net.branches], dtype=np.int32)
        k["br_to"] = np.array([b.to_bus for b in net.branches], dtype=np.int32)
        k["br_y"] = np.ascontiguousarray(two_port_table(net))
        k["m_type"] = np.ascontiguousarray(ms.mtype, dtype=np.int32)
        k["m_target"] = np.ascontiguousarray(ms.target, dtype=np.int32)
        k["m_z"] = np.ascontiguousarray(ms.z, dtype=np.float64)
        k["m_w"] = np.ascontiguousarray(ms.weight, dtype=np.float64)
        k["area"] = np.ascontiguousarray(area_of_bus, dtype=np.int32)
        self.n_bus = len(net.buses)
        self.n_areas = int(k["area"].max()) + 1 if self.n_bus else 0
        d = _Desc()
        d.n_bus, d.n_branch, d.n_rows = self.n_bus, len(net.branches), len(k["m_z"])
        d.n_areas, d.slack = self.n_areas, int(net.slack)
        d.dense_threshold = int(dense_threshold)
        d.slack_va = float(net.buses[net.slack].va_true)
        for name, t in (("y_ptr", _i32p), ("y_idx", _i32p), ("y_g", _f64p), ("y_b", _f64p),
                        ("br_from", _i32p), ("br_to", _i32p), ("br_y", _f64p),
                        ("m_type", _i32p), ("m_target", _i32p), ("m_z", _f64p), ("m_w", _f64p)):
            setattr(d, name, _p(k[name], t))
        d.area_of_bus = _p(k["area"], _i32p)
        self._h = lib.orc_create(C.byref(d))
        self.n_gamma = lib.orc_n_gamma(self._h)

    # -- sizes / arrays ------------------------------------------------------
    def dims(self, a):
        out = np.zeros(8, dtype=np.int32)
        _lib().orc_area_dims(self._h, a, _p(out, _i32p))
        keys = ("n_i", "n_b", "n_rows", "n_slots", "nnz_ii", "nnz_ib", "nnz_l", "dense")
        return dict(zip(keys, (int(v) for v in out)))

    def _ints(self, a, which, n):
        ptr = _lib().orc_area_int(self._h, a, which)
        return np.ctypeslib.as_array(ptr, shape=(n,)).copy() if n else np.zeros(0, dtype=np.int32)

    def _f64(self, a, which, n):
        ptr = _lib().orc_area_f64(self._h, a, which)
        return np.ctypeslib.as_array(ptr, shape=(n,)).copy() if n else np.zeros(0)

    def blocks(self, a):
        """Normal-equation blocks of area ``a`` in the reference layout."""
        d = self.dims(a)
        ni, nb = d["n_i"], d["n_b"]
        return {
            "ii_ptr": self._ints(a, 0, ni + 1), "ii_idx": self._ints(a, 1, d["nnz_ii"]),
            "ib_ptr": self._ints(a, 2, ni + 1), "ib_idx": self._ints(a, 3, d["nnz_ib"]),
            "data_ii": self._f64(a, 0, d["nnz_ii"]), "data_ib": self._f64(a, 1, d["nnz_ib"]),
            "g_bb": self._f64(a, 2, nb * nb).reshape(nb, nb),
            "b_i": self._f64(a, 3, ni), "b_b": self._f64(a, 4, nb),
        }

    def schur(self, a):
        nb = self.dims(a)["n_b"]
        return self._f64(a, 5, nb * nb).reshape(nb, nb), self._f64(a, 6, nb)

    def selector(self, a):
        return self._ints(a, 4, self.dims(a)["n_b"])

    def interior_delta(self, a):
        return self._f64(a, 7, self.dims(a)["n_i"])

    def boundary_system(self):
        ng = self.n_gamma
        get = _lib().orc_gamma_f64

        def arr(which, n):
            return np.ctypeslib.as_array(get(self._h, which), shape=(n,)).copy() if n else np.zeros(0)
        return arr(0, ng * ng).reshape(ng, ng), arr(1, ng), arr(2, ng)

    def _raise(self):
        e = np.zeros(3, dtype=np.int32)
        _lib().orc_last_error(self._h, _p(e, _i32p))
        raise OracleError(int(e[0]), int(e[1]), int(e[2]))

    # -- phases --------------------------------------------------------------
    def assemble(self, va, vm):
        va = np.ascontiguousarray(va, dtype=np.float64)
        vm = np.ascontiguousarray(vm, dtype=np.float64)
        _lib().orc_assemble_only(self._h, _p(va, _f64p), _p(vm, _f64p))

    def local(self, va, vm, threads=1):
        va = np.ascontiguousarray(va, dtype=np.float64)
        vm = np.ascontiguousarray(vm, dtype=np.float64)
        if _lib().orc_local(self._h, _p(va, _f64p), _p(vm, _f64p), threads):
            self._raise()

    def boundary(self):
        if _lib().orc_boundary(self._h):
            self._raise()

    def recover(self, va, vm, threads=1):
        """In-place state update; returns the update's infinity norm."""
        assert va.dtype == np.float64 and vm.dtype == np.float64
        return float(_lib().orc_recover(self._h, _p(va, _f64p), _p(vm, _f64p), threads))

    # -- area-sharded variants (multi-process driver tests) -----------------------------------
    def local_masked(self, va, vm, mine):
        lib = _lib()
        lib.orc_local_masked.argtypes = [C.c_void_p, _f64p, _f64p, _i32p]
        mine = np.ascontiguousarray(mine, dtype=np.int32)
        if lib.orc_local_masked(self._h, _p(np.ascontiguousarray(va), _f64p),
                                _p(np.ascontiguousarray(vm), _f64p), _p(mine, _i32p)):
            self._raise()

    def set_schur(self, a, s_b, b_hat):
        lib = _lib()
        lib.orc_set_schur.argtypes = [C.c_void_p, C.c_int, _f64p, _f64p]
        s_b = np.ascontiguousarray(s_b, dtype=np.float64)
        b_hat = np.ascontiguousarray(b_hat, dtype=np.float64)
        lib.orc_set_schur(self._h, a, _p(s_b, _f64p), _p(b_hat, _f64p))

    def set_dx_gamma(self, dx):
        lib = _lib()
        lib.orc_set_dx_gamma.argtypes = [C.c_void_p, _f64p]
        dx = np.ascontiguousarray(dx, dtype=np.float64)
        lib.orc_set_dx_gamma(self._h, _p(dx, _f64p))

    def recover_masked(self, va, vm, mine):
        lib = _lib()
        lib.orc_recover_masked.restype = C.c_double
        lib.orc_recover_masked.argtypes = [C.c_void_p, _f64p, _f64p, _i32p]
        mine = np.ascontiguousarray(mine, dtype=np.int32)
        return float(lib.orc_recover_masked(self._h, _p(va, _f64p), _p(vm, _f64p), _p(mine, _i32p)))

    def inner_step_masked(self, va, vm, mine):
        """In-place interior-only GN step of the areas flagged in ``mine``; returns max |dx_i|."""
        lib = _lib()
        lib.orc_inner_step_masked.restype = C.c_double
        lib.orc_inner_step_masked.argtypes = [C.c_void_p, _f64p, _f64p, _i32p]
        mine = np.ascontiguousarray(mine, dtype=np.int32)
        d = float(lib.orc_inner_step_masked(self._h, _p(va, _f64p), _p(vm, _f64p), _p(mine, _i32p)))
        if d < 0:
            self._raise()
        return d

    def objective(self, va, vm):
        va = np.ascontiguousarray(va, dtype=np.float64)
        vm = np.ascontiguousarray(vm, dtype=np.float64)
        return float(_lib().orc_objective(self._h, _p(va, _f64p), _p(vm, _f64p)))

    def solve(self, max_iter=10, tol=1e-6, threads=1, trace=False, inner=1):
        """Flat-start GN loop -> dict(va, vm, iterations, converged, deltas, J[, trace])."""
        nb = self.n_bus
        va, vm = np.zeros(nb), np.zeros(nb)
        deltas = np.zeros(max_iter)
        tva = np.zeros((max_iter, nb)) if trace else None
        tvm = np.zeros((max_iter, nb)) if trace else None
        conv = np.zeros(1, dtype=np.int32)
        it = _lib().orc_solve_inner(
            self._h, max_iter, inner, tol, _p(va, _f64p), _p(vm, _f64p), threads, _p(deltas, _f64p),
            _p(tva, _f64p) if trace else None, _p(tvm, _f64p) if trace else None,
            _p(conv, _i32p))
        if it < 0:
            self._raise()
        out = {"va": va, "vm": vm, "iterations": int(it), "converged": bool(conv[0]),
               "deltas": deltas[:it].copy(), "objective": self.objective(va, vm)}
        if trace:
            out["trace_va"], out["trace_vm"] = tva[:it].copy(), tvm[:it].copy()
        return out


def dense_cholesky_solve(a, b):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.zeros_like(b)
    info = _lib().orc_dense_cholesky_solve(_p(a, _f64p), _p(b, _f64p), len(b), _p(x, _f64p))
    if info:
        raise OracleError(2, -1, info - 1)
    return x


def max_threads():
    return int(_lib().orc_max_threads())
