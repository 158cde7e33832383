"""TEST-ONLY host interpreter of the device program (see hostsim.cpp)."""

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(os.path.dirname(_HERE))
_SO = os.path.join(_HERE, "_hostsim.so")
_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        srcs = [os.path.join(_HERE, "hostsim.cpp"),
                os.path.join(_ROOT, "paper_2604_23175_b200", "csrc", "symbolic.cpp")]
        deps = srcs + [os.path.join(_ROOT, "paper_2604_23175_b200", "csrc", "plan.hpp")]
        if not os.path.exists(_SO) or any(os.path.getmtime(s) > os.path.getmtime(_SO) for s in deps):
            subprocess.run(["/usr/bin/g++", "-std=c++17", "-O2", "-ffp-contract=off", "-shared", "-fPIC", "-pthread",
                            "-o", _SO, *srcs], check=True)
        L = C.CDLL(_SO)
        L.hostsim_create.restype = C.c_void_p
        L.hostsim_iterate.restype = C.c_longlong
        L.hostsim_n_ref.restype = C.c_longlong
        _LIB = L
    return _LIB


class HostSim:
    def __init__(self, net, ms, part, bord, maps, dense=False, leaf=0, pmax=0, rank=0, world=1,
                 area_rank=None, boundary_mode=0):
        from paper_2604_23175_b200._native import make_desc
        L = _lib()
        self.desc, self.keep = make_desc(net, ms, part, bord, maps)
        msg = C.create_string_buffer(256)
        ar = None
        if area_rank is not None:
            self.keep["ar"] = np.ascontiguousarray(area_rank, dtype=np.int32)
            ar = self.keep["ar"].ctypes.data_as(C.POINTER(C.c_int32))
        self.h = C.c_void_p(L.hostsim_create(C.byref(self.desc), int(dense), leaf, pmax, rank, world, ar, msg, 256, int(boundary_mode)))
        if not self.h:
            raise RuntimeError(msg.value.decode())
        self.net, self.maps, self.n_gamma = net, maps, bord.n_gamma

    def stats(self):
        out = np.zeros(12)
        _lib().hostsim_stats(self.h, out.ctypes.data_as(C.POINTER(C.c_double)))
        keys = ("fronts", "levels", "max_front", "lbuf", "ubuf", "pairs", "gval", "flops", "tasks", "bwd_levels", "chain_pivots", "boundary_chain_pivots")
        return dict(zip(keys, out))

    def iterate(self, va, vm):
        d = C.c_double()
        code = _lib().hostsim_iterate(self.h, va.ctypes.data_as(C.POINTER(C.c_double)),
                                      vm.ctypes.data_as(C.POINTER(C.c_double)), C.byref(d))
        return int(code), d.value

    def area_schur(self, a):
        nb = self.maps[a].n_boundary
        s = np.zeros((nb, nb))
        b = np.zeros(nb)
        _lib().hostsim_area_schur(self.h, a, s.ctypes.data_as(C.POINTER(C.c_double)),
                                  b.ctypes.data_as(C.POINTER(C.c_double)))
        return s, b

    def ref_blocks(self):
        n = _lib().hostsim_n_ref(self.h)
        out = np.zeros(max(n, 1))
        _lib().hostsim_ref_blocks(self.h, out.ctypes.data_as(C.POINTER(C.c_double)))
        off = np.zeros(len(self.maps) + 1, dtype=np.int64)
        _lib().hostsim_ref_off(self.h, off.ctypes.data_as(C.POINTER(C.c_longlong)))
        return out[:n], off

    def solve(self, max_iter=10, tol=1e-6):
        net = self.net
        va = np.zeros(net.n_bus)
        va[net.slack] = net.buses[net.slack].va_true
        vm = np.ones(net.n_bus)
        deltas = []
        for it in range(1, max_iter + 1):
            code, d = self.iterate(va, vm)
            if code >= 0:
                raise RuntimeError(f"not SPD: front {code >> 32} pivot {code & 0xffffffff}")
            deltas.append(d)
            if d < tol:
                return va, vm, it, True, deltas
        return va, vm, max_iter, False, deltas
