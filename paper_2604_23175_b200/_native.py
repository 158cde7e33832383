"""ctypes binding of ``libgridse_b200.so`` (C ABI: ``include/gridse_b200.h``).

The product path has no CPU fallback: ``lib()`` raises when the shared library is
missing (it is built in-tree by ``paper_2604_23175_b200/build.py``) and
``Plan`` raises ``NoDeviceError`` when no CUDA device is visible.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgridse_b200.so")

i32p = C.POINTER(C.c_int32)
f64p = C.POINTER(C.c_double)
i64p = C.POINTER(C.c_int64)

GSE_OK = 0
GSE_E_INVALID = -1
GSE_E_CUDA = -2
GSE_E_NOT_SPD_AREA = -3
GSE_E_NOT_SPD_BOUNDARY = -4
GSE_E_NO_DEVICE = -5


class ProblemDesc(C.Structure):
    _fields_ = [
        ("n_bus", C.c_int32), ("n_branch", C.c_int32), ("n_rows", C.c_int32),
        ("n_areas", C.c_int32), ("n_gamma", C.c_int32), ("slack", C.c_int32),
        ("y_ptr", i32p), ("y_idx", i32p), ("y_g", f64p), ("y_b", f64p),
        ("br_from", i32p), ("br_to", i32p), ("br_y", f64p),
        ("m_type", i32p), ("m_target", i32p), ("m_z", f64p), ("m_w", f64p),
        ("area_of_bus", i32p),
        ("ia_ptr", i32p), ("ia_bus", i32p), ("im_ptr", i32p), ("im_bus", i32p),
        ("ba_ptr", i32p), ("ba_bus", i32p), ("bm_ptr", i32p), ("bm_bus", i32p),
        ("sel_ptr", i32p), ("sel", i32p),
        ("gamma_bus", i32p), ("gamma_quant", i32p),
    ]


class Options(C.Structure):
    _fields_ = [
        ("device", C.c_int32), ("backend_dense", C.c_int32), ("leaf_buses", C.c_int32),
        ("max_pivots", C.c_int32), ("rank", C.c_int32), ("world", C.c_int32),
        ("area_rank", i32p), ("persistent", C.c_int32), ("tile_rows", C.c_int32),
        ("boundary_mode", C.c_int32),
        ("stream", C.c_void_p),
        ("max_ctas", C.c_int32),
    ]


class PeerInfo(C.Structure):
    """gse_peer_info: what a rank publishes for the peer-linked solve (plain bytes, exchanged by the host layer)."""
    _fields_ = [
        ("rank", C.c_int32), ("world", C.c_int32), ("n_gamma_fronts", C.c_int32), ("device", C.c_int32),
        ("pid", C.c_int64),
        ("ubuf", C.c_uint64), ("xsol", C.c_uint64), ("sync", C.c_uint64),
        ("ipc", (C.c_uint8 * 64) * 3),
        ("ipc_off", C.c_int64 * 3),
    ]


class Config(C.Structure):
    _fields_ = [("max_outer_iterations", C.c_int32), ("convergence_tol", C.c_double),
                ("time_phases", C.c_int32)]


class Report(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("converged", C.c_int32), ("objective", C.c_double),
                ("delta_inf", C.c_double * 64), ("phase_s", C.c_double * 5), ("loop_s", C.c_double),
                ("gpu_s", C.c_double)]


class Error(C.Structure):
    _fields_ = [("code", C.c_int32), ("area", C.c_int32), ("pivot", C.c_int32),
                ("message", C.c_char * 200)]


class NativeError(RuntimeError):
    def __init__(self, code, area, pivot, message):
        super().__init__(message)
        self.code, self.area, self.pivot = code, area, pivot


class NoDeviceError(NativeError):
    pass


_LIB = None


def lib():
    """Load the engine; the product fails loudly when it is absent."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2604_23175_b200.build` "
            "(gridse-b200 has no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp = C.c_void_p
    L.gse_version.restype = C.c_char_p
    L.gse_plan_create.argtypes = [C.POINTER(ProblemDesc), C.POINTER(Options), C.POINTER(vp)]
    L.gse_plan_destroy.argtypes = [vp]
    L.gse_plan_destroy.restype = None
    L.gse_last_error.argtypes = [vp]
    L.gse_last_error.restype = C.POINTER(Error)
    L.gse_set_weights.argtypes = [vp, f64p]
    L.gse_set_measurements.argtypes = [vp, f64p]
    L.gse_solve.argtypes = [vp, C.POINTER(Config), vp, vp, C.POINTER(Report)]
    L.gse_solve_io.argtypes = [vp, C.POINTER(Config), vp, vp, vp, vp, C.POINTER(Report)]
    L.gse_iterate.argtypes = [vp, vp, vp, f64p]
    L.gse_inner_step.argtypes = [vp, vp, vp, f64p]
    L.gse_phase_local_async.argtypes = [vp, vp, vp]
    L.gse_phase_boundary_async.argtypes = [vp]
    L.gse_phase_recover_async.argtypes = [vp, vp, vp]
    L.gse_partition_attempt.argtypes = [C.c_int32, i32p, i32p, C.c_int32, i32p, i32p, C.c_int32, C.c_int32, i32p, i32p]
    L.gse_partition_thin_cuts.argtypes = [C.c_int32, i32p, i32p, C.c_int32, i32p, i32p, C.c_int32, i32p]
    L.gse_set_rows_pinned.argtypes = [vp, vp, vp]
    L.gse_matrix_plan_create.argtypes = [C.c_int32, C.c_int32, i32p, i32p, i32p, i32p, C.POINTER(Options), C.POINTER(vp)]
    L.gse_matrix_set_values.argtypes = [vp, f64p, f64p, f64p, f64p, f64p]
    L.gse_matrix_condense.argtypes = [vp]
    L.gse_matrix_recover.argtypes = [vp, f64p, f64p]
    L.gse_matrix_perm.argtypes = [vp, i32p]
    L.gse_matrix_forward_get.argtypes = [vp, f64p]
    L.gse_matrix_backward.argtypes = [vp, f64p, f64p]
    L.gse_assemble_boundary.argtypes = [C.c_int32, C.c_int32, i32p, i32p, f64p, f64p, f64p, f64p]
    L.gse_phase_assemble.argtypes = [vp, vp, vp]
    L.gse_phase_condense.argtypes = [vp]
    L.gse_phase_boundary.argtypes = [vp]
    L.gse_phase_recover.argtypes = [vp, vp, vp, f64p]
    L.gse_check.argtypes = [vp]
    L.gse_objective.argtypes = [vp, vp, vp, f64p]
    L.gse_area_dims.argtypes = [vp, C.c_int32, i32p]
    L.gse_area_pattern.argtypes = [vp, C.c_int32, i32p, i32p, i32p, i32p]
    L.gse_area_blocks.argtypes = [vp, C.c_int32, f64p, f64p, f64p, f64p, f64p]
    L.gse_area_schur.argtypes = [vp, C.c_int32, f64p, f64p]
    L.gse_area_templates.argtypes = [vp, C.c_int32, i32p, i32p, i32p, f64p, f64p]
    L.gse_area_delta.argtypes = [vp, C.c_int32, f64p]
    L.gse_boundary_system.argtypes = [vp, f64p, f64p, f64p]
    L.gse_set_boundary_delta.argtypes = [vp, f64p]
    L.gse_exchange_buffer_dev.argtypes = [vp, i64p]
    L.gse_exchange_buffer_dev.restype = vp
    L.gse_exchange_offsets.argtypes = [vp, i64p]
    L.gse_boundary_delta_dev.argtypes = [vp]
    L.gse_boundary_delta_dev.restype = vp
    L.gse_status_dev.argtypes = [vp]
    L.gse_status_dev.restype = vp
    L.gse_plan_stats.argtypes = [vp, f64p, C.c_int32]
    L.gse_stream.argtypes = [vp]
    L.gse_stream.restype = vp
    L.gse_peer_info_get.argtypes = [vp, C.POINTER(PeerInfo)]
    L.gse_peer_link.argtypes = [vp, C.POINTER(PeerInfo)]
    L.gse_peer_solve_prepare.argtypes = [vp]
    _LIB = L
    return L


EXPORTED = [
    "gse_plan_create", "gse_plan_destroy", "gse_last_error", "gse_set_weights",
    "gse_set_measurements", "gse_set_rows_pinned", "gse_solve", "gse_iterate", "gse_inner_step", "gse_phase_assemble",
    "gse_phase_condense", "gse_phase_boundary", "gse_phase_recover", "gse_check", "gse_objective",
    "gse_area_dims", "gse_area_pattern", "gse_area_blocks", "gse_area_schur", "gse_area_delta",
    "gse_boundary_system", "gse_set_boundary_delta", "gse_exchange_buffer_dev",
    "gse_exchange_offsets", "gse_boundary_delta_dev", "gse_status_dev", "gse_plan_stats",
    "gse_version", "gse_stream", "gse_matrix_plan_create", "gse_matrix_set_values", "gse_matrix_condense",
    "gse_matrix_recover", "gse_assemble_boundary", "gse_phase_local_async", "gse_phase_boundary_async",
    "gse_phase_recover_async", "gse_debug_trace", "gse_solve_layout", "gse_partition_attempt", "gse_partition_thin_cuts",
    "gse_peer_info_get", "gse_peer_link", "gse_peer_solve_prepare",
    "gse_matrix_perm", "gse_matrix_forward_get", "gse_matrix_backward", "gse_area_templates", "gse_solve_io",
]


def _ip(a):
    return a.ctypes.data_as(i32p)


def _fp(a):
    return a.ctypes.data_as(f64p)


def two_port_table(net):
    arr = net.branch_arrays()
    out = np.empty((net.n_branch, 8))
    for c, key in enumerate(("y_ff", "y_ft", "y_tf", "y_tt")):
        out[:, 2 * c] = arr[key].real
        out[:, 2 * c + 1] = arr[key].imag
    return out


def make_desc(net, ms, part, bord, maps):
    """Flatten (net, ms, part, (bord, maps)) into a ``gse_problem_desc``.

    Returns (desc, keepalive dict of the numpy arrays the struct points into).
    """
    k = {}
    y = net.ybus
    k["y_ptr"] = np.ascontiguousarray(y.indptr, dtype=np.int32)
    k["y_idx"] = np.ascontiguousarray(y.indices, dtype=np.int32)
    k["y_g"] = np.ascontiguousarray(y.data.real, dtype=np.float64)
    k["y_b"] = np.ascontiguousarray(y.data.imag, dtype=np.float64)
    if net.n_branch:
        arr = net.branch_arrays()
        k["br_from"] = np.ascontiguousarray(arr["from"], dtype=np.int32)
        k["br_to"] = np.ascontiguousarray(arr["to"], dtype=np.int32)
        k["br_y"] = np.ascontiguousarray(two_port_table(net))
    else:
        k["br_from"] = np.zeros(1, dtype=np.int32)
        k["br_to"] = np.zeros(1, dtype=np.int32)
        k["br_y"] = np.zeros(8)
    k["m_type"] = np.ascontiguousarray(ms.mtype, dtype=np.int32)
    k["m_target"] = np.ascontiguousarray(ms.target, dtype=np.int32)
    k["m_z"] = np.ascontiguousarray(ms.z, dtype=np.float64)
    k["m_w"] = np.ascontiguousarray(ms.weight, dtype=np.float64)
    k["area_of_bus"] = np.ascontiguousarray(part.area_of_bus, dtype=np.int32)

    def ragged(name, lists):
        ptr = np.zeros(len(lists) + 1, dtype=np.int32)
        ptr[1:] = np.cumsum([len(x) for x in lists])
        flat = (np.concatenate([np.asarray(x, dtype=np.int32) for x in lists])
                if ptr[-1] else np.zeros(1, dtype=np.int32))
        k[name + "_ptr"] = ptr
        k[name] = np.ascontiguousarray(flat, dtype=np.int32)

    ragged("ia", [m.interior_angle_buses for m in maps])
    ragged("im", [m.interior_mag_buses for m in maps])
    ragged("ba", [m.local_boundary_angle_buses() for m in maps])
    ragged("bm", [m.local_boundary_buses for m in maps])
    ragged("sel", [m.boundary_selector for m in maps])
    ng = bord.n_gamma
    k["gamma_bus"] = np.array([b for b, _ in bord.entries] or [0], dtype=np.int32)
    k["gamma_quant"] = np.array([0 if q == "va" else 1 for _, q in bord.entries] or [0],
                                dtype=np.int32)
    d = ProblemDesc()
    d.n_bus, d.n_branch, d.n_rows = net.n_bus, net.n_branch, ms.m
    d.n_areas, d.n_gamma, d.slack = len(maps), ng, net.slack
    for name in ("y_ptr", "y_idx", "br_from", "br_to", "m_type", "m_target", "area_of_bus",
                 "ia_ptr", "im_ptr", "ba_ptr", "bm_ptr", "sel_ptr", "sel", "gamma_bus",
                 "gamma_quant"):
        setattr(d, name, _ip(k[name]))
    d.ia_bus, d.im_bus, d.ba_bus, d.bm_bus = _ip(k["ia"]), _ip(k["im"]), _ip(k["ba"]), _ip(k["bm"])
    for name in ("y_g", "y_b", "br_y", "m_z", "m_w"):
        setattr(d, name, _fp(k[name]))
    return d, k


class Plan:
    """Owner of one ``gse_plan`` (analysis + device program of one problem)."""

    def __init__(self, net, ms, part, bord, maps, *, device=0, dense=False, leaf_buses=0,
                 max_pivots=0, rank=0, world=1, area_rank=None, tile_rows=0, boundary_mode=0, stream=None,
                 max_ctas=0):
        L = lib()
        self._desc, self._keep = make_desc(net, ms, part, bord, maps)
        opt = Options()
        opt.device, opt.backend_dense = int(device), int(bool(dense))
        opt.leaf_buses, opt.max_pivots = int(leaf_buses), int(max_pivots)
        opt.rank, opt.world = int(rank), int(world)
        opt.tile_rows = int(tile_rows)
        opt.boundary_mode = int(boundary_mode)
        opt.max_ctas = int(max_ctas)
        opt.stream = int(stream) if stream else None      # cudaStream_t of the caller (e.g. torch's current stream)
        if area_rank is not None:
            self._keep["area_rank"] = np.ascontiguousarray(area_rank, dtype=np.int32)
            opt.area_rank = _ip(self._keep["area_rank"])
        self._h = C.c_void_p()
        rc = L.gse_plan_create(C.byref(self._desc), C.byref(opt), C.byref(self._h))
        self.n_bus, self.n_areas, self.n_gamma, self.n_rows = net.n_bus, len(maps), bord.n_gamma, ms.m
        self.device = int(device)
        if rc != GSE_OK:
            err = self._error()
            self.close()
            raise err

    # -- plumbing ------------------------------------------------------------------
    def _error(self):
        e = lib().gse_last_error(self._h).contents
        cls = NoDeviceError if e.code == GSE_E_NO_DEVICE else NativeError
        return cls(e.code, e.area, e.pivot, e.message.decode(errors="replace"))

    def _call(self, rc):
        if rc != GSE_OK:
            raise self._error()

    def close(self):
        if getattr(self, "_h", None) is not None and self._h:
            lib().gse_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- inputs --------------------------------------------------------------------
    def set_weights(self, w):
        w = np.ascontiguousarray(w, dtype=np.float64)
        assert w.shape == (self.n_rows,)
        self._call(lib().gse_set_weights(self._h, _fp(w)))

    def set_rows_pinned(self, z_ptr, w_ptr):
        """Async refresh from pinned host memory (raw addresses, 0 = skip)."""
        self._call(lib().gse_set_rows_pinned(self._h, C.c_void_p(z_ptr or None), C.c_void_p(w_ptr or None)))

    def set_measurements(self, z):
        z = np.ascontiguousarray(z, dtype=np.float64)
        assert z.shape == (self.n_rows,)
        self._call(lib().gse_set_measurements(self._h, _fp(z)))

    # -- solve ---------------------------------------------------------------------
    def solve(self, va_ptr, vm_ptr, max_iter=10, tol=1e-6, time_phases=False):
        cfg = Config(int(max_iter), float(tol), int(bool(time_phases)))
        rep = Report()
        self._call(lib().gse_solve(self._h, C.byref(cfg), va_ptr, vm_ptr, C.byref(rep)))
        return rep

    def solve_io(self, init_ptr, va_ptr, vm_ptr, out_pinned_ptr, max_iter=10, tol=1e-6, time_phases=False):
        """``solve`` with the start-state copy (device) and the result copy (pinned host) in the same enqueue."""
        cfg = Config(int(max_iter), float(tol), int(bool(time_phases)))
        rep = Report()
        self._call(lib().gse_solve_io(self._h, C.byref(cfg), C.c_void_p(init_ptr or None), va_ptr, vm_ptr,
                                      C.c_void_p(out_pinned_ptr or None), C.byref(rep)))
        return rep

    # -- peer-linked multi-rank solve (exchanges inside the persistent kernel) ---------
    def peer_info(self):
        """This rank's ``gse_peer_info`` as bytes (for an all-gather through the host layer)."""
        info = PeerInfo()
        self._call(lib().gse_peer_info_get(self._h, C.byref(info)))
        return bytes(info)

    def peer_link(self, infos):
        """``infos``: the records of all ranks, ordered by rank (bytes as returned by ``peer_info``)."""
        arr = (PeerInfo * len(infos))()
        for k, raw in enumerate(infos):
            C.memmove(C.byref(arr[k]), raw, C.sizeof(PeerInfo))
        self._call(lib().gse_peer_link(self._h, arr))

    def peer_solve_prepare(self):
        self._call(lib().gse_peer_solve_prepare(self._h))

    def iterate(self, va_ptr, vm_ptr):
        d = C.c_double()
        self._call(lib().gse_iterate(self._h, va_ptr, vm_ptr, C.byref(d)))
        return d.value

    def inner_step(self, va_ptr, vm_ptr):
        d = C.c_double()
        self._call(lib().gse_inner_step(self._h, va_ptr, vm_ptr, C.byref(d)))
        return d.value

    def objective(self, va_ptr, vm_ptr):
        j = C.c_double()
        self._call(lib().gse_objective(self._h, va_ptr, vm_ptr, C.byref(j)))
        return j.value

    # -- phases, enqueue-only (multi-GPU driver) ------------------------------------
    def phase_local_async(self, va_ptr, vm_ptr):
        self._call(lib().gse_phase_local_async(self._h, va_ptr, vm_ptr))

    def phase_boundary_async(self):
        self._call(lib().gse_phase_boundary_async(self._h))

    def phase_recover_async(self, va_ptr, vm_ptr):
        self._call(lib().gse_phase_recover_async(self._h, va_ptr, vm_ptr))

    def check(self):
        self._call(lib().gse_check(self._h))

    # -- phases ----------------------------------------------------------------------
    def phase_assemble(self, va_ptr, vm_ptr):
        self._call(lib().gse_phase_assemble(self._h, va_ptr, vm_ptr))

    def phase_condense(self):
        self._call(lib().gse_phase_condense(self._h))

    def phase_boundary(self):
        self._call(lib().gse_phase_boundary(self._h))

    def phase_recover(self, va_ptr, vm_ptr):
        d = C.c_double()
        self._call(lib().gse_phase_recover(self._h, va_ptr, vm_ptr, C.byref(d)))
        return d.value

    # -- readback ----------------------------------------------------------------------
    def area_dims(self, a):
        out = np.zeros(8, dtype=np.int32)
        self._call(lib().gse_area_dims(self._h, a, _ip(out)))
        return {"n_i": int(out[0]), "n_b": int(out[1]), "nnz_ii": int(out[2]),
                "nnz_ib": int(out[3]), "rows": int(out[4]), "slots": int(out[5]), "fronts": int(out[6]),
                "factor_nnz": int(out[7])}

    def area_templates(self, a):
        """Template layer of area ``a`` after ``phase_assemble``: (rows, slot_ptr, slot_var, g, w*r)."""
        d = self.area_dims(a)
        rows = np.zeros(max(d["rows"], 1), dtype=np.int32)
        slot_ptr = np.zeros(d["rows"] + 1, dtype=np.int32)
        slot_var = np.zeros(max(d["slots"], 1), dtype=np.int32)
        g, wr = np.zeros(max(d["slots"], 1)), np.zeros(max(d["rows"], 1))
        self._call(lib().gse_area_templates(self._h, a, _ip(rows), _ip(slot_ptr), _ip(slot_var), _fp(g), _fp(wr)))
        return rows[:d["rows"]], slot_ptr, slot_var[:d["slots"]], g[:d["slots"]], wr[:d["rows"]]

    def area_pattern(self, a):
        d = self.area_dims(a)
        ii_ptr = np.zeros(d["n_i"] + 1, dtype=np.int32)
        ii_idx = np.zeros(max(d["nnz_ii"], 1), dtype=np.int32)
        ib_ptr = np.zeros(d["n_i"] + 1, dtype=np.int32)
        ib_idx = np.zeros(max(d["nnz_ib"], 1), dtype=np.int32)
        self._call(lib().gse_area_pattern(self._h, a, _ip(ii_ptr), _ip(ii_idx), _ip(ib_ptr),
                                          _ip(ib_idx)))
        return ii_ptr, ii_idx[: d["nnz_ii"]], ib_ptr, ib_idx[: d["nnz_ib"]]

    def area_blocks(self, a):
        d = self.area_dims(a)
        ni, nb = d["n_i"], d["n_b"]
        data_ii = np.zeros(max(d["nnz_ii"], 1))
        data_ib = np.zeros(max(d["nnz_ib"], 1))
        g_bb = np.zeros(max(nb * nb, 1))
        b_i = np.zeros(max(ni, 1))
        b_b = np.zeros(max(nb, 1))
        self._call(lib().gse_area_blocks(self._h, a, _fp(data_ii), _fp(data_ib), _fp(g_bb),
                                         _fp(b_i), _fp(b_b)))
        return (data_ii[: d["nnz_ii"]], data_ib[: d["nnz_ib"]], g_bb[: nb * nb].reshape(nb, nb),
                b_i[:ni], b_b[:nb])

    def area_schur(self, a):
        nb = self.area_dims(a)["n_b"]
        s_b = np.zeros(max(nb * nb, 1))
        b_hat = np.zeros(max(nb, 1))
        self._call(lib().gse_area_schur(self._h, a, _fp(s_b), _fp(b_hat)))
        return s_b[: nb * nb].reshape(nb, nb), b_hat[:nb]

    def area_delta(self, a):
        ni = self.area_dims(a)["n_i"]
        dx = np.zeros(max(ni, 1))
        self._call(lib().gse_area_delta(self._h, a, _fp(dx)))
        return dx[:ni]

    def boundary_system(self):
        ng = self.n_gamma
        s = np.zeros(max(ng * ng, 1))
        b = np.zeros(max(ng, 1))
        dx = np.zeros(max(ng, 1))
        self._call(lib().gse_boundary_system(self._h, _fp(s), _fp(b), _fp(dx)))
        return s[: ng * ng].reshape(ng, ng), b[:ng], dx[:ng]

    def set_boundary_delta(self, dx):
        dx = np.ascontiguousarray(dx, dtype=np.float64)
        assert dx.shape == (self.n_gamma,)
        if self.n_gamma:
            self._call(lib().gse_set_boundary_delta(self._h, _fp(dx)))

    # -- exchange buffers (multi-GPU driver) ---------------------------------------------
    def exchange_buffer(self):
        n = C.c_int64()
        ptr = lib().gse_exchange_buffer_dev(self._h, C.byref(n))
        off = np.zeros(self.n_areas + 1, dtype=np.int64)
        lib().gse_exchange_offsets(self._h, off.ctypes.data_as(i64p))
        return ptr, int(n.value), off

    def boundary_delta_ptr(self):
        return lib().gse_boundary_delta_dev(self._h)

    def status_ptr(self):
        return lib().gse_status_dev(self._h)

    def stats(self):
        s = np.zeros(16)
        lib().gse_plan_stats(self._h, _fp(s), 16)
        keys = ("launches_last", "fronts", "levels", "tasks", "max_front", "factor_doubles",
                "update_doubles", "pair_contributions", "slots", "alg_bytes", "dense_flops",
                "launches_per_iter", "persistent", "solve_ctas", "solve_smem_bytes", "items_per_iteration")
        return dict(zip(keys, (float(v) for v in s)))


class MatrixPlan:
    """One-area Schur-mode plan on caller-supplied blocks (``gse_matrix_*``): the device engine
    behind ``linalg.symbolic_analyze / numeric_refactor / schur_condense / interior_recover /
    dense_cholesky_solve``."""

    def __init__(self, n_i, n_b, ii_ptr, ii_idx, ib_ptr=None, ib_idx=None, *, dense=False, device=0):
        L = lib()
        self.n_i, self.n_b = int(n_i), int(n_b)
        self._keep = [np.ascontiguousarray(a, dtype=np.int32) if a is not None else None
                      for a in (ii_ptr, ii_idx, ib_ptr, ib_idx)]
        for i in (1, 3):        # ctypes needs a non-null buffer even for empty index lists
            if self._keep[i] is not None and self._keep[i].size == 0:
                self._keep[i] = np.zeros(1, dtype=np.int32)
        opt = Options()
        opt.device, opt.backend_dense = int(device), int(bool(dense))
        self._h = C.c_void_p()
        args = [(_ip(a) if a is not None else None) for a in self._keep]
        rc = L.gse_matrix_plan_create(self.n_i, self.n_b, *args, C.byref(opt), C.byref(self._h))
        if rc != GSE_OK:
            if not self._h:
                raise NativeError(rc, -1, -1, "invalid matrix pattern")
            err = self._error()
            self.close()
            raise err

    _error = Plan._error
    _call = Plan._call
    close = Plan.close
    __del__ = Plan.__del__

    @staticmethod
    def _opt(a):
        if a is None:
            return None, None
        a = np.ascontiguousarray(a, dtype=np.float64)
        return a, (_fp(a) if a.size else None)

    def set_values(self, data_ii=None, data_ib=None, g_bb=None, b_i=None, b_b=None):
        keep = [self._opt(a) for a in (data_ii, data_ib, g_bb, b_i, b_b)]
        self._call(lib().gse_matrix_set_values(self._h, *[k[1] for k in keep]))

    def condense(self):
        self._call(lib().gse_matrix_condense(self._h))

    def schur(self):
        s_b, b_hat = np.zeros((self.n_b, self.n_b)), np.zeros(self.n_b)
        if self.n_b:
            self._call(lib().gse_area_schur(self._h, 0, _fp(s_b), _fp(b_hat)))
        return s_b, b_hat

    def perm(self):
        """perm[e] = original index of elimination position e (the reference's ``cache.perm``)."""
        out = np.zeros(max(self.n_i, 1), dtype=np.int32)
        self._call(lib().gse_matrix_perm(self._h, _ip(out)))
        return out[:self.n_i]

    def forward_get(self):
        """y = L^-1 P b of the right-hand side given to the last set_values + condense."""
        y = np.zeros(max(self.n_i, 1))
        self._call(lib().gse_matrix_forward_get(self._h, _fp(y)))
        return y[:self.n_i]

    def backward(self, y):
        y = np.ascontiguousarray(y, dtype=np.float64)
        x = np.zeros(max(self.n_i, 1))
        self._call(lib().gse_matrix_backward(self._h, _fp(y) if y.size else None, _fp(x)))
        return x[:self.n_i]

    def recover(self, dx_b=None):
        dx_i = np.zeros(max(self.n_i, 1))
        k = self._opt(dx_b)
        self._call(lib().gse_matrix_recover(self._h, k[1], _fp(dx_i)))
        return dx_i[:self.n_i]


def assemble_boundary_device(s_blocks, b_hats, selectors, n_gamma):
    """``gse_assemble_boundary``: S_Gamma / b_Gamma summed on the device in area order."""
    sel_ptr = np.zeros(len(selectors) + 1, dtype=np.int32)
    sel_ptr[1:] = np.cumsum([len(s) for s in selectors])
    sel = np.ascontiguousarray(np.concatenate([np.asarray(s, dtype=np.int32) for s in selectors] or [np.zeros(0, np.int32)]))
    sb = np.ascontiguousarray(np.concatenate([np.asarray(s, dtype=np.float64).ravel() for s in s_blocks] or [np.zeros(0)]))
    bh = np.ascontiguousarray(np.concatenate([np.asarray(b, dtype=np.float64).ravel() for b in b_hats] or [np.zeros(0)]))
    if sel.size == 0:
        sel = np.zeros(1, dtype=np.int32)
    if sb.size == 0:
        sb = np.zeros(1)
    if bh.size == 0:
        bh = np.zeros(1)
    s_gamma, b_gamma = np.zeros((n_gamma, n_gamma)), np.zeros(n_gamma)
    out_s = s_gamma if n_gamma else np.zeros((1, 1))
    out_b = b_gamma if n_gamma else np.zeros(1)
    rc = lib().gse_assemble_boundary(int(n_gamma), len(selectors), _ip(sel_ptr), _ip(sel), _fp(sb), _fp(bh), _fp(out_s), _fp(out_b))
    if rc == GSE_E_NO_DEVICE:
        raise NoDeviceError(rc, -1, -1, "no CUDA device visible: gridse-b200 has no CPU fallback")
    if rc != GSE_OK:
        raise NativeError(rc, -1, -1, "gse_assemble_boundary failed")
    return s_gamma, b_gamma
