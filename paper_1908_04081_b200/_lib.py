"""ctypes binding of the C ABI declared in include/sscg.h.

The library is loaded on first use from paper_1908_04081_b200/_lib/libsscg.so
(built in-tree by `paper_1908_04081_b200.build`).  A missing library or a
machine without a CUDA device is an error: there is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SSCG_LIB") or os.path.join(HERE, "_lib", "libsscg.so")

# keep in sync with include/sscg.h
ABI_VERSION = 2
MAX_SIGMA = 16
OK, EINVAL, ECUDA, ENOMEM, EPARAM, ENODEV, EBREAKDOWN, EFORMAT = range(8)
RUNNING, CONVERGED, STAGNATED, DIVERGED, EXHAUSTED = range(5)
SOLVER_ADAPTIVE, SOLVER_FIXED = 0, 1
LOG_CAP_OUTER, LOG_CAP_ITERS = 1 << 18, 1 << 21  # include/sscg.h SSCG_LOG_CAP_*
BASIS = {"monomial": 0, "newton": 1, "chebyshev": 2}
BASIS_NAMES = {v: k for k, v in BASIS.items()}
CSTRAT = {"adaptive": 0, "unit": 1, "kappa-estimate": 2, "full-bound": 3}
REC_K, REC_SBAR, REC_STILDE, REC_SACTUAL, REC_BREAKJ, REC_MARK, REC_PKIND = range(7)
REC_NI = 8
RECD_PHI, RECD_BLHS, RECD_BRHS, RECD_GEN_LO, RECD_GEN_HI, RECD_TRUE, RECD_RREL, RECD_C = range(8)
RECD_ND = 8
IT_ALPHA, IT_BETA, IT_TRUE, IT_UPD, IT_GAP, IT_XI, IT_LMIN, IT_LMAX, IT_PSI, IT_EST = range(10)
IT_N = 10

EXPORTS = (
    "sscg_last_error", "sscg_abi_version", "sscg_device_count", "sscg_plan_create",
    "sscg_plan_destroy", "sscg_plan_device_bytes", "sscg_solve", "sscg_load", "sscg_run",
    "sscg_fetch", "sscg_set_profiling", "sscg_get_profile", "sscg_get_small_phases",
    "sscg_plan_mpk_schedule", "sscg_set_basis_params", "sscg_hscg",
    "sscg_mm_parse", "sscg_mm_take", "sscg_mm_free", "sscg_mm_error_line", "sscg_power_iteration",
    "sscg_spmv", "sscg_build_block",
    "sscg_gram", "sscg_recover", "sscg_nested_conds", "sscg_select_s_tilde",
    "sscg_leja_points", "sscg_params_for", "sscg_ritz_sequence", "sscg_sym_eig",
    "sscg_nccl_unique_id", "sscg_plan_create_part", "sscg_vgroup_run",
    "sscg_plan_collectives", "sscg_group_create", "sscg_group_solve", "sscg_hscg_ex",
    "sscg_vgroup_hscg", "sscg_host_alloc", "sscg_host_free",
)
HSCG_MODES = {"reference": 0, "production": 1}


class SscgConfig(C.Structure):
    _fields_ = [
        ("sigma", C.c_int32), ("s_bar0", C.c_int32), ("f", C.c_int32),
        ("basis_kind", C.c_int32), ("c_strategy", C.c_int32), ("variant", C.c_int32),
        ("max_outer", C.c_int32), ("leja_grid", C.c_int32), ("has_bounds", C.c_int32),
        ("trace_full", C.c_int32), ("n_a", C.c_int32), ("solver", C.c_int32),
        ("eps_star", C.c_double), ("bound_lo", C.c_double), ("bound_hi", C.c_double),
        ("norm_a", C.c_double), ("norm_abs_a", C.c_double), ("kappa_a", C.c_double),
    ]


_DP = C.POINTER(C.c_double)
_IP = C.POINTER(C.c_int32)


class SscgLogs(C.Structure):
    _fields_ = [
        ("cap_iters", C.c_int64), ("cap_outer", C.c_int64),
        ("iters", _DP), ("rec_i", _IP), ("rec_d", _DP), ("conds", _DP),
        ("thetas", _DP), ("gammas", _DP), ("mus", _DP), ("outer_true", _DP),
        ("first_gram", _DP),
        ("status", C.c_int32), ("total_iters", C.c_int32), ("total_outer", C.c_int32),
        ("n_records", C.c_int32), ("outer_launched", C.c_int32), ("reserved", C.c_int32),
        ("device_ms", C.c_double),
    ]


class SscgPart(C.Structure):
    _fields_ = [
        ("n_own", C.c_int64), ("n_rows", C.c_int64), ("n_local", C.c_int64), ("nnz", C.c_int64),
        ("depth", C.c_int32), ("rank", C.c_int32), ("world", C.c_int32), ("n_peers", C.c_int32),
        ("row_ptr", C.POINTER(C.c_int64)), ("col_idx", C.POINTER(C.c_int32)),
        ("values", C.POINTER(C.c_double)), ("lvl_rows", C.POINTER(C.c_int64)),
        ("peer_rank", C.POINTER(C.c_int32)), ("send_off", C.POINTER(C.c_int64)),
        ("recv_off", C.POINTER(C.c_int64)), ("send_idx", C.POINTER(C.c_int32)),
        ("recv_idx", C.POINTER(C.c_int32)), ("nccl_id", C.c_void_p), ("nccl_lib", C.c_char_p),
        ("global_rows", C.POINTER(C.c_int64)),
    ]


class SscgError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"sscg error {code}: {msg}")
        self.code = code


_lock = threading.Lock()
_lib = None


def _declare(lib):
    vp = C.c_void_p
    i32, i64, dbl = C.c_int32, C.c_int64, C.c_double
    sig = {
        "sscg_last_error": (C.c_char_p, []),
        "sscg_abi_version": (C.c_int, []),
        "sscg_device_count": (C.c_int, [_IP]),
        "sscg_plan_create": (C.c_int, [C.POINTER(vp), i32, i64, i64, C.POINTER(i64), _IP, _DP]),
        "sscg_plan_destroy": (C.c_int, [vp]),
        "sscg_plan_device_bytes": (C.c_int, [vp, C.POINTER(i64)]),
        "sscg_solve": (C.c_int, [vp, C.POINTER(SscgConfig), _DP, _DP, _DP, C.POINTER(SscgLogs)]),
        "sscg_load": (C.c_int, [vp, _DP, _DP]),
        "sscg_run": (C.c_int, [vp, C.POINTER(SscgConfig), C.POINTER(SscgLogs)]),
        "sscg_fetch": (C.c_int, [vp, _DP, C.POINTER(SscgLogs)]),
        "sscg_set_profiling": (C.c_int, [vp, i32]),
        "sscg_get_profile": (C.c_int, [vp, _DP, C.POINTER(i64)]),
        "sscg_get_small_phases": (C.c_int, [vp, C.POINTER(i64)]),
        "sscg_plan_mpk_schedule": (C.c_int, [vp, i32, _IP]),
        "sscg_set_basis_params": (C.c_int, [vp, i32, _DP, _DP, _DP]),
        "sscg_hscg": (C.c_int, [vp, _DP, _DP, dbl, i64, _DP, C.POINTER(SscgLogs)]),
        "sscg_mm_parse": (C.c_int, [C.c_char_p, i64, C.POINTER(vp), C.POINTER(i64),
                                    C.POINTER(i64), _IP]),
        "sscg_mm_take": (C.c_int, [vp, C.POINTER(i64), _IP, _DP]),
        "sscg_mm_free": (None, [vp]),
        "sscg_mm_error_line": (C.c_int, []),
        "sscg_power_iteration": (C.c_int, [vp, i32, dbl, _DP, i32, dbl, _DP, _IP, _IP]),
        "sscg_spmv": (C.c_int, [vp, _DP, _DP]),
        "sscg_build_block": (C.c_int, [vp, _DP, _DP, i32, _DP, _DP, _DP, _DP, _DP]),
        "sscg_gram": (C.c_int, [i32, i64, i32, _DP, _DP]),
        "sscg_recover": (C.c_int, [i32, i64, i32, _DP, _DP, _DP, _DP, _DP, _DP, _DP, _DP]),
        "sscg_nested_conds": (C.c_int, [i32, _DP, i32, _DP]),
        "sscg_select_s_tilde": (C.c_int, [i32, _DP, i32, dbl, dbl, dbl, dbl, _IP, _DP]),
        "sscg_leja_points": (C.c_int, [i32, dbl, dbl, i32, i32, _DP]),
        "sscg_params_for": (C.c_int, [i32, i32, i32, i32, dbl, dbl, i32, _DP, _DP, _DP, _IP]),
        "sscg_ritz_sequence": (C.c_int, [i32, i32, _DP, _DP, _DP]),
        "sscg_sym_eig": (C.c_int, [i32, i32, _DP, _DP]),
        "sscg_nccl_unique_id": (C.c_int, [C.c_char_p, C.c_void_p]),
        "sscg_plan_create_part": (C.c_int, [C.POINTER(vp), i32, C.POINTER(SscgPart)]),
        "sscg_vgroup_run": (C.c_int, [C.POINTER(vp), i32, C.POINTER(SscgConfig),
                                      C.POINTER(_DP), C.POINTER(_DP), C.POINTER(SscgLogs)]),
        "sscg_plan_collectives": (C.c_int, [vp, _IP]),
        "sscg_hscg_ex": (C.c_int, [vp, _DP, _DP, dbl, i64, i32, _DP, C.POINTER(SscgLogs)]),
        "sscg_vgroup_hscg": (C.c_int, [C.POINTER(vp), i32, C.POINTER(_DP), C.POINTER(_DP), dbl,
                                       i64, i32, C.POINTER(SscgLogs)]),
        "sscg_host_alloc": (C.c_int, [C.POINTER(vp), i64]),
        "sscg_host_free": (C.c_int, [vp]),
        "sscg_group_create": (C.c_int, [C.POINTER(vp), i32, _IP, C.POINTER(SscgPart)]),
        "sscg_group_solve": (C.c_int, [C.POINTER(vp), i32, C.POINTER(SscgConfig), C.POINTER(_DP),
                                       C.POINTER(_DP), C.POINTER(_DP),
                                       C.POINTER(C.POINTER(SscgLogs))]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args


def load(path=LIB_PATH):
    """Load (once) and return the ctypes handle of libsscg.so."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise RuntimeError(
                    f"{path} is missing: build it with `python -m paper_1908_04081_b200.build` "
                    "(there is no CPU fallback)")
            lib = C.CDLL(path)
            _declare(lib)
            if lib.sscg_abi_version() != ABI_VERSION:
                raise RuntimeError("libsscg ABI version mismatch")
            _lib = lib
    return _lib


class _PinnedBlock:
    """One page-locked host block behind a result vector; back to the pool when
    the last array viewing it is gone."""

    def __init__(self, pool, ptr, nbytes):
        self._pool, self.ptr, self.nbytes = pool, ptr, nbytes
        self.__array_interface__ = {"shape": (nbytes // 8,), "typestr": "<f8",
                                    "data": (ptr, False), "version": 3}

    def __del__(self):
        pool = self._pool
        if pool is not None:
            pool._give_back(self.ptr, self.nbytes)


class PinnedPool:
    """Result vectors in page-locked host memory (sscg_host_alloc): the solve's
    device-to-host copy of x is then one DMA instead of a staged copy into a
    freshly faulted-in numpy array.  Blocks return to the pool when the arrays
    handed out are garbage collected; at most `max_bytes` are ever pinned --
    past that (or for small vectors) callers get a plain numpy array."""

    def __init__(self, min_bytes=16 << 20, max_bytes=1 << 30):
        self.min_bytes, self.max_bytes = min_bytes, max_bytes
        self._free = {}  # nbytes -> [ptr]
        self._pinned = 0
        self._mu = threading.Lock()

    def vector(self, n):
        nbytes = 8 * int(n)
        if nbytes < self.min_bytes:
            return np.empty(n)
        with self._mu:
            lst = self._free.get(nbytes)
            ptr = lst.pop() if lst else None
            if ptr is None:
                if self._pinned + nbytes > self.max_bytes:
                    self._trim_locked()
                if self._pinned + nbytes > self.max_bytes:
                    return np.empty(n)
                out = C.c_void_p()
                if load().sscg_host_alloc(C.byref(out), nbytes) != OK or not out.value:
                    return np.empty(n)
                ptr = out.value
                self._pinned += nbytes
                # the first block of a size brings a spare: `x, tr, co = solve(...)`
                # in a loop holds the last x while the next solve fills another
                # block, and page-locking costs ~0.2 ms per MB -- not inside a solve
                if lst is None and self._pinned + nbytes <= self.max_bytes:
                    spare = C.c_void_p()
                    if load().sscg_host_alloc(C.byref(spare), nbytes) == OK and spare.value:
                        self._free.setdefault(nbytes, []).append(spare.value)
                        self._pinned += nbytes
        return np.asarray(_PinnedBlock(self, ptr, nbytes))

    def _give_back(self, ptr, nbytes):
        try:
            with self._mu:
                self._free.setdefault(nbytes, []).append(ptr)
        except Exception:  # interpreter shutdown
            pass

    def _trim_locked(self):
        lib = load()
        for nbytes, lst in self._free.items():
            while lst:
                lib.sscg_host_free(lst.pop())
                self._pinned -= nbytes


result_pool = PinnedPool()


def check(rc):
    if rc != OK:
        msg = load().sscg_last_error().decode(errors="replace")
        raise SscgError(rc, msg)


def dptr(a):
    return a.ctypes.data_as(_DP)


def iptr(a):
    return a.ctypes.data_as(_IP)


def f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def device_count():
    n = C.c_int32(0)
    rc = load().sscg_device_count(C.byref(n))
    return n.value if rc == OK else 0


def require_device(device=0):
    n = device_count()
    if device >= n:
        raise SscgError(ENODEV, f"no CUDA device {device} ({n} visible); this build has no CPU path")


def plan_collectives(lib, handle):
    """What one outer loop of a plan's captured graph contains
    (sscg_plan_collectives): allreduce calls, halo exchange groups, NCCL
    kernel nodes, kernel nodes, graph nodes (-1 before the first solve)."""
    out = np.zeros(5, dtype=np.int32)
    check(lib.sscg_plan_collectives(handle, iptr(out)))
    keys = ("allreduce_per_outer", "halo_exchanges_per_outer", "nccl_kernel_nodes",
            "kernel_nodes", "graph_nodes")
    return {k: int(v) for k, v in zip(keys, out)}


class Plan:
    """Device copy of one CSR operator (owns the sscg_plan handle)."""

    def __init__(self, n, row_ptr, col_idx, values, device=0):
        lib = load()
        require_device(device)
        rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
        ci = np.ascontiguousarray(col_idx, dtype=np.int32)
        va = f64(values)
        h = C.c_void_p()
        check(lib.sscg_plan_create(C.byref(h), int(device), int(n), int(len(va)),
                                   rp.ctypes.data_as(C.POINTER(C.c_int64)), iptr(ci), dptr(va)))
        self.handle = h
        self.n = int(n)
        self.nnz = int(len(va))
        self.device = int(device)
        self._lib = lib

    def close(self):
        if getattr(self, "handle", None) is not None and self.handle.value:
            self._lib.sscg_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def device_bytes(self):
        v = C.c_int64(0)
        check(self._lib.sscg_plan_device_bytes(self.handle, C.byref(v)))
        return v.value

    def mpk_schedule(self, sigma):
        """Matrix-powers schedule for `sigma` (see `plan_mpk_schedule`)."""
        return plan_mpk_schedule(self._lib, self.handle, sigma)

    def collectives(self):
        return plan_collectives(self._lib, self.handle)


def plan_mpk_schedule(lib, handle, sigma):
    """sscg_plan_mpk_schedule of a plan handle:
    {"kind": "csr"|"pattern"|"stencil values", "form": pattern kernel form ("table" walk,
    "superset" mask, plane "march", TMA-fed "tma march") or None, "ctas": G, "patterns": P (pattern),
    "slots": union size (stencil values), "planes": value planes streamed per level (the
    symmetric form stores the diagonal and the upper offsets only), "passes": [(1, 0)] * sigma
    (one launch per level)}."""
    out = np.zeros(4 + 2 * 16, dtype=np.int32)
    check(lib.sscg_plan_mpk_schedule(handle, int(sigma), iptr(out)))
    npass = int(out[3])
    kind = ("csr", "csr", "pattern", "stencil values")[int(out[0])]
    form = ("table", "superset", "march", "tma march")[int(out[-1])] if kind == "pattern" else None
    slots = int(out[2]) if kind == "stencil values" else 0
    if kind == "stencil values" and int(out[-1]) == 1:
        form = "symmetric"  # the diagonal's and the upper offsets' planes only
    return {"kind": kind, "form": form, "ctas": int(out[1]),
            "patterns": int(out[2]) if kind == "pattern" else 0,
            "slots": slots,
            "planes": (slots + 1) // 2 if form == "symmetric" else slots,
            "passes": [(int(out[4 + 2 * q]), int(out[5 + 2 * q])) for q in range(npass)]}
