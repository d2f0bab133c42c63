"""TEST INFRASTRUCTURE ONLY -- ctypes access to the CPU oracle.

Two libraries, both built by ``oracle/Makefile``:

* ``oracle/libktune_oracle.so``: the plain-C restatement of the reference's
  SpMV path (``oracle/ktune_oracle.c``; each function cites the reference
  file:line it follows).
* ``oracle/_ref/libktune_ref.so``: the UNMODIFIED reference headers
  (``/root/reference/proj/include/ktune``) behind ``extern "C"`` forwarding
  wrappers (``oracle/ref_shim.cpp``). Built only where the reference tree
  exists; the prebuilt file travels to the GPU box with the repo snapshot.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference`` arm) may import this module, and
only as the checker / the CPU baseline. The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libktune_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libktune_ref.so")

_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_I64 = C.c_int64


def build() -> None:
    """Compile the oracle (and oracle/_ref when the reference is present)."""
    import subprocess

    subprocess.run(["make", "-s", "-C", HERE], check=True)


_ora = None
_ref = None


def lib():
    global _ora
    if _ora is None:
        if not os.path.exists(ORACLE_SO):
            build()
        L = C.CDLL(ORACLE_SO)
        L.ko_error_message.restype = C.c_char_p
        L.ko_validate.argtypes = [_I64, _i64p, _I64, _i64p, C.c_int]
        L.ko_spmv_ref.argtypes = [_I64, _i64p, _i64p, _f64p, _f64p, _f64p]
        L.ko_expand_symmetric_nnz.argtypes = [_I64, _i64p, _i64p]
        L.ko_expand_symmetric_nnz.restype = _I64
        L.ko_expand_symmetric.argtypes = [_I64, _i64p, _i64p, _f64p, _i64p, _i64p, _f64p]
        L.ko_build_row_partition.argtypes = [_i64p, _I64, C.c_int, C.c_int, _i64p]
        L.ko_build_reduction_regions.argtypes = [_I64, _i64p, _i64p, C.c_int, _i64p, _i64p, _i64p]
        L.ko_bss_count.argtypes = [_I64, _i64p, _I64, C.POINTER(_I64), C.POINTER(_I64)]
        L.ko_bss_fill.argtypes = [_I64, _i64p, _I64, _i64p, _i64p, _i64p, _i64p, _i64p, _u8p]
        L.ko_spmv_row_blocks.argtypes = [_I64, _i64p, _i64p, _f64p, C.c_int, _i64p, _f64p, _f64p]
        L.ko_spmv_bss.argtypes = [C.c_int, _I64, _i64p, _f64p, _I64, _i64p, _i64p, _i64p, _i64p,
                                  _u8p, _f64p, _f64p, _f64p]
        L.ko_spmv_sym.argtypes = [C.c_int, _I64, _i64p, _i64p, _f64p, C.c_int, _i64p, _i64p,
                                  _i64p, C.c_int, _f64p, _f64p, _f64p]
        L.ko_seeded_vector.argtypes = [_I64, C.c_uint64, _f64p]
        L.ko_probe_vector.argtypes = [_I64, _f64p]
        L.ko_outputs_match.argtypes = [_I64, _f64p, _f64p]
        L.ko_dot.argtypes = [_I64, _f64p, _f64p]
        L.ko_dot.restype = C.c_double
        L.ko_norm2.argtypes = [_I64, _f64p]
        L.ko_norm2.restype = C.c_double
        L.ko_gmres_mgs.argtypes = [_I64, _i64p, _i64p, _f64p, _f64p, _I64, C.c_double, _I64,
                                   _f64p, _f64p, C.c_void_p]
        L.ko_ilu0_factorize.argtypes = [_I64, _i64p, _i64p, _f64p, _i64p]
        L.ko_ilu0_factorize.restype = _I64
        L.ko_ilu0_apply.argtypes = [_I64, _i64p, _i64p, _f64p, _i64p, _f64p, _f64p]
        _ora = L
    return _ora


# The reference compiled three ways (oracle/Makefile): "parity" (-O2
# -ffp-contract=off: bitwise with the restatement, the checker), "release"
# (the reference's own CMake Release: -O3 -DNDEBUG) and "native" (Release +
# -march=native); the last two are CPU baselines only.
REF_VARIANTS = {"parity": REF_SO,
                "release": os.path.join(HERE, "_ref", "libktune_ref_rel.so"),
                "native": os.path.join(HERE, "_ref", "libktune_ref_native.so")}
REF_FLAGS = {"parity": "g++ -O2 -std=c++20 -fopenmp -ffp-contract=off",
             "release": "g++ -O3 -DNDEBUG -std=c++20 -fopenmp (the reference's CMake Release)",
             "native": "g++ -O3 -DNDEBUG -march=native -std=c++20 -fopenmp"}
_refs: dict = {}


def ref_available(variant: str = "parity") -> bool:
    return os.path.exists(REF_VARIANTS[variant])


def ref(variant: str = "parity"):
    global _ref
    if variant not in _refs:
        path = REF_VARIANTS[variant]
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where the "
                                    "reference tree is present")
        L = C.CDLL(path)
        L.kr_last_error.restype = C.c_char_p
        L.kr_validate.argtypes = [_I64, _i64p, _i64p, _f64p, C.c_int]
        L.kr_spmv_ref.argtypes = [_I64, _i64p, _i64p, _f64p, _f64p, _f64p]
        L.kr_expand_symmetric.argtypes = [_I64, _i64p, _i64p, _f64p, _I64, _i64p, _i64p, _f64p]
        L.kr_build_row_partition.argtypes = [_I64, _i64p, C.c_int, C.c_int, _i64p]
        L.kr_build_reduction_regions.argtypes = [_I64, _i64p, _i64p, _f64p, C.c_int, C.c_int,
                                                 _i64p, _i64p]
        L.kr_bss_create.argtypes = [_I64, _i64p, _i64p, _f64p, _I64, C.POINTER(C.c_void_p)]
        L.kr_bss_info.argtypes = [C.c_void_p, C.POINTER(_I64), C.POINTER(_I64)]
        L.kr_bss_copy.argtypes = [C.c_void_p, _i64p, _i64p, _i64p, _i64p, _i64p, _u8p]
        L.kr_bss_destroy.argtypes = [C.c_void_p]
        L.kr_spmv_unsym.argtypes = [C.c_int, _I64, _i64p, _i64p, _f64p, C.c_int, _I64, _f64p,
                                    _f64p]
        L.kr_spmv_sym.argtypes = [C.c_int, _I64, _i64p, _i64p, _f64p, C.c_int, _f64p, _f64p]
        L.kr_seeded_vector.argtypes = [_I64, C.c_uint64, _f64p]
        L.kr_probe_vector.argtypes = [_I64, _f64p]
        L.kr_select.argtypes = [C.c_int, _I64, _i64p, _i64p, _f64p, C.c_int, C.c_int,
                                C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                C.c_void_p, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.kr_engine_create.argtypes = [C.c_int, _I64, _i64p, _i64p, _f64p, C.c_int,
                                       C.POINTER(C.c_void_p)]
        L.kr_engine_selected.argtypes = [C.c_void_p, C.c_char_p, C.POINTER(_I64),
                                         C.POINTER(C.c_int), C.POINTER(C.c_double)]
        L.kr_engine_apply.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.kr_engine_destroy.argtypes = [C.c_void_p]
        L.kr_gmres.argtypes = [_I64, _i64p, _i64p, _f64p, _f64p, _I64, C.c_double, _I64,
                               C.c_int, C.c_int, _f64p, _f64p] + [C.c_void_p] * 8
        L.kr_max_threads.restype = C.c_int
        L.kr_ilu0_factorize.argtypes = [_I64, _i64p, _i64p, _f64p, _f64p, _i64p]
        L.kr_ilu0_apply.argtypes = [_I64, _i64p, _i64p, _f64p, _i64p, _f64p, _f64p]
        L.kr_gmres_ilu0.argtypes = [_I64, _i64p, _i64p, _f64p, _f64p, _I64, C.c_double, _I64,
                                    C.c_int, _f64p] + [C.c_void_p] * 4
        L.kr_mm_probe.argtypes = [C.c_char_p, C.POINTER(_I64), C.POINTER(_I64),
                                  C.POINTER(C.c_int)]
        L.kr_mm_load.argtypes = [C.c_char_p, C.c_int, C.POINTER(C.c_void_p)]
        L.kr_mm_info.argtypes = [C.c_void_p, C.POINTER(_I64), C.POINTER(_I64),
                                 C.POINTER(C.c_int)]
        L.kr_mm_copy.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.kr_mm_destroy.argtypes = [C.c_void_p]
        L.kr_mm_write.argtypes = [C.c_char_p, _I64, _i64p, _i64p, _f64p, C.c_int]
        L.kr_engine_create_stencil7.argtypes = [_I64, _I64, _I64, C.c_double, C.c_double,
                                                C.c_int, C.POINTER(C.c_void_p)]
        L.kr_engine_report.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.POINTER(C.c_int),
                                       C.POINTER(C.c_int)]
        _refs[variant] = L
        if variant == "parity":
            _ref = L
    return _refs[variant]


class OracleError(RuntimeError):
    pass


REF_EIG_SO = os.path.join(os.path.dirname(REF_SO), "libktune_ref_eig.so")
_ref_eig = None


def ref_eig_available() -> bool:
    return os.path.exists(REF_EIG_SO)


def ref_eig():
    """The reference's Lanczos (oracle/ref_shim_eig.cpp, LAPACKE from the
    python env's bundled OpenBLAS)."""
    global _ref_eig
    if _ref_eig is None:
        L = C.CDLL(REF_EIG_SO)
        L.kre_last_error.restype = C.c_char_p
        L.kre_lanczos.argtypes = [_I64, _i64p, _i64p, _f64p, _I64, _I64, C.c_double, _I64,
                                  C.c_int, C.c_uint64, _f64p, _f64p] + [C.c_void_p] * 4
        _ref_eig = L
    return _ref_eig


def ref_lanczos(n, rp, ci, v, k, m=30, tol=1e-8, max_iters=10000, ortho_kind=1, seed=20080517):
    """lanczos_restarted(SymCsrMatrix, k, cfg) of the reference (sym upper
    storage in) -> (eigenvalues, residuals, info dict)."""
    rp, ci, v = _csr(rp, ci, v)
    ev, rs = np.zeros(k), np.zeros(k)
    nf, its, rst = _I64(), _I64(), _I64()
    conv = C.c_int()
    rc = ref_eig().kre_lanczos(n, rp, ci, v, k, m, tol, max_iters, ortho_kind, seed, ev, rs,
                               C.byref(nf), C.byref(its), C.byref(rst), C.byref(conv))
    if rc:
        raise OracleError(ref_eig().kre_last_error().decode())
    return ev[: nf.value], rs[: nf.value], dict(iterations=its.value, restarts=rst.value,
                                                converged=bool(conv.value))


def _chk_ref(rc: int, L=None) -> None:
    if rc != 0:
        raise OracleError((L or ref()).kr_last_error().decode())


def _csr(rp, ci, v):
    return (np.ascontiguousarray(rp, np.int64), np.ascontiguousarray(ci, np.int64),
            np.ascontiguousarray(v, np.float64))


# ---------------------------------------------------------------- restatement
def validate(n, rp, ci, upper_only=False) -> str | None:
    rp, ci, _ = _csr(rp, ci, np.zeros(len(ci)))
    rc = lib().ko_validate(n, rp, len(ci), ci, 1 if upper_only else 0)
    return None if rc == 0 else lib().ko_error_message(rc).decode()


def spmv_ref(n, rp, ci, v, x):
    rp, ci, v = _csr(rp, ci, v)
    y = np.empty(n, np.float64)
    lib().ko_spmv_ref(n, rp, ci, v, np.ascontiguousarray(x, np.float64), y)
    return y


def expand_symmetric(n, rp, ci, v):
    rp, ci, v = _csr(rp, ci, v)
    nnz = lib().ko_expand_symmetric_nnz(n, rp, ci)
    orp = np.empty(n + 1, np.int64)
    oci = np.empty(nnz, np.int64)
    ov = np.empty(nnz, np.float64)
    lib().ko_expand_symmetric(n, rp, ci, v, orp, oci, ov)
    return orp, oci, ov


def build_row_partition(rp, num_workers, scheme):
    rp = np.ascontiguousarray(rp, np.int64)
    out = np.empty(max(num_workers, 0) + 1, np.int64)
    rc = lib().ko_build_row_partition(rp, len(rp) - 1, num_workers, scheme, out)
    if rc:
        raise OracleError(lib().ko_error_message(rc).decode())
    return out


def build_reduction_regions(n, rp, ci, boundaries):
    rp, ci, _ = _csr(rp, ci, np.zeros(len(ci)))
    P = len(boundaries) - 1
    lo = np.empty(P, np.int64)
    hi = np.empty(P, np.int64)
    lib().ko_build_reduction_regions(n, rp, ci, P, np.ascontiguousarray(boundaries, np.int64),
                                     lo, hi)
    return lo, hi


@dataclass
class BssPlan:
    jl: int
    slice_start: np.ndarray
    slice_len: np.ndarray
    slice_row: np.ndarray
    lane_slice_ptr: np.ndarray
    row_slice_ptr: np.ndarray
    row_start_flag: np.ndarray


def build_bss_plan(n, rp, jl) -> BssPlan:
    rp = np.ascontiguousarray(rp, np.int64)
    jle, tot = _I64(), _I64()
    rc = lib().ko_bss_count(n, rp, jl, C.byref(jle), C.byref(tot))
    if rc:
        raise OracleError(lib().ko_error_message(rc).decode())
    T, J = tot.value, jle.value
    p = BssPlan(J, np.empty(T, np.int64), np.empty(T, np.int64), np.empty(T, np.int64),
                np.empty(J + 1, np.int64), np.empty(n + 1, np.int64),
                np.empty(int(rp[n]), np.uint8))
    lib().ko_bss_fill(n, rp, J, p.slice_start, p.slice_len, p.slice_row, p.lane_slice_ptr,
                      p.row_slice_ptr, p.row_start_flag)
    return p


def spmv_row_blocks(n, rp, ci, v, boundaries, x):
    rp, ci, v = _csr(rp, ci, v)
    y = np.empty(n, np.float64)
    lib().ko_spmv_row_blocks(n, rp, ci, v, len(boundaries) - 1,
                             np.ascontiguousarray(boundaries, np.int64),
                             np.ascontiguousarray(x, np.float64), y)
    return y


def spmv_bss(n, rp, ci, v, plan: BssPlan, x, u4=False):
    rp, ci, v = _csr(rp, ci, v)
    y = np.empty(n, np.float64)
    sums = np.empty(max(len(plan.slice_start), 1), np.float64)
    lib().ko_spmv_bss(1 if u4 else 0, n, ci, v, plan.jl, plan.slice_start, plan.slice_len,
                      plan.lane_slice_ptr, plan.row_slice_ptr, plan.row_start_flag,
                      np.ascontiguousarray(x, np.float64), sums, y)
    return y


def spmv_sym(kernel, n, rp, ci, v, num_workers, x, pool_size=None):
    """kernel: 0=s1 (row-based), 1=s2 (nnz-balanced), 2=s3 (zero-omission)."""
    rp, ci, v = _csr(rp, ci, v)
    b = build_row_partition(rp, num_workers, 0 if kernel == 0 else 1)
    lo, hi = build_reduction_regions(n, rp, ci, b)
    y = np.empty(n, np.float64)
    scratch = np.full(num_workers * max(n, 1), np.nan)
    lib().ko_spmv_sym(kernel, n, rp, ci, v, num_workers, b, lo, hi,
                      pool_size or num_workers, np.ascontiguousarray(x, np.float64), y, scratch)
    return y


def seeded_vector(n, seed):
    out = np.empty(n, np.float64)
    lib().ko_seeded_vector(n, seed, out)
    return out


def probe_vector(n):
    out = np.empty(n, np.float64)
    lib().ko_probe_vector(n, out)
    return out


def outputs_match(y, ref_y) -> bool:
    return bool(lib().ko_outputs_match(len(y), np.ascontiguousarray(y, np.float64),
                                       np.ascontiguousarray(ref_y, np.float64)))


class _GmresRes(C.Structure):
    _fields_ = [("iterations", _I64), ("restarts", _I64), ("spmv_calls", _I64),
                ("converged", C.c_int), ("breakdown", C.c_int), ("fault_convergence", C.c_int),
                ("recurrence_residual", C.c_double), ("true_residual", C.c_double)]


def gmres_mgs(n, rp, ci, v, b, m=30, tol=1e-8, max_iters=3000):
    rp, ci, v = _csr(rp, ci, v)
    x = np.empty(n, np.float64)
    hist = np.zeros(max(max_iters, 1), np.float64)
    r = _GmresRes()
    rc = lib().ko_gmres_mgs(n, rp, ci, v, np.ascontiguousarray(b, np.float64), m, tol,
                            max_iters, x, hist, C.byref(r))
    if rc:
        raise OracleError(lib().ko_error_message(rc).decode())
    res = {f: getattr(r, f) for f, _ in _GmresRes._fields_}
    res["history"] = hist[: r.iterations].copy()
    return x, res


def ilu0_factorize(n, rp, ci, v):
    """ilu0.hpp:23-69 -> (values, diag_ptr); raises OracleError with the
    reference's message on a missing diagonal / zero pivot."""
    rp, ci, v = _csr(rp, ci, v)
    vals = v.copy()
    diag = np.empty(max(n, 1), np.int64)
    rc = lib().ko_ilu0_factorize(n, rp, ci, vals, diag)
    if rc < 0:
        raise OracleError(f"ilu0: structurally missing diagonal in row {-rc - 1}")
    if rc > 0:
        raise OracleError(f"ilu0: zero pivot at row {rc - 1}")
    return vals, diag[:n]


def ilu0_apply(n, rp, ci, fv, diag, r):
    rp, ci, fv = _csr(rp, ci, fv)
    z = np.empty(n, np.float64)
    lib().ko_ilu0_apply(n, rp, ci, fv, np.ascontiguousarray(diag, np.int64),
                        np.ascontiguousarray(r, np.float64), z)
    return z


# ------------------------------------------------------------------ reference
class _Cand(C.Structure):
    _fields_ = [("name", C.c_char * 8), ("ordinal", C.c_int), ("jl", _I64),
                ("workers", C.c_int), ("correct", C.c_int), ("executions", C.c_int),
                ("n_trials", C.c_int), ("best_seconds", C.c_double),
                ("trial_seconds", C.c_double * 8)]


NOW_FN = C.CFUNCTYPE(C.c_double, C.c_void_p)


class Ref:
    """Namespace of thin wrappers over oracle/_ref/libktune_ref.so."""

    @staticmethod
    def validate(n, rp, ci, v, upper=False):
        rp, ci, v = _csr(rp, ci, v)
        rc = ref().kr_validate(n, rp, ci, v, 1 if upper else 0)
        return None if rc == 0 else ref().kr_last_error().decode()

    @staticmethod
    def spmv_ref(n, rp, ci, v, x):
        rp, ci, v = _csr(rp, ci, v)
        y = np.empty(n, np.float64)
        _chk_ref(ref().kr_spmv_ref(n, rp, ci, v, np.ascontiguousarray(x, np.float64), y))
        return y

    @staticmethod
    def expand_symmetric(n, rp, ci, v):
        rp, ci, v = _csr(rp, ci, v)
        diag = int(np.sum(ci == np.repeat(np.arange(n), np.diff(rp))))
        nnz = 2 * len(ci) - diag
        orp, oci, ov = np.empty(n + 1, np.int64), np.empty(nnz, np.int64), np.empty(nnz)
        _chk_ref(ref().kr_expand_symmetric(n, rp, ci, v, nnz, orp, oci, ov))
        return orp, oci, ov

    @staticmethod
    def build_row_partition(rp, P, scheme):
        rp = np.ascontiguousarray(rp, np.int64)
        out = np.empty(P + 1, np.int64)
        _chk_ref(ref().kr_build_row_partition(len(rp) - 1, rp, P, scheme, out))
        return out

    @staticmethod
    def build_reduction_regions(n, rp, ci, v, P, scheme=1):
        rp, ci, v = _csr(rp, ci, v)
        lo, hi = np.empty(P, np.int64), np.empty(P, np.int64)
        _chk_ref(ref().kr_build_reduction_regions(n, rp, ci, v, P, scheme, lo, hi))
        return lo, hi

    @staticmethod
    def build_bss_plan(n, rp, ci, v, jl) -> BssPlan:
        rp, ci, v = _csr(rp, ci, v)
        h = C.c_void_p()
        _chk_ref(ref().kr_bss_create(n, rp, ci, v, jl, C.byref(h)))
        try:
            J, T = _I64(), _I64()
            ref().kr_bss_info(h, C.byref(J), C.byref(T))
            p = BssPlan(J.value, np.empty(T.value, np.int64), np.empty(T.value, np.int64),
                        np.empty(T.value, np.int64), np.empty(J.value + 1, np.int64),
                        np.empty(n + 1, np.int64), np.empty(len(ci), np.uint8))
            ref().kr_bss_copy(h, p.slice_start, p.slice_len, p.slice_row, p.lane_slice_ptr,
                              p.row_slice_ptr, p.row_start_flag)
            return p
        finally:
            ref().kr_bss_destroy(h)

    @staticmethod
    def spmv_unsym(kernel, n, rp, ci, v, workers, jl, x):
        rp, ci, v = _csr(rp, ci, v)
        y = np.empty(n, np.float64)
        _chk_ref(ref().kr_spmv_unsym(kernel, n, rp, ci, v, workers, jl,
                                     np.ascontiguousarray(x, np.float64), y))
        return y

    @staticmethod
    def spmv_sym(kernel, n, rp, ci, v, workers, x):
        rp, ci, v = _csr(rp, ci, v)
        y = np.empty(n, np.float64)
        _chk_ref(ref().kr_spmv_sym(kernel, n, rp, ci, v, workers,
                                   np.ascontiguousarray(x, np.float64), y))
        return y

    @staticmethod
    def seeded_vector(n, seed):
        out = np.empty(n, np.float64)
        ref().kr_seeded_vector(n, seed, out)
        return out

    @staticmethod
    def probe_vector(n):
        out = np.empty(n, np.float64)
        ref().kr_probe_vector(n, out)
        return out

    @staticmethod
    def select(sym, n, rp, ci, v, pool_size, timed_trials=3, jl_candidates=None, sweep=False,
               now=None):
        """Returns (candidates as dicts, selected index). `now` is an optional
        Python callable used as the injected timer (autotune.hpp:164)."""
        rp, ci, v = _csr(rp, ci, v)
        cands = (_Cand * 256)()
        nout, sel = C.c_int(), C.c_int()
        jl_arr = None if jl_candidates is None else np.ascontiguousarray(jl_candidates, np.int64)
        cb = NOW_FN(lambda _ctx: float(now())) if now else None
        _chk_ref(ref().kr_select(1 if sym else 0, n, rp, ci, v, pool_size, timed_trials,
                                 None if jl_arr is None else jl_arr.ctypes.data,
                                 0 if jl_arr is None else len(jl_arr), 1 if sweep else 0,
                                 C.cast(cb, C.c_void_p) if cb else None, None, cands, 256,
                                 C.byref(nout), C.byref(sel)))
        out = []
        for i in range(min(nout.value, 256)):
            c = cands[i]
            out.append(dict(name=c.name.decode(), ordinal=c.ordinal, jl=c.jl, workers=c.workers,
                            correct=bool(c.correct), executions=c.executions,
                            best_seconds=c.best_seconds,
                            trial_seconds=list(c.trial_seconds[: c.n_trials])))
        return out, sel.value

    @staticmethod
    def gmres(n, rp, ci, v, b, m=30, tol=1e-8, max_iters=3000, ortho_kind=1, engine_workers=0):
        rp, ci, v = _csr(rp, ci, v)
        x = np.empty(n, np.float64)
        hist = np.zeros(max_iters + 1, np.float64)
        its, rs, calls = _I64(), _I64(), _I64()
        conv = C.c_int()
        rec, tru, sec, ssec = C.c_double(), C.c_double(), C.c_double(), C.c_double()
        _chk_ref(ref().kr_gmres(n, rp, ci, v, np.ascontiguousarray(b, np.float64), m, tol,
                                max_iters, ortho_kind, engine_workers, x, hist,
                                C.byref(its), C.byref(rs), C.byref(calls), C.byref(conv),
                                C.byref(rec), C.byref(tru), C.byref(sec), C.byref(ssec)))
        return x, dict(iterations=its.value, restarts=rs.value, spmv_calls=calls.value,
                       converged=bool(conv.value), recurrence_residual=rec.value,
                       true_residual=tru.value, seconds=sec.value, spmv_seconds=ssec.value,
                       history=hist[: its.value].copy())

    @staticmethod
    def ilu0_factorize(n, rp, ci, v):
        rp, ci, v = _csr(rp, ci, v)
        vals = np.empty(max(len(v), 1), np.float64)
        diag = np.empty(max(n, 1), np.int64)
        _chk_ref(ref().kr_ilu0_factorize(n, rp, ci, v, vals, diag))
        return vals[: len(v)], diag[:n]

    @staticmethod
    def ilu0_apply(n, rp, ci, fv, diag, r):
        rp, ci, fv = _csr(rp, ci, fv)
        z = np.empty(n, np.float64)
        _chk_ref(ref().kr_ilu0_apply(n, rp, ci, fv, np.ascontiguousarray(diag, np.int64),
                                     np.ascontiguousarray(r, np.float64), z))
        return z

    @staticmethod
    def gmres_ilu0(n, rp, ci, v, b, m=30, tol=1e-8, max_iters=3000, ortho_kind=1):
        """The reference's gmres_m with Precond = its ilu0_apply."""
        rp, ci, v = _csr(rp, ci, v)
        x = np.empty(n, np.float64)
        its, rs = _I64(), _I64()
        conv, tru = C.c_int(), C.c_double()
        _chk_ref(ref().kr_gmres_ilu0(n, rp, ci, v, np.ascontiguousarray(b, np.float64), m, tol,
                                     max_iters, ortho_kind, x, C.byref(its), C.byref(rs),
                                     C.byref(conv), C.byref(tru)))
        return x, dict(iterations=its.value, restarts=rs.value, converged=bool(conv.value),
                       true_residual=tru.value)

    @staticmethod
    def mm_probe(path):
        n, e, sym = _I64(), _I64(), C.c_int()
        _chk_ref(ref().kr_mm_probe(os.fsencode(path), C.byref(n), C.byref(e), C.byref(sym)))
        return n.value, e.value, bool(sym.value)

    @staticmethod
    def mm_load(path, want_symmetric):
        """load_matrix_market -> (kind, n, row_ptr, col_idx, values); kind 1 =
        SymCsrMatrix. Raises OracleError with the reference's message."""
        h = C.c_void_p()
        _chk_ref(ref().kr_mm_load(os.fsencode(path), 1 if want_symmetric else 0, C.byref(h)))
        try:
            n, nnz, kind = _I64(), _I64(), C.c_int()
            ref().kr_mm_info(h, C.byref(n), C.byref(nnz), C.byref(kind))
            rp = np.empty(n.value + 1, np.int64)
            ci = np.empty(max(nnz.value, 1), np.int64)
            v = np.empty(max(nnz.value, 1), np.float64)
            ref().kr_mm_copy(h, rp.ctypes.data, ci.ctypes.data, v.ctypes.data)
            return kind.value, n.value, rp, ci[: nnz.value], v[: nnz.value]
        finally:
            ref().kr_mm_destroy(h)

    @staticmethod
    def mm_write(path, n, rp, ci, v, sym):
        rp, ci, v = _csr(rp, ci, v)
        _chk_ref(ref().kr_mm_write(os.fsencode(path), n, rp, ci, v, 1 if sym else 0))


class RefEngine:
    """The reference's tuned engine (select_spmv_* + Unsym/SymEngine::op).
    ``select_seconds`` is the wall time of the reference's selection (plan
    builds + every candidate's warm-up and timed runs)."""

    def __init__(self, sym, n, rp, ci, v, pool_size, variant="parity", _handle=None):
        import time

        self.variant = variant
        self.L = ref(variant)
        t0 = time.perf_counter()
        if _handle is None:
            self._keep = _csr(rp, ci, v)
            h = C.c_void_p()
            _chk_ref(self.L.kr_engine_create(1 if sym else 0, n, *self._keep, pool_size,
                                             C.byref(h)), self.L)
        else:
            h = _handle
        self.select_seconds = time.perf_counter() - t0
        self.n = n
        self.nnz = int(rp[-1]) if rp is not None else None
        self.h = h
        name = C.create_string_buffer(8)
        jl, w, best = _I64(), C.c_int(), C.c_double()
        self.L.kr_engine_selected(h, name, C.byref(jl), C.byref(w), C.byref(best))
        self.selected = dict(name=name.value.decode(), jl=jl.value, workers=w.value,
                             best_seconds=best.value)

    @classmethod
    def stencil7(cls, nx, ny, nz, diag=6.0, off=-1.0, pool_size=1, variant="parity"):
        """The engine over the 7-point stencil built in place by the shim
        (kr_engine_create_stencil7): configs 1 and 4 at full size."""
        import time

        L = ref(variant)
        h = C.c_void_p()
        t0 = time.perf_counter()
        _chk_ref(L.kr_engine_create_stencil7(nx, ny, nz, diag, off, pool_size, C.byref(h)), L)
        e = cls(False, nx * ny * nz, None, None, None, pool_size, variant, _handle=h)
        e.select_seconds = time.perf_counter() - t0
        e.nnz = 7 * nx * ny * nz - 2 * (nx * ny + ny * nz + nx * nz)
        return e

    def report(self):
        """The TuningReport candidates (autotune.hpp:216-259)."""
        out = (_Cand * 64)()
        n, sel = C.c_int(), C.c_int()
        self.L.kr_engine_report(self.h, out, 64, C.byref(n), C.byref(sel))
        return [dict(name=c.name.decode(), jl=c.jl, workers=c.workers, correct=bool(c.correct),
                     best_seconds=c.best_seconds) for c in out[:n.value]], sel.value

    def apply(self, x: np.ndarray, y: np.ndarray) -> None:
        _chk_ref(self.L.kr_engine_apply(self.h, x.ctypes.data, y.ctypes.data), self.L)

    def close(self):
        if self.h:
            self.L.kr_engine_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
