"""Host-side mirror of the reference's SpMV operator interface (namespace
``ktune``, /root/reference/proj/include/ktune/*.hpp) running on the B200
engine behind the C ABI (include/ktb.h).

Same names, argument meaning and error wording as the reference:

===========================  ==============================================
reference                    here
===========================  ==============================================
CsrMatrix / SymCsrMatrix     CsrMatrix / SymCsrMatrix (csr.hpp:13-65)
build_row_partition          build_row_partition (partition.hpp:28-55)
build_reduction_regions      build_reduction_regions (partition.hpp:73-96)
build_bss_plan               build_bss_plan (bss.hpp:34-69)
expand_symmetric             expand_symmetric (csr.hpp:88-123)
spmv_unsym / spmv_sym        spmv_unsym / spmv_sym (spmv.hpp:111-234)
select_spmv_unsym / _sym     select_spmv_unsym / _sym (autotune.hpp:267-377)
UnsymEngine / SymEngine      UnsymEngine / SymEngine (meta.hpp:20-82)
LinOp, make_ref_op           LinOp (solver_types.hpp:17-31)
ktune::Error                 Error
===========================  ==============================================

Every plan artefact (partition boundaries, regions, BSS flags/slices) is
computed by device kernels and is bit-exact with the reference builders;
every SpMV runs on the GPU. There is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import enum
import threading
import time
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from . import _lib

_DEV_LOCK = threading.Lock()  # lazy device uploads (CsrMatrix.dev)

I64 = C.c_int64


class Error(RuntimeError):
    """ktune::Error (common.hpp:18-21): contract violations."""


class CudaError(RuntimeError):
    pass


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = _lib.load().ktb_last_error().decode()
    if rc == 1:
        raise Error(msg)
    if rc == 3:
        raise Error(msg)
    raise CudaError(msg)


def require(cond: bool, msg: str) -> None:  # common.hpp:23-25
    if not cond:
        raise Error(msg)


class UnsymKernel(enum.IntEnum):  # spmv.hpp:15
    u1_row = 0
    u2_nnz = 1
    u3_bss = 2
    u4_ss = 3


class SymKernel(enum.IntEnum):  # spmv.hpp:16 (ABI tags 16..18)
    s1_row = 16
    s2_nnz = 17
    s3_nnz_zero_omit = 18


class PartitionScheme(enum.IntEnum):  # partition.hpp:12
    row_based = 0
    nnz_balanced = 1


def kernel_name(k) -> str:  # spmv.hpp:18-35
    return {0: "u1", 1: "u2", 2: "u3", 3: "u4", 16: "s1", 17: "s2", 18: "s3"}[int(k)]


# ------------------------------------------------------------------ storage
class _DeviceMatrix:
    """Owner of a ktb_matrix handle."""

    def __init__(self, handle: C.c_void_p, owned: bool = True):
        self.h = handle
        self.owned = owned  # borrowed handles (e.g. a ktb_dist's A_d) are not destroyed here
        n, nnz, mx, bw = I64(), I64(), I64(), I64()
        kind = C.c_int()
        _check(_lib.load().ktb_matrix_info(handle, C.byref(n), C.byref(nnz), C.byref(kind),
                                           C.byref(mx), C.byref(bw)))
        self.n, self.nnz, self.kind = n.value, nnz.value, kind.value
        self.max_row_nnz, self.bandwidth = mx.value, bw.value

    def close(self):
        if getattr(self, "h", None):
            if self.owned:
                _lib.load().ktb_matrix_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def download(self):
        rp = np.empty(self.n + 1, np.int32)
        ci = np.empty(max(self.nnz, 1), np.int32)
        v = np.empty(max(self.nnz, 1), np.float64)
        _check(_lib.load().ktb_matrix_download(self.h, rp.ctypes.data, ci.ctypes.data,
                                               v.ctypes.data))
        return rp, ci[: self.nnz], v[: self.nnz]


@dataclass
class CsrMatrix:
    """csr.hpp:13-55: square CRS, int64 indices, fp64 values. Construction
    validates (csr.hpp:38-54) and uploads to the device once."""

    n: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray
    device: int = 0
    _kind: int = field(default=0, repr=False)
    _dev: Optional[_DeviceMatrix] = field(default=None, repr=False)

    def __post_init__(self):
        self.row_ptr = np.ascontiguousarray(self.row_ptr, np.int64)
        self.col_idx = np.ascontiguousarray(self.col_idx, np.int64)
        self.values = np.ascontiguousarray(self.values, np.float64)

    def nnz(self) -> int:
        return len(self.values)

    def row_nnz(self, i: int) -> int:
        return int(self.row_ptr[i + 1] - self.row_ptr[i])

    def max_row_nnz(self) -> int:
        return int(np.max(np.diff(self.row_ptr))) if self.n > 0 else 0

    def storage_bytes(self) -> int:  # csr.hpp:30-33
        return 8 * (len(self.row_ptr) + len(self.col_idx) + len(self.values))

    @property
    def dev(self) -> _DeviceMatrix:
        if self._dev is not None:
            return self._dev
        with _DEV_LOCK:  # one upload even when several threads ask at once
            if self._dev is not None:
                return self._dev
            # csr.hpp:39-43 length checks the C ABI cannot see
            require(self.n >= 0, "csr: negative dimension")
            require(len(self.row_ptr) == self.n + 1, "csr: row_ptr length != n+1")
            require(len(self.col_idx) == len(self.values), "csr: col_idx/values length mismatch")
            require(self.row_ptr[0] == 0, "csr: row_ptr[0] != 0")
            require(self.row_ptr[-1] == len(self.values), "csr: row_ptr[n] != nnz")
            h = C.c_void_p()
            _check(_lib.load().ktb_matrix_create(self.n, self.row_ptr.ctypes.data,
                                                 self.col_idx.ctypes.data,
                                                 self.values.ctypes.data, self._kind,
                                                 self.device, C.byref(h)))
            self._dev = _DeviceMatrix(h)
            return self._dev

    def validate(self) -> None:
        _ = self.dev


@dataclass
class SymCsrMatrix(CsrMatrix):
    """csr.hpp:57-65: diagonal + strict upper; A = U + U^T - diag(U)."""

    _kind: int = field(default=1, repr=False)

    def spmv_flops(self) -> int:  # csr.hpp:64
        return 4 * self.nnz() - 2 * self.n


class DeviceCsr:
    """A matrix generated directly on the device (SURVEY.md §8d recipes);
    behaves like CsrMatrix/SymCsrMatrix for every call here."""

    def __init__(self, handle: C.c_void_p, sym: bool, owner=None):
        self._owner = owner  # keeps the owner of a borrowed handle alive
        self._dev = _DeviceMatrix(handle, owned=owner is None)
        self._kind = 1 if sym else 0
        self.n = self._dev.n

    @property
    def dev(self):
        return self._dev

    def nnz(self) -> int:
        return self._dev.nnz

    def spmv_flops(self) -> int:
        return 4 * self.nnz() - 2 * self.n if self._kind else 2 * self.nnz()

    def to_host(self):
        rp, ci, v = self._dev.download()
        return rp.astype(np.int64), ci.astype(np.int64), v

    def slice_rows(self, r0: int, r1: int) -> "DeviceCsr":
        """Rows [r0, r1) as a new device matrix (same column space)."""
        h = C.c_void_p()
        _check(_lib.load().ktb_matrix_slice(self._dev.h, r0, r1, C.byref(h)))
        return DeviceCsr(h, False)


def stencil7(nx, ny, nz, diag=6.0, off=-1.0, c_xm=None, c_xp=None, device=0) -> DeviceCsr:
    h = C.c_void_p()
    _check(_lib.load().ktb_gen_stencil7(nx, ny, nz, diag, off, off if c_xm is None else c_xm,
                                        off if c_xp is None else c_xp, device, C.byref(h)))
    return DeviceCsr(h, False)


def stencil27_upper(nx, ny, nz, diag=26.0, off=-1.0, device=0) -> DeviceCsr:
    h = C.c_void_p()
    _check(_lib.load().ktb_gen_stencil27_upper(nx, ny, nz, diag, off, device, C.byref(h)))
    return DeviceCsr(h, True)


def powerlaw(n=4_000_000, seed=3, target_nnz=40_000_000, empty_frac=0.1, max_len=65536,
             device=0) -> DeviceCsr:
    """Config 3 (BASELINE.json configs[2]): irregular power-law matrix."""
    h = C.c_void_p()
    _check(_lib.load().ktb_gen_powerlaw(n, seed, target_nnz, empty_frac, max_len, device,
                                        C.byref(h)))
    return DeviceCsr(h, False)


def powerlaw_host(n=4_000_000, seed=3, target_nnz=40_000_000, empty_frac=0.1, max_len=65536):
    """Host arrays of the same matrix (int64 row_ptr, int64 cols, fp64 values)."""
    L = _lib.load()
    rp = np.empty(n + 1, np.int64)
    _check(L.ktb_gen_powerlaw_host(n, seed, target_nnz, empty_frac, max_len, rp.ctypes.data,
                                   None, None))
    nnz = int(rp[-1])
    ci = np.empty(max(nnz, 1), np.int32)
    v = np.empty(max(nnz, 1), np.float64)
    _check(L.ktb_gen_powerlaw_host(n, seed, target_nnz, empty_frac, max_len, rp.ctypes.data,
                                   ci.ctypes.data, v.ctypes.data))
    return n, rp, ci[:nnz].astype(np.int64), v[:nnz]


def stencil7_slab(nx, ny, nz, z0, z1, diag=6.0, off=-1.0, device=0) -> DeviceCsr:
    h = C.c_void_p()
    _check(_lib.load().ktb_gen_stencil7_slab(nx, ny, nz, z0, z1, diag, off, device,
                                             C.byref(h)))
    return DeviceCsr(h, False)


# ---------------------------------------------------------- Matrix Market
@dataclass
class MmInfo:  # matrix_market.hpp:18-22
    n: int = 0
    entries: int = 0
    symmetric: bool = False


def _path(path) -> bytes:
    import os

    return os.fsencode(path)


def probe_matrix_market(path) -> MmInfo:  # matrix_market.hpp:154-158
    n, e, s = I64(), I64(), C.c_int()
    _check(_lib.load().ktb_mm_probe(_path(path), C.byref(n), C.byref(e), C.byref(s)))
    return MmInfo(n.value, e.value, bool(s.value))


class _HostCsr:
    """Owner of a ktb_csr_host handle (the parsed file, int64 host CRS)."""

    def __init__(self, path, want_symmetric: bool):
        self.h = C.c_void_p()
        _check(_lib.load().ktb_mm_read(_path(path), int(bool(want_symmetric)), C.byref(self.h)))
        n, nnz, kind = I64(), I64(), C.c_int()
        _check(_lib.load().ktb_csr_host_info(self.h, C.byref(n), C.byref(nnz), C.byref(kind)))
        self.n, self.nnz, self.kind = n.value, nnz.value, kind.value

    def arrays(self):
        rp = np.empty(self.n + 1, np.int64)
        ci = np.empty(max(self.nnz, 1), np.int64)
        v = np.empty(max(self.nnz, 1), np.float64)
        _check(_lib.load().ktb_csr_host_copy(self.h, rp.ctypes.data, ci.ctypes.data,
                                             v.ctypes.data))
        return rp, ci[: self.nnz], v[: self.nnz]

    def __del__(self):
        if getattr(self, "h", None):
            _lib.load().ktb_csr_host_destroy(self.h)
            self.h = None


def load_matrix_market(path, want_symmetric: bool, device: int = 0):
    """matrix_market.hpp:165-194: SymCsrMatrix when want_symmetric (a general
    file must then be exactly symmetric), else CsrMatrix (a symmetric file is
    expanded). Same messages as the reference."""
    h = _HostCsr(path, want_symmetric)
    rp, ci, v = h.arrays()
    cls = SymCsrMatrix if h.kind == 1 else CsrMatrix
    return cls(h.n, rp, ci, v, device=device)


def load_matrix_market_general(path, device: int = 0) -> CsrMatrix:  # :196-198
    return load_matrix_market(path, False, device)


def load_matrix_market_symmetric(path, device: int = 0) -> SymCsrMatrix:  # :200-202
    return load_matrix_market(path, True, device)


def load_matrix_market_device(path, want_symmetric: bool, device: int = 0) -> DeviceCsr:
    """Parse and upload straight to the device (no numpy copy of the CRS)."""
    h = _HostCsr(path, want_symmetric)
    d = C.c_void_p()
    _check(_lib.load().ktb_csr_host_upload(h.h, device, C.byref(d)))
    return DeviceCsr(d, h.kind == 1)


def write_matrix_market(path, a) -> None:
    """matrix_market.hpp:223-239: a CsrMatrix writes "general", a
    SymCsrMatrix its upper storage transposed ("symmetric", lower form)."""
    if isinstance(a, DeviceCsr):
        rp, ci, v = a.to_host()
        n, kind = a.n, a._kind
    else:
        rp, ci, v, n, kind = a.row_ptr, a.col_idx, a.values, a.n, a._kind
    rp = np.ascontiguousarray(rp, np.int64)
    require(len(rp) == n + 1, "csr: row_ptr length != n+1")
    ci = np.ascontiguousarray(ci, np.int64)
    v = np.ascontiguousarray(v, np.float64)
    require(len(ci) == len(v), "csr: col_idx/values length mismatch")
    require(rp[-1] == len(v), "csr: row_ptr[n] != nnz")
    _check(_lib.load().ktb_mm_write(_path(path), n, rp.ctypes.data, ci.ctypes.data,
                                    v.ctypes.data, kind))


# ----------------------------------------------------------------- ILU(0)
class IluFactors:
    """ilu0.hpp:14-18 IluFactors, resident on the device (ktb_ilu): the
    combined unit-L / U factors on A's pattern plus the level schedules of
    the two triangular sweeps."""

    def __init__(self, handle, a):
        self.h, self.a = handle, a
        n, nl, nu, la = I64(), I64(), I64(), I64()
        _check(_lib.load().ktb_ilu0_info(handle, C.byref(n), C.byref(nl), C.byref(nu),
                                         C.byref(la)))
        self.n, self.lower_levels, self.upper_levels = n.value, nl.value, nu.value
        self.launches_per_apply = la.value

    def download(self):
        """(diag_ptr int64[n], values fp64[nnz]) -- the reference's fields."""
        nnz = self.a.nnz()
        d = np.empty(max(self.n, 1), np.int32)
        v = np.empty(max(nnz, 1), np.float64)
        _check(_lib.load().ktb_ilu0_download(self.h, d.ctypes.data, v.ctypes.data))
        return d[: self.n].astype(np.int64), v[:nnz]

    def apply(self, r, z) -> None:
        if isinstance(r, np.ndarray):
            require(len(r) == self.n and len(z) == self.n, "ilu0: dimension mismatch")
            r = np.ascontiguousarray(r, np.float64)
            _check(_lib.load().ktb_ilu0_apply(self.h, r.ctypes.data, z.ctypes.data, 0, None))
        else:
            import torch

            require(r.shape[0] == self.n and z.shape[0] == self.n, "ilu0: dimension mismatch")
            s = torch.cuda.current_stream(r.device).cuda_stream
            _check(_lib.load().ktb_ilu0_apply(self.h, _dptr(r), _dptr(z), 1, s))

    def __del__(self):
        if getattr(self, "h", None):
            try:
                _lib.load().ktb_ilu0_destroy(self.h)
            except Exception:
                pass
            self.h = None


def ilu0_factorize(a) -> IluFactors:
    """ilu0.hpp:23-69 on the device; same failure messages."""
    h = C.c_void_p()
    _check(_lib.load().ktb_ilu0_create(a.dev.h, None, C.byref(h)))
    return IluFactors(h, a)


def ilu0_apply(f: IluFactors, r, z=None):
    """ilu0.hpp:73-93: z = (LU)^{-1} r (allocating form when z is None)."""
    if z is None:
        z = np.empty(f.n, np.float64) if isinstance(r, np.ndarray) else _like(r, f.n)
    f.apply(r, z)
    return z


# -------------------------------------------------------------- artefacts
@dataclass
class RowPartition:  # partition.hpp:15-23
    num_workers: int
    boundaries: np.ndarray
    scheme: PartitionScheme
    n: int = -1

    def lo(self, p):
        return int(self.boundaries[p])

    def hi(self, p):
        return int(self.boundaries[p + 1])

    def rows(self):
        return int(self.boundaries[-1])


@dataclass
class ReductionRegions:  # partition.hpp:60-71
    num_workers: int
    lo: np.ndarray
    hi: np.ndarray

    def total_width(self) -> int:
        return int(np.sum(self.hi - self.lo))


@dataclass
class BssPlan:  # bss.hpp:19-32
    jl: int
    n: int
    nnz: int
    slice_start: np.ndarray
    slice_len: np.ndarray
    slice_row: np.ndarray
    lane_slice_ptr: np.ndarray
    row_slice_ptr: np.ndarray
    row_start_flag: np.ndarray

    def total_slices(self) -> int:
        return len(self.slice_start)


def build_row_partition(a, num_workers: int, scheme) -> RowPartition:
    """partition.hpp:28-55 on the device. `a` is a matrix (the reference takes
    its row_ptr span)."""
    require(num_workers >= 1, "row partition: num_workers must be >= 1")
    out = np.empty(num_workers + 1, np.int64)
    _check(_lib.load().ktb_row_partition(a.dev.h, num_workers, int(scheme), out.ctypes.data))
    return RowPartition(num_workers, out, PartitionScheme(int(scheme)), a.n)


def build_reduction_regions(a, part: RowPartition) -> ReductionRegions:
    require(part.rows() == a.n, "reduction regions: partition/matrix dimension mismatch")
    P = part.num_workers
    lo, hi = np.empty(P, np.int64), np.empty(P, np.int64)
    b = np.ascontiguousarray(part.boundaries, np.int64)
    _check(_lib.load().ktb_reduction_regions(a.dev.h, P, b.ctypes.data, lo.ctypes.data,
                                             hi.ctypes.data))
    return ReductionRegions(P, lo, hi)


def build_bss_plan(a, jl: int) -> BssPlan:
    require(jl >= 1, "bss plan: jl must be >= 1")
    require(a.nnz() > 0, "bss plan: empty matrix")
    L = _lib.load()
    je, tot = I64(), I64()
    _check(L.ktb_bss_plan_size(a.dev.h, jl, C.byref(je), C.byref(tot)))
    T, J, n, nnz = tot.value, je.value, a.n, a.nnz()
    arr = [np.empty(T, np.int64) for _ in range(3)]
    lane = np.empty(J + 1, np.int64)
    rsp = np.empty(n + 1, np.int64)
    flag = np.empty(nnz, np.uint8)
    _check(L.ktb_bss_plan_copy(a.dev.h, jl, arr[0].ctypes.data, arr[1].ctypes.data,
                               arr[2].ctypes.data, lane.ctypes.data, rsp.ctypes.data,
                               flag.ctypes.data))
    return BssPlan(J, n, nnz, arr[0], arr[1], arr[2], lane, rsp, flag)


def expand_symmetric(a) -> DeviceCsr:
    require(a._kind == 1, "expand_symmetric: matrix is not symmetric storage")
    h = C.c_void_p()
    _check(_lib.load().ktb_expand_symmetric(a.dev.h, C.byref(h)))
    return DeviceCsr(h, False)


# ------------------------------------------------------------------ plans
class DevicePlan:
    """ktb_plan: a kernel bound to its device decomposition and stream."""

    def __init__(self, a, kernel: int, param: int = 0, workers: int = 0, stream=None,
                 handle=None):
        self.a = a  # keep the matrix alive (engines hold a reference, meta.hpp:44)
        self.n = a.n
        if handle is None:
            h = C.c_void_p()
            _check(_lib.load().ktb_plan_create(a.dev.h, int(kernel), int(param), int(workers),
                                               stream, C.byref(h)))
            handle = h
        self.h = handle
        k, prm, ctas, launches, extra = C.c_int(), I64(), I64(), C.c_int(), I64()
        _check(_lib.load().ktb_plan_info(self.h, C.byref(k), C.byref(prm), C.byref(ctas),
                                         C.byref(launches), C.byref(extra)))
        self.kernel, self.param, self.ctas = k.value, prm.value, ctas.value
        self.launches, self.extra_bytes = launches.value, extra.value

    def s3_info(self) -> dict:
        """S3 layout facts (ktb_plan_s3_info): far entries, long rows, patch
        target rows, spill doubles, window length, SELL slots."""
        v = [I64() for _ in range(4)]
        w, slots = C.c_int(), I64()
        _check(_lib.load().ktb_plan_s3_info(self.h, *[C.byref(q) for q in v], C.byref(w),
                                            C.byref(slots)))
        return dict(far=v[0].value, long_rows=v[1].value, patch_rows=v[2].value,
                    spill=v[3].value, window=w.value, slots=slots.value)

    def set_stream(self, stream) -> None:
        _check(_lib.load().ktb_plan_set_stream(self.h, stream))
        self._stream = stream

    def apply(self, x, y) -> None:
        """y = A x. numpy arrays -> host-span mode (copies, synchronous);
        torch CUDA tensors or raw device pointers (int) -> device mode."""
        if isinstance(x, np.ndarray):
            require(x.dtype == np.float64 and y.dtype == np.float64 and x.flags.c_contiguous
                    and y.flags.c_contiguous, "spmv: dimension mismatch")
            _check(_lib.load().ktb_spmv(self.h, x.ctypes.data, y.ctypes.data, 0))
        else:
            self._follow_torch_stream(x)
            _check(_lib.load().ktb_spmv(self.h, _dptr(x), _dptr(y), 1))

    def _follow_torch_stream(self, t) -> None:
        """Device mode runs on the caller's current torch stream so it is
        ordered with the producer of x and the consumer of y."""
        if hasattr(t, "data_ptr"):
            import torch

            s = torch.cuda.current_stream(t.device).cuda_stream
            if s != getattr(self, "_stream", None):
                self.set_stream(s)
                self._stream = s

    def apply_host_pipelined(self, x, y, count=None) -> None:
        """y_k = A x_k for host vectors (rows of 2-D float64 arrays, or one
        1-D vector reused `count` times -- still copied every time): host->
        device copy of k+1 and device->host copy of k-1 overlap the SpMV of k
        (ktb_spmv_host_pipelined). Pinned host memory gives the overlap."""
        x, y = np.asarray(x), np.asarray(y)
        require(x.dtype == np.float64 and y.dtype == np.float64 and x.flags.c_contiguous
                and y.flags.c_contiguous, "spmv: dimension mismatch")
        if x.ndim == 1:
            require(count is not None and x.shape[0] == self.a.n, "spmv: dimension mismatch")
            cnt, ldx = int(count), 0
        else:
            cnt, ldx = x.shape[0], x.shape[1]
            require(ldx == self.a.n, "spmv: dimension mismatch")
        if y.ndim == 1:
            require(y.shape[0] == self.a.n, "spmv: dimension mismatch")
            ldy = 0
        else:
            require(y.shape[0] == cnt and y.shape[1] == self.a.n, "spmv: dimension mismatch")
            ldy = y.shape[1]
        _check(_lib.load().ktb_spmv_host_pipelined(self.h, cnt, x.ctypes.data, ldx,
                                                   y.ctypes.data, ldy))

    def apply_rows(self, r0, r1, x, y) -> None:
        self._follow_torch_stream(x)
        _check(_lib.load().ktb_spmv_rows(self.h, r0, r1, _dptr(x), _dptr(y)))

    def time(self, x, y, reps=20, flush_bytes=0):
        self._follow_torch_stream(x)
        avg, mn = C.c_double(), C.c_double()
        _check(_lib.load().ktb_time_spmv(self.h, _dptr(x), _dptr(y), reps, flush_bytes,
                                         C.byref(avg), C.byref(mn)))
        return avg.value, mn.value

    def close(self):
        if getattr(self, "h", None):
            _lib.load().ktb_plan_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _dptr(t) -> int:
    if isinstance(t, int):
        return t
    if hasattr(t, "data_ptr"):
        require(bool(getattr(t, "is_cuda", False)), "spmv: device mode needs CUDA tensors")
        return int(t.data_ptr())
    raise Error("spmv: unsupported vector type")


_plan_cache: dict = {}


def _plan_for(a, kernel, param=0, workers=0) -> DevicePlan:
    key = (id(a.dev), int(kernel), int(param), int(workers))
    p = _plan_cache.get(key)
    if p is None or p.a is not a:
        p = DevicePlan(a, kernel, param, workers)
        _plan_cache[key] = p
    return p


def _len(v) -> int:
    return int(v.shape[0]) if hasattr(v, "shape") else len(v)


def spmv_unsym(kernel, a, part: Optional[RowPartition], plan: Optional[BssPlan], x, y=None):
    """spmv.hpp:111-170: same contract checks and messages, then the GPU
    kernel for the variant (U1 vector-per-row, U2 merge-path, U3 BSS, U4 flag
    scan). Allocating form when y is None (spmv.hpp:238-244)."""
    kernel = UnsymKernel(int(kernel))
    if y is None:
        y = np.empty(a.n, np.float64) if isinstance(x, np.ndarray) else _like(x, a.n)
    require(_len(x) == a.n and _len(y) == a.n, "spmv: dimension mismatch")
    if kernel in (UnsymKernel.u1_row, UnsymKernel.u2_nnz):
        require(part is not None, "spmv: U1/U2 need a row partition")
        require(part.rows() == a.n, "spmv: partition built for a different matrix")
        want = (PartitionScheme.row_based if kernel == UnsymKernel.u1_row
                else PartitionScheme.nnz_balanced)
        require(part.scheme == want, "spmv: partition scheme does not match kernel")
        _plan_for(a, kernel).apply(x, y)
    else:
        require(plan is not None, "spmv: U3/U4 need a bss plan")
        require(plan.n == a.n and plan.nnz == a.nnz(), "spmv: plan built for a different matrix")
        _plan_for(a, kernel).apply(x, y)
    return y


def spmv_sym(kernel, a, part: RowPartition, regions: Optional[ReductionRegions], x, y=None):
    """spmv.hpp:180-234 contract, GPU kernels S1/S2 (atomic full-range) and
    S3 (zero-omission smem window)."""
    kernel = SymKernel(int(kernel))
    if y is None:
        y = np.empty(a.n, np.float64) if isinstance(x, np.ndarray) else _like(x, a.n)
    require(_len(x) == a.n and _len(y) == a.n, "spmv: dimension mismatch")
    require(part.rows() == a.n, "spmv: partition built for a different matrix")
    want = PartitionScheme.row_based if kernel == SymKernel.s1_row else PartitionScheme.nnz_balanced
    require(part.scheme == want, "spmv: partition scheme does not match kernel")
    omit = kernel == SymKernel.s3_nnz_zero_omit
    require(not omit or regions is not None, "spmv: S3 needs reduction regions")
    if omit:
        require(regions.num_workers == part.num_workers,
                "spmv: regions built for a different partition")
    _plan_for(a, kernel).apply(x, y)
    return y


def _like(x, n):
    import torch

    return torch.empty(n, dtype=torch.float64, device=x.device)


# --------------------------------------------------------------- selector
@dataclass
class TuningCandidate:  # autotune.hpp:130-139
    name: str
    ordinal: int
    jl: int
    workers: int
    trial_seconds: list
    best_seconds: float
    correct: bool
    executions: int
    cta_threads: int = 0       # launch shape timed (0 = the kernel's default)
    setup_seconds: float = 0.0  # plan build before the warm-up


@dataclass
class TuningReport:  # autotune.hpp:141-158
    candidates: list
    selected: int = -1
    trials_per_candidate: int = 3
    forced: bool = False

    def max_executions(self) -> int:
        return max((c.executions for c in self.candidates), default=0)

    def selected_candidate(self) -> TuningCandidate:
        require(0 <= self.selected < len(self.candidates), "tuning report: nothing selected")
        return self.candidates[self.selected]


@dataclass
class SelectOptions:  # autotune.hpp:160-165
    jl_candidates: Optional[list] = None  # GPU: nonzeros per BSS lane (jl = nnz / E)
    timed_trials: int = 3
    sweep_workers: bool = False
    now: Optional[Callable[[], float]] = None
    warm_trials: bool = False  # True: back-to-back trials (the reference's protocol)


class _Cand(C.Structure):
    _fields_ = [("name", C.c_char * 8), ("ordinal", C.c_int), ("param", I64),
                ("workers", C.c_int), ("correct", C.c_int), ("executions", C.c_int),
                ("n_trials", C.c_int), ("best_seconds", C.c_double),
                ("trial_seconds", C.c_double * 8), ("cta_threads", C.c_int),
                ("setup_seconds", C.c_double)]


class _Opts(C.Structure):
    _fields_ = [("params", C.c_void_p), ("n_params", C.c_int), ("timed_trials", C.c_int),
                ("workers", C.c_int), ("now", C.c_void_p), ("now_ctx", C.c_void_p),
                ("warm_trials", C.c_int)]


_NOW = C.CFUNCTYPE(C.c_double, C.c_void_p)


@dataclass
class UnsymChoice:  # autotune.hpp:168-175
    kernel: UnsymKernel
    jl: int
    workers: int
    plan: DevicePlan


@dataclass
class SymChoice:  # autotune.hpp:177-183
    kernel: SymKernel
    workers: int
    plan: DevicePlan


def _select(a, opts: Optional[SelectOptions]):
    require(a.n > 0 and a.nnz() > 0, "kernel selection: empty matrix")
    opts = opts or SelectOptions()
    o = _Opts()
    params = None
    if opts.jl_candidates:
        params = np.ascontiguousarray(opts.jl_candidates, np.int64)
        o.params, o.n_params = params.ctypes.data, len(params)
    o.timed_trials = opts.timed_trials
    o.warm_trials = int(bool(opts.warm_trials))
    cb = None
    if opts.now is not None:
        cb = _NOW(lambda _ctx: float(opts.now()))
        o.now = C.cast(cb, C.c_void_p)
    cands = (_Cand * 64)()
    nc, sel = C.c_int(), C.c_int()
    h = C.c_void_p()
    _check(_lib.load().ktb_select(a.dev.h, C.byref(o), None, C.byref(h), cands, 64,
                                  C.byref(nc), C.byref(sel)))
    rep = TuningReport([], sel.value, opts.timed_trials)
    for i in range(nc.value):
        c = cands[i]
        rep.candidates.append(TuningCandidate(c.name.decode(), c.ordinal, c.param, c.workers,
                                              list(c.trial_seconds[: c.n_trials]),
                                              c.best_seconds, bool(c.correct), c.executions,
                                              c.cta_threads, c.setup_seconds))
    return DevicePlan(a, 0, handle=h), rep


def select_spmv_unsym(a, pool=None, opts: Optional[SelectOptions] = None):
    """autotune.hpp:267-330 on device time; returns (UnsymChoice, TuningReport)."""
    plan, rep = _select(a, opts)
    w = rep.selected_candidate()
    return UnsymChoice(UnsymKernel(plan.kernel), w.jl, w.workers, plan), rep


def select_spmv_sym(a, pool=None, opts: Optional[SelectOptions] = None):
    """autotune.hpp:333-377 on device time; returns (SymChoice, TuningReport)."""
    plan, rep = _select(a, opts)
    w = rep.selected_candidate()
    return SymChoice(SymKernel(plan.kernel), w.workers, plan), rep


# ----------------------------------------------------------------- engines
@dataclass
class LinOp:  # solver_types.hpp:17-20
    n: int
    apply: Callable


class _Engine:
    def __init__(self, a, choice):
        self.a = a
        self.choice = choice
        self._calls = 0
        self._seconds = 0.0

    def op(self) -> LinOp:
        """meta.hpp:25-35: a LinOp that runs the tuned kernel, counting calls
        and in-kernel seconds (host spans -> H2D/D2H inside)."""

        def apply(x, y):
            t0 = time.perf_counter()
            self.choice.plan.apply(x, y)
            self._seconds += time.perf_counter() - t0
            self._calls += 1

        return LinOp(self.a.n, apply)

    def calls(self) -> int:
        return self._calls

    def kernel_seconds(self) -> float:
        return self._seconds

    def workers(self) -> int:
        return self.choice.workers


class UnsymEngine(_Engine):  # meta.hpp:20-49
    def flops_per_call(self) -> float:
        return 2.0 * self.a.nnz()


class SymEngine(_Engine):  # meta.hpp:51-82
    def flops_per_call(self) -> float:
        return float(self.a.spmv_flops())


def make_ref_op(a) -> LinOp:
    """solver_types.hpp:29-31 -- here backed by the device U1 kernel; the
    CPU oracle lives in oracle/ (tests only)."""
    plan = _plan_for(a, SymKernel.s3_nnz_zero_omit if a._kind else UnsymKernel.u1_row)
    return LinOp(a.n, plan.apply)


# ------------------------------------------------------------------ GMRES
@dataclass
class KrylovConfig:  # solver_types.hpp:44-57 (MGS, no restart adaptation)
    restart_m: int = 30
    m_max: int = 30
    tol: float = 1e-8
    max_iters: int = 10000


@dataclass
class SolverResult:  # solver_types.hpp:64-77
    x: np.ndarray
    converged: bool
    breakdown: bool
    fault_convergence: bool
    iterations: int
    restarts: int
    recurrence_residual: float
    true_residual: float
    residual_history: np.ndarray
    elapsed_seconds: float
    spmv_calls: int
    spmv_seconds: float


class _GmresRes(C.Structure):
    _fields_ = [("iterations", I64), ("restarts", I64), ("spmv_calls", I64),
                ("converged", C.c_int), ("breakdown", C.c_int), ("fault_convergence", C.c_int),
                ("recurrence_residual", C.c_double), ("true_residual", C.c_double),
                ("seconds", C.c_double), ("spmv_seconds", C.c_double)]


def gmres_m(a, b, cfg: KrylovConfig = KrylovConfig(), plan: Optional[DevicePlan] = None,
            precond: Optional["IluFactors"] = None):
    """gmres.hpp:16-173 (GMRES(m), MGS, x0 = 0) with every vector in HBM and
    the SpMV on `plan` (default: the device-time selected kernel); `precond`
    = ILU(0) factors (ilu0_factorize) as the right preconditioner."""
    require(len(b) == a.n, "gmres: dimension mismatch")
    require(1 <= cfg.restart_m <= cfg.m_max, "gmres: need 1 <= m <= m_max")
    require(cfg.tol > 0.0, "gmres: tol must be positive")
    if plan is None:
        plan = select_spmv_unsym(a)[0].plan
    b = np.ascontiguousarray(b, np.float64)
    x = np.empty(a.n, np.float64)
    hist = np.zeros(max(cfg.max_iters, 1), np.float64)
    r = _GmresRes()
    if precond is None:
        _check(_lib.load().ktb_gmres(plan.h, b.ctypes.data, x.ctypes.data, cfg.restart_m,
                                     cfg.tol, cfg.max_iters, hist.ctypes.data, C.byref(r)))
    else:
        _check(_lib.load().ktb_gmres_ilu0(plan.h, precond.h, b.ctypes.data, x.ctypes.data,
                                          cfg.restart_m, cfg.tol, cfg.max_iters,
                                          hist.ctypes.data, C.byref(r)))
    return SolverResult(x, bool(r.converged), bool(r.breakdown), bool(r.fault_convergence),
                        r.iterations, r.restarts, r.recurrence_residual, r.true_residual,
                        hist[: r.iterations].copy(), r.seconds, r.spmv_calls, r.spmv_seconds)
