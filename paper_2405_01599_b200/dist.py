"""Row-block sharding of SpMV across GPUs: the
Python face of libktb's native data plane (csrc/ktb_comm.cu).

The reference has no distributed path; this is the B200
framework's scale-out of spmv_unsym (spmv.hpp:111): each rank owns a
contiguous row block and the same entries of x and y (y stays row-sharded:
no reduction collective). Two operators, both native C++ behind the C ABI:

* ``DistSpMV`` (config 4): z-slab of the 3-D 7-point stencil, local x laid
  out [halo_lo plane | owned planes | halo_hi plane]; per apply one NCCL
  group (send the owned edge planes, receive the halos in place) on a
  high-priority stream, overlapped with the interior rows; the boundary
  planes run after an event wait (ktb_halo_spmv).
* ``DistCsrSpMV`` (any CRS): NNZ_BALANCED row blocks split into A_d (owned
  columns, any tuned kernel) and A_o (ghost columns); ghost lists exchanged
  once; per apply pack -> NCCL ghost exchange overlapped with A_d x ->
  y += A_o x_ghost (ktb_dist_spmv).

The communicator is ``Comm``: NCCL (``Comm.nccl``; torch.distributed only
hands the unique id around) or, for single-GPU checks of the same native
code, an in-process loopback world (``Comm.loopback`` + ``run_ranks``).

``SlabLayout`` / ``halo_plan`` / ``halo_exchange`` / ``exchange_ghost_lists``
restate the native protocol in Python over torch.distributed so that the
multi-rank logic is testable on CPU ranks with the gloo backend.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class SlabLayout:
    nx: int
    ny: int
    nz: int
    rank: int
    world: int

    @property
    def plane(self) -> int:
        return self.nx * self.ny

    @property
    def z0(self) -> int:
        return self.rank * self.nz // self.world

    @property
    def z1(self) -> int:
        return (self.rank + 1) * self.nz // self.world

    @property
    def has_lo(self) -> bool:
        return self.z0 > 0

    @property
    def has_hi(self) -> bool:
        return self.z1 < self.nz

    @property
    def n_local(self) -> int:
        return (self.z1 - self.z0) * self.plane

    @property
    def row0(self) -> int:  # first owned global row
        return self.z0 * self.plane

    @property
    def owned_offset(self) -> int:  # owned x starts here in the local x buffer
        return self.plane if self.has_lo else 0

    @property
    def x_local_len(self) -> int:
        return self.n_local + self.plane * (int(self.has_lo) + int(self.has_hi))

    @property
    def col_base(self) -> int:
        return self.row0 - self.owned_offset

    def interior_rows(self) -> tuple[int, int]:
        """Local rows whose stencil touches no halo plane."""
        lo = self.plane if self.has_lo else 0
        hi = self.n_local - (self.plane if self.has_hi else 0)
        return lo, max(lo, hi)

    def boundary_ranges(self) -> list[tuple[int, int]]:
        lo, hi = self.interior_rows()
        out = []
        if lo > 0:
            out.append((0, lo))
        if hi < self.n_local:
            out.append((hi, self.n_local))
        return out


def slab_layout(nx: int, ny: int, nz: int, rank: int, world: int) -> SlabLayout:
    if not (1 <= world <= nz):
        raise ValueError("slab: need 1 <= world <= nz")
    return SlabLayout(nx, ny, nz, rank, world)


def halo_plan(L: SlabLayout):
    """(peer, send_slice, recv_slice) per neighbour, slices into local x."""
    p, o, n = L.plane, L.owned_offset, L.n_local
    plan = []
    if L.has_lo:
        plan.append((L.rank - 1, slice(o, o + p), slice(0, p)))
    if L.has_hi:
        plan.append((L.rank + 1, slice(o + n - p, o + n), slice(o + n, o + n + p)))
    return plan


def halo_exchange(L: SlabLayout, xloc, group=None):
    """Issue the halo send/recv pairs as one batch (NCCL group over NVLink on
    GPUs, gloo on CPU); returns the request list (wait() them)."""
    import torch.distributed as dist

    ops = []
    for peer, s, r in halo_plan(L):
        ops.append(dist.P2POp(dist.isend, xloc[s], peer, group))
        ops.append(dist.P2POp(dist.irecv, xloc[r], peer, group))
    if not ops:
        return []
    return dist.batch_isend_irecv(ops)


def slab_csr_numpy(L: SlabLayout, diag=6.0, off=-1.0):
    """Host restatement of the local slab CSR (local columns) used by the
    CPU tests; the device builds the same bytes in ktb_gen_stencil7_slab."""
    nx, ny, nz, p = L.nx, L.ny, L.nz, L.plane
    rows = np.arange(L.row0, L.row0 + L.n_local, dtype=np.int64)
    z, rem = np.divmod(rows, p)
    y, x = np.divmod(rem, nx)
    offs = [(-p, z > 0), (-nx, y > 0), (-1, x > 0), (0, np.ones(len(rows), bool)),
            (1, x < nx - 1), (nx, y < ny - 1), (p, z < nz - 1)]
    cnt = sum(m.astype(np.int64) for _, m in offs)
    rp = np.zeros(L.n_local + 1, np.int64)
    np.cumsum(cnt, out=rp[1:])
    ci = np.empty(rp[-1], np.int64)
    v = np.empty(rp[-1], np.float64)
    pos = rp[:-1].copy()
    for d, m in offs:
        idx = np.nonzero(m)[0]
        ci[pos[idx]] = rows[idx] + d - L.col_base
        v[pos[idx]] = diag if d == 0 else off
        pos[idx] += 1
    return L.n_local, rp, ci, v


class Comm:
    """ktb_comm: the native communicator of the data plane (include/ktb.h).

    NCCL (the product path): ``Comm.nccl(group, device)`` -- rank 0 draws
    the NCCL unique id inside libktb, torch.distributed (any backend, here
    only as the out-of-band channel) hands it to every rank, and every rank
    calls ncclCommInitRank through ``ktb_comm_create``. ``Comm.loopback``:
    W ranks inside one process (one host thread per rank) for single-GPU
    checks of the native exchange code (see ktb_comm.cu)."""

    def __init__(self, handle, keep=None):
        import ctypes as C

        from . import _lib
        from .ktune import _check

        self.h, self._keep, self._L, self._check = handle, keep, _lib.load(), _check
        v = [C.c_int() for _ in range(5)]
        _check(self._L.ktb_comm_info(self.h, *[C.byref(x) for x in v]))
        self.world, self.rank, self.device, self.nccl_version, nccl = [x.value for x in v]
        self.is_nccl = bool(nccl)

    @classmethod
    def nccl(cls, group=None, device=None) -> "Comm":
        import ctypes as C

        import torch
        import torch.distributed as dist

        from . import _lib
        from .ktune import _check

        L = _lib.load()
        dev = torch.cuda.current_device() if device is None else int(device)
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        uid = (C.c_uint8 * 128)()
        if rank == 0:
            _check(L.ktb_comm_id(uid))
        if world > 1:
            box = [bytes(uid)]
            dist.broadcast_object_list(box, src=0, group=group)
            C.memmove(uid, box[0], 128)
        h = C.c_void_p()
        _check(L.ktb_comm_create(uid, world, rank, dev, C.byref(h)))
        return cls(h)

    @classmethod
    def wrap(cls, nccl_comm_ptr: int, device: int = -1) -> "Comm":
        """Borrow an existing ncclComm_t (e.g. ProcessGroupNCCL._comm_ptr())."""
        import ctypes as C

        from . import _lib
        from .ktune import _check

        h = C.c_void_p()
        _check(_lib.load().ktb_comm_wrap(C.c_void_p(nccl_comm_ptr), device, C.byref(h)))
        return cls(h)

    @classmethod
    def loopback(cls, world: int, device: int = 0) -> list:
        import ctypes as C

        from . import _lib
        from .ktune import _check

        L = _lib.load()
        w = C.c_void_p()
        _check(L.ktb_loopback_world_create(world, C.byref(w)))
        keep = _LoopWorld(w)
        out = []
        for r in range(world):
            h = C.c_void_p()
            _check(L.ktb_comm_create_loopback(w, r, device, C.byref(h)))
            out.append(cls(h, keep))
        return out

    def _stream(self, stream=None) -> int:
        import torch

        if stream is not None:
            return int(stream)
        return torch.cuda.current_stream(self.device).cuda_stream

    def allreduce(self, t, op: str = "sum", stream=None) -> None:
        """In place over a float64 CUDA tensor (deterministic on loopback)."""
        self._check(self._L.ktb_comm_allreduce(self.h, t.data_ptr(), t.numel(),
                                               1 if op == "max" else 0, self._stream(stream)))

    def allgather(self, send, recv, stream=None) -> None:
        self._check(self._L.ktb_comm_allgather(self.h, send.data_ptr(), recv.data_ptr(),
                                               send.numel() * send.element_size(),
                                               self._stream(stream)))

    def barrier(self) -> None:
        """Host barrier: a one-element all-reduce, then wait for it."""
        import torch

        t = torch.zeros(1, dtype=torch.float64, device=f"cuda:{self.device}")
        self.allreduce(t)
        torch.cuda.current_stream(self.device).synchronize()

    def close(self):
        if getattr(self, "h", None):
            self._L.ktb_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class _LoopWorld:
    def __init__(self, h):
        from . import _lib

        self.h, self._L = h, _lib.load()

    def __del__(self):
        try:
            self._L.ktb_loopback_world_destroy(self.h)
        except Exception:
            pass


def run_ranks(world: int, fn):
    """fn(rank) on `world` host threads at once (collective native calls on
    loopback communicators); returns the results in rank order and re-raises
    the first failure."""
    import threading

    out, errs = [None] * world, [None] * world

    def body(r):
        try:
            import torch

            torch.cuda.set_device(0)
            out[r] = fn(r)
        except BaseException as e:  # noqa: BLE001 (re-raised below)
            errs[r] = e
            # the other ranks may now wait for this one forever: say why at once
            import sys
            import traceback

            print(f"run_ranks: rank {r} failed:", file=sys.stderr)
            traceback.print_exc()

    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for e in errs:
        if e is not None:
            raise e
    return out


class DistSpMV:
    """Config-4 sharded SpMV on this rank's GPU, native end to end (ktb_halo:
    the slab generated on the device, interior/boundary row plans, the NCCL
    halo group on a high-priority stream overlapped with the interior rows).
    Collective: every rank of ``comm`` constructs it together."""

    def __init__(self, nx, ny, nz, comm: Comm, seed=4, diag=6.0, off=-1.0, kernel=0, param=106):
        import ctypes as C

        import torch

        from . import _lib
        from .ktune import _check

        self.comm, self._L, self._check = comm, _lib.load(), _check
        self.L = slab_layout(nx, ny, nz, comm.rank, comm.world)
        self.device = comm.device
        h = C.c_void_p()
        _check(self._L.ktb_halo_create_stencil7(nx, ny, nz, diag, off, comm.h, int(kernel),
                                                int(param), C.byref(h)))
        self.h = h
        v = [C.c_int64() for _ in range(6)] + [C.c_int()]
        _check(self._L.ktb_halo_info(self.h, *[C.byref(x) for x in v]))
        (self.n_local, self.x_len, self.owned_offset, self.interior_begin, self.interior_end,
         self._nnz, self._launches) = [x.value for x in v]
        assert (self.n_local, self.x_len, self.owned_offset) == (
            self.L.n_local, self.L.x_local_len, self.L.owned_offset)
        dev = f"cuda:{self.device}"
        self.x = torch.zeros(self.x_len, dtype=torch.float64, device=dev)
        self.y = torch.empty(self.n_local, dtype=torch.float64, device=dev)
        owned = self.x[self.owned_offset:self.owned_offset + self.n_local]
        _check(self._L.ktb_seeded_vector(self.n_local, seed, self.L.row0, owned.data_ptr(),
                                         torch.cuda.current_stream(self.device).cuda_stream))

    @property
    def nnz(self) -> int:
        return self._nnz

    def parts(self):
        """(interior_rows, interior_nnz, boundary_rows, boundary_nnz)."""
        import ctypes as C

        v = [C.c_int64() for _ in range(4)]
        self._check(self._L.ktb_halo_parts(self.h, *[C.byref(x) for x in v]))
        return tuple(x.value for x in v)

    def plan_params(self):
        """(interior, boundary) U1 variants the plans resolved to after the
        create call's fallbacks (106 -> 105 -> 104 -> 100); -1 = no rows."""
        import ctypes as C

        v = [C.c_int64() for _ in range(2)]
        self._check(self._L.ktb_halo_plan_params(self.h, *[C.byref(x) for x in v]))
        return tuple(x.value for x in v)

    def _s(self, stream=None):
        import torch

        return int(stream) if stream is not None else \
            torch.cuda.current_stream(self.device).cuda_stream

    def apply(self, stream=None):
        """One sharded y = A x (ktb_halo_spmv) on the current torch stream."""
        self._check(self._L.ktb_halo_spmv(self.h, self.x.data_ptr(), self.y.data_ptr(),
                                          self._s(stream)))
        return self.y

    def apply_host(self, x_owned, y, chunks: int = 16) -> None:
        """y = A x with host arrays (owned x in, owned y out; pinned memory
        for the in-call copy/compute overlap), synchronous
        (ktb_halo_spmv_host)."""
        x_owned, y = np.asarray(x_owned), np.asarray(y)
        assert x_owned.dtype == np.float64 and y.dtype == np.float64
        assert x_owned.shape == (self.n_local,) and y.shape == (self.n_local,)
        assert x_owned.flags.c_contiguous and y.flags.c_contiguous
        self._check(self._L.ktb_halo_spmv_host(self.h, x_owned.ctypes.data, y.ctypes.data,
                                               int(chunks)))

    def exchange_only(self, stream=None):
        """The halo exchange of one apply alone (ktb_halo_exchange)."""
        self._check(self._L.ktb_halo_exchange(self.h, self.x.data_ptr(), self._s(stream)))

    def launches_per_apply(self) -> int:
        return self._launches

    def set_timing(self, on: bool = True) -> None:
        self._check(self._L.ktb_halo_set_timing(self.h, int(on)))

    def last_times(self):
        """(interior_ms, boundary_ms) of the last apply (set_timing first)."""
        import ctypes as C

        a, b = C.c_double(), C.c_double()
        self._check(self._L.ktb_halo_timing(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def close(self):
        if getattr(self, "h", None):
            self._L.ktb_halo_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def local_exchange(layouts, xs) -> None:
    """Single-process stand-in for halo_exchange over all ranks' buffers (the
    same send/recv slices, done as plain copies): lets one GPU check the
    sharded result without running ranks that wait on each other."""
    for L, x in zip(layouts, xs):
        for peer, s, r in halo_plan(L):
            src_L, src_x = layouts[peer], xs[peer]
            # what `peer` sends to this rank lands in this rank's recv slice
            for pp, ss, _ in halo_plan(src_L):
                if pp == L.rank:
                    x[r] = src_x[ss]


# ======================================================================
# General row-block sharding of an arbitrary CRS.
# The split and ghost bookkeeping are native (libktb ktb_dist_*, host-only
# until upload); the exchange is native too (ktb_dist_connect/spmv).
# ======================================================================
def nnz_balanced_boundaries(row_ptr, world: int) -> np.ndarray:
    """partition.hpp:28-55 NNZ_BALANCED on host: boundary p is the smallest
    row r with row_ptr[r] * P >= p * nnz (exact int64), r < n."""
    rp = np.ascontiguousarray(row_ptr, np.int64)
    n, nnz = len(rp) - 1, int(rp[-1])
    out = np.empty(world + 1, np.int64)
    out[0], out[world] = 0, n
    scaled = rp[:-1] * world
    for p in range(1, world):
        out[p] = np.searchsorted(scaled, p * nnz, side="left")
    return out


class DistCsr:
    """One rank's share of a row-block sharded CRS (ktb_dist handle).
    row_ptr/col_idx/values: this rank's rows (local row_ptr, GLOBAL columns)."""

    def __init__(self, n_global, boundaries, rank, world, row_ptr, col_idx, values):
        import ctypes as C

        from . import _lib
        from .ktune import _check

        self._C, self._L, self._check = C, _lib.load(), _check
        self.boundaries = np.ascontiguousarray(boundaries, np.int64)
        self.rank, self.world, self.n_global = rank, world, n_global
        rp = np.ascontiguousarray(row_ptr, np.int64)
        ci = np.ascontiguousarray(col_idx, np.int64)
        v = np.ascontiguousarray(values, np.float64)
        self.h = C.c_void_p()
        _check(self._L.ktb_dist_create(n_global, world, self.boundaries.ctypes.data, rank,
                                       rp.ctypes.data, ci.ctypes.data, v.ctypes.data,
                                       C.byref(self.h)))
        vals = [C.c_int64() for _ in range(5)]
        _check(self._L.ktb_dist_info(self.h, *[C.byref(x) for x in vals]))
        (self.n_local, self.n_ghost, self.nnz_local, self.nnz_ghost,
         self.ghost_rows) = [x.value for x in vals]
        self.ghosts = np.empty(max(self.n_ghost, 1), np.int64)
        self.recv_counts = np.empty(world, np.int64)
        _check(self._L.ktb_dist_ghosts(self.h, self.ghosts.ctypes.data,
                                       self.recv_counts.ctypes.data))
        self.ghosts = self.ghosts[: self.n_ghost]
        self.send_counts = None
        self.send_cols = None

    @property
    def row0(self) -> int:
        return int(self.boundaries[self.rank])

    def recv_offsets(self) -> np.ndarray:
        return np.concatenate([[0], np.cumsum(self.recv_counts)])

    def send_offsets(self) -> np.ndarray:
        return np.concatenate([[0], np.cumsum(self.send_counts)])

    def set_sends(self, counts, cols) -> None:
        self.send_counts = np.ascontiguousarray(counts, np.int64)
        self.send_cols = np.ascontiguousarray(cols, np.int64)
        self._check(self._L.ktb_dist_set_sends(self.h, self.send_counts.ctypes.data,
                                               self.send_cols.ctypes.data))

    def local_csr(self):
        rp = np.empty(self.n_local + 1, np.int32)
        ci = np.empty(max(self.nnz_local, 1), np.int32)
        v = np.empty(max(self.nnz_local, 1), np.float64)
        self._check(self._L.ktb_dist_local_csr(self.h, rp.ctypes.data, ci.ctypes.data,
                                               v.ctypes.data))
        return rp, ci[: self.nnz_local], v[: self.nnz_local]

    def ghost_csr(self):
        rows = np.empty(max(self.ghost_rows, 1), np.int32)
        rp = np.empty(self.ghost_rows + 1, np.int32)
        ci = np.empty(max(self.nnz_ghost, 1), np.int32)
        v = np.empty(max(self.nnz_ghost, 1), np.float64)
        self._check(self._L.ktb_dist_ghost_csr(self.h, rows.ctypes.data, rp.ctypes.data,
                                               ci.ctypes.data, v.ctypes.data))
        return rows[: self.ghost_rows], rp, ci[: self.nnz_ghost], v[: self.nnz_ghost]

    def upload(self, device: int):
        """Both blocks to `device`; returns A_d as a (borrowed) DeviceCsr."""
        from .ktune import DeviceCsr

        self._check(self._L.ktb_dist_upload(self.h, device))
        m = self._C.c_void_p()
        self._check(self._L.ktb_dist_local_matrix(self.h, self._C.byref(m)))
        return DeviceCsr(m, False, owner=self)

    def close(self):
        if getattr(self, "h", None):
            self._L.ktb_dist_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def exchange_ghost_lists(dc: DistCsr, group=None, device=None):
    """Python restatement of ktb_dist_connect's list exchange over
    torch.distributed (CPU gloo tests of the protocol): every rank learns
    which of its owned columns each peer needs. Counts by all_gather (world x world), lists by one batch of
    point-to-point transfers. Returns (send_counts, send_cols)."""
    import torch
    import torch.distributed as dist

    W, r = dc.world, dc.rank
    if W == 1:  # nothing to exchange (and no process group is required)
        return np.zeros(1, np.int64), np.zeros(0, np.int64)
    dev = "cpu" if device is None else f"cuda:{device}"
    mine = torch.as_tensor(dc.recv_counts, dtype=torch.int64, device=dev)
    allc = [torch.empty(W, dtype=torch.int64, device=dev) for _ in range(W)]
    dist.all_gather(allc, mine, group=group)
    send_counts = np.array([int(allc[p][r]) for p in range(W)], np.int64)
    ro = dc.recv_offsets()
    so = np.concatenate([[0], np.cumsum(send_counts)])
    ghosts = torch.as_tensor(dc.ghosts, dtype=torch.int64, device=dev)
    out = torch.empty(int(so[-1]), dtype=torch.int64, device=dev)
    ops = []
    for p in range(W):
        if p == r:
            continue
        if dc.recv_counts[p]:
            ops.append(dist.P2POp(dist.isend, ghosts[ro[p]:ro[p + 1]], p, group))
        if send_counts[p]:
            ops.append(dist.P2POp(dist.irecv, out[so[p]:so[p + 1]], p, group))
    if ops:
        for q in dist.batch_isend_irecv(ops):
            q.wait()
    return send_counts, out.cpu().numpy()


class DistCsrSpMV:
    """y = A x for an arbitrary CRS sharded by rows over a communicator (one
    rank per GPU), native end to end: ktb_dist_connect exchanges the ghost
    lists over the communicator once; every apply is ktb_dist_spmv (pack ->
    grouped NCCL send/recv of the ghosts on a high-priority stream,
    overlapped with the A_d plan -> y += A_o x_ghost). Collective: every rank
    constructs it together. kernel None: A_d's plan comes from the selector
    (select_spmv_unsym on device time) and is handed to the split."""

    def __init__(self, n_global, boundaries, comm: Comm, row_ptr=None, col_idx=None, values=None,
                 kernel=None, param=0, dc=None):
        import ctypes as C

        from . import ktune as K

        self.comm = comm
        self.dc = dc or DistCsr(n_global, boundaries, comm.rank, comm.world, row_ptr, col_idx,
                                values)
        L, chk = self.dc._L, self.dc._check
        k0, p0 = (0, 100) if kernel is None else (int(kernel), int(param))
        chk(L.ktb_dist_connect(self.dc.h, comm.h, k0, p0))
        self.device = comm.device
        m = C.c_void_p()
        chk(L.ktb_dist_local_matrix(self.dc.h, C.byref(m)))
        self.A_d = K.DeviceCsr(m, False, owner=self.dc)
        self.report = None
        self.plan = None
        if kernel is None and self.A_d.nnz() > 0:
            choice, self.report = K.select_spmv_unsym(self.A_d)
            self.plan = choice.plan
            chk(L.ktb_dist_set_plan(self.dc.h, self.plan.h))
        # the lists the native connect derived (for reporting and parity tests)
        cnt = np.empty(comm.world, np.int64)
        chk(L.ktb_dist_sends(self.dc.h, cnt.ctypes.data, None))
        cols = np.empty(max(int(cnt.sum()), 1), np.int64)
        chk(L.ktb_dist_sends(self.dc.h, None, cols.ctypes.data))
        self.dc.send_counts, self.dc.send_cols = cnt, cols[:int(cnt.sum())]

    @property
    def n_local(self) -> int:
        return self.dc.n_local

    def _stream(self, stream=None):
        import torch

        return int(stream) if stream is not None else \
            torch.cuda.current_stream(self.device).cuda_stream

    def apply(self, x_owned, y, stream=None):
        """One sharded y = A x (CUDA tensors of length n_local)."""
        self.dc._check(self.dc._L.ktb_dist_spmv(self.dc.h, x_owned.data_ptr(), y.data_ptr(),
                                                self._stream(stream)))
        return y

    def exchange_only(self, x_owned, stream=None):
        """Pack + ghost exchange of one apply alone (for timing it)."""
        self.dc._check(self.dc._L.ktb_dist_exchange(self.dc.h, x_owned.data_ptr(),
                                                    self._stream(stream)))

    def launches_per_apply(self) -> int:
        import ctypes as C

        n = C.c_int()
        self.dc._check(self.dc._L.ktb_dist_launches(self.dc.h, C.byref(n)))
        return n.value

    def kernel_name(self) -> str:
        if self.plan is not None:
            return "u%d" % (self.plan.kernel + 1)
        return "u1/u2 default" if self.A_d.nnz() else "none"


def local_send_lists(dcs):
    """What exchange_ghost_lists returns on each rank, computed in one
    process from all ranks' DistCsr objects."""
    W = len(dcs)
    out = []
    for r in range(W):
        counts = np.zeros(W, np.int64)
        cols = []
        for p in range(W):
            if p == r:
                continue
            ro = dcs[p].recv_offsets()
            seg = dcs[p].ghosts[ro[r]:ro[r + 1]]
            counts[p] = len(seg)
            cols.append(seg)
        out.append((counts, np.concatenate(cols) if cols else np.zeros(0, np.int64)))
    return out
