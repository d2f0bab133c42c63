"""Row-block (z-slab) sharding of the config-4 SpMV across GPUs with a
one-plane x halo exchanged by NCCL point-to-point.

The reference has no distributed path; this is the B200
framework's scale-out of spmv_unsym (spmv.hpp:111): rank r of P owns the
z-planes [r*nz/P, (r+1)*nz/P) of the 3-D 7-point stencil, i.e. a contiguous
row block, and y stays row-sharded (no reduction collective).

Local x layout on each rank:  [halo_lo plane | owned planes | halo_hi plane]
(end ranks omit the missing neighbour's plane). Local column index =
global column - col_base, col_base = first owned row - (plane if halo_lo).

Per apply:
  1. the two boundary planes of owned x are sent to the neighbours and the
     halo planes received, as one batch of NCCL send/recv (batch_isend_irecv);
  2. the interior rows (which touch no halo) run on the compute stream while
     NCCL moves the halos over NVLink;
  3. the compute stream waits for the exchange and runs the two boundary
     planes.

Host-side layout logic (SlabLayout, halo_ops) is plain Python so the
multi-rank protocol is testable on CPU with the gloo backend.
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


class DistSpMV:
    """Config-4 sharded SpMV on this rank's GPU (torch.distributed, NCCL).
    The slab is split once into its interior rows (no halo columns) and the
    boundary planes, each a device matrix with its own plan over the same
    local x; both default to U1 over the warp-sliced copy (param 100)."""

    def __init__(self, nx, ny, nz, rank, world, device, seed=4, diag=6.0, off=-1.0,
                 interior_kernel=0, interior_param=100, boundary_param=100):
        import torch

        from . import _lib
        from . import ktune as K

        self.L = slab_layout(nx, ny, nz, rank, world)
        self.device = device
        slab = K.stencil7_slab(nx, ny, nz, self.L.z0, self.L.z1, diag, off, device=device)
        self._nnz = slab.nnz()
        lo, hi = self.L.interior_rows()
        self.parts = []  # (r0, r1, plan)
        if hi > lo:
            a = slab.slice_rows(lo, hi)
            self.parts.append((lo, hi, K.DevicePlan(a, int(interior_kernel), int(interior_param))))
        self.boundary = []
        for b0, b1 in self.L.boundary_ranges():
            a = slab.slice_rows(b0, b1)
            self.boundary.append((b0, b1, K.DevicePlan(a, K.UnsymKernel.u1_row,
                                                       int(boundary_param))))
        del slab
        self.x = torch.empty(self.L.x_local_len, dtype=torch.float64, device=f"cuda:{device}")
        self.y = torch.empty(self.L.n_local, dtype=torch.float64, device=f"cuda:{device}")
        owned = self.x[self.L.owned_offset:self.L.owned_offset + self.L.n_local]
        rc = _lib.load().ktb_seeded_vector(self.L.n_local, seed, self.L.row0, owned.data_ptr(),
                                           torch.cuda.current_stream(device).cuda_stream)
        if rc != 0:
            raise RuntimeError(_lib.load().ktb_last_error().decode())

    @property
    def nnz(self) -> int:
        return self._nnz

    def _run(self, parts):
        for r0, r1, plan in parts:
            plan.apply(self.x, self.y[r0:r1])

    def apply(self):
        """One sharded y = A x with halo/interior overlap (see module doc)."""
        reqs = halo_exchange(self.L, self.x)
        self._run(self.parts)
        for r in reqs:
            r.wait()  # the current stream waits for the NCCL transfers
        self._run(self.boundary)
        return self.y

    def exchange_only(self):
        """The halo exchange of one apply alone (for timing it): the two
        one-plane messages, waited on by the current stream."""
        for r in halo_exchange(self.L, self.x):
            r.wait()

    def compute_local(self):
        """The local rows only (halos assumed in place): interior + boundary."""
        self._run(self.parts)
        self._run(self.boundary)
        return self.y

    def launches_per_apply(self) -> int:
        return sum(p.launches for _, _, p in self.parts + self.boundary)


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
# until upload); this layer exchanges the ghost lists once and drives the
# per-apply pack -> NCCL send/recv -> A_d x (overlapped) -> y += A_o x_g.
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
    """Once per matrix: every rank learns which of its owned columns each peer
    needs. Counts by all_gather (world x world), lists by one batch of
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
    """y = A x for an arbitrary CRS sharded by rows over the process group
    (one rank per GPU, NCCL). x and y are row-sharded like A; the local
    diagonal block runs the selected/tuned kernel, overlapped with the ghost
    exchange; the off-diagonal block accumulates after it."""

    def __init__(self, n_global, boundaries, rank, world, row_ptr, col_idx, values, device,
                 kernel=None, group=None, sends=None, dc=None):
        import torch

        from . import ktune as K

        self.dc = dc or DistCsr(n_global, boundaries, rank, world, row_ptr, col_idx, values)
        if sends is None:
            counts, cols = exchange_ghost_lists(self.dc, group, device)
        else:  # precomputed (single-process emulation: local_send_lists)
            counts, cols = sends
        self.dc.set_sends(counts, cols)
        self.device, self.group = device, group
        self.A_d = self.dc.upload(device)
        if kernel is None and self.A_d.nnz() > 0:
            choice, self.report = K.select_spmv_unsym(self.A_d)
            self.plan = choice.plan
        else:
            self.plan = K.DevicePlan(self.A_d, int(kernel if kernel is not None else 0))
            self.report = None
        dev = f"cuda:{device}"
        self.xg = torch.zeros(max(self.dc.n_ghost, 1), dtype=torch.float64, device=dev)
        self.send = torch.empty(max(int(counts.sum()), 1), dtype=torch.float64, device=dev)
        self._ro, self._so = self.dc.recv_offsets(), self.dc.send_offsets()

    @property
    def n_local(self) -> int:
        return self.dc.n_local

    def _stream(self):
        import torch

        return torch.cuda.current_stream(self.device).cuda_stream

    def pack(self, x_owned) -> None:
        self.dc._check(self.dc._L.ktb_dist_pack(self.dc.h, x_owned.data_ptr(),
                                                self.send.data_ptr(), self._stream()))

    def exchange(self):
        import torch.distributed as dist

        ops = []
        for p in range(self.dc.world):
            if p == self.dc.rank:
                continue
            if self.dc.send_counts[p]:
                ops.append(dist.P2POp(dist.isend, self.send[self._so[p]:self._so[p + 1]], p,
                                      self.group))
            if self.dc.recv_counts[p]:
                ops.append(dist.P2POp(dist.irecv, self.xg[self._ro[p]:self._ro[p + 1]], p,
                                      self.group))
        return dist.batch_isend_irecv(ops) if ops else []

    def ghost_spmv(self, y) -> None:
        self.dc._check(self.dc._L.ktb_dist_ghost_spmv(self.dc.h, self.xg.data_ptr(),
                                                      y.data_ptr(), self._stream()))

    def apply(self, x_owned, y):
        """One sharded y = A x (torch CUDA tensors of length n_local)."""
        self.pack(x_owned)
        reqs = self.exchange()
        if self.A_d.nnz() > 0:
            self.plan.apply(x_owned, y)
        else:
            y.zero_()
        for q in reqs:
            q.wait()
        self.ghost_spmv(y)
        return y

    def exchange_only(self, x_owned):
        """Pack + ghost exchange of one apply alone (for timing it)."""
        self.pack(x_owned)
        for q in self.exchange():
            q.wait()

    def launches_per_apply(self) -> int:
        return int(self.dc.send_counts.sum() > 0) + self.plan.launches + int(self.dc.ghost_rows > 0)


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


def local_ghost_exchange(spmvs, xs) -> None:
    """Single-process stand-in for the per-apply exchange over all ranks'
    DistCsrSpMV objects on one device (plain copies of the same slices)."""
    for s, x in zip(spmvs, xs):
        s.pack(x)
    for s in spmvs:
        r = s.dc.rank
        for p in range(s.dc.world):
            if p == r or not s.dc.recv_counts[p]:
                continue
            src = spmvs[p]
            so = src._so
            s.xg[s._ro[p]:s._ro[p + 1]] = src.send[so[r]:so[r + 1]]
