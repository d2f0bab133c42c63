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
    """Config-4 sharded SpMV on this rank's GPU (torch.distributed, NCCL)."""

    def __init__(self, nx, ny, nz, rank, world, device, seed=4, diag=6.0, off=-1.0):
        import torch

        from . import _lib
        from . import ktune as K

        self.L = slab_layout(nx, ny, nz, rank, world)
        self.device = device
        self.A = K.stencil7_slab(nx, ny, nz, self.L.z0, self.L.z1, diag, off, device=device)
        self.plan = K.DevicePlan(self.A, K.UnsymKernel.u1_row)
        self.x = torch.empty(self.L.x_local_len, dtype=torch.float64, device=f"cuda:{device}")
        self.y = torch.empty(self.L.n_local, dtype=torch.float64, device=f"cuda:{device}")
        owned = self.x[self.L.owned_offset:self.L.owned_offset + self.L.n_local]
        rc = _lib.load().ktb_seeded_vector(self.L.n_local, seed, self.L.row0, owned.data_ptr(),
                                           torch.cuda.current_stream(device).cuda_stream)
        if rc != 0:
            raise RuntimeError(_lib.load().ktb_last_error().decode())

    @property
    def nnz(self) -> int:
        return self.A.nnz()

    def apply(self):
        """One sharded y = A x with halo/interior overlap (see module doc)."""
        reqs = halo_exchange(self.L, self.x)
        lo, hi = self.L.interior_rows()
        if hi > lo:
            self.plan.apply_rows(lo, hi, self.x, self.y)
        for r in reqs:
            r.wait()  # the current stream waits for the NCCL transfers
        for b0, b1 in self.L.boundary_ranges():
            self.plan.apply_rows(b0, b1, self.x, self.y)
        return self.y

    def compute_local(self):
        """The local rows only (halos assumed in place): interior + boundary."""
        lo, hi = self.L.interior_rows()
        if hi > lo:
            self.plan.apply_rows(lo, hi, self.x, self.y)
        for b0, b1 in self.L.boundary_ranges():
            self.plan.apply_rows(b0, b1, self.x, self.y)
        return self.y

    def launches_per_apply(self) -> int:
        lo, hi = self.L.interior_rows()
        return int(hi > lo) + len(self.L.boundary_ranges())


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
