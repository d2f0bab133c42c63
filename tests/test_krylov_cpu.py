"""Distributed GMRES(m) (paper_2405_01599_b200.krylov) on
CPU ranks with gloo: the library's host loop (Arnoldi, the four
orthogonalisers with their all-reduces, Givens, restarts) driven with a
torch-CPU stand-in for the device BLAS-1 (test infrastructure) and a CPU
operator built on the native row-block split (ktb_dist_*) with the same
ghost exchange protocol. Checked against the reference's own gmres_m
(oracle/_ref): same iteration count within +-2, true residual < tol,
solution close.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import matgen
from oracle import oracle as O
from paper_2405_01599_b200 import dist as D
from paper_2405_01599_b200 import krylov as KR

GRID = (12, 11, 10)
KINDS = {"cgs": 0, "mgs": 1, "dgks": 2, "bcgs": 3}


def _matrix():
    return matgen.stencil7(*GRID, xp=-0.7, xm=-1.3)  # config-5 convection-diffusion


class CpuVecOps:
    """torch-CPU stand-in for DeviceVecOps (same method contract)."""

    def __init__(self, n_global=None):
        self.n_global = n_global

    def copy(self, src, dst):
        dst.copy_(src)

    def seeded(self, seed, offset, out):
        full = O.seeded_vector(self.n_global, seed)
        out.copy_(torch.from_numpy(full[offset:offset + out.shape[0]].copy()))

    def empty(self, *s):
        return torch.empty(*s, dtype=torch.float64)

    def zeros(self, *s):
        return torch.zeros(*s, dtype=torch.float64)

    def mdot(self, V, k, w, out):
        for j in range(k):
            out[j] = torch.dot(V[j], w)

    def maxpy(self, V, k, coef, alpha, w):
        for j in range(k):
            w.add_(V[j], alpha=float(alpha * coef[j]))

    def axpby(self, a, x, b, y):
        y.copy_(a * x + b * y)

    def scale(self, s, x, divide=False):
        if divide:
            x.div_(s)
        else:
            x.mul_(s)

    def to_host(self, t):
        return t.tolist()

    def from_host(self, vals, out):
        out.copy_(torch.tensor(vals, dtype=torch.float64))


class CpuDistOp:
    """y = A x on this rank's rows: A_d x_owned + A_o x_ghost, the ghosts
    exchanged with one batch of gloo send/recv (the DistCsrSpMV protocol)."""

    def __init__(self, n, rp, ci, v, rank, world):
        b = D.nnz_balanced_boundaries(rp, world)
        r0, r1 = int(b[rank]), int(b[rank + 1])
        self.dc = D.DistCsr(n, b, rank, world, rp[r0:r1 + 1] - rp[r0], ci[rp[r0]:rp[r1]],
                            v[rp[r0]:rp[r1]])
        self.counts, self.cols = D.exchange_ghost_lists(self.dc)
        self.dc.set_sends(self.counts, self.cols)
        self.r0, self.n_local, self.world, self.rank = r0, r1 - r0, world, rank
        drp, dci, dv = self.dc.local_csr()
        self.d_rows = np.repeat(np.arange(self.n_local), np.diff(drp))
        self.dci, self.dv = dci.astype(np.int64), dv
        orows, orp, oci, ov = self.dc.ghost_csr()
        self.o_rows = np.repeat(orows, np.diff(orp)).astype(np.int64)
        self.oci, self.ov = oci.astype(np.int64), ov

    def apply(self, x, y):
        xn = x.numpy()
        send = torch.from_numpy(np.ascontiguousarray(xn[self.cols - self.r0]))
        xg = torch.zeros(max(self.dc.n_ghost, 1), dtype=torch.float64)
        ro, so = self.dc.recv_offsets(), self.dc.send_offsets()
        ops = []
        for p in range(self.world):
            if p != self.rank and self.counts[p]:
                ops.append(dist.P2POp(dist.isend, send[so[p]:so[p + 1]], p))
            if p != self.rank and self.dc.recv_counts[p]:
                ops.append(dist.P2POp(dist.irecv, xg[ro[p]:ro[p + 1]], p))
        if ops:
            for q in dist.batch_isend_irecv(ops):
                q.wait()
        out = np.bincount(self.d_rows, weights=self.dv * xn[self.dci], minlength=self.n_local)
        if len(self.o_rows):
            out += np.bincount(self.o_rows, weights=self.ov * xg.numpy()[self.oci],
                               minlength=self.n_local)
        y.copy_(torch.from_numpy(out))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir, kind, m):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, rp, ci, v = _matrix()
        bg = O.spmv_ref(n, rp, ci, v, np.ones(n))
        op = CpuDistOp(n, rp, ci, v, rank, world)
        b = torch.from_numpy(bg[op.r0:op.r0 + op.n_local].copy())
        res = KR.gmres_m_dist(op, b, m=m, tol=1e-8, max_iters=500, ortho=kind, ops=CpuVecOps())
        np.save(os.path.join(out_dir, f"x{rank}.npy"), res.x.numpy())
        np.save(os.path.join(out_dir, f"s{rank}.npy"),
                np.array([res.iterations, res.converged, res.true_residual, res.allreduces,
                          len(res.restarts)]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,kind,m", [(2, "mgs", 30), (3, "mgs", 12), (2, "cgs", 30),
                                          (3, "dgks", 20), (2, "bcgs", 30)])
def test_gloo_gmres_matches_reference(world, kind, m, tmp_path):
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    mp.spawn(_worker, args=(world, _port(), str(tmp_path), kind, m), nprocs=world, join=True)
    n, rp, ci, v = _matrix()
    b = O.spmv_ref(n, rp, ci, v, np.ones(n))
    xr, rr = O.Ref.gmres(n, rp, ci, v, b, m=m, tol=1e-8, max_iters=500, ortho_kind=KINDS[kind])
    stats = [np.load(tmp_path / f"s{r}.npy") for r in range(world)]
    its = int(stats[0][0])
    assert all(int(s[0]) == its for s in stats)  # every rank ran the same loop
    assert bool(stats[0][1]) and stats[0][2] < 1e-8
    assert abs(its - rr["iterations"]) <= 2, (its, rr["iterations"])
    x = np.concatenate([np.load(tmp_path / f"x{r}.npy") for r in range(world)])
    assert np.max(np.abs(x - 1.0)) < 1e-5 and np.max(np.abs(x - xr)) < 1e-5


def test_single_rank_loop_and_allreduce_counts():
    """World 1 (no process group): identical loop; all-reduce counts per
    Arnoldi step follow the orthogoniser's structure."""
    n, rp, ci, v = _matrix()
    bg = O.spmv_ref(n, rp, ci, v, np.ones(n))

    class Op:
        n_local = n

        def apply(self, x, y):
            y.copy_(torch.from_numpy(O.spmv_ref(n, rp, ci, v, x.numpy())))

    res = {}
    for kind in KINDS:
        r = KR.gmres_m_dist(Op(), torch.from_numpy(bg.copy()), m=30, tol=1e-8, max_iters=500,
                            ortho=kind, ops=CpuVecOps(), allreduce=lambda t: None)
        xr, rr = O.Ref.gmres(n, rp, ci, v, bg, m=30, tol=1e-8, max_iters=500,
                             ortho_kind=KINDS[kind]) if O.ref_available() else (None, None)
        assert r.converged and r.true_residual < 1e-8
        if rr:
            assert abs(r.iterations - rr["iterations"]) <= 2
        res[kind] = r
    # mgs: per step k = j+1 projections + 2 norms; cgs 3; dgks 4 (+ 1 per restart
    # for beta, + b's norm, + the final true residual)
    cyc = len(res["mgs"].restarts) + 1
    it = res["mgs"].iterations
    assert res["cgs"].allreduces == 3 * res["cgs"].iterations + (len(res["cgs"].restarts) + 1) + 2
    assert res["dgks"].allreduces == 4 * res["dgks"].iterations + (len(res["dgks"].restarts) + 1) + 2
    assert res["mgs"].allreduces > 3 * it and cyc >= 1
    with pytest.raises(ValueError, match="unknown kind"):
        KR.gmres_m_dist(Op(), torch.from_numpy(bg.copy()), ortho="householder", ops=CpuVecOps(),
                        allreduce=lambda t: None)


def test_single_rank_ilu0_right_preconditioning_matches_reference():
    """The host loop with a right preconditioner (here the oracle's ILU(0),
    test infrastructure) reproduces the reference's gmres_m + ilu0 pairing."""
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    n, rp, ci, v = _matrix()
    bg = O.spmv_ref(n, rp, ci, v, np.ones(n))
    fv, diag = O.ilu0_factorize(n, rp, ci, v)

    class Op:
        n_local = n

        def apply(self, x, y):
            y.copy_(torch.from_numpy(O.spmv_ref(n, rp, ci, v, x.numpy())))

    def pc(r, z):
        z.copy_(torch.from_numpy(O.ilu0_apply(n, rp, ci, fv, diag, r.numpy())))

    res = KR.gmres_m_dist(Op(), torch.from_numpy(bg.copy()), m=30, tol=1e-8, max_iters=500,
                          ops=CpuVecOps(), allreduce=lambda t: None, precond=pc)
    xr, rr = O.Ref.gmres_ilu0(n, rp, ci, v, bg)
    assert res.converged and res.true_residual < 1e-8
    assert abs(res.iterations - rr["iterations"]) <= 2, (res.iterations, rr["iterations"])
    assert res.iterations < 0.5 * KR.gmres_m_dist(
        Op(), torch.from_numpy(bg.copy()), m=30, tol=1e-8, max_iters=500, ops=CpuVecOps(),
        allreduce=lambda t: None).iterations
