"""General row-block sharding of an arbitrary CRS on CPU
ranks with gloo: the native split (libktb ktb_dist_*: ghost discovery, owner
grouping, renumbering, send lists) plus the exchange protocol reproduce the
global SpMV. Per rank y = A_d x_owned + A_o x_ghost is evaluated with numpy
here (test infrastructure); the device kernels run in test_dist_general_gpu.

Bar: |y - y_ref| <= 1e-12 (|A||x|)_i (the split changes the summation
order of a row: owned-column terms first, then ghost terms)."""
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

TOL = 1e-12


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _matrix(kind):
    if kind == "random":
        return matgen.random_csr(700, 0.01, np.random.default_rng(11), empty_frac=0.1)
    if kind == "skew":
        return matgen.random_csr(900, 0.0, np.random.default_rng(12), skew=True, empty_frac=0.2)
    if kind == "stencil":
        return matgen.stencil7(7, 6, 9)
    if kind == "powerlaw":
        return matgen.powerlaw(3000, 5, 30000, 0.1, 2000)
    raise ValueError(kind)


def _bounds(rp, world, kind):
    if kind == "nnz":
        return D.nnz_balanced_boundaries(rp, world)
    n = len(rp) - 1  # a rank with no rows in the middle
    b = np.linspace(0, n, world + 1).astype(np.int64)
    if world >= 3:
        b[2] = b[1]
    return b


def _local_spmv(dc, x_owned, xg):
    rp, ci, v = dc.local_csr()
    y = O.spmv_ref(dc.n_local, rp.astype(np.int64), ci.astype(np.int64), v, x_owned) \
        if dc.n_local else np.zeros(0)
    rows, orp, oci, ov = dc.ghost_csr()
    for g, r in enumerate(rows):
        s = 0.0
        for k in range(orp[g], orp[g + 1]):
            s += ov[k] * xg[oci[k]]
        y[r] += s
    return y


def _worker(rank, world, port, out_dir, mkind, bkind):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, rp, ci, v = _matrix(mkind)
        b = _bounds(rp, world, bkind)
        r0, r1 = int(b[rank]), int(b[rank + 1])
        lrp = rp[r0:r1 + 1] - rp[r0]
        lci, lv = ci[rp[r0]:rp[r1]], v[rp[r0]:rp[r1]]
        dc = D.DistCsr(n, b, rank, world, lrp, lci, lv)
        counts, cols = D.exchange_ghost_lists(dc)
        dc.set_sends(counts, cols)
        # per-apply protocol: pack the send list, one batch of send/recv
        x = O.seeded_vector(n, 21)
        x_owned = x[r0:r1]
        send = torch.from_numpy(np.ascontiguousarray(x_owned[cols - r0]))
        xg = torch.zeros(max(dc.n_ghost, 1), dtype=torch.float64)
        ro, so = dc.recv_offsets(), dc.send_offsets()
        ops = []
        for p in range(world):
            if p != rank and counts[p]:
                ops.append(dist.P2POp(dist.isend, send[so[p]:so[p + 1]], p))
            if p != rank and dc.recv_counts[p]:
                ops.append(dist.P2POp(dist.irecv, xg[ro[p]:ro[p + 1]], p))
        if ops:
            for q in dist.batch_isend_irecv(ops):
                q.wait()
        xg = xg.numpy()[: dc.n_ghost]
        assert np.array_equal(xg, x[dc.ghosts])  # the receive buffer IS x[ghosts]
        y = _local_spmv(dc, x_owned, xg)
        np.save(os.path.join(out_dir, f"y{rank}.npy"), y)
        np.save(os.path.join(out_dir, f"g{rank}.npy"), dc.ghosts)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,mkind,bkind", [(2, "random", "nnz"), (3, "skew", "nnz"),
                                               (3, "stencil", "uneven"), (4, "powerlaw", "nnz"),
                                               (2, "powerlaw", "uneven")])
def test_gloo_general_sharding_reproduces_global_spmv(world, mkind, bkind, tmp_path):
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), mkind, bkind), nprocs=world,
             join=True)
    n, rp, ci, v = _matrix(mkind)
    x = O.seeded_vector(n, 21)
    y_ref = O.spmv_ref(n, rp, ci, v, x)
    bound = TOL * O.spmv_ref(n, rp, ci, np.abs(v), np.abs(x))
    y = np.concatenate([np.load(tmp_path / f"y{r}.npy") for r in range(world)])
    assert len(y) == n
    assert np.all(np.abs(y - y_ref) <= bound)
    b = _bounds(rp, world, bkind)
    for r in range(world):  # ghosts: exactly the off-block columns of the rank's rows
        g = np.load(tmp_path / f"g{r}.npy")
        c = ci[rp[b[r]]:rp[b[r + 1]]]
        want = np.unique(c[(c < b[r]) | (c >= b[r + 1])])
        assert np.array_equal(g, want)


def test_nnz_boundaries_match_reference_partition():
    for mk in ("random", "skew", "powerlaw"):
        n, rp, ci, v = _matrix(mk)
        for w in (1, 2, 3, 7, 148):
            assert np.array_equal(D.nnz_balanced_boundaries(rp, w),
                                  O.build_row_partition(rp, w, 1))


def test_split_structure_and_contract_messages():
    n, rp, ci, v = _matrix("random")
    b = D.nnz_balanced_boundaries(rp, 3)
    r0, r1 = int(b[1]), int(b[2])
    lrp = rp[r0:r1 + 1] - rp[r0]
    dc = D.DistCsr(n, b, 1, 3, lrp, ci[rp[r0]:rp[r1]], v[rp[r0]:rp[r1]])
    drp, dci, dv = dc.local_csr()
    rows, orp, oci, ov = dc.ghost_csr()
    assert dc.nnz_local + dc.nnz_ghost == rp[r1] - rp[r0]
    assert np.all((dci >= 0) & (dci < r1 - r0))
    assert np.all(np.diff(rows) > 0) and np.all(np.diff(orp) > 0)
    assert int(dc.recv_counts[1]) == 0 and dc.recv_counts.sum() == dc.n_ghost
    # contract checks of the native split
    with pytest.raises(Exception, match="column index out of range"):
        bad = ci[rp[r0]:rp[r1]].copy()
        bad[0] = n
        D.DistCsr(n, b, 1, 3, lrp, bad, v[rp[r0]:rp[r1]])
    with pytest.raises(Exception, match="boundaries must span"):
        D.DistCsr(n + 1, b, 1, 3, lrp, ci[rp[r0]:rp[r1]], v[rp[r0]:rp[r1]])
    with pytest.raises(Exception, match="not owned by this rank"):
        dc.set_sends(np.array([1, 0, 0]), np.array([0]))
    with pytest.raises(Exception, match="does not send to itself"):
        dc.set_sends(np.array([0, 1, 0]), np.array([r0]))
