"""General row-block sharding on the device through the
native exchange (ktb_dist_connect / ktb_dist_spmv, csrc/ktb_comm.cu): P
in-process loopback ranks on one GPU (one host thread each; messages matched
on the host, never ranks waiting on each other inside a kernel), each
running k_pack, the grouped ghost send/recv, its A_d plan (every
unsymmetric kernel, and the selector) and k_ghost_acc. The concatenated y
matches the oracle: |y - y_ref| <= 1e-12 (|A||x|)_i. The ghost lists the
native connect derives equal the Python restatement's."""
import numpy as np
import pytest

import matgen
from oracle import oracle as O

pytestmark = pytest.mark.gpu

TOL = 1e-12


def _run(n, rp, ci, v, world, kernel, reps=2):
    import torch

    from paper_2405_01599_b200 import dist as D

    b = D.nnz_balanced_boundaries(rp, world)
    comms = D.Comm.loopback(world)
    x = O.seeded_vector(n, 8)

    def rank(r):
        r0, r1 = int(b[r]), int(b[r + 1])
        sp = D.DistCsrSpMV(n, b, comms[r], rp[r0:r1 + 1] - rp[r0], ci[rp[r0]:rp[r1]],
                           v[rp[r0]:rp[r1]], kernel=kernel)
        xo = torch.from_numpy(x[r0:r1].copy()).cuda()
        y = torch.empty(max(sp.n_local, 1), dtype=torch.float64, device="cuda")
        for _ in range(reps):
            sp.apply(xo, y[:sp.n_local])
        torch.cuda.current_stream().synchronize()
        return sp, y[:sp.n_local].cpu().numpy()

    outs = D.run_ranks(world, rank)
    return b, [o[0] for o in outs], np.concatenate([o[1] for o in outs]), x


def _check(y, n, rp, ci, v, x):
    y_ref = O.spmv_ref(n, rp, ci, v, x)
    bound = TOL * O.spmv_ref(n, rp, ci, np.abs(v), np.abs(x))
    bad = np.nonzero(np.abs(y - y_ref) > bound)[0]
    assert bad.size == 0, bad[:5]


@pytest.mark.parametrize("kernel", [0, 1, 2, None])
@pytest.mark.parametrize("world", [2, 5])
def test_virtual_ranks_random(kernel, world):
    n, rp, ci, v = matgen.random_csr(3000, 0.003, np.random.default_rng(3), empty_frac=0.1)
    b, sp, y, x = _run(n, rp, ci, v, world, kernel)
    _check(y, n, rp, ci, v, x)


def test_native_send_lists_equal_restatement():
    from paper_2405_01599_b200 import dist as D

    n, rp, ci, v = matgen.random_csr(2000, 0.004, np.random.default_rng(5), empty_frac=0.05)
    world = 4
    b, sp, y, x = _run(n, rp, ci, v, world, 0, reps=1)
    want = D.local_send_lists([s.dc for s in sp])
    for s, (counts, cols) in zip(sp, want):
        # what each rank's native connect received = what its peers need
        assert np.array_equal(s.dc.send_counts, counts)
        assert np.array_equal(s.dc.send_cols, cols)
    _check(y, n, rp, ci, v, x)


def test_virtual_ranks_powerlaw_8():
    n, rp, ci, v = matgen.powerlaw(200_000, 3, 2_000_000, 0.1, 65536)
    b, sp, y, x = _run(n, rp, ci, v, 8, None)
    _check(y, n, rp, ci, v, x)
    # ghost volume: every rank needs a large share of x on this matrix
    assert all(s.dc.n_ghost > 0 for s in sp)


def test_single_rank_has_no_ghosts():
    n, rp, ci, v = matgen.stencil7(10, 9, 8)
    b, sp, y, x = _run(n, rp, ci, v, 1, 0)
    assert sp[0].dc.n_ghost == 0 and sp[0].dc.ghost_rows == 0
    _check(y, n, rp, ci, v, x)


def test_nccl_world1_general_split():
    """The general split over the real NCCL communicator at world 1."""
    import torch

    from paper_2405_01599_b200 import dist as D

    n, rp, ci, v = matgen.random_csr(1500, 0.005, np.random.default_rng(9))
    c = D.Comm.nccl(device=0)
    sp = D.DistCsrSpMV(n, D.nnz_balanced_boundaries(rp, 1), c, rp, ci, v, kernel=None)
    x = O.seeded_vector(n, 8)
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    sp.apply(torch.from_numpy(x).cuda(), y)
    torch.cuda.synchronize()
    _check(y.cpu().numpy(), n, rp, ci, v, x)
