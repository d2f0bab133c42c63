"""General row-block sharding on the device: P virtual
ranks on one GPU (the exchange done as plain copies by local_ghost_exchange,
never ranks that wait on each other), each running k_pack, its A_d plan
(every unsymmetric kernel, and the selector) and k_ghost_acc. The
concatenated y matches the oracle: |y - y_ref| <= 1e-12 (|A||x|)_i."""
import numpy as np
import pytest

import matgen
from oracle import oracle as O

pytestmark = pytest.mark.gpu

TOL = 1e-12


def _setup(n, rp, ci, v, world, kernel):
    import torch

    from paper_2405_01599_b200 import dist as D

    b = D.nnz_balanced_boundaries(rp, world)
    dcs = []
    for r in range(world):
        r0, r1 = int(b[r]), int(b[r + 1])
        dcs.append(D.DistCsr(n, b, r, world, rp[r0:r1 + 1] - rp[r0], ci[rp[r0]:rp[r1]],
                             v[rp[r0]:rp[r1]]))
    sends = D.local_send_lists(dcs)
    sp = [D.DistCsrSpMV(n, b, r, world, None, None, None, 0, kernel=kernel, sends=sends[r],
                        dc=dcs[r]) for r in range(world)]
    x = O.seeded_vector(n, 8)
    xs = [torch.from_numpy(x[int(b[r]):int(b[r + 1])].copy()).cuda() for r in range(world)]
    return b, sp, xs, x


def _run(sp, xs):
    import torch

    from paper_2405_01599_b200 import dist as D

    D.local_ghost_exchange(sp, xs)
    ys = []
    for s, x in zip(sp, xs):
        y = torch.empty(s.n_local, dtype=torch.float64, device="cuda")
        if s.A_d.nnz() > 0:
            s.plan.apply(x, y)
        else:
            y.zero_()
        s.ghost_spmv(y)
        ys.append(y)
    torch.cuda.synchronize()
    return np.concatenate([y.cpu().numpy() for y in ys])


def _check(y, n, rp, ci, v, x):
    y_ref = O.spmv_ref(n, rp, ci, v, x)
    bound = TOL * O.spmv_ref(n, rp, ci, np.abs(v), np.abs(x))
    bad = np.nonzero(np.abs(y - y_ref) > bound)[0]
    assert bad.size == 0, bad[:5]


@pytest.mark.parametrize("kernel", [0, 1, 2, None])
@pytest.mark.parametrize("world", [2, 5])
def test_virtual_ranks_random(kernel, world):
    n, rp, ci, v = matgen.random_csr(3000, 0.003, np.random.default_rng(3), empty_frac=0.1)
    b, sp, xs, x = _setup(n, rp, ci, v, world, kernel)
    _check(_run(sp, xs), n, rp, ci, v, x)


def test_virtual_ranks_powerlaw_8():
    n, rp, ci, v = matgen.powerlaw(200_000, 3, 2_000_000, 0.1, 65536)
    b, sp, xs, x = _setup(n, rp, ci, v, 8, None)
    _check(_run(sp, xs), n, rp, ci, v, x)
    # ghost volume: every rank needs a large share of x on this matrix
    assert all(s.dc.n_ghost > 0 for s in sp)


def test_single_rank_has_no_ghosts():
    n, rp, ci, v = matgen.stencil7(10, 9, 8)
    b, sp, xs, x = _setup(n, rp, ci, v, 1, 0)
    assert sp[0].dc.n_ghost == 0 and sp[0].dc.ghost_rows == 0
    _check(_run(sp, xs), n, rp, ci, v, x)
