"""Config-5 consumer: device-resident GMRES(30)+MGS against the reference's own
solver (golden fixture from oracle/_ref, and the C restatement at 32^3).
Dot products are reduced in parallel (not the reference's serial order), so
the iteration count may move by +-2 (SURVEY.md §7 hard part 7); the true
residual must meet tol."""
import os

import numpy as np
import pytest

import matgen
from oracle import oracle as O

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _solve(n, rp, ci, v, b, max_iters=3000):
    from paper_2405_01599_b200 import ktune as K

    a = K.CsrMatrix(n, rp, ci, v)
    plan = K.DevicePlan(a, K.UnsymKernel.u1_row)
    return K.gmres_m(a, b, K.KrylovConfig(30, 30, 1e-8, max_iters), plan=plan)


def test_gmres_golden_16cubed():
    g = np.load(os.path.join(GOLD, "stencil.npz"))
    rp, ci, v, b = g["cd_rp"], g["cd_ci"], g["cd_v"], g["cd_b"]
    r = _solve(len(rp) - 1, rp, ci, v, b)
    assert r.converged and not r.fault_convergence
    assert abs(r.iterations - int(g["cd_iterations"])) <= 2
    assert r.true_residual < 1e-8
    assert np.max(np.abs(r.x - g["cd_x"])) < 1e-6  # both within tol of x = ones
    k = min(len(r.residual_history), len(g["cd_hist"])) - 3
    assert np.allclose(r.residual_history[:k], g["cd_hist"][:k], rtol=1e-6, atol=0)


def test_gmres_32cubed_vs_restatement():
    n, rp, ci, v = matgen.stencil7(32, 32, 32, xp=-0.7, xm=-1.3)
    b = O.spmv_ref(n, rp, ci, v, np.ones(n))
    xo, ro = O.gmres_mgs(n, rp, ci, v, b)
    r = _solve(n, rp, ci, v, b)
    assert r.converged and abs(r.iterations - ro["iterations"]) <= 2
    assert r.true_residual < 1e-8
    assert r.spmv_calls == r.iterations + r.restarts + 2
    assert np.max(np.abs(r.x - 1.0)) < 1e-5


def test_gmres_max_iters_and_zero_rhs():
    n, rp, ci, v = matgen.stencil7(8, 8, 8, xp=-0.7, xm=-1.3)
    b = O.spmv_ref(n, rp, ci, v, np.ones(n))
    r = _solve(n, rp, ci, v, b, max_iters=5)
    assert not r.converged and r.iterations == 5
    r = _solve(n, rp, ci, v, np.zeros(n))
    assert r.converged and r.iterations == 0 and not r.x.any()


def test_gmres_both_mgs_kernels_and_config5(monkeypatch):
    """The resident-w MGS (default) and the streaming MGS (KTB_GMRES_STREAM_MGS,
    used when a slice does not fit on chip) against the C restatement, plus
    config 5 at full size: the reference's 653 iterations +-2, true residual
    < tol, one SpMV per iteration + one per restart cycle + the final check."""
    from paper_2405_01599_b200 import ktune as K

    n, rp, ci, v = matgen.stencil7(24, 20, 16, xp=-0.7, xm=-1.3)
    b = O.spmv_ref(n, rp, ci, v, np.ones(n))
    xo, ro = O.gmres_mgs(n, rp, ci, v, b)
    for env in ("", "1"):
        if env:
            monkeypatch.setenv("KTB_GMRES_STREAM_MGS", env)
        r = _solve(n, rp, ci, v, b)
        assert r.converged and abs(r.iterations - ro["iterations"]) <= 2, env
        assert r.true_residual < 1e-8
    monkeypatch.delenv("KTB_GMRES_STREAM_MGS")
    a = K.stencil7(128, 128, 128, c_xm=-1.3, c_xp=-0.7)
    plan = K.DevicePlan(a, K.UnsymKernel.u1_row, 100)
    import torch

    ones = torch.ones(a.n, dtype=torch.float64, device="cuda")
    bd = torch.empty_like(ones)
    plan.apply(ones, bd)
    torch.cuda.synchronize()
    r = K.gmres_m(a, bd.cpu().numpy(), K.KrylovConfig(30, 30, 1e-8, 3000), plan=plan)
    assert r.converged and abs(r.iterations - 653) <= 2 and r.true_residual < 1e-8
    assert r.spmv_calls == r.iterations + r.restarts + 2


@pytest.mark.parametrize("dims", [(24, 20, 16), (96, 64, 40), (130, 128, 126)])
def test_mgs_bulk_copy_kernel_bitwise_equals_resident_kernel(monkeypatch, dims):
    """k_mgs_dma (even n: w in registers, basis columns double-buffered in
    shared memory by bulk copies, slots one per line) keeps k_mgs_res's
    element-to-thread mapping, update arithmetic and reduction trees: the
    two solves agree in every iteration and bit for bit in x, for slices of
    1, 2 and 14 elements per thread (the last with a ragged final CTA)."""
    n, rp, ci, v = matgen.stencil7(*dims, xp=-0.7, xm=-1.3)
    assert n % 2 == 0
    b = O.spmv_ref(n, rp, ci, v, np.ones(n))
    r_dma = _solve(n, rp, ci, v, b)
    monkeypatch.setenv("KTB_GMRES_NO_DMA_MGS", "1")
    r_res = _solve(n, rp, ci, v, b)
    monkeypatch.delenv("KTB_GMRES_NO_DMA_MGS")
    assert r_dma.converged and r_dma.iterations == r_res.iterations
    assert np.array_equal(r_dma.x, r_res.x)
    assert np.array_equal(r_dma.residual_history, r_res.residual_history)


@pytest.mark.parametrize("stream_mgs", ["0", "1"])
@pytest.mark.parametrize("kernel,param", [(0, 100), (1, 8)])
def test_gmres_odd_n_unaligned_columns(monkeypatch, stream_mgs, kernel, param):
    """Odd n: basis column j starts at V + j*n, only 8-byte aligned for odd j
    (the L2 bulk prefetch must widen to 16-byte bounds). Both MGS
    kernels, two SpMV kernels; against the C restatement."""
    from paper_2405_01599_b200 import ktune as K

    if stream_mgs == "1":
        monkeypatch.setenv("KTB_GMRES_STREAM_MGS", "1")
    n, rp, ci, v = matgen.stencil7(15, 13, 11, xp=-0.7, xm=-1.3)
    assert n % 2 == 1
    b = O.spmv_ref(n, rp, ci, v, np.ones(n))
    xo, ro = O.gmres_mgs(n, rp, ci, v, b)
    a = K.CsrMatrix(n, rp, ci, v)
    plan = K.DevicePlan(a, kernel, param)
    r = K.gmres_m(a, b, K.KrylovConfig(30, 30, 1e-8, 3000), plan=plan)
    assert r.converged and abs(r.iterations - ro["iterations"]) <= 2
    assert r.true_residual < 1e-8


def test_s3_odd_n_unaligned_x():
    """S3's x front prefetch on an 8-byte-aligned x (a basis-column-like
    offset view): same y as on an aligned copy."""
    import torch

    from paper_2405_01599_b200 import ktune as K

    n, rp, ci, v = matgen.stencil27_upper(23, 19, 17)
    s = K.SymCsrMatrix(n, rp, ci, v)
    plan = K.DevicePlan(s, K.SymKernel.s3_nnz_zero_omit)
    x = O.seeded_vector(n, 2)
    buf = torch.zeros(n + 1, dtype=torch.float64, device="cuda")
    buf[1:] = torch.from_numpy(x).cuda()
    xa = torch.from_numpy(x).cuda()
    y0 = torch.empty(n, dtype=torch.float64, device="cuda")
    y1 = torch.empty_like(y0)
    plan.apply(xa, y0)
    plan.apply(buf[1:], y1)  # data_ptr % 16 == 8
    torch.cuda.synchronize()
    assert buf[1:].data_ptr() % 16 == 8
    assert torch.equal(y0, y1)
