"""Small invocations of the kernels with hand-written synchronisation, for
compute-sanitizer (tools/sanitize.sh): racecheck (shared-memory hazards),
synccheck (barrier / mbarrier misuse), memcheck (out-of-bounds, misaligned).

    python tools/sanitize_cases.py s3|mgs|ilu|unsym|halo
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import matgen  # noqa: E402
from oracle import oracle as O  # noqa: E402


def case_s3():
    """k_s3 (TMA ring, mbarriers, window rounds) + k_s3_fixup + k_s3_patch."""
    from paper_2405_01599_b200 import ktune as K

    mats = [matgen.stencil27_upper(48, 40, 36)]
    rng = np.random.default_rng(1)
    n = 60_000
    rows = [np.unique(np.concatenate([[i], np.minimum(i + rng.integers(1, 30_000, 3), n - 1)]))
            for i in range(n)]
    rp = np.zeros(n + 1, np.int64)
    rp[1:] = np.cumsum([len(r) for r in rows])
    mats.append((n, rp, np.concatenate(rows), rng.uniform(-1, 1, int(rp[-1]))))
    for n, rp, ci, v in mats:
        s = K.SymCsrMatrix(n, rp, ci, v)
        p = K.DevicePlan(s, K.SymKernel.s3_nnz_zero_omit)
        x = O.seeded_vector(n, 2)
        y = np.empty(n)
        for _ in range(2):
            p.apply(x, y)
        erp, eci, ev = O.expand_symmetric(n, rp, ci, v)
        ref = O.spmv_ref(n, erp, eci, ev, x)
        assert np.allclose(y, ref, rtol=1e-12, atol=1e-12), "s3"
        print("s3", n, p.s3_info())


def case_mgs():
    """k_mgs_res (cross-CTA tagged slots, resident w) on odd and even n."""
    from paper_2405_01599_b200 import ktune as K

    for dims in ((15, 13, 11), (16, 16, 12)):
        n, rp, ci, v = matgen.stencil7(*dims, xp=-0.7, xm=-1.3)
        b = O.spmv_ref(n, rp, ci, v, np.ones(n))
        a = K.CsrMatrix(n, rp, ci, v)
        r = K.gmres_m(a, b, K.KrylovConfig(30, 30, 1e-8, 200),
                      plan=K.DevicePlan(a, K.UnsymKernel.u1_row, 100))
        print("mgs", n, r.iterations, r.true_residual)


def case_ilu():
    """k_ilu_sweep_cluster (16-CTA cluster barrier per level) and the
    level-scheduled factorisation."""
    from paper_2405_01599_b200 import ktune as K

    n, rp, ci, v = matgen.stencil7(20, 18, 16, xp=-0.7, xm=-1.3)
    a = K.CsrMatrix(n, rp, ci, v)
    f = K.ilu0_factorize(a)
    r = O.seeded_vector(n, 3)
    z = np.empty(n)
    for _ in range(2):
        K.ilu0_apply(f, r, z)
    print("ilu", n, float(np.abs(z).max()))


def case_unsym():
    """U1 warp-sliced (3 shapes), U2 warp tiles (2 shapes) + merge path,
    U3 lanes and warp tiles, U4."""
    from paper_2405_01599_b200 import ktune as K

    n, rp, ci, v = matgen.random_csr(3000, 0.004, np.random.default_rng(4), skew=True,
                                     empty_frac=0.1)
    a = K.CsrMatrix(n, rp, ci, v)
    x = O.seeded_vector(n, 1)
    ref = O.spmv_ref(n, rp, ci, v, x)
    S = 1 << 16
    for k, prm in ((0, 0), (0, 100 | 64 * S), (0, 100 | 256 * S), (0, 101), (1, 8),
                   (1, 8 | 256 * S), (1, 108), (2, 8), (2, 1008), (2, 1008 | 256 * S), (3, 8)):
        y = np.empty(n)
        K.DevicePlan(a, k, prm).apply(x, y)
        assert np.allclose(y, ref, rtol=1e-12, atol=1e-12), (k, prm)
    print("unsym ok")


def case_halo():
    """The native halo operator over 3 loopback ranks (host-chunked path too)."""
    import torch

    from paper_2405_01599_b200 import dist as D

    comms = D.Comm.loopback(3)

    def rank(r):
        s = D.DistSpMV(16, 14, 12, comms[r])
        s.apply()
        xo = s.x[s.owned_offset:s.owned_offset + s.n_local].cpu().numpy().copy()
        yh = np.empty(s.n_local)
        s.apply_host(xo, yh, chunks=4)
        torch.cuda.synchronize()
        return s.y.cpu().numpy()

    D.run_ranks(3, rank)
    print("halo ok")


if __name__ == "__main__":
    globals()["case_" + sys.argv[1]]()
