"""Deterministic-kernel results for the race-stress comparison
(tests/test_chaos_gpu.py): run once with libktb.so and once with
libktb_chaos.so (KTB_LIB_NAME) and compare the saved arrays bitwise.

    KTB_LIB_NAME=libktb_chaos.so python tools/chaos_cases.py out.npz [reps]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import matgen  # noqa: E402
from oracle import oracle as O  # noqa: E402


def main():
    import torch

    from paper_2405_01599_b200 import _lib
    from paper_2405_01599_b200 import dist as D
    from paper_2405_01599_b200 import ktune as K

    out_path = sys.argv[1]
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    res = {"lib": np.array(os.path.basename(_lib.LIB_PATH))}
    S = 1 << 16

    def rep_apply(plan, x, n, tag):
        ys = []
        for _ in range(reps):
            y = np.full(n, np.nan)
            plan.apply(x, y)
            ys.append(y)
        for y in ys[1:]:  # reproducible within the run
            assert np.array_equal(y, ys[0]), tag
        res[tag] = ys[0]

    # S3: config 2 at full size (TMA ring, mbarriers, window rounds, fixup)
    a2 = K.stencil27_upper(128, 128, 128)
    x2 = O.seeded_vector(a2.n, 2)
    rep_apply(K.DevicePlan(a2, K.SymKernel.s3_nnz_zero_omit), x2, a2.n, "s3_cfg2")
    # S3 with far entries and long rows (patch pass)
    rng = np.random.default_rng(1)
    n = 60_000
    rows = []
    for i in range(n):
        c = np.minimum(i + rng.integers(1, 30_000, 3), n - 1)
        if i % 4999 == 0:
            c = np.concatenate([c, rng.integers(i, n, 300)])
        rows.append(np.unique(np.concatenate([[i], c])))
    rp = np.zeros(n + 1, np.int64)
    rp[1:] = np.cumsum([len(r) for r in rows])
    s = K.SymCsrMatrix(n, rp, np.concatenate(rows), rng.uniform(-1, 1, int(rp[-1])))
    rep_apply(K.DevicePlan(s, K.SymKernel.s3_nnz_zero_omit), O.seeded_vector(n, 3), n, "s3_far")
    # persistent coded slices: register-pipelined (104), bulk-copy staged (105),
    # and with coded values (106)
    a5 = K.stencil7(96, 80, 64, c_xm=-1.3, c_xp=-0.7)
    x5 = O.seeded_vector(a5.n, 5)
    for prm in (104, 105, 106):
        rep_apply(K.DevicePlan(a5, 0, prm), x5, a5.n, f"u1_{prm}")
    # S1 106: the expanded 27-point stencil's pair-coded records (27 slots, 4 batches)
    a27 = K.stencil27_upper(48, 40, 36)
    rep_apply(K.DevicePlan(a27, K.SymKernel.s1_row, 106), O.seeded_vector(a27.n, 2), a27.n,
              "s1_106")
    # warp tiles (smem products, swizzled row-end maps, carries), both shapes
    n, rp, ci, v = matgen.powerlaw(300_000, 3, 3_000_000, 0.1, 65536)
    a3 = K.CsrMatrix(n, rp, ci, v)
    x3 = O.seeded_vector(n, 3)
    for k, prm, tag in ((1, 8, "u2w4"), (1, 8 | 256 * S, "u2w8"), (2, 1008, "u3w4"),
                        (2, 1008 | 256 * S, "u3w8"), (2, 8, "u3"), (1, 108, "u2mp"),
                        (0, 101, "u1sorted")):
        rep_apply(K.DevicePlan(a3, k, prm), x3, n, tag)
    # MGS tag exchange: GMRES on odd n and on a 48^3 convection-diffusion
    # (odd n: k_mgs_res; even n: k_mgs_dma with 1 and 8 elements per thread)
    for dims, tag in (((15, 13, 11), "gmres_odd"), ((48, 48, 48), "gmres_48"),
                      ((96, 96, 96), "gmres_96")):
        n, rp, ci, v = matgen.stencil7(*dims, xp=-0.7, xm=-1.3)
        b = O.spmv_ref(n, rp, ci, v, np.ones(n))
        a = K.CsrMatrix(n, rp, ci, v)
        xs = []
        for _ in range(max(2, reps // 2)):
            r = K.gmres_m(a, b, K.KrylovConfig(30, 30, 1e-8, 3000),
                          plan=K.DevicePlan(a, K.UnsymKernel.u1_row, 100))
            xs.append((r.iterations, r.x.copy()))
        assert all(it == xs[0][0] and np.array_equal(x, xs[0][1]) for it, x in xs), tag
        res[tag] = xs[0][1]
        res[tag + "_its"] = np.array(xs[0][0])
    # ILU(0) cluster sweep
    n, rp, ci, v = matgen.stencil7(40, 36, 30, xp=-0.7, xm=-1.3)
    f = K.ilu0_factorize(K.CsrMatrix(n, rp, ci, v))
    r = O.seeded_vector(n, 5)
    zs = [K.ilu0_apply(f, r) for _ in range(reps)]
    assert all(np.array_equal(z, zs[0]) for z in zs)
    res["ilu"] = zs[0]
    # halo operator over 3 loopback ranks (NCCL-group protocol, overlap events)
    comms = D.Comm.loopback(3)

    def rank(k):
        sp = D.DistSpMV(64, 60, 48, comms[k])
        for _ in range(reps):
            sp.apply()
        torch.cuda.current_stream().synchronize()
        return sp.y.cpu().numpy()

    res["halo"] = np.concatenate(D.run_ranks(3, rank))
    np.savez(out_path, **res)
    print("chaos cases ok:", res["lib"], len(res) - 1, "arrays")


if __name__ == "__main__":
    main()
