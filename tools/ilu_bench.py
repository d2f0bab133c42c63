"""ILU(0) on config 5's operator (128^3 convection-diffusion): device
factorisation / apply / preconditioned GMRES(30) vs the reference's own
ilu0_factorize / ilu0_apply / gmres_m + ilu0 (oracle/_ref, one host thread:
the reference's ILU is sequential)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import numpy as np  # noqa: E402
import torch  # noqa: E402

import matgen  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2405_01599_b200 import ktune as K  # noqa: E402


def main():
    n, rp, ci, v = matgen.stencil7(128, 128, 128, xp=-0.7, xm=-1.3)
    a = K.CsrMatrix(n, rp, ci, v)
    _ = a.dev
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f = K.ilu0_factorize(a)
    torch.cuda.synchronize()
    t_fac = time.perf_counter() - t0
    r = torch.from_numpy(O.seeded_vector(n, 13)).cuda()
    z = torch.empty_like(r)
    for _ in range(3):
        f.apply(r, z)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    for _ in range(reps):
        f.apply(r, z)
    e1.record()
    e1.synchronize()
    t_apply = e0.elapsed_time(e1) / reps * 1e-3
    choice, _ = K.select_spmv_unsym(a)
    b = O.spmv_ref(n, rp, ci, v, np.ones(n))
    cfg = K.KrylovConfig(30, 30, 1e-8, 3000)
    K.gmres_m(a, b, cfg, plan=choice.plan, precond=f)
    t0 = time.perf_counter()
    g = K.gmres_m(a, b, cfg, plan=choice.plan, precond=f)
    t_gm = time.perf_counter() - t0
    print(f"device: factor {t_fac * 1e3:.1f} ms (incl. level analysis), apply {t_apply * 1e6:.0f} us "
          f"({f.lower_levels}+{f.upper_levels} levels, {f.launches_per_apply} launches), "
          f"gmres+ilu0 {g.iterations} its in {t_gm * 1e3:.1f} ms (true res {g.true_residual:.2e})")
    if O.ref_available():
        t0 = time.perf_counter()
        fv, diag = O.Ref.ilu0_factorize(n, rp, ci, v)
        t_rf = time.perf_counter() - t0
        rr = r.cpu().numpy()
        t0 = time.perf_counter()
        for _ in range(3):
            O.Ref.ilu0_apply(n, rp, ci, fv, diag, rr)
        t_ra = (time.perf_counter() - t0) / 3
        t0 = time.perf_counter()
        _, res = O.Ref.gmres_ilu0(n, rp, ci, v, b)
        t_rg = time.perf_counter() - t0
        print(f"reference (1 host thread): factor {t_rf * 1e3:.1f} ms, apply {t_ra * 1e3:.1f} ms, "
              f"gmres+ilu0 {res['iterations']} its in {t_rg:.2f} s")
        print(f"speed-up: factor {t_rf / t_fac:.1f}x, apply {t_ra / t_apply:.1f}x, "
              f"solve {t_rg / t_gm:.1f}x")


if __name__ == "__main__":
    main()
