"""Randomised check of the device Lanczos path (krylov.lanczos_restarted_dist
on an S3 plan, lanczos.hpp:54-192) against a dense eigendecomposition: random
symmetric matrices small enough for numpy (27-point stencils on random grids,
random sparse symmetric with a dominant diagonal; n up to ~1,500), the k
largest-magnitude eigenvalues to 1e-8 relative, residuals below tol.

    python tools/fuzz_lanczos.py [cases] [seed]
"""
import faulthandler
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import matgen  # noqa: E402
from paper_2405_01599_b200 import krylov as KR  # noqa: E402
from paper_2405_01599_b200 import ktune as K  # noqa: E402


class PlanOp:
    def __init__(self, plan, n):
        self.plan, self.n_local, self.device = plan, n, 0

    def apply(self, x, y):
        self.plan.apply(x, y)


def main():
    faulthandler.enable()
    if os.environ.get("FUZZ_WATCHDOG"):
        faulthandler.dump_traceback_later(int(os.environ["FUZZ_WATCHDOG"]), exit=True)
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 12
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    rng = np.random.default_rng(seed)
    done = 0
    for c in range(cases):
        if c % 2 == 0:
            g = [int(q) for q in rng.integers(3, 12, 3)]
            n, rp, ci, v = matgen.stencil27_upper(*g)
        else:
            n = int(rng.choice([40, 300, 1200]))
            cnt = 4 * n  # strict upper entries at random places + every diagonal
            i = rng.integers(0, n, cnt)
            j = rng.integers(0, n, cnt)
            keep = i < j
            pairs = np.unique(np.stack([i[keep], j[keep]], 1), axis=0)
            rows = np.concatenate([np.arange(n), pairs[:, 0]])
            cols = np.concatenate([np.arange(n), pairs[:, 1]])
            vals = np.concatenate([rng.uniform(1.0, 30.0, n), rng.uniform(-1, 1, len(pairs))])
            o = np.lexsort((cols, rows))
            rows, ci, v = rows[o], cols[o].astype(np.int64), vals[o]
            rp = np.zeros(n + 1, np.int64)
            np.add.at(rp, rows + 1, 1)
            rp = np.cumsum(rp)
        dense = matgen.csr_to_dense(n, rp, ci, v)
        dense = dense + dense.T - np.diag(np.diag(dense))
        w = np.linalg.eigvalsh(dense)
        k = int(rng.integers(1, 5))
        order = np.argsort(-np.abs(w))
        want = w[order[:k]]
        gap = np.abs(w[order[k - 1]]) - np.abs(w[order[k]]) if k < n else 1.0
        if gap < 1e-6 * max(1.0, np.abs(w).max()):
            continue  # the k-th and (k+1)-th magnitudes tie: the set is not unique
        a = K.SymCsrMatrix(n, rp, ci, v)
        plan = K.DevicePlan(a, K.SymKernel.s3_nnz_zero_omit)
        m = int(rng.choice([20, 30]))
        if m >= n:
            continue
        res = KR.lanczos_restarted_dist(PlanOp(plan, n), k, m=m, tol=1e-9, max_iters=60000)
        tag = (c, n, k, m, res.iterations)
        assert res.converged and res.max_residual < 1e-8 * max(1.0, np.abs(w).max()), tag
        got = np.sort(np.asarray(res.eigenvalues))
        assert np.allclose(got, np.sort(want), rtol=1e-8, atol=1e-8 * np.abs(w).max()), (tag, got, want)
        done += 1
    print(f"fuzz_lanczos: seed {seed}: {done} eigenproblems, the k largest-magnitude eigenvalues equal to the "
          "dense decomposition's to 1e-8")


if __name__ == "__main__":
    main()
