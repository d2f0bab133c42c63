"""Randomised parity of every device plan variant against the oracle on
mid-sized random matrices (uniform random, skewed rows, banded, power-law,
runs of empty rows, one very long row; n from 1 to ~200,000): every U1 form
(lanes, 100-106), the U2 / U3 / U4 variants in both CTA shapes, S1 / S2 / S3
(both shapes) and S1 106. A plan either builds -- then |y - y_ref| <= 1e-12
(|A||x|)_i on every row, bitwise for U1 100, 102-106 and S1 106, and bitwise
reproducible on a second apply, U1 row sub-ranges leave the other rows
untouched, the pipelined host batch agrees -- or is refused with a ktune error.

    python tools/fuzz_all.py [cases] [seed]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import matgen  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2405_01599_b200 import ktune as K  # noqa: E402

S = 1 << 16
UNSYM_PLANS = [(0, 0), (0, 1), (0, 4), (0, 32), (0, 100), (0, 100 | 64 * S), (0, 100 | 256 * S),
               (0, 101), (0, 102), (0, 103), (0, 104), (0, 105), (0, 106),
               (1, 0), (1, 4), (1, 8 | 256 * S), (1, 108), (2, 4), (2, 8), (2, 16), (2, 1008),
               (2, 1008 | 256 * S), (3, 8)]
BITWISE = {100, 102, 103, 104, 105, 106}  # (101: rows > 256 are summed in tile order)
SYM_PLANS = [(16, 0), (16, 106), (17, 0), (18, 0), (18, 512 * S)]


def gen_unsym(rng, c):
    kind = c % 6
    if kind == 0:
        n = int(rng.choice([1, 2, 33, 1000, 30000]))
        return matgen.random_csr(n, float(rng.choice([0.0005, 0.003, 0.02])) if n > 100 else 0.5, rng,
                                 skew=bool(rng.integers(0, 2)), empty_frac=float(rng.choice([0, 0.3])))
    if kind == 1:
        return matgen.powerlaw(int(rng.choice([5000, 60000, 200000])), int(rng.integers(1, 99)),
                               int(rng.choice([40000, 600000, 1500000])), 0.1, 65536)
    if kind == 2:  # banded, few deltas, palette values (the coded forms build)
        n = int(rng.choice([100, 4097, 50000]))
        d = sorted(set(int(x) for x in rng.integers(-300, 301, int(rng.integers(1, 9)))))
        rows = np.repeat(np.arange(n), len(d))
        cols = rows + np.tile(d, n)
        ok = (cols >= 0) & (cols < n) & (rng.random(len(cols)) < 0.9)
        rows, cols = rows[ok], cols[ok]
        pal = rng.uniform(-1, 1, 5)
        vals = pal[(rows // 64 + cols) % 5]
        rp = np.zeros(n + 1, np.int64)
        np.add.at(rp, rows + 1, 1)
        return n, np.cumsum(rp), cols.astype(np.int64), vals
    if kind == 3:  # one very long row among short ones and runs of empty rows
        n = int(rng.choice([3000, 80000]))
        lens = rng.integers(0, 4, n)
        lens[rng.integers(0, n)] = min(n, 70000)
        lens[n // 3:n // 3 + 500] = 0
        rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        ci = np.concatenate([np.sort(rng.choice(n, int(l), replace=False)) for l in lens if l] or
                            [np.zeros(0, np.int64)]).astype(np.int64)
        return n, rp, ci, rng.uniform(-1, 1, len(ci))
    if kind == 4:
        g = [int(x) for x in rng.integers(3, 40, 3)]
        return matgen.stencil7(*g, xp=-0.7, xm=-1.3)
    n = int(rng.choice([257, 2048, 9999]))
    return matgen.random_csr(n, 0.01, rng, skew=True, empty_frac=0.1)


def check(what, y, yref, absax, bitwise):
    if bitwise:
        assert np.array_equal(y, yref), (what, "bitwise", np.flatnonzero(y != yref)[:5])
    else:
        err = np.abs(y - yref)
        assert (err <= 1e-12 * absax).all(), (what, float(err.max()))


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 60
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    rng = np.random.default_rng(seed)
    built = refused = subranges = batches = 0
    for c in range(cases):
        n, rp, ci, v = gen_unsym(rng, c)
        a = K.CsrMatrix(n, rp, ci, v)
        x = O.seeded_vector(n, 100 + c)
        yref = O.spmv_ref(n, rp, ci, v, x)
        absax = O.spmv_ref(n, rp, ci, np.abs(v), np.abs(x))
        for kern, prm in UNSYM_PLANS:
            if kern >= 2 and rp[-1] == 0:
                continue
            try:
                plan = K.DevicePlan(a, kern, prm)
            except K.Error:
                refused += 1
                continue
            y, y2 = np.full(n, np.nan), np.full(n, np.nan)
            plan.apply(x, y)
            plan.apply(x, y2)
            check((c, n, kern, prm), y, yref, absax, kern == 0 and (prm & (S - 1)) in BITWISE)
            assert np.array_equal(y, y2), (c, n, kern, prm, "not reproducible")
            built += 1
            base = prm & (S - 1)
            if kern == 0 and base != 101 and n > 1:  # row sub-range: rows outside stay untouched
                import torch

                r0 = int(rng.integers(0, n))
                r1 = int(rng.integers(r0, n + 1))
                xd = torch.from_numpy(x).cuda()
                yd = torch.full((n,), float("nan"), dtype=torch.float64, device="cuda")
                plan.apply_rows(r0, r1, xd, yd)
                got = yd.cpu().numpy()
                check((c, n, kern, prm, "rows", r0, r1), got[r0:r1], yref[r0:r1], absax[r0:r1],
                      base in BITWISE)
                assert np.isnan(got[:r0]).all() and np.isnan(got[r1:]).all(), (c, n, kern, prm, r0, r1)
                subranges += 1
            if (c + len(UNSYM_PLANS) + prm) % 7 == 0:  # the pipelined host batch: 3 vectors
                X = np.stack([O.seeded_vector(n, 300 + c + k) for k in range(3)])
                Y = np.full((3, n), np.nan)
                plan.apply_host_pipelined(X, Y)
                for k in range(3):
                    yk = O.spmv_ref(n, rp, ci, v, X[k])
                    ak = O.spmv_ref(n, rp, ci, np.abs(v), np.abs(X[k]))
                    check((c, n, kern, prm, "batch", k), Y[k], yk, ak, kern == 0 and base in BITWISE)
                batches += 1
        if c % 3 == 0:  # symmetric: the upper triangle of a random pattern, or a stencil
            if c % 2:
                g = [int(q) for q in rng.integers(3, 30, 3)]
                ns, srp, sci, sv = matgen.stencil27_upper(*g)
            else:
                ns = int(rng.choice([50, 3000, 40000]))
                ns, srp, sci, sv = matgen.random_csr(ns, float(rng.choice([0.001, 0.01])), rng,
                                                     upper=True, skew=bool(rng.integers(0, 2)))
            s = K.SymCsrMatrix(ns, srp, sci, sv)
            xs = O.seeded_vector(ns, 7 + c)
            erp, eci, ev = O.expand_symmetric(ns, srp, sci, sv)
            yref = O.spmv_ref(ns, erp, eci, ev, xs)
            absax = O.spmv_ref(ns, erp, eci, np.abs(ev), np.abs(xs))
            for kern, prm in SYM_PLANS:
                try:
                    plan = K.DevicePlan(s, kern, prm)
                except K.Error:
                    refused += 1
                    continue
                y, y2 = np.full(ns, np.nan), np.full(ns, np.nan)
                plan.apply(xs, y)
                plan.apply(xs, y2)
                check((c, ns, kern, prm), y, yref, absax, prm == 106)
                if kern == 18 or prm == 106:  # S3 and S1 106 are deterministic
                    assert np.array_equal(y, y2), (c, ns, kern, prm, "not reproducible")
                built += 1
    print(f"fuzz_all: {cases} cases, seed {seed}: {built} plans built and checked ({subranges} row sub-ranges, "
          f"{batches} pipelined host batches), {refused} refused; all within "
          "1e-12 (|A||x|)_i of the oracle (U1 100, 102-106 and S1 106 bitwise), all reproducible")


if __name__ == "__main__":
    main()
