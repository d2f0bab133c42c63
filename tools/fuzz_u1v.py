"""Randomised bitwise check of the pair-coded record kernels against the
oracle: U1 param 106 on random banded matrices (random delta sets of 1-32
offsets, values from palettes that change per block of rows, dropped entries,
empty rows, any n) and S1 param 106 on random symmetric banded matrices. A
case either builds a plan -- then y must equal spmv_ref (resp.
spmv_ref(expand_symmetric)) bit for bit, whole and on a random row sub-range
-- or is refused with the documented error (more than 63 pairs per record).

    python tools/fuzz_u1v.py [cases] [seed]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2405_01599_b200 import ktune as K  # noqa: E402


def banded(rng, n, deltas, palette, block, keep, empty):
    """CSR with row i holding columns i + d (d in deltas, in range, kept with
    probability keep); the value of (row, delta k) is drawn from the 1-3
    palette entries that delta k may take in the row's block."""
    d = np.array(sorted(deltas), np.int64)
    rows = np.repeat(np.arange(n, dtype=np.int64), len(d))
    cols = rows + np.tile(d, n)
    k = np.tile(np.arange(len(d)), n)
    ok = (cols >= 0) & (cols < n) & (rng.random(len(cols)) < keep)
    if empty:
        ok &= (rows % empty) != 3
    rows, cols, k = rows[ok], cols[ok], k[ok]
    blk = rows // block
    choice = rng.integers(0, 3, len(rows))
    pal_idx = (blk * 7 + k * 3 + choice * (rng.integers(0, 2, len(rows)))) % len(palette)
    vals = palette[pal_idx]
    rp = np.zeros(n + 1, np.int64)
    np.add.at(rp, rows + 1, 1)
    return n, np.cumsum(rp), cols, vals


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    rng = np.random.default_rng(seed)
    special = np.array([0.0, -0.0, 5e-324, -1.7e308, 1e300, 2.0 ** -1060])
    built = refused = sym_built = sym_refused = 0
    for c in range(cases):
        n = int(rng.choice([1, 2, 31, 32, 33, 63, 64, 65, 127, 1000, 4097, 20011, 70001]))
        nd = int(rng.integers(1, 33))
        span = int(rng.choice([3, 40, 700, 5000]))
        deltas = set(int(x) for x in rng.integers(-span, span + 1, nd))
        npal = int(rng.choice([1, 2, 5, 12, 30, 80]))
        palette = np.concatenate([rng.uniform(-2, 2, npal), special[:int(rng.integers(0, 7))]])
        block = int(rng.choice([32, 64, 100, 1000]))
        keep = float(rng.choice([1.0, 0.9, 0.5]))
        empty = int(rng.choice([0, 0, 5, 64]))
        sym = c % 4 == 3
        if sym:  # diagonal + strict upper, every row with its diagonal
            deltas = {abs(d) for d in deltas} | {0}
            keep, empty = 1.0, 0
        n, rp, ci, v = banded(rng, n, deltas, palette, block, keep, empty)
        if len(ci) == 0:
            continue
        x = O.seeded_vector(n, 7 + c)
        try:
            if sym:
                a = K.SymCsrMatrix(n, rp, ci, v)
                plan = K.DevicePlan(a, K.SymKernel.s1_row, 106)
                erp, eci, ev = O.expand_symmetric(n, rp, ci, v)
                with np.errstate(all="ignore"):
                    yref = O.spmv_ref(n, erp, eci, ev, x)
            else:
                a = K.CsrMatrix(n, rp, ci, v)
                plan = K.DevicePlan(a, K.UnsymKernel.u1_row, 106)
                with np.errstate(all="ignore"):
                    yref = O.spmv_ref(n, rp, ci, v, x)
        except K.Error as e:
            msg = str(e)
            assert "pairs" in msg or "width" in msg or "slices" in msg or "triple" in msg, msg
            if sym:
                sym_refused += 1
            else:
                refused += 1
            continue
        y = np.full(n, np.nan)
        plan.apply(x, y)
        good = np.array_equal(y.view(np.int64), yref.view(np.int64)) or \
            (np.array_equal(y, yref, equal_nan=True) and np.isnan(yref).any())
        assert good, (c, sym, n, sorted(deltas), npal, block, keep, empty,
                      np.flatnonzero(y.view(np.int64) != yref.view(np.int64))[:8])
        if not sym and n > 1:
            r0 = int(rng.integers(0, n))
            r1 = int(rng.integers(r0, n + 1))
            xd = torch.from_numpy(x).cuda()
            yd = torch.full((n,), float("nan"), dtype=torch.float64, device="cuda")
            plan.apply_rows(r0, r1, xd, yd)
            got = yd.cpu().numpy()
            assert np.array_equal(got[r0:r1], yref[r0:r1], equal_nan=True), (c, n, r0, r1)
            assert np.isnan(got[:r0]).all() and np.isnan(got[r1:]).all(), (c, n, r0, r1)
        if sym:
            sym_built += 1
        else:
            built += 1
    print(f"fuzz_u1v: {cases} cases, seed {seed}: u1 106 built {built} refused {refused}; "
          f"s1 106 built {sym_built} refused {sym_refused}; all built plans bitwise equal to the oracle")


if __name__ == "__main__":
    main()
