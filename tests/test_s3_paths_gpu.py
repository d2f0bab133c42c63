"""S3 (zero-omission window, spmv.hpp:180-234 S3) on the inputs that leave
the shared-memory window layout ("a test naming the inputs on
which S3 uses the nondeterministic far path"). Since round 2 those entries
go through the per-target patch pass (k_s3_patch: fixed-order sums, one add
per target row), so S3 is deterministic on EVERY input; each case below
names which path it exercises (ktb_plan_s3_info), checks every row against
spmv_ref(expand_symmetric(A)) within 1e-12 (|A||x|)_i and checks that
repeated applies and independently built plans give bitwise the same y.

The three triggers (ktb_sym.cu s3_setup):
  * far:       an upper entry (i, j) with j - (sub-tile start) >= window
               (bandwidth beyond the ring, ~18k doubles of shared memory);
  * congested: a window slot targeted in all 64 rounds of a sub-tile
               (one column shared by more than 64 rows of a 2048-row tile);
  * long row:  more than max(32, min(64, 4 mean + 8)) stored entries.
Config 2 uses none of them."""
import numpy as np
import pytest

import matgen
from oracle import oracle as O

pytestmark = pytest.mark.gpu
TOL = 1e-12


def _sym_csr(n, rows):
    rp = np.zeros(n + 1, np.int64)
    rp[1:] = np.cumsum([len(r) for r in rows])
    ci = np.concatenate(rows).astype(np.int64)
    v = np.random.default_rng(n).uniform(-1, 1, len(ci))
    return n, rp, ci, v


def _run(n, rp, ci, v, seed=2):
    from paper_2405_01599_b200 import ktune as K

    s = K.SymCsrMatrix(n, rp, ci, v)
    x = O.seeded_vector(n, seed)
    erp, eci, ev = O.expand_symmetric(n, rp, ci, v)
    yref = O.spmv_ref(n, erp, eci, ev, x)
    absax = O.spmv_ref(n, erp, eci, np.abs(ev), np.abs(x))
    ys, infos = [], []
    for _ in range(2):  # two independently built plans
        p = K.DevicePlan(s, K.SymKernel.s3_nnz_zero_omit)
        infos.append(p.s3_info())
        for _ in range(2):
            y = np.full(n, np.nan)
            p.apply(x, y)
            ys.append(y)
    bad = np.flatnonzero(np.abs(ys[0] - yref) > TOL * absax)
    assert bad.size == 0, bad[:5]
    for y in ys[1:]:
        assert np.array_equal(y, ys[0])  # deterministic
    assert infos[0] == infos[1]
    return infos[0]


def test_config_like_stencil_uses_window_only():
    n, rp, ci, v = matgen.stencil27_upper(40, 36, 30)
    info = _run(n, rp, ci, v)
    assert info["far"] == 0 and info["long_rows"] == 0 and info["patch_rows"] == 0


def test_far_entries_beyond_the_window():
    """A band of width ~60k (> the ~18k-double window): far entries."""
    rng = np.random.default_rng(1)
    n = 120_000
    rows = []
    for i in range(n):
        off = rng.integers(1, 60_000, size=4)
        rows.append(np.unique(np.concatenate([[i], np.minimum(i + off, n - 1)])))
    info = _run(n, *_sym_csr(n, rows)[1:])
    assert info["far"] > 0 and info["patch_rows"] > 0


def test_congested_slot():
    """Every row of a 2048-row tile also touches one column just past the
    tile: one window slot targeted by far more than 64 rows of a sub-tile
    (n large enough that the 148 blocks hold whole sub-tiles)."""
    n = 148 * 4096
    rows = []
    for i in range(n):
        c = [i, min(i + 1, n - 1), min((i // 2048) * 2048 + 2048 + 100, n - 1)]
        rows.append(np.unique(np.array(c, np.int64)))
    info = _run(n, *_sym_csr(n, rows)[1:])
    assert info["far"] > 0


def test_long_rows():
    """Arrow-like rows with hundreds of entries (above the long-row cutoff)
    mixed with short rows."""
    rng = np.random.default_rng(7)
    n = 20_000
    rows = []
    for i in range(n):
        if i % 997 == 0:
            c = np.concatenate([[i], i + rng.choice(np.arange(1, n - i), size=min(400, n - i - 1),
                                                     replace=False)]) if i < n - 1 else [i]
        else:
            c = [i, min(i + 1, n - 1), min(i + 128, n - 1)]
        rows.append(np.unique(np.asarray(c, np.int64)))
    info = _run(n, *_sym_csr(n, rows)[1:])
    assert info["long_rows"] > 0 and info["patch_rows"] > 0


def test_random_wide_symmetric_families():
    rng = np.random.default_rng(5)
    for t in range(6):
        n = int(rng.integers(2000, 30_000))
        n, rp, ci, v = matgen.random_csr(n, 3.0 / n, rng, upper=True, skew=bool(t % 2))
        _run(n, rp, ci, v, seed=t + 1)
