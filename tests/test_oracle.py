"""CPU tests: the oracle restatement (oracle/ktune_oracle.c) pinned against
the reference's own outputs (tests/golden/*.npz, produced by
tests/golden/make_golden.py from the unmodified reference headers) and the
SPEC.md known-answer examples. No GPU needed."""
import os

import numpy as np
import pytest

import matgen
from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")
WORKERS = (1, 2, 3, 4, 8)
JLS = (1, 8, 16, 32, 64, 128, 256)


def load(name):
    return np.load(os.path.join(GOLD, name))


def cases(g):
    for c in range(int(g["count"])):
        p = f"c{c}_"
        yield c, p, int(g[p + "n"]), g[p + "rp"], g[p + "ci"], g[p + "v"], g[p + "x"]


# --------------------------------------------------------- golden pinning
def test_unsym_golden_bitwise():
    g = load("unsym.npz")
    for c, p, n, rp, ci, v, x in cases(g):
        assert np.array_equal(O.spmv_ref(n, rp, ci, v, x), g[p + "y_ref"]), c
        for P in WORKERS:
            b_row = O.build_row_partition(rp, P, 0)
            b_nnz = O.build_row_partition(rp, P, 1)
            assert np.array_equal(b_row, g[p + f"part_row_{P}"]), (c, P)
            assert np.array_equal(b_nnz, g[p + f"part_nnz_{P}"]), (c, P)
            assert np.array_equal(O.spmv_row_blocks(n, rp, ci, v, b_row, x), g[p + f"y_u1_{P}"])
            assert np.array_equal(O.spmv_row_blocks(n, rp, ci, v, b_nnz, x), g[p + f"y_u2_{P}"])
        if rp[-1] == 0:
            continue
        for jl in JLS:
            plan = O.build_bss_plan(n, rp, jl)
            assert plan.jl == int(g[p + f"bss{jl}_jl"])
            for f in ("slice_start", "slice_len", "slice_row", "lane_slice_ptr",
                      "row_slice_ptr", "row_start_flag"):
                assert np.array_equal(getattr(plan, f), g[p + f"bss{jl}_{f}"]), (c, jl, f)
            assert np.array_equal(O.spmv_bss(n, rp, ci, v, plan, x), g[p + f"y_u3_{jl}"])
            assert np.array_equal(O.spmv_bss(n, rp, ci, v, plan, x, u4=True),
                                  g[p + f"y_u4_{jl}"])


def test_sym_golden_bitwise():
    g = load("sym.npz")
    for c, p, n, rp, ci, v, x in cases(g):
        erp, eci, ev = O.expand_symmetric(n, rp, ci, v)
        assert np.array_equal(erp, g[p + "full_rp"]) and np.array_equal(eci, g[p + "full_ci"])
        assert np.array_equal(ev, g[p + "full_v"])
        assert np.array_equal(O.spmv_ref(n, erp, eci, ev, x), g[p + "y_ref"])
        for P in WORKERS:
            lo, hi = O.build_reduction_regions(n, rp, ci, O.build_row_partition(rp, P, 1))
            assert np.array_equal(lo, g[p + f"reg_lo_{P}"]) and np.array_equal(hi, g[p + f"reg_hi_{P}"])
            for k in range(3):
                y = O.spmv_sym(k, n, rp, ci, v, P, x)
                assert np.array_equal(y, g[p + f"y_s{k + 1}_{P}"]), (c, P, k)


def test_stencil_and_generators_golden():
    g = load("stencil.npz")
    n, rp, ci, v = matgen.stencil7(8, 8, 8)
    assert np.array_equal(rp, g["s7_rp"]) and np.array_equal(ci, g["s7_ci"])
    assert np.array_equal(v, g["s7_v"])
    assert np.array_equal(O.spmv_ref(n, rp, ci, v, g["s7_x"]), g["s7_y"])
    n, rp, ci, v = matgen.stencil27_upper(8, 8, 8)
    assert np.array_equal(rp, g["s27_rp"]) and np.array_equal(ci, g["s27_ci"])
    erp, eci, ev = O.expand_symmetric(n, rp, ci, v)
    assert np.array_equal(O.spmv_ref(n, erp, eci, ev, g["s27_x"]), g["s27_y"])
    assert np.array_equal(O.seeded_vector(64, 1), g["seeded_1_64"])
    assert np.array_equal(O.seeded_vector(64, 3), g["seeded_3_64"])
    big = O.seeded_vector(1 << 20, 2)
    assert np.sum(big) == g["seeded_2_sum"] and np.array_equal(big[-8:], g["seeded_2_last"])
    assert np.array_equal(O.probe_vector(64), g["probe_64"])
    assert np.sum(O.probe_vector(1 << 20)) == g["probe_sum_1m"]


def test_gmres_known_answer_bitwise():
    """config-5 recipe at 16^3: the restated GMRES(30)+MGS reproduces the
    reference's iterates, residual history and counts exactly."""
    g = load("stencil.npz")
    rp, ci, v, b = g["cd_rp"], g["cd_ci"], g["cd_v"], g["cd_b"]
    n = len(rp) - 1
    x, res = O.gmres_mgs(n, rp, ci, v, b, m=30, tol=1e-8, max_iters=3000)
    assert res["iterations"] == int(g["cd_iterations"])
    assert res["restarts"] == int(g["cd_restarts"])
    assert res["spmv_calls"] == int(g["cd_spmv_calls"])
    assert res["recurrence_residual"] == float(g["cd_rec"])
    assert res["true_residual"] == float(g["cd_true"])
    assert np.array_equal(x, g["cd_x"]) and np.array_equal(res["history"], g["cd_hist"])


# ---------------------------------------------------------------- SPEC KATs
def test_spec_partition_examples():
    # SPEC.md:75-77
    rp = np.array([0, 10, 11, 12, 22])
    assert list(O.build_row_partition(rp, 2, 1)) == [0, 2, 4]
    assert list(O.build_row_partition(rp, 1, 1)) == [0, 4]
    assert list(O.build_row_partition(np.array([0, 1, 2, 3, 4]), 2, 0)) == [0, 2, 4]
    with pytest.raises(O.OracleError, match="num_workers must be >= 1"):
        O.build_row_partition(rp, 0, 0)


def test_spec_regions_examples():
    # tridiagonal upper n=8, P=2 -> [1,5), [5,8)
    a = np.diag(np.full(8, 2.0)) + np.diag(np.full(7, -1.0), 1)
    n, rp, ci, v = matgen.dense_to_csr(a, upper=True)
    lo, hi = O.build_reduction_regions(n, rp, ci, np.array([0, 4, 8]))
    assert list(lo) == [1, 5] and list(hi) == [5, 8]
    n, rp, ci, v = matgen.dense_to_csr(np.diag(np.arange(1.0, 6.0)), upper=True)
    lo, hi = O.build_reduction_regions(n, rp, ci, O.build_row_partition(rp, 3, 1))
    assert not lo.any() and not hi.any()
    a = np.eye(6)
    a[0, :] = 1.0
    n, rp, ci, v = matgen.dense_to_csr(a, upper=True)
    lo, hi = O.build_reduction_regions(n, rp, ci, np.array([0, 3, 6]))
    assert hi[0] == 6


def test_spec_bss_examples():
    # SPEC.md:95-97
    n, rp, ci, v = matgen.dense_to_csr(np.diag([1.0, 2.0, 3.0]))
    p = O.build_bss_plan(n, rp, 1)
    assert len(p.slice_start) == 3 and list(p.lane_slice_ptr) == [0, 3]
    n, rp, ci, v = 1, np.array([0, 8]), np.arange(1)[[0] * 8] * 0 + np.arange(8), np.ones(8)
    # single dense row of 8 nonzeros needs an 8x8 matrix; use row 0 of an 8x8
    a = np.zeros((8, 8))
    a[0, :] = 1.0
    n, rp, ci, v = matgen.dense_to_csr(a)
    p = O.build_bss_plan(n, rp, 2)
    assert list(p.slice_len) == [4, 4] and list(p.slice_row) == [0, 0]
    with pytest.raises(O.OracleError, match="jl must be >= 1"):
        O.build_bss_plan(n, rp, 0)


def test_spec_spmv_examples():
    # SPEC.md:158-160, :178
    n, rp, ci, v = matgen.dense_to_csr(np.eye(3))
    assert list(O.spmv_ref(n, rp, ci, v, np.array([1.0, 2.0, 3.0]))) == [1, 2, 3]
    n, rp, ci, v = matgen.dense_to_csr([[2, 1], [0, 3]])
    assert list(O.spmv_ref(n, rp, ci, v, np.ones(2))) == [3, 3]
    n, rp, ci, v = matgen.dense_to_csr([[1, 0], [0, 0]])
    assert O.spmv_ref(n, rp, ci, v, np.ones(2))[1] == 0.0
    n, rp, ci, v = matgen.dense_to_csr([[2, 1], [1, 2]], upper=True)
    for k in range(3):
        assert list(O.spmv_sym(k, n, rp, ci, v, 2, np.array([1.0, 2.0]))) == [4, 5]


def test_validate_messages():
    assert O.validate(2, [0, 1, 2], [1, 0]) is None
    assert O.validate(2, [0, 2, 2], [1, 0]) == "csr: columns not strictly increasing"
    assert O.validate(2, [0, 1, 2], [0, 5]) == "csr: column index out of range"
    assert O.validate(2, [0, 1, 2], [0, 0], upper_only=True) == "sym csr: entry below the diagonal"


def test_outputs_match_rule():
    # autotune.hpp:198-204: absolute 1e-10 * max(1, ||ref||_inf)
    ref = np.array([1e6, 1.0])
    assert O.outputs_match(ref + np.array([9e-5, 0.0]), ref)
    assert not O.outputs_match(ref + np.array([0.0, 2e-4]), ref)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_restatement_matches_reference_random():
    """Randomised (SPEC.md:559-570 style) restatement == reference, bitwise."""
    R = O.Ref
    rng = np.random.default_rng(123)
    for t in range(40):
        n = int(rng.integers(1, 300))
        n, rp, ci, v = matgen.random_csr(n, float(rng.choice([0.01, 0.05, 0.2])), rng,
                                         skew=bool(t % 2), empty_frac=0.15 * (t % 3))
        x = rng.uniform(-1, 1, n)
        assert np.array_equal(O.spmv_ref(n, rp, ci, v, x), R.spmv_ref(n, rp, ci, v, x))
        for P in (1, 2, 5, 8, 16):
            for s in (0, 1):
                assert np.array_equal(O.build_row_partition(rp, P, s), R.build_row_partition(rp, P, s))
        if rp[-1]:
            for jl in (1, 3, 8, 64, 256, 10**6):
                a, b = O.build_bss_plan(n, rp, jl), R.build_bss_plan(n, rp, ci, v, jl)
                assert a.jl == b.jl and np.array_equal(a.slice_start, b.slice_start)
                assert np.array_equal(a.slice_row, b.slice_row)
                assert np.array_equal(a.row_slice_ptr, b.row_slice_ptr)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_selector_golden_with_injected_timer():
    """The reference selector driven by a scripted clock (autotune.hpp:164):
    the selections recorded in the fixture reproduce."""
    g = load("select.npz")
    assert int(g["u_u2fast_sel"]) == 1   # u2 fastest -> u2
    assert int(g["u_tie_sel"]) == 0      # exact tie u1/u2 -> lowest ordinal
    assert int(g["u_u3fast_sel"]) == 2   # u3 fastest -> smallest jl among ties
    assert int(g["s_s3fast_sel"]) == 2
    assert int(g["s_tie23_sel"]) == 0
    assert (g["u_u2fast_exec"] <= 4).all()


def test_ilu0_restatement_pinned_bitwise():
    """oracle ko_ilu0_factorize / ko_ilu0_apply == the reference's
    ilu0_factorize / ilu0_apply (tests/golden/ilu0.npz) bit for bit, and the
    same failure messages."""
    g = np.load(os.path.join(GOLD, "ilu0.npz"))
    for c in range(int(g["count"])):
        p = f"c{c}_"
        n, rp, ci, v = int(g[p + "n"]), g[p + "rp"], g[p + "ci"], g[p + "v"]
        fv, diag = O.ilu0_factorize(n, rp, ci, v)
        assert np.array_equal(diag, g[p + "diag"])
        assert np.array_equal(fv.view(np.int64), g[p + "fv"].view(np.int64)), c
        z = O.ilu0_apply(n, rp, ci, fv, diag, g[p + "r"])
        assert np.array_equal(z.view(np.int64), g[p + "z"].view(np.int64)), c
    errs = []
    for n, rp, ci, v in [
            (3, np.array([0, 2, 3, 5]), np.array([0, 1, 0, 1, 2]), np.ones(5)),
            (2, np.array([0, 2, 4]), np.array([0, 1, 0, 1]), np.ones(4)),
            (2, np.array([0, 2, 4]), np.array([0, 1, 0, 1]), np.array([0.0, 1.0, 1.0, 1.0]))]:
        with pytest.raises(O.OracleError) as e:
            O.ilu0_factorize(n, rp, ci, v)
        errs.append(str(e.value))
    assert errs == list(g["errors"])
