"""GPU parity tests: the CUDA path (through the C ABI) against the CPU oracle
and the reference's golden fixtures.

Bars (BASELINE.json north_star):
  * integer artefacts (partition boundaries, reduction regions, BSS flags /
    slices / row assignment, expand_symmetric structure) bit-exact;
  * fp64 outputs |y_i - y_ref_i| <= 1e-12 * (|A||x|)_i on every row.
"""
import os

import numpy as np
import pytest

import matgen
from oracle import oracle as O

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")
TOL = 1e-12
WORKERS = (1, 2, 3, 4, 8)
JLS = (1, 8, 16, 32, 64, 128, 256)


@pytest.fixture(scope="module")
def K():
    from paper_2405_01599_b200 import ktune

    return ktune


def load(name):
    return np.load(os.path.join(GOLD, name))


def cases(g):
    for c in range(int(g["count"])):
        p = f"c{c}_"
        yield c, p, int(g[p + "n"]), g[p + "rp"], g[p + "ci"], g[p + "v"], g[p + "x"]


def assert_close(y, y_ref, absax, what=""):
    err = np.abs(np.asarray(y) - y_ref)
    bound = TOL * absax
    bad = np.nonzero(err > bound)[0]
    assert bad.size == 0, (what, bad[:5], err[bad[:5]], bound[bad[:5]])


def absax_of(n, rp, ci, v, x):
    return O.spmv_ref(n, rp, ci, np.abs(v), np.abs(x))


UNSYM = ("u1_row", "u2_nnz", "u3_bss", "u4_ss")
SYM = ("s1_row", "s2_nnz", "s3_nnz_zero_omit")


# ------------------------------------------------------------ artefacts
def test_partitions_and_bss_plans_bit_exact(K):
    g = load("unsym.npz")
    for c, p, n, rp, ci, v, x in cases(g):
        a = K.CsrMatrix(n, rp, ci, v)
        for P in WORKERS:
            part = K.build_row_partition(a, P, K.PartitionScheme.row_based)
            assert np.array_equal(part.boundaries, g[p + f"part_row_{P}"]), (c, P)
            part = K.build_row_partition(a, P, K.PartitionScheme.nnz_balanced)
            assert np.array_equal(part.boundaries, g[p + f"part_nnz_{P}"]), (c, P)
        if rp[-1] == 0:
            continue
        for jl in JLS:
            plan = K.build_bss_plan(a, jl)
            assert plan.jl == int(g[p + f"bss{jl}_jl"])
            for f in ("slice_start", "slice_len", "slice_row", "lane_slice_ptr",
                      "row_slice_ptr", "row_start_flag"):
                assert np.array_equal(getattr(plan, f), g[p + f"bss{jl}_{f}"]), (c, jl, f)


def test_regions_and_expand_symmetric_bit_exact(K):
    g = load("sym.npz")
    for c, p, n, rp, ci, v, x in cases(g):
        a = K.SymCsrMatrix(n, rp, ci, v)
        for P in WORKERS:
            part = K.build_row_partition(a, P, K.PartitionScheme.nnz_balanced)
            r = K.build_reduction_regions(a, part)
            assert np.array_equal(r.lo, g[p + f"reg_lo_{P}"]), (c, P)
            assert np.array_equal(r.hi, g[p + f"reg_hi_{P}"]), (c, P)
            part = K.build_row_partition(a, P, K.PartitionScheme.row_based)
            r = K.build_reduction_regions(a, part)
            assert np.array_equal(r.lo, g[p + f"regrow_lo_{P}"])
            assert np.array_equal(r.hi, g[p + f"regrow_hi_{P}"])
        if n and rp[-1]:
            full = K.expand_symmetric(a)
            frp, fci, fv = full.to_host()
            assert np.array_equal(frp, g[p + "full_rp"]) and np.array_equal(fci, g[p + "full_ci"])
            assert np.array_equal(fv, g[p + "full_v"])


# ------------------------------------------------------------ SpMV parity
def _run_unsym(K, a, kernel, x):
    k = K.UnsymKernel[kernel]
    part = K.build_row_partition(a, 4, K.PartitionScheme.row_based if k == 0
                                 else K.PartitionScheme.nnz_balanced)
    plan = K.build_bss_plan(a, 8) if k >= 2 else None
    return K.spmv_unsym(k, a, part if k < 2 else None, plan, x)


def test_unsym_variants_golden(K):
    g = load("unsym.npz")
    for c, p, n, rp, ci, v, x in cases(g):
        a = K.CsrMatrix(n, rp, ci, v)
        absax = absax_of(n, rp, ci, v, x)
        for kern in UNSYM:
            if kern in ("u3_bss", "u4_ss") and rp[-1] == 0:
                continue
            y = _run_unsym(K, a, kern, x)
            assert_close(y, g[p + "y_ref"], absax, (c, kern))


def test_u3_equals_u4_bitwise(K):
    g = load("unsym.npz")
    for c, p, n, rp, ci, v, x in cases(g):
        if rp[-1] == 0:
            continue
        a = K.CsrMatrix(n, rp, ci, v)
        assert np.array_equal(_run_unsym(K, a, "u3_bss", x), _run_unsym(K, a, "u4_ss", x)), c


def _run_sym(K, a, kernel, x):
    k = K.SymKernel[kernel]
    part = K.build_row_partition(a, 4, K.PartitionScheme.row_based if kernel == "s1_row"
                                 else K.PartitionScheme.nnz_balanced)
    regions = K.build_reduction_regions(a, part) if kernel == "s3_nnz_zero_omit" else None
    return K.spmv_sym(k, a, part, regions, x)


def test_sym_variants_golden(K):
    g = load("sym.npz")
    for c, p, n, rp, ci, v, x in cases(g):
        a = K.SymCsrMatrix(n, rp, ci, v)
        absax = absax_of(n, g[p + "full_rp"], g[p + "full_ci"], g[p + "full_v"], x)
        for kern in SYM:
            y = _run_sym(K, a, kern, x)
            assert_close(y, g[p + "y_ref"], absax, (c, kern))


def test_s3_is_deterministic(K):
    n, rp, ci, v = matgen.stencil27_upper(24, 20, 18)
    a = K.SymCsrMatrix(n, rp, ci, v)
    x = O.seeded_vector(n, 2)
    y0 = _run_sym(K, a, "s3_nnz_zero_omit", x)
    for _ in range(3):
        assert np.array_equal(_run_sym(K, a, "s3_nnz_zero_omit", x), y0)
    # both CTA shapes (256 x 8, 512 x 4 rows): same rounds, same sums
    for t in (256, 512):
        y = np.full(n, np.nan)
        K.DevicePlan(a, K.SymKernel.s3_nnz_zero_omit, t << 16).apply(x, y)
        assert np.array_equal(y, y0), t


def test_random_families_all_variants(K):
    """SPEC.md:559-570 style sweep: random matrices incl. skewed rows, empty
    rows, single rows, against the oracle."""
    rng = np.random.default_rng(99)
    for t in range(30):
        n = int(rng.integers(1, 700))
        n, rp, ci, v = matgen.random_csr(n, float(rng.choice([0.002, 0.02, 0.1])), rng,
                                         skew=bool(t % 2), empty_frac=0.2 * (t % 3 == 2))
        x = rng.uniform(-1, 1, n)
        a = K.CsrMatrix(n, rp, ci, v)
        yref, absax = O.spmv_ref(n, rp, ci, v, x), absax_of(n, rp, ci, v, x)
        for kern in UNSYM:
            if kern in ("u3_bss", "u4_ss") and rp[-1] == 0:
                continue
            assert_close(_run_unsym(K, a, kern, x), yref, absax, (t, kern))
        n, rp, ci, v = matgen.random_csr(n, float(rng.choice([0.005, 0.05])), rng, upper=True,
                                         skew=bool(t % 2))
        s = K.SymCsrMatrix(n, rp, ci, v)
        erp, eci, ev = O.expand_symmetric(n, rp, ci, v)
        yref, absax = O.spmv_ref(n, erp, eci, ev, x), absax_of(n, erp, eci, ev, x)
        for kern in SYM:
            assert_close(_run_sym(K, s, kern, x), yref, absax, (t, kern))


def test_long_rows_and_empty_rows(K):
    """Row-length extremes: one row holding most nonzeros (generate.hpp:73-96
    skewed_rows regime), runs of empty rows, trailing empties."""
    n = 5000
    rows = [np.arange(0, n, dtype=np.int64)]
    rows += [np.array([i], np.int64) for i in range(1, n // 2)]
    rows += [np.array([], np.int64)] * 700
    rows += [np.array([3, 17, n - 1], np.int64)]
    rows += [np.array([], np.int64)] * (n - len(rows))
    assert len(rows) == n
    rp = np.zeros(n + 1, np.int64)
    rp[1:] = np.cumsum([len(r) for r in rows])
    ci = np.concatenate(rows).astype(np.int64)
    v = np.random.default_rng(3).uniform(-1, 1, len(ci))
    x = O.seeded_vector(n, 5)
    a = K.CsrMatrix(n, rp, ci, v)
    yref, absax = O.spmv_ref(n, rp, ci, v, x), absax_of(n, rp, ci, v, x)
    for kern in UNSYM:
        assert_close(_run_unsym(K, a, kern, x), yref, absax, kern)


# ------------------------------------------------------------ configs
def test_generators_match_recipes(K):
    for dims in ((8, 8, 8), (5, 7, 3)):
        d = K.stencil7(*dims)
        rp, ci, v = d.to_host()
        n, rp2, ci2, v2 = matgen.stencil7(*dims)
        assert np.array_equal(rp, rp2) and np.array_equal(ci, ci2) and np.array_equal(v, v2)
        d = K.stencil27_upper(*dims)
        rp, ci, v = d.to_host()
        n, rp2, ci2, v2 = matgen.stencil27_upper(*dims)
        assert np.array_equal(rp, rp2) and np.array_equal(ci, ci2) and np.array_equal(v, v2)
    d = K.stencil7(6, 5, 4, diag=6.0, c_xm=-1.3, c_xp=-0.7)
    rp, ci, v = d.to_host()
    n, rp2, ci2, v2 = matgen.stencil7(6, 5, 4, xp=-0.7, xm=-1.3)
    assert np.array_equal(v, v2)


def test_config1_full_size_all_unsym(K):
    """config 1 (64^3 7-pt, n=262,144, nnz=1,810,432) on every row."""
    import torch

    a = K.stencil7(64, 64, 64)
    assert a.n == 262144 and a.nnz() == 1810432
    rp, ci, v = a.to_host()
    x = O.seeded_vector(a.n, 1)
    yref, absax = O.spmv_ref(a.n, rp, ci, v, x), absax_of(a.n, rp, ci, v, x)
    xd = torch.from_numpy(x).cuda()
    for kern in UNSYM:
        y = _run_unsym(K, a, kern, xd)
        assert_close(y.cpu().numpy(), yref, absax, kern)
    # the bench's kernel for configs 1 and 5 (U1 106, pair-coded records): bitwise
    for prm in (105, 106):
        y = torch.full_like(xd, float("nan"))
        K.DevicePlan(a, K.UnsymKernel.u1_row, prm).apply(xd, y)
        assert np.array_equal(y.cpu().numpy(), yref), prm
    a5 = K.stencil7(128, 128, 128, c_xm=-1.3, c_xp=-0.7)
    rp, ci, v = a5.to_host()
    x5 = O.seeded_vector(a5.n, 5)
    xd5 = torch.from_numpy(x5).cuda()
    y = torch.full_like(xd5, float("nan"))
    K.DevicePlan(a5, K.UnsymKernel.u1_row, 106).apply(xd5, y)
    assert np.array_equal(y.cpu().numpy(), O.spmv_ref(a5.n, rp, ci, v, x5))


def test_config2_full_size_sym(K):
    """config 2 (128^3 27-pt upper, n=2,097,152, nnz_s=28,920,060) on every
    row, all three symmetric kernels, against spmv_ref(expand_symmetric(A))."""
    import torch

    a = K.stencil27_upper(128, 128, 128)
    assert a.n == 2097152 and a.nnz() == 28920060
    rp, ci, v = a.to_host()
    erp, eci, ev = O.expand_symmetric(a.n, rp, ci, v)
    assert len(ev) == 55742968
    x = O.seeded_vector(a.n, 2)
    yref, absax = O.spmv_ref(a.n, erp, eci, ev, x), absax_of(a.n, erp, eci, ev, x)
    xd = torch.from_numpy(x).cuda()
    for kern in SYM:
        y = _run_sym(K, a, kern, xd)
        assert_close(y.cpu().numpy(), yref, absax, kern)
    # S1 106 (the bench's selected kernel: gathers over the expanded pair-coded
    # records): bitwise equal to spmv_ref(expand_symmetric(A)) on every row
    y = torch.full_like(xd, float("nan"))
    K.DevicePlan(a, K.SymKernel.s1_row, 106).apply(xd, y)
    assert np.array_equal(y.cpu().numpy(), yref)


def test_seeded_vector_device_bitwise(K):
    import ctypes as C

    import torch

    from paper_2405_01599_b200 import _lib

    n = 100003
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    assert _lib.load().ktb_seeded_vector(n, 7, 0, out.data_ptr(), None) == 0
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), O.seeded_vector(n, 7))
    part = torch.empty(100, dtype=torch.float64, device="cuda")
    assert _lib.load().ktb_seeded_vector(100, 7, 500, part.data_ptr(), None) == 0
    torch.cuda.synchronize()
    assert np.array_equal(part.cpu().numpy(), O.seeded_vector(600, 7)[500:])


# ------------------------------------------------------------ selector
def test_selector_unsym_and_sym(K):
    n, rp, ci, v = matgen.random_csr(3000, 0.004, np.random.default_rng(1), skew=True)
    a = K.CsrMatrix(n, rp, ci, v)
    choice, rep = K.select_spmv_unsym(a)
    assert rep.selected >= 0 and rep.selected_candidate().correct
    assert rep.max_executions() <= 4
    names = [c.name for c in rep.candidates]
    # U1 (lanes, warp-sliced x 3 CTA shapes, row-sorted x 3), U2 (warp tiles x
    # 2 shapes, merge path), U3 (lanes per E, warp tiles x 2 shapes)
    assert names[:17] == ["u1"] * 14 + ["u2"] * 3 and set(names[17:]) == {"u3"}
    assert all(c.correct for c in rep.candidates[14:])  # U2 and every U3 form
    # param slot (reference name jl): the warp-sliced U1, its column-coded,
    # persistent and row-sorted forms
    assert [c.jl for c in rep.candidates[1:14]] == ([100] * 3 + [102] * 3 + [106, 105, 104, 103]
                                                    + [101] * 3)
    assert [c.cta_threads for c in rep.candidates[1:7]] == [128, 64, 256] * 2
    x = O.seeded_vector(n, 1)
    y = np.empty(n)
    choice.plan.apply(x, y)
    assert_close(y, O.spmv_ref(n, rp, ci, v, x), absax_of(n, rp, ci, v, x))
    n, rp, ci, v = matgen.stencil27_upper(16, 16, 16)
    s = K.SymCsrMatrix(n, rp, ci, v)
    choice, rep = K.select_spmv_sym(s)
    assert [c.name for c in rep.candidates] == ["s1", "s1", "s2", "s3", "s3"]
    assert [c.jl for c in rep.candidates[:2]] == [rep.candidates[0].jl, 106]
    assert [c.cta_threads for c in rep.candidates[3:]] == [256, 512]
    assert all(c.correct for c in rep.candidates)
    # S1 106 (transposed products gathered from the expanded pair-coded slices):
    # bitwise equal to spmv_ref(expand_symmetric(A))
    x = O.seeded_vector(n, 2)
    y = np.full(n, np.nan)
    K.DevicePlan(s, K.SymKernel.s1_row, 106).apply(x, y)
    erp, eci, ev = O.expand_symmetric(n, rp, ci, v)
    assert np.array_equal(y, O.spmv_ref(n, erp, eci, ev, x))
    # random symmetric values: too many pairs per slice -> refused, the selector skips it
    rs = K.SymCsrMatrix(n, rp, ci, np.random.default_rng(5).uniform(-1, 1, len(ci)))
    with pytest.raises(K.Error):
        K.DevicePlan(rs, K.SymKernel.s1_row, 106)
    _, rep = K.select_spmv_sym(rs)
    assert not rep.candidates[1].correct and rep.selected_candidate().correct


def test_selector_injected_timer_and_tie_break(K):
    """autotune.hpp:164 injected timer; tie -> lowest ordinal."""
    n, rp, ci, v = matgen.random_csr(400, 0.03, np.random.default_rng(2))
    a = K.CsrMatrix(n, rp, ci, v)
    clock = {"t": 0.0}

    def now():
        clock["t"] += 1.0  # every trial measures exactly 1 s -> all tie
        return clock["t"]

    choice, rep = K.select_spmv_unsym(a, opts=K.SelectOptions(now=now))
    assert rep.selected == 0 and choice.kernel == K.UnsymKernel.u1_row
    assert all(c.best_seconds == 1.0 for c in rep.candidates if c.correct)


# ------------------------------------------------------------ contract
def test_contract_messages(K):
    n, rp, ci, v = matgen.random_csr(50, 0.1, np.random.default_rng(4))
    a = K.CsrMatrix(n, rp, ci, v)
    part = K.build_row_partition(a, 2, K.PartitionScheme.row_based)
    with pytest.raises(K.Error, match="dimension mismatch"):
        K.spmv_unsym(K.UnsymKernel.u1_row, a, part, None, np.ones(n + 1))
    with pytest.raises(K.Error, match="U1/U2 need a row partition"):
        K.spmv_unsym(K.UnsymKernel.u1_row, a, None, None, np.ones(n))
    with pytest.raises(K.Error, match="partition scheme does not match kernel"):
        K.spmv_unsym(K.UnsymKernel.u2_nnz, a, part, None, np.ones(n))
    with pytest.raises(K.Error, match="U3/U4 need a bss plan"):
        K.spmv_unsym(K.UnsymKernel.u3_bss, a, None, None, np.ones(n))
    n2, rp2, ci2, v2 = matgen.random_csr(51, 0.1, np.random.default_rng(5))
    b = K.CsrMatrix(n2, rp2, ci2, v2)
    with pytest.raises(K.Error, match="partition built for a different matrix"):
        K.spmv_unsym(K.UnsymKernel.u1_row, b, part, None, np.ones(n2))
    with pytest.raises(K.Error, match="plan built for a different matrix"):
        K.spmv_unsym(K.UnsymKernel.u3_bss, b, None, K.build_bss_plan(a, 8), np.ones(n2))
    s = K.SymCsrMatrix(*matgen.random_csr(40, 0.1, np.random.default_rng(6), upper=True))
    sp = K.build_row_partition(s, 2, K.PartitionScheme.nnz_balanced)
    with pytest.raises(K.Error, match="S3 needs reduction regions"):
        K.spmv_sym(K.SymKernel.s3_nnz_zero_omit, s, sp, None, np.ones(40))
    with pytest.raises(K.Error, match="bss plan: jl must be >= 1"):
        K.build_bss_plan(a, 0)


def test_engine_linop_counts(K):
    n, rp, ci, v = matgen.stencil7(10, 10, 10)
    a = K.CsrMatrix(n, rp, ci, v)
    choice, rep = K.select_spmv_unsym(a)
    eng = K.UnsymEngine(a, choice)
    op = eng.op()
    x = O.seeded_vector(n, 9)
    y = np.empty(n)
    for _ in range(3):
        op.apply(x, y)
    assert eng.calls() == 3 and eng.kernel_seconds() > 0
    assert_close(y, O.spmv_ref(n, rp, ci, v, x), absax_of(n, rp, ci, v, x))


def test_config3_full_size_all_unsym(K):
    """config 3 (power-law, n=4,000,000, nnz=39,552,727, 10% empty rows, rows
    up to 65,536) on every row, U1/U2/U3/U4, against the oracle."""
    import torch

    a = K.powerlaw()
    assert a.n == 4_000_000 and a.nnz() == 39_552_727
    rp, ci, v = a.to_host()
    x = O.seeded_vector(a.n, 3)
    yref, absax = O.spmv_ref(a.n, rp, ci, v, x), absax_of(a.n, rp, ci, v, x)
    xd = torch.from_numpy(x).cuda()
    for kern in UNSYM:
        y = _run_unsym(K, a, kern, xd)
        assert_close(y.cpu().numpy(), yref, absax, kern)


def test_config4_properties_full_size(K):
    """config 4 (512^3, 937,951,232 nnz) is too large for the oracle at full
    size: size-independent properties instead. A*ones = row sums (exact:
    6 - #neighbours), linearity A(2x + z) = 2Ax + Az, and a z-slab of the
    full product equals the oracle on the same slab."""
    import torch

    from paper_2405_01599_b200 import dist as D

    a = K.stencil7(512, 512, 512)
    assert a.nnz() == 937_951_232
    plan = K.DevicePlan(a, K.UnsymKernel.u1_row)
    n = a.n
    ones = torch.ones(n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(ones)
    plan.apply(ones, y)
    torch.cuda.synchronize()
    # interior rows: 6 - 6 = 0; boundary rows count missing neighbours
    idx = torch.arange(n, device="cuda", dtype=torch.int64)
    z, r = idx // (512 * 512), idx % (512 * 512)
    yy, xx = r // 512, r % 512
    missing = sum(((c == 0) | (c == 511)).to(torch.float64) for c in (xx, yy, z))
    assert torch.equal(y, missing)
    del missing, idx, z, r, yy, xx
    x = torch.from_numpy(O.seeded_vector(n, 4)).cuda()
    zz = torch.from_numpy(O.seeded_vector(n, 5)).cuda()
    ax, az, ac = torch.empty_like(x), torch.empty_like(x), torch.empty_like(x)
    plan.apply(x, ax)
    plan.apply(zz, az)
    plan.apply(2.0 * x + zz, ac)
    torch.cuda.synchronize()
    scale = (2.0 * ax.abs() + az.abs() + 16.0)
    assert ((ac - (2.0 * ax + az)).abs() <= 1e-12 * scale * 8).all()
    # slab 200..203 of the full product vs the oracle on that slab
    L = D.slab_layout(512, 512, 512, 100, 128)  # planes 400..403
    nl, rp, ci, v = D.slab_csr_numpy(L)
    xl = O.seeded_vector(n, 4)[L.col_base:L.col_base + L.x_local_len]
    yl = O.spmv_ref(nl, rp, ci, v, xl)
    absl = O.spmv_ref(nl, rp, ci, np.abs(v), np.abs(xl))
    got = ax[L.row0:L.row0 + nl].cpu().numpy()
    assert_close(got, yl, absl, "cfg4 slab")


SHAPE = 1 << 16  # param bits 16..31: CTA threads (launch-shape candidates)


def test_u2_all_tile_variants(K):
    """Every U2 implementation (warp tiles IPT 4/8 in 4- and 8-warp CTAs,
    merge path 104/108/112) on random, skewed, empty-row and long-row
    matrices; the two CTA shapes of the warp tiles are bitwise equal."""
    rng = np.random.default_rng(7)
    mats = []
    for t in range(8):
        n = int(rng.integers(1, 3000))
        mats.append(matgen.random_csr(n, float(rng.choice([0.001, 0.01, 0.05])), rng,
                                      skew=bool(t % 2), empty_frac=0.3 * (t % 3 == 2)))
    n = 6000  # one huge row, singletons, a run of empties, trailing empties
    rows = [np.arange(0, n, dtype=np.int64)] + [np.array([i], np.int64) for i in range(1, 3000)]
    rows += [np.array([], np.int64)] * 1500 + [np.array([5, 9], np.int64)] * 1000
    rows += [np.array([], np.int64)] * (n - len(rows))
    rp = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int64)
    mats.append((n, rp, np.concatenate(rows), rng.uniform(-1, 1, int(rp[-1]))))
    mats.append((4, np.zeros(5, np.int64), np.zeros(0, np.int64), np.zeros(0)))  # all empty
    for n, rp, ci, v in mats:
        x = rng.uniform(-1, 1, n)
        a = K.CsrMatrix(n, rp, ci, v)
        yref, absax = O.spmv_ref(n, rp, ci, v, x), absax_of(n, rp, ci, v, x)
        ys = {}
        for prm in (4, 8, 4 | 256 * SHAPE, 8 | 128 * SHAPE, 8 | 256 * SHAPE, 104, 108, 112):
            plan = K.DevicePlan(a, K.UnsymKernel.u2_nnz, prm)
            y = np.full(n, np.nan)
            plan.apply(x, y)
            assert_close(y, yref, absax, (n, prm))
            ys[prm] = y
        assert np.array_equal(ys[8], ys[8 | 256 * SHAPE]), n
        assert np.array_equal(ys[8], ys[8 | 128 * SHAPE]), n
        assert np.array_equal(ys[4], ys[4 | 256 * SHAPE]), n


def test_launch_shapes(K):
    """The selector's launch-shape candidates: U1 warp-sliced at 64/128/256
    threads (bitwise = spmv_ref), U3 warp tiles at 4/8 warps (bitwise equal
    to each other), each plan reporting its shape; bad shapes are refused."""
    n, rp, ci, v = matgen.stencil7(30, 20, 18, xp=-0.7, xm=-1.3)
    a = K.CsrMatrix(n, rp, ci, v)
    x = O.seeded_vector(n, 6)
    yref = O.spmv_ref(n, rp, ci, v, x)
    for t in (64, 128, 256):
        for base in (100, 101, 102):
            p = K.DevicePlan(a, K.UnsymKernel.u1_row, base | t * SHAPE)
            assert p.param == base | t * SHAPE
            y = np.full(n, np.nan)
            p.apply(x, y)
            assert np.array_equal(y, yref), (base, t)
    n, rp, ci, v = matgen.random_csr(4000, 0.003, np.random.default_rng(2), skew=True,
                                     empty_frac=0.1)
    a = K.CsrMatrix(n, rp, ci, v)
    x = O.seeded_vector(n, 7)
    yref, absax = O.spmv_ref(n, rp, ci, v, x), absax_of(n, rp, ci, v, x)
    ys = []
    for t in (128, 256):
        y = np.full(n, np.nan)
        K.DevicePlan(a, K.UnsymKernel.u3_bss, 1008 | t * SHAPE).apply(x, y)
        assert_close(y, yref, absax, t)
        ys.append(y)
    assert np.array_equal(ys[0], ys[1])
    for k, prm in ((K.UnsymKernel.u1_row, 4 | 128 * SHAPE), (K.UnsymKernel.u1_row, 100 | 96 * SHAPE),
                   (K.UnsymKernel.u3_bss, 8 | 128 * SHAPE), (K.UnsymKernel.u2_nnz, 108 | 256 * SHAPE)):
        with pytest.raises(K.Error):
            K.DevicePlan(a, k, prm)


def test_selector_times_launch_shapes_and_keeps_one_plan(K):
    """ktb_select's candidate list crosses the reference's kernels with the
    GPU variants and their CTA shapes (the GPU worker-count sweep); every
    candidate runs <= 4 times; each reports its plan-setup seconds."""
    n, rp, ci, v = matgen.stencil7(40, 40, 40)
    a = K.CsrMatrix(n, rp, ci, v)
    choice, rep = K.select_spmv_unsym(a)
    shapes = {(c.name, c.cta_threads) for c in rep.candidates}
    assert {("u1", 64), ("u1", 128), ("u1", 256), ("u2", 128), ("u2", 256),
            ("u3", 128), ("u3", 256)} <= shapes
    assert all(c.executions <= 4 for c in rep.candidates)
    assert all(c.setup_seconds >= 0 for c in rep.candidates if c.correct)
    x = O.seeded_vector(n, 1)
    y = np.empty(n)
    choice.plan.apply(x, y)
    assert_close(y, O.spmv_ref(n, rp, ci, v, x), absax_of(n, rp, ci, v, x))


def test_u1_warp_sliced_bitwise_reference(K):
    """U1 param 100 (thread per row over the SELL-32 copy) sums every row
    left to right with unfused multiply-add, exactly like the reference's U1
    worker and spmv_ref: y is bitwise equal to the oracle on random, skewed
    and empty-row matrices, config 1 and config 5 at full size, and on row
    sub-ranges. A layout whose padding would more than triple the matrix is
    refused."""
    import torch

    rng = np.random.default_rng(11)
    mats = []
    for t in range(8):
        n = int(rng.integers(1, 3000))
        mats.append(matgen.random_csr(n, float(rng.choice([0.001, 0.01, 0.05])), rng,
                                      skew=False, empty_frac=0.3 * (t % 3 == 2)))
    mats.append((4, np.zeros(5, np.int64), np.zeros(0, np.int64), np.zeros(0)))  # all empty
    mats.append((1, np.array([0, 1], np.int64), np.array([0], np.int64), np.array([2.5])))
    for n, rp, ci, v in mats:
        x = rng.uniform(-1, 1, n)
        a = K.CsrMatrix(n, rp, ci, v)
        plan = K.DevicePlan(a, K.UnsymKernel.u1_row, 100)
        assert plan.param == 100
        y = np.full(n, np.nan)
        plan.apply(x, y)
        assert np.array_equal(y, O.spmv_ref(n, rp, ci, v, x)), n
    for a, seed in ((K.stencil7(64, 64, 64), 1),
                    (K.stencil7(128, 128, 128, c_xm=-1.3, c_xp=-0.7), 5)):
        rp, ci, v = a.to_host()
        x = O.seeded_vector(a.n, seed)
        yref = O.spmv_ref(a.n, rp, ci, v, x)
        plan = K.DevicePlan(a, K.UnsymKernel.u1_row, 100)
        xd = torch.from_numpy(x).cuda()
        yd = torch.full((a.n,), float("nan"), dtype=torch.float64, device="cuda")
        plan.apply(xd, yd)
        torch.cuda.synchronize()
        assert np.array_equal(yd.cpu().numpy(), yref)
        yd.fill_(float("nan"))
        r0, r1 = 4133, a.n - 77  # unaligned to the 32-row slices
        plan.apply_rows(r0, r1, xd, yd)
        torch.cuda.synchronize()
        got = yd.cpu().numpy()
        assert np.array_equal(got[r0:r1], yref[r0:r1])
        assert np.isnan(got[:r0]).all() and np.isnan(got[r1:]).all()
    # one 6000-long row among singletons: padding 32x the matrix -> refused
    n = 6000
    rows = [np.arange(0, n, dtype=np.int64)] + [np.array([i], np.int64) for i in range(1, n)]
    rp = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int64)
    a = K.CsrMatrix(n, rp, np.concatenate(rows), rng.uniform(-1, 1, int(rp[-1])))
    with pytest.raises(Exception):
        K.DevicePlan(a, K.UnsymKernel.u1_row, 100)


def test_u1_column_coded_slices(K):
    """U1 param 102: the warp-sliced copy with each slice's columns coded as
    4-bit indices into a <= 15-entry dictionary of column deltas (col - row).
    Same entries, order and arithmetic: bitwise equal to spmv_ref on the
    stencils (configs 1 and 5 at full size, row sub-ranges), on banded
    matrices with exactly 15 distinct deltas per slice, and on empty rows;
    16 distinct deltas in one slice and random columns are refused."""
    import torch

    for a, seed in ((K.stencil7(64, 64, 64), 1),
                    (K.stencil7(128, 128, 128, c_xm=-1.3, c_xp=-0.7), 5)):
        rp, ci, v = a.to_host()
        x = O.seeded_vector(a.n, seed)
        yref = O.spmv_ref(a.n, rp, ci, v, x)
        for t in (64, 128, 256, 103, 104, 106, 105):
            plan = K.DevicePlan(a, K.UnsymKernel.u1_row,
                                t if t in (103, 104, 105, 106) else 102 | t * SHAPE)
            xd = torch.from_numpy(x).cuda()
            yd = torch.full((a.n,), float("nan"), dtype=torch.float64, device="cuda")
            plan.apply(xd, yd)
            torch.cuda.synchronize()
            assert np.array_equal(yd.cpu().numpy(), yref), t
        yd.fill_(float("nan"))
        r0, r1 = 4133, a.n - 77
        plan.apply_rows(r0, r1, xd, yd)
        torch.cuda.synchronize()
        got = yd.cpu().numpy()
        assert np.array_equal(got[r0:r1], yref[r0:r1]) and np.isnan(got[:r0]).all()

    def banded(n, deltas, rng, empty_every=0):
        rows = []
        for i in range(n):
            if empty_every and i % empty_every == 3:
                rows.append(np.zeros(0, np.int64))
                continue
            c = np.array([i + d for d in deltas if 0 <= i + d < n], np.int64)
            keep = rng.random(len(c)) < 0.8
            rows.append(np.unique(c[keep]))
        rp = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int64)
        ci = np.concatenate(rows).astype(np.int64)
        return n, rp, ci, rng.uniform(-1, 1, len(ci))

    rng = np.random.default_rng(21)
    ok15 = [-700, -300, -64, -33, -5, -2, -1, 0, 1, 2, 7, 40, 129, 512, 999]
    for n, rp, ci, v in (banded(5000, ok15, rng), banded(3000, ok15[:7], rng, empty_every=5)):
        a = K.CsrMatrix(n, rp, ci, v)
        x = O.seeded_vector(n, 4)
        y = np.full(n, np.nan)
        K.DevicePlan(a, K.UnsymKernel.u1_row, 102).apply(x, y)
        assert np.array_equal(y, O.spmv_ref(n, rp, ci, v, x))
    n, rp, ci, v = banded(4000, ok15 + [2000], rng)  # 16 deltas
    with pytest.raises(K.Error, match="15 distinct column deltas"):
        K.DevicePlan(K.CsrMatrix(n, rp, ci, v), K.UnsymKernel.u1_row, 102)
    n, rp, ci, v = matgen.random_csr(3000, 0.01, rng)
    with pytest.raises(K.Error):
        K.DevicePlan(K.CsrMatrix(n, rp, ci, v), K.UnsymKernel.u1_row, 102)


def test_u1_value_coded_slices(K):
    """U1 param 106: one record per warp slice -- a dictionary of <= 63
    (column delta, fp64 bit pattern) pairs and one 8-bit pair code per slot. The multiplied values are the stored bit patterns and the sum
    keeps spmv_ref's order: bitwise equal on banded matrices with exactly 15
    distinct pairs per slice (incl. -0.0 next to 0.0, denormals, huge
    values), with per-slice value sets that differ from slice to slice, empty
    rows, row sub-ranges, n not a multiple of 32, 27-slot rows, 63 pairs; 64
    distinct pairs in one slice, random values and rows longer than 32 are
    refused (the callers fall back to 105)."""
    import torch

    rng = np.random.default_rng(106)
    deltas = [-300, -33, -1, 0, 1, 40, 512]

    def banded(n, vals_of, empty_every=0):
        """vals_of(slice, delta index) -> the values that delta may take there."""
        rows, vals = [], []
        for i in range(n):
            if empty_every and i % empty_every == 3:
                rows.append(np.zeros(0, np.int64))
                vals.append(np.zeros(0))
                continue
            keep = [k for k, d in enumerate(deltas) if 0 <= i + d < n and rng.random() < 0.85]
            rows.append(np.array([i + deltas[k] for k in keep], np.int64))
            vals.append(np.array([rng.choice(vals_of(i // 32, k)) for k in keep], np.float64))
        rp = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int64)
        return n, rp, np.concatenate(rows).astype(np.int64), np.concatenate(vals)

    special = np.array([0.0, -0.0, 5e-324, -1.7e308, 1.0, -1.0, 6.0, 26.0, 1 / 3, -0.7, -1.3,
                        2.0 ** -40, 3.5, 1e100, 7.25])
    assert len(set(special.view(np.int64).tolist())) == 15
    # 7 deltas x 2 values + a third value on the diagonal = 15 pairs per slice
    two = lambda s, k: special[2 * k:2 * k + 2] if k != 3 else special[[6, 7, 14]]  # noqa: E731
    own = lambda s, k: np.random.default_rng(1000 * s + k).uniform(-1, 1, 2)  # noqa: E731
    cases = [banded(5003, two), banded(3000, lambda s, k: special[k:k + 1], empty_every=5),
             banded(4001, own)]  # every slice its own values
    for n, rp, ci, v in cases:
        a = K.CsrMatrix(n, rp, ci, v)
        x = O.seeded_vector(n, 4)
        yref = O.spmv_ref(n, rp, ci, v, x)
        plan = K.DevicePlan(a, K.UnsymKernel.u1_row, 106)
        y = np.full(n, np.nan)
        plan.apply(x, y)
        assert np.array_equal(y.view(np.int64), yref.view(np.int64))  # incl. the sign of zero
        xd = torch.from_numpy(x).cuda()
        yd = torch.full((n,), float("nan"), dtype=torch.float64, device="cuda")
        r0, r1 = 37, n - 45
        plan.apply_rows(r0, r1, xd, yd)
        torch.cuda.synchronize()
        got = yd.cpu().numpy()
        assert np.array_equal(got[r0:r1], yref[r0:r1]) and np.isnan(got[:r0]).all() \
            and np.isnan(got[r1:]).all()
    # an infinite x entry next to padding slots must not leak a NaN (0 * inf)
    n, rp, ci, v = cases[1]
    x = O.seeded_vector(n, 4)
    x[[0, 77, n - 1]] = np.inf
    y = np.full(n, np.nan)
    K.DevicePlan(K.CsrMatrix(n, rp, ci, v), K.UnsymKernel.u1_row, 106).apply(x, y)
    with np.errstate(invalid="ignore"):
        yref = O.spmv_ref(n, rp, ci, v, x)
    # (NaN sign/payload differs between x86 and the GPU: compare as numbers)
    assert np.array_equal(y, yref, equal_nan=True) and np.isnan(yref).sum() < 40
    # wide rows and bigger dictionaries: the expanded 27-point stencil (27 slots, 27 pairs),
    # 16 pairs, and 9 deltas x 7 values = 63 pairs
    e27 = O.expand_symmetric(*matgen.stencil27_upper(20, 17, 13))
    n27 = 20 * 17 * 13
    deltas = [-300, -33, -7, -1, 0, 1, 40, 512, 1000]
    wide = [(n27, *e27),
            banded(4000, lambda s, k: (special[2 * k:2 * k + 2] if k < 7 else special[k:k + 1])
                   if k != 3 else special[[6, 7, 14, 13]]),
            banded(3000, lambda s, k: special[k:k + 7])]
    for n, rp, ci, v in wide:
        x = O.seeded_vector(n, 4)
        y = np.full(n, np.nan)
        K.DevicePlan(K.CsrMatrix(n, rp, ci, v), K.UnsymKernel.u1_row, 106).apply(x, y)
        assert np.array_equal(y.view(np.int64), O.spmv_ref(n, rp, ci, v, x).view(np.int64))
    # 64 distinct pairs in one slice, random values (config 3's kind), rows longer than 32
    n, rp, ci, v = banded(3000, lambda s, k: special[k:k + 7] if k else special[:8])
    with pytest.raises(K.Error, match="63 distinct .column delta, value. pairs"):
        K.DevicePlan(K.CsrMatrix(n, rp, ci, v), K.UnsymKernel.u1_row, 106)
    n, rp, ci, v = banded(3000, lambda s, k: rng.uniform(-1, 1, 64))
    with pytest.raises(K.Error):
        K.DevicePlan(K.CsrMatrix(n, rp, ci, v), K.UnsymKernel.u1_row, 106)
    n, rp, ci, v = matgen.random_csr(2000, 0.03, rng)
    with pytest.raises(K.Error):
        K.DevicePlan(K.CsrMatrix(n, rp, ci, v), K.UnsymKernel.u1_row, 106)


def test_u1_sorted_slices(K):
    """U1 param 101: rows of length <= 256 sorted by length into warp slices
    (bitwise equal to spmv_ref on those rows: same left-to-right unfused sum),
    longer rows through U2 warp tiles on a compact sub-matrix (tolerance);
    random, skewed, empty-row and very long-row matrices, config 3 at full
    size."""
    import torch

    rng = np.random.default_rng(13)
    mats = []
    for t in range(6):
        n = int(rng.integers(1, 3000))
        mats.append(matgen.random_csr(n, float(rng.choice([0.001, 0.01, 0.05])), rng,
                                      skew=bool(t % 2), empty_frac=0.3 * (t % 3 == 2)))
    n = 6000  # one huge row, singletons, empties, rows just around the cap
    rows = [np.arange(0, n, dtype=np.int64)] + [np.array([i], np.int64) for i in range(1, 2000)]
    rows += [np.array([], np.int64)] * 1500
    rows += [np.sort(rng.choice(n, 256 + (i % 3) - 1, replace=False)).astype(np.int64)
             for i in range(60)]
    rows += [np.array([5, 9], np.int64)] * (n - len(rows))
    rp = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int64)
    mats.append((n, rp, np.concatenate(rows), rng.uniform(-1, 1, int(rp[-1]))))
    mats.append((4, np.zeros(5, np.int64), np.zeros(0, np.int64), np.zeros(0)))  # all empty
    mats.append((1, np.array([0, 1], np.int64), np.array([0], np.int64), np.array([2.5])))
    for n, rp, ci, v in mats:
        x = rng.uniform(-1, 1, n)
        a = K.CsrMatrix(n, rp, ci, v)
        plan = K.DevicePlan(a, K.UnsymKernel.u1_row, 101)
        y = np.full(n, np.nan)
        plan.apply(x, y)
        yref, absax = O.spmv_ref(n, rp, ci, v, x), absax_of(n, rp, ci, v, x)
        assert_close(y, yref, absax, (n, 101))
        short = np.diff(rp) <= 256
        assert np.array_equal(y[short], yref[short]), n
    a = K.powerlaw()
    rp, ci, v = a.to_host()
    x = O.seeded_vector(a.n, 3)
    yref, absax = O.spmv_ref(a.n, rp, ci, v, x), absax_of(a.n, rp, ci, v, x)
    plan = K.DevicePlan(a, K.UnsymKernel.u1_row, 101)
    y = torch.full((a.n,), float("nan"), dtype=torch.float64, device="cuda")
    plan.apply(torch.from_numpy(x).cuda(), y)
    torch.cuda.synchronize()
    got = y.cpu().numpy()
    assert_close(got, yref, absax, "cfg3 101")
    short = np.diff(rp) <= 256
    assert np.array_equal(got[short], yref[short])


def test_host_pipelined_batch(K):
    """ktb_spmv_host_pipelined: every vector's result equals the single-call
    host path (same plan), for distinct inputs (2-D) and a reused input."""
    import torch

    for a, kern, prm in ((K.stencil7(40, 30, 20), K.UnsymKernel.u1_row, 100),
                         (K.stencil27_upper(24, 20, 16), K.SymKernel.s3_nnz_zero_omit, 0)):
        plan = K.DevicePlan(a, kern, prm)
        rng = np.random.default_rng(5)
        X = torch.from_numpy(rng.uniform(-1, 1, (7, a.n))).pin_memory()
        Y = torch.full((7, a.n), float("nan"), dtype=torch.float64).pin_memory()
        plan.apply_host_pipelined(X.numpy(), Y.numpy())
        for k in range(7):
            yk = np.empty(a.n)
            plan.apply(X.numpy()[k].copy(), yk)
            assert np.array_equal(Y.numpy()[k], yk), k
        y1 = np.full(a.n, np.nan)
        plan.apply_host_pipelined(X.numpy()[3].copy(), y1, count=5)
        assert np.array_equal(y1, Y.numpy()[3])


def test_u3_warp_bss_tiles(K):
    """U3 param 1008: the branchless segmented scan as a flag-driven warp-level
    scan over 256-nonzero tiles (row starts from the reference's flag bits,
    rows from the nonempty-row map), within tolerance of spmv_ref on random,
    skewed, empty-row, leading-empty and long-row matrices and config 3, and
    of the U2 warp tiles (same tiles; a row ending exactly at a tile boundary
    is closed by the next tile, so its partial sums associate differently)."""
    import torch

    rng = np.random.default_rng(17)
    mats = []
    for t in range(8):
        n = int(rng.integers(1, 3000))
        mats.append(matgen.random_csr(n, float(rng.choice([0.001, 0.01, 0.05])), rng,
                                      skew=bool(t % 2), empty_frac=0.3 * (t % 3 == 2)))
    n = 6000  # one huge row, singletons, a run of empties, trailing empties
    rows = [np.arange(0, n, dtype=np.int64)] + [np.array([i], np.int64) for i in range(1, 3000)]
    rows += [np.array([], np.int64)] * 1500 + [np.array([5, 9], np.int64)] * 1000
    rows += [np.array([], np.int64)] * (n - len(rows))
    rp = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int64)
    mats.append((n, rp, np.concatenate(rows), rng.uniform(-1, 1, int(rp[-1]))))
    rows = [np.array([], np.int64)] * 50 + [np.array([3], np.int64)]  # leading empties
    rp = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int64)
    mats.append((51, rp, np.concatenate(rows), np.array([1.5])))
    for n, rp, ci, v in mats:
        if rp[-1] == 0:
            continue
        x = rng.uniform(-1, 1, n)
        a = K.CsrMatrix(n, rp, ci, v)
        y3, y2 = np.full(n, np.nan), np.full(n, np.nan)
        K.DevicePlan(a, K.UnsymKernel.u3_bss, 1008).apply(x, y3)
        K.DevicePlan(a, K.UnsymKernel.u2_nnz, 8).apply(x, y2)
        absax = absax_of(n, rp, ci, v, x)
        assert_close(y3, O.spmv_ref(n, rp, ci, v, x), absax, (n, "u3w"))
        assert_close(y3, y2, absax, (n, "u3w vs u2"))
    a = K.powerlaw()
    rp, ci, v = a.to_host()
    x = O.seeded_vector(a.n, 3)
    xd = torch.from_numpy(x).cuda()
    y = torch.full((a.n,), float("nan"), dtype=torch.float64, device="cuda")
    K.DevicePlan(a, K.UnsymKernel.u3_bss, 1008).apply(xd, y)
    torch.cuda.synchronize()
    assert_close(y.cpu().numpy(), O.spmv_ref(a.n, rp, ci, v, x), absax_of(a.n, rp, ci, v, x),
                 "cfg3 u3w")


def test_plans_of_one_kernel_with_different_shared_memory_needs(K):
    """The dynamic shared-memory opt-in is a per-kernel attribute, not a
    per-plan one: a plan built later with a smaller need must not lower it
    under an earlier plan's launches (U1 105 / 106 with different widths, S3
    with different windows; found by tools/fuzz_dist.py as "invalid argument"
    on loopback ranks)."""
    rng = np.random.default_rng(8)

    def banded(n, deltas):
        rows = np.repeat(np.arange(n), len(deltas))
        cols = rows + np.tile(deltas, n)
        ok = (cols >= 0) & (cols < n)
        rows, cols = rows[ok], cols[ok]
        rp = np.zeros(n + 1, np.int64)
        np.add.at(rp, rows + 1, 1)
        return n, np.cumsum(rp), cols.astype(np.int64), np.where(rows == cols, 6.0, -1.0)

    wide = banded(9000, [-600, -40, -3, -1, 0, 1, 3, 40])   # width 8
    narrow = banded(9000, [-1, 0])                          # width 2
    for prm in (105, 106):
        plans, refs = [], []
        for n, rp, ci, v in (wide, narrow):
            plans.append((K.DevicePlan(K.CsrMatrix(n, rp, ci, v), K.UnsymKernel.u1_row, prm), n))
            refs.append((n, rp, ci, v))
        for (plan, n), (n_, rp, ci, v) in zip(plans, refs):  # the wide plan runs after the narrow setup
            x = O.seeded_vector(n, 3)
            y = np.full(n, np.nan)
            plan.apply(x, y)
            assert np.array_equal(y, O.spmv_ref(n, rp, ci, v, x)), prm
    # S3: a wide-band symmetric matrix (large window), then a tridiagonal one
    s_wide = matgen.stencil27_upper(20, 18, 16)
    n2 = 7000
    rp2 = np.arange(0, 2 * n2 + 1, 2, dtype=np.int64)
    rp2[-1] = 2 * n2 - 1
    ci2 = np.stack([np.arange(n2), np.arange(1, n2 + 1)], 1).ravel()[:2 * n2 - 1].astype(np.int64)
    v2 = rng.uniform(-1, 1, len(ci2))
    pa = K.DevicePlan(K.SymCsrMatrix(*s_wide), K.SymKernel.s3_nnz_zero_omit)
    pb = K.DevicePlan(K.SymCsrMatrix(n2, rp2, ci2, v2), K.SymKernel.s3_nnz_zero_omit)
    for plan, (n, rp, ci, v) in ((pa, s_wide), (pb, (n2, rp2, ci2, v2))):
        x = O.seeded_vector(n, 5)
        y = np.full(n, np.nan)
        plan.apply(x, y)
        erp, eci, ev = O.expand_symmetric(n, rp, ci, v)
        assert_close(y, O.spmv_ref(n, erp, eci, ev, x), absax_of(n, erp, eci, ev, x), "s3")
