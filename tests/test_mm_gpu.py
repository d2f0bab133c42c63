"""Matrix Market file -> device -> SpMV: the ingest row feeding
every kernel, checked against the oracle's spmv_ref on the same file's CRS
(|y - y_ref| <= 1e-12 (|A||x|)_i, BASELINE.json north_star)."""
import numpy as np
import pytest

import matgen
from oracle import oracle as O

pytestmark = pytest.mark.gpu

TOL = 1e-12


@pytest.fixture(scope="module")
def K():
    from paper_2405_01599_b200 import ktune

    return ktune


def _check(y, n, rp, ci, v, x):
    y_ref = O.spmv_ref(n, rp, ci, v, x)
    bound = TOL * O.spmv_ref(n, rp, ci, np.abs(v), np.abs(x))
    bad = np.nonzero(np.abs(np.asarray(y) - y_ref) > bound)[0]
    assert bad.size == 0, bad[:5]


def test_symmetric_file_all_kernels(K, tmp_path):
    n, rp, ci, v = matgen.random_csr(3000, 0.004, np.random.default_rng(5), upper=True,
                                     empty_frac=0.05)
    path = str(tmp_path / "s.mtx")
    K.write_matrix_market(path, K.SymCsrMatrix(n, rp, ci, v))
    a = K.load_matrix_market_device(path, True)
    assert a.n == n and a.nnz() == len(ci)
    frp, fci, fv = O.expand_symmetric(n, rp, ci, v)
    x = O.seeded_vector(n, 9)
    for k in K.SymKernel:
        for w in (1, 4, 148):
            sch = (K.PartitionScheme.row_based if k == K.SymKernel.s1_row
                   else K.PartitionScheme.nnz_balanced)
            part = K.build_row_partition(a, w, sch)
            reg = K.build_reduction_regions(a, part)
            _check(K.spmv_sym(k, a, part, reg, x), n, frp, fci, fv, x)
    g = K.load_matrix_market_device(path, False)  # expanded on the host
    assert g.nnz() == len(fci)
    for k in K.UnsymKernel:
        sch = (K.PartitionScheme.row_based if k == K.UnsymKernel.u1_row
               else K.PartitionScheme.nnz_balanced)
        part = K.build_row_partition(g, 8, sch)
        plan = K.build_bss_plan(g, 16) if k in (K.UnsymKernel.u3_bss, K.UnsymKernel.u4_ss) else None
        _check(K.spmv_unsym(k, g, part, plan, x), n, frp, fci, fv, x)


def test_general_file_engine(K, tmp_path):
    n, rp, ci, v = matgen.random_csr(2000, 0.005, np.random.default_rng(6), skew=True)
    path = str(tmp_path / "g.mtx")
    O.Ref.mm_write(path, n, rp, ci, v, sym=False) if O.ref_available() else \
        K.write_matrix_market(path, K.CsrMatrix(n, rp, ci, v))
    a = K.load_matrix_market(path, False)
    choice, rep = K.select_spmv_unsym(a)
    x = O.seeded_vector(n, 4)
    y = np.empty(n)
    K.UnsymEngine(a, choice).op().apply(x, y)
    _check(y, n, rp, ci, v, x)


def test_upload_ring_bytes_and_stats(K, tmp_path):
    """ktb_csr_host_upload (pinned staging ring, parallel narrowing) gives the
    same device bytes and row statistics as ktb_matrix_create, on a file big
    enough to cross several 32 MB staging chunks."""
    n, rp, ci, v = matgen.stencil27_upper(100, 100, 100)  # 13.7M stored entries
    v = v + np.random.default_rng(2).standard_normal(len(v))
    path = str(tmp_path / "big.mtx")
    K.write_matrix_market(path, K.SymCsrMatrix(n, rp, ci, v))
    d = K.load_matrix_market_device(path, True)
    ref = K.SymCsrMatrix(n, rp, ci, v).dev
    got = d.dev.download()
    want = ref.download()
    for a, b in zip(got, want):
        assert np.array_equal(a, b)
    assert (d.dev.max_row_nnz, d.dev.bandwidth) == (ref.max_row_nnz, ref.bandwidth)
