"""Matrix Market ingest: libktb's parallel loader vs
the reference's own load_matrix_market / write_matrix_market
(proj/include/ktune/matrix_market.hpp, run through oracle/_ref).

Host-only: ktb_mm_* never touch the GPU, so these run in the CPU suite.
Every accepted file must give bit-identical CRS arrays and the same return
alternative; every rejected file the same message.
"""
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2405_01599_b200 import ktune as K

import matgen

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def _ours(path, want_sym):
    try:
        a = K.load_matrix_market(path, want_sym)
    except K.Error as e:
        return ("err", str(e))
    return (int(isinstance(a, K.SymCsrMatrix)), a.n, a.row_ptr, a.col_idx, a.values)


def _ref(path, want_sym):
    try:
        return O.Ref.mm_load(path, want_sym)
    except O.OracleError as e:
        return ("err", str(e))


def _same(path, want_sym):
    a, b = _ours(path, want_sym), _ref(path, want_sym)
    if b[0] == "err" or a[0] == "err":
        assert a == b, (path, want_sym)
        return a
    assert a[0] == b[0] and a[1] == b[1], (a[:2], b[:2])
    for x, y in zip(a[2:], b[2:]):
        assert x.dtype == y.dtype and np.array_equal(x.view(np.int64), y.view(np.int64))
    return a


def _write(tmp_path, name, text):
    p = tmp_path / name
    p.write_bytes(text.encode() if isinstance(text, str) else text)
    return str(p)


HDR = "%%MatrixMarket matrix coordinate real general\n"
SYM = "%%MatrixMarket matrix coordinate real symmetric\n"


# ------------------------------------------------------------ round trips
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_general_roundtrip(tmp_path, seed):
    n, rp, ci, v = matgen.random_csr(300 + 50 * seed, 0.03, np.random.default_rng(seed),
                                     empty_frac=0.1)
    v = v * np.random.default_rng(seed).choice([1e-300, 1e-7, 1.0, 3e5, 1e300], len(v))
    ref_file, our_file = str(tmp_path / "r.mtx"), str(tmp_path / "o.mtx")
    O.Ref.mm_write(ref_file, n, rp, ci, v, sym=False)
    K.write_matrix_market(our_file, K.CsrMatrix(n, rp, ci, v))
    assert open(ref_file, "rb").read() == open(our_file, "rb").read()
    r = _same(our_file, False)
    assert np.array_equal(r[2], rp) and np.array_equal(r[3], ci) and np.array_equal(r[4], v)
    _same(our_file, True)  # not exactly symmetric -> same message


@pytest.mark.parametrize("seed", [3, 4])
def test_symmetric_roundtrip(tmp_path, seed):
    n, urp, uci, uv = matgen.random_csr(400, 0.02, np.random.default_rng(seed), upper=True,
                                        empty_frac=0.1)
    cnt = np.diff(urp)
    ref_file, our_file = str(tmp_path / "r.mtx"), str(tmp_path / "o.mtx")
    O.Ref.mm_write(ref_file, n, urp, uci, uv, sym=True)
    K.write_matrix_market(our_file, K.SymCsrMatrix(n, urp, uci, uv))
    assert open(ref_file, "rb").read() == open(our_file, "rb").read()
    s = _same(our_file, True)
    assert s[0] == 1 and np.array_equal(s[3], uci)
    g = _same(our_file, False)  # expanded to the full matrix
    assert g[0] == 0 and len(g[3]) == 2 * len(uci) - int(np.sum(uci == np.repeat(np.arange(n), cnt)))
    # the expanded general file, read back with want_symmetric, folds to the same upper
    full = str(tmp_path / "full.mtx")
    K.write_matrix_market(full, K.CsrMatrix(n, g[2], g[3], g[4]))
    f = _same(full, True)
    assert f[0] == 1 and np.array_equal(f[3], uci) and np.array_equal(f[4], uv)


# --------------------------------------------------------- accepted edges
ACCEPT = {
    "comments_blank": HDR + "% c1\n%\n\n3 3 3\n% mid\n1 1 1.5\n\n2 3 -2\n%x\n3 2 4e-3\n",
    "upper_banner": "%%MatrixMarket MATRIX Coordinate REAL General\n2 2 1\n2 1 7\n",
    "crlf_header": "%%MatrixMarket matrix coordinate real general\r\n2 2 1\r\n1 2 3.25\r\n",
    "signs_tabs": HDR + "3 3 3\n+1\t+2\t+0.5\n\t2   3 -.25\n3\t3\t+7.E+2\n",
    "trailing": HDR + "2 2 2\n1 1 1.0 extra tokens\n2 2 3abc\n",
    "adjacent_sign": HDR + "3 3 1\n1 2-3.5\n",
    "exponents": HDR + "2 2 4\n1 1 1e5\n1 2 -2.5E-3\n2 1 1.7976931348623157e308\n2 2 4.9e-324\n",
    "underflow": HDR + "2 2 2\n1 1 1e-400\n2 2 -1e-330\n",
    "dup_two": HDR + "2 2 4\n1 1 0.1\n2 2 1\n1 1 0.2\n2 1 5\n",
    "unsorted": HDR + "4 4 5\n4 1 1\n1 4 2\n2 2 3\n1 1 4\n4 4 5\n",
    "empty_matrix": HDR + "5 5 0\n",
    "empty_rows": HDR + "6 6 2\n6 6 1\n1 6 2\n",
    "no_final_newline": HDR + "2 2 2\n1 1 1\n2 2 2",
    "size_line_junk": HDR + "3 3 x\n",
    "leading_zeros": HDR + "3 3 1\n003 0002 000.5\n",
    "sym_mixed_triangles": SYM + "3 3 4\n1 1 2\n2 1 -1\n2 3 -1\n3 3 2\n",
    "sym_dup_across": SYM + "3 3 3\n2 1 1.5\n1 2 2.5\n3 3 1\n",
    "sym_banner_case": "%%MatrixMarket matrix coordinate real SYMMETRIC\n2 2 2\n2 1 1\n1 1 2\n",
    "general_symmetric": HDR + "3 3 5\n1 1 4\n1 2 -1\n2 1 -1\n2 2 4\n3 3 1\n",
}


@pytest.mark.parametrize("name", sorted(ACCEPT))
@pytest.mark.parametrize("want_sym", [False, True])
def test_accept_cases(tmp_path, name, want_sym):
    _same(_write(tmp_path, name + ".mtx", ACCEPT[name]), want_sym)


# ------------------------------------------------------- rejected inputs
REJECT = {
    "empty": ("", "empty file"),
    "banner": ("%MatrixMarket matrix coordinate real general\n1 1 0\n", "malformed header"),
    "array": ("%%MatrixMarket matrix array real general\n1 1\n1\n", "only coordinate"),
    "vector": ("%%MatrixMarket vector coordinate real general\n1 1 0\n", "only coordinate"),
    "pattern": ("%%MatrixMarket matrix coordinate pattern general\n1 1 1\n1 1\n", "pattern"),
    "complex": ("%%MatrixMarket matrix coordinate Complex general\n1 1 0\n", "complex"),
    "integer": ("%%MatrixMarket matrix coordinate integer general\n1 1 0\n", "only real"),
    "hermitian": ("%%MatrixMarket matrix coordinate real hermitian\n1 1 0\n", "unsupported symmetry"),
    "skew": ("%%MatrixMarket matrix coordinate real skew-symmetric\n1 1 0\n", "unsupported symmetry"),
    "no_symmetry": ("%%MatrixMarket matrix coordinate real\n1 1 0\n", "unsupported symmetry"),
    "no_size": (HDR + "% only comments\n", "malformed size"),
    "size_two": (HDR + "3 3\n", "malformed size"),
    "size_zero": (HDR + "0 0 0\n", "malformed size"),
    "size_neg": (HDR + "3 3 -1\n", "malformed size"),
    "size_cr_line": (HDR + "\r\n3 3 0\n", "malformed size"),
    "not_square": (HDR + "3 4 0\n", "not square"),
    "entry_short": (HDR + "2 2 1\n1 2\n", "malformed entry"),
    "entry_alpha": (HDR + "2 2 1\n1 x 3\n", "malformed entry"),
    "entry_float_idx": (HDR + "2 2 1\n1.5 2 3\n", "malformed entry"),
    "entry_inf": (HDR + "2 2 1\n1 2 inf\n", "malformed entry"),
    "entry_nan": (HDR + "2 2 1\n1 2 nan\n", "malformed entry"),
    "entry_overflow": (HDR + "2 2 1\n1 2 1e400\n", "malformed entry"),
    "entry_dot": (HDR + "2 2 1\n1 2 .\n", "malformed entry"),
    "entry_bare_e": (HDR + "2 2 1\n1 2 1e\n", "malformed entry"),
    "entry_e_sign": (HDR + "2 2 1\n1 2 1e+\n", "malformed entry"),
    "entry_double_sign": (HDR + "2 2 1\n1 2 +-1\n", "malformed entry"),
    "entry_plus_minus_idx": (HDR + "2 2 1\n+-1 2 1\n", "malformed entry"),
    "entry_idx_overflow": (HDR + "2 2 1\n99999999999999999999 1 1\n", "malformed entry"),
    "cr_only_line": (HDR + "2 2 1\n1 1 1\n\r\n", "malformed entry"),
    "spaces_line": (HDR + "2 2 1\n1 1 1\n   \n", "malformed entry"),
    "indented_comment": (HDR + "2 2 1\n %c\n1 1 1\n", "malformed entry"),
    "idx_zero": (HDR + "2 2 1\n0 1 1\n", "index out of range"),
    "idx_big": (HDR + "2 2 1\n1 3 1\n", "index out of range"),
    "idx_neg": (HDR + "2 2 1\n-1 1 1\n", "index out of range"),
    "too_few": (HDR + "2 2 3\n1 1 1\n2 2 2\n", "entry count"),
    "too_many": (HDR + "2 2 1\n1 1 1\n2 2 2\n", "entry count"),
    "first_error_wins": (HDR + "2 2 2\n1 x 1\n5 5 5\n", "malformed entry"),
    "first_error_wins2": (HDR + "2 2 2\n5 5 5\n1 x 1\n", "index out of range"),
    "general_unsym": (HDR + "2 2 2\n1 2 1\n2 1 2\n", None),  # only with want_symmetric
}


@pytest.mark.parametrize("name", sorted(REJECT))
@pytest.mark.parametrize("want_sym", [False, True])
def test_reject_cases(tmp_path, name, want_sym):
    text, frag = REJECT[name]
    path = _write(tmp_path, name + ".mtx", text)
    r = _same(path, want_sym)
    if frag is None:
        assert (r[0] == "err") == want_sym
        if want_sym:
            assert r[1] == "matrix market: general file is not numerically symmetric: " + path
        return
    assert r[0] == "err" and frag in r[1] and r[1].endswith(path)


def test_missing_and_directory(tmp_path):
    for p in [str(tmp_path / "nope.mtx")]:
        assert _ours(p, False) == _ref(p, False) == ("err", "matrix market: cannot open " + p)
    with pytest.raises(K.Error, match="cannot open"):
        K.load_matrix_market(str(tmp_path), False)
    with pytest.raises(K.Error, match="cannot open"):
        K.probe_matrix_market(str(tmp_path / "nope.mtx"))


def test_probe(tmp_path):
    p = _write(tmp_path, "a.mtx", SYM + "% c\n7 7 3\n1 1 1\n")  # entries not read
    info = K.probe_matrix_market(p)
    assert (info.n, info.entries, info.symmetric) == O.Ref.mm_probe(p) == (7, 3, True)


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("sym", [False, True])
def test_many_duplicates_match_reference_bitwise(tmp_path, seed, sym):
    """Coordinates repeated 3-6 times in shuffled files well above std::sort's
    16-element insertion-sort cut-off, values spanning 1e-3..1e16 so the
    summation order shows in the last bits: the CRS equals the reference
    loader's bit for bit (the exact std::sort path takes over
    when a run has 3+ copies)."""
    rng = np.random.default_rng(seed)
    n = 40
    coords = [(int(rng.integers(0, n)), int(rng.integers(0, n))) for _ in range(60)]
    entries = []
    for (i, j) in coords:
        for _ in range(int(rng.integers(1, 7))):
            entries.append((i, j, float(rng.choice([1e-3, 0.1, 1.0, 3.0, 1e8, 1e16]) *
                                        rng.uniform(-1, 1))))
    rng.shuffle(entries)
    text = (SYM if sym else HDR) + f"{n} {n} {len(entries)}\n" + "".join(
        f"{i + 1} {j + 1} {v!r}\n" for i, j, v in entries)
    path = _write(tmp_path, f"dup{seed}.mtx", text)
    for want in (False, True):
        _same(path, want)


# ------------------------------------------------------------------ fuzz
def _token(rng):
    parts = []
    if rng.random() < 0.3:
        parts.append(rng.choice(["+", "-", "+-", "--"]) if rng.random() < 0.2 else
                     rng.choice(["+", "-"]))
    if rng.random() < 0.85:
        parts.append(str(rng.integers(0, 10 ** rng.integers(1, 6))))
    if rng.random() < 0.4:
        parts.append("." + (str(rng.integers(0, 1000)) if rng.random() < 0.8 else ""))
    if rng.random() < 0.3:
        parts.append(rng.choice(["e", "E"]) + rng.choice(["", "+", "-"]) +
                     (str(rng.integers(0, 400)) if rng.random() < 0.85 else ""))
    if rng.random() < 0.05:
        parts.append(rng.choice(["x", "inf", "nan", "0x1p3", "d", ","]))
    return "".join(parts) or "."


def test_fuzz_entry_tokens(tmp_path):
    """Seeded token fuzz against libstdc++'s `>> index_t >> index_t >> double`
    as the reference uses it: same accept/reject, same values, bit for bit."""
    rng = np.random.default_rng(2405)
    n = 50
    for t in range(400):
        lines = []
        k = int(rng.integers(1, 5))
        for _ in range(k):
            i = rng.integers(1, n + 1) if rng.random() < 0.9 else _token(rng)
            j = rng.integers(1, n + 1) if rng.random() < 0.9 else _token(rng)
            ws = [rng.choice([" ", "\t", "  ", " \t", "\v", "\f"]) for _ in range(3)]
            lines.append(f"{i}{ws[0]}{j}{ws[1]}{_token(rng)}{ws[2] if rng.random() < 0.2 else ''}")
        path = _write(tmp_path, f"f{t}.mtx", HDR + f"{n} {n} {k}\n" + "\n".join(lines) + "\n")
        _same(path, False)


# ------------------------------------------------------- parallel ranges
def test_large_file_parallel_split(tmp_path):
    """~25 MB of entries: several parser threads, line cuts mid-file; the
    result and the earliest-error rule match the reference."""
    rng = np.random.default_rng(7)
    n, m = 200_000, 1_000_000
    r = rng.integers(1, n + 1, m)
    c = rng.integers(1, n + 1, m)
    v = rng.standard_normal(m) * 10.0 ** rng.integers(-20, 20, m)
    body = "\n".join(f"{a} {b} {x!r}" for a, b, x in zip(r.tolist(), c.tolist(), v.tolist()))
    path = _write(tmp_path, "big.mtx", HDR + "% generated\n" + f"{n} {n} {m}\n" + body + "\n")
    assert os.path.getsize(path) > 16 << 20
    _same(path, False)
    lines = body.split("\n")
    lines[m // 2] = "1 x 1"
    lines[(3 * m) // 4] = f"{n + 1} 1 1"
    bad = _write(tmp_path, "bad.mtx", HDR + f"{n} {n} {m}\n" + "\n".join(lines) + "\n")
    assert _same(bad, False)[1].startswith("matrix market: malformed entry line")


@pytest.mark.parametrize("sym", [True, False])
def test_large_sorted_files_parallel_assembly(tmp_path, sym):
    """Writer-ordered files (the parallel assembly path, with rows straddling
    the thread cuts), symmetric and general, both return alternatives."""
    n, rp, ci, v = matgen.stencil27_upper(40, 40, 40)
    v = v + np.random.default_rng(1).standard_normal(len(v))
    path = str(tmp_path / "s.mtx")
    if sym:
        K.write_matrix_market(path, K.SymCsrMatrix(n, rp, ci, v))
    else:
        frp, fci, fv = O.expand_symmetric(n, rp, ci, v)
        K.write_matrix_market(path, K.CsrMatrix(n, frp, fci, fv))
    assert os.path.getsize(path) > 8 << 20
    s = _same(path, True)
    assert s[0] == 1 and np.array_equal(s[2], rp) and np.array_equal(s[3], ci)
    _same(path, False)
