"""Test-side matrix generators (numpy). Independent restatements of the
BASELINE.json config recipes at small sizes, plus random CSR
families used by the SPEC property tests."""
from __future__ import annotations

import numpy as np


def stencil7(nx, ny, nz, diag=6.0, off=-1.0, xp=None, xm=None):
    """3-D 7-point Dirichlet stencil, full CRS, columns sorted
    (-z,-y,-x,diag,+x,+y,+z). xp/xm override the +x/-x coefficients
    (convection-diffusion, config 5)."""
    xp = off if xp is None else xp
    xm = off if xm is None else xm
    n = nx * ny * nz
    rows, cols, vals = [], [], []
    idx = np.arange(n, dtype=np.int64)
    z, rem = np.divmod(idx, nx * ny)
    y, x = np.divmod(rem, nx)
    offs = [(-nx * ny, z > 0, off), (-nx, y > 0, off), (-1, x > 0, xm), (0, np.ones(n, bool), diag),
            (1, x < nx - 1, xp), (nx, y < ny - 1, off), (nx * ny, z < nz - 1, off)]
    for d, mask, val in offs:
        r = idx[mask]
        rows.append(r)
        cols.append(r + d)
        vals.append(np.full(len(r), val))
    return _coo_to_csr(n, rows, cols, vals)


def stencil27_upper(nx, ny, nz, diag=26.0, off=-1.0):
    """3-D 27-point stencil, diagonal + strict upper triangle (config 2)."""
    n = nx * ny * nz
    idx = np.arange(n, dtype=np.int64)
    z, rem = np.divmod(idx, nx * ny)
    y, x = np.divmod(rem, nx)
    rows, cols, vals = [], [], []
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                d = (dz * ny + dy) * nx + dx
                if d < 0:
                    continue
                mask = ((x + dx >= 0) & (x + dx < nx) & (y + dy >= 0) & (y + dy < ny)
                        & (z + dz >= 0) & (z + dz < nz))
                r = idx[mask]
                rows.append(r)
                cols.append(r + d)
                vals.append(np.full(len(r), diag if d == 0 else off))
    return _coo_to_csr(n, rows, cols, vals)


def _coo_to_csr(n, rows, cols, vals):
    r = np.concatenate(rows)
    c = np.concatenate(cols)
    v = np.concatenate(vals)
    order = np.lexsort((c, r))
    r, c, v = r[order], c[order], v[order]
    rp = np.zeros(n + 1, np.int64)
    np.add.at(rp, r + 1, 1)
    rp = np.cumsum(rp)
    return n, rp, c.astype(np.int64), v.astype(np.float64)


def random_csr(n, density, rng, skew=False, empty_frac=0.0, upper=False, val_range=(-1, 1)):
    """Random square CRS; skew=True draws heavy-tailed row lengths."""
    rows = []
    for i in range(n):
        if empty_frac and rng.random() < empty_frac:
            rows.append(np.empty(0, np.int64))
            continue
        lo = i if upper else 0
        width = n - lo
        if skew:
            L = int(min(width, np.floor((1 - rng.random()) ** (-1 / 1.2))))
        else:
            L = int(rng.binomial(width, density))
        cols = np.sort(rng.choice(width, size=L, replace=False)) + lo
        if upper and (len(cols) == 0 or cols[0] != i) and rng.random() < 0.8:
            cols = np.unique(np.concatenate([[i], cols]))
        rows.append(cols.astype(np.int64))
    rp = np.zeros(n + 1, np.int64)
    rp[1:] = np.cumsum([len(c) for c in rows])
    ci = np.concatenate(rows) if rp[-1] else np.empty(0, np.int64)
    v = rng.uniform(val_range[0], val_range[1], size=len(ci))
    return n, rp, ci, v


def dense_to_csr(a, upper=False):
    a = np.asarray(a, np.float64)
    n = a.shape[0]
    rp = [0]
    ci, v = [], []
    for i in range(n):
        for j in range(i if upper else 0, n):
            if a[i, j] != 0:
                ci.append(j)
                v.append(a[i, j])
        rp.append(len(ci))
    return n, np.array(rp, np.int64), np.array(ci, np.int64), np.array(v, np.float64)


def csr_to_dense(n, rp, ci, v):
    a = np.zeros((n, n))
    for i in range(n):
        a[i, ci[rp[i]:rp[i + 1]]] = v[rp[i]:rp[i + 1]]
    return a


# ------------------------------------------------------------------ config 3
_G = np.uint64(0x9E3779B97F4A7C15)
_H = np.uint64(0xD1B54A32D192ED03)
_V = np.uint64(0xA5A5A5A5A5A5A5A5)


def _mix(z):
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def _unif(s, k):
    k = np.asarray(k, np.uint64)
    return (_mix(s + (k + np.uint64(1)) * _G) >> np.uint64(11)).astype(np.float64) * (
        1.0 / 9007199254740992.0)


def powerlaw(n=4_000_000, seed=3, target=40_000_000, empty_frac=0.1, max_len=65536):
    """Config 3 recipe, independent numpy restatement of
    paper_2405_01599_b200/csrc/ktb_gen.cu; bit-identical output."""
    with np.errstate(over="ignore"):
        i = np.arange(n, dtype=np.uint64)
        s = _mix(np.uint64(seed) + (i + np.uint64(1)) * _H)
        empty = _unif(s, 0) < empty_frac
        w1 = 1.0 - _unif(s, 1)
        w = w1 * w1
        L = np.floor(np.power(w1, -2.0 / 3.0)).astype(np.int64)
        L = np.clip(L, 1, max_len + 1)

        def le1(l):
            lf = l.astype(np.float64)
            return (lf * lf * lf) * w <= 1.0

        while True:
            up = (L <= max_len) & le1(L + 1)
            if not up.any():
                break
            L += up
        while True:
            dn = (L > 1) & ~le1(L)
            if not dn.any():
                break
            L -= dn
        L = np.minimum(L, max_len)
        L[empty] = 0
        total = int(L.sum())
        q = (L.astype(np.float64) * float(target)) / float(total)
        lens = np.clip(np.floor(q + 0.5).astype(np.int64), 1, min(max_len, n))
        lens[L == 0] = 0
        rp = np.zeros(n + 1, np.int64)
        np.cumsum(lens, out=rp[1:])
        nnz = int(rp[-1])
        row = np.repeat(np.arange(n, dtype=np.int64), lens)
        k = (np.arange(nnz, dtype=np.int64) - rp[row]).astype(np.uint64)
        zz = _mix(s[row] + (k + np.uint64(3)) * _G)
        cand = ((zz >> np.uint64(32)) * np.uint64(n)) >> np.uint64(32)
        cand = cand.astype(np.int64)
        order = np.lexsort((cand, row))
        col = cand[order]
        dup = np.nonzero((col[1:] == col[:-1]) & (row[1:] == row[:-1]))[0]
        for r in np.unique(row[dup + 1]):  # rows whose first l candidates collide
            lo, l = rp[r], rp[r + 1] - rp[r]
            taken = sorted(set(col[lo:lo + l].tolist()))
            kk = l
            while len(taken) < l:
                z = _mix(np.uint64(s[r]) + (np.uint64(kk) + np.uint64(3)) * _G)
                c = int((int(z) >> 32) * n >> 32)
                if c not in taken:
                    taken.append(c)
                    taken.sort()
                kk += 1
            col[lo:lo + l] = taken
        pos = k  # position within the sorted row
        val = 2.0 * _unif(s[row] ^ _V, pos) - 1.0
    return n, rp, col, val
