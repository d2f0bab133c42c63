"""Matrix Market ingest timing: libktb's parallel loader (ktb_mm_read) vs the
reference's load_matrix_market (oracle/_ref), same file, same host.

  python tools/mm_bench.py [--nx 100] [--sym] [--ref] [--keep PATH]

Writes the config-2 27-point stencil (diag + upper, --sym: symmetric file;
else the expanded general matrix) with ktb_mm_write, then times the reads.
Host-only (no GPU needed)."""
import argparse
import os
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

from oracle import oracle as O  # noqa: E402
from paper_2405_01599_b200 import ktune as K  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nx", type=int, default=100)
    ap.add_argument("--sym", action="store_true")
    ap.add_argument("--ref", action="store_true", help="also time the reference loader")
    ap.add_argument("--keep", default=None)
    ap.add_argument("--device", action="store_true", help="also time file -> device matrix")
    a = ap.parse_args()
    import matgen  # tests/matgen.py

    n, rp, ci, v = matgen.stencil27_upper(a.nx, a.nx, a.nx)
    m = K.SymCsrMatrix(n, rp, ci, v)
    if not a.sym:
        frp, fci, fv = O.expand_symmetric(n, rp, ci, v)
        m = K.CsrMatrix(n, frp, fci, fv)
    path = a.keep or os.path.join(tempfile.mkdtemp(), "a.mtx")
    t0 = time.perf_counter()
    K.write_matrix_market(path, m)
    tw = time.perf_counter() - t0
    size = os.path.getsize(path)
    print(f"file {size / 1e6:.1f} MB, n={n}, entries={m.nnz()}, write {tw:.2f}s")
    best = 1e9
    for _ in range(3):
        t0 = time.perf_counter()
        b = K.load_matrix_market(path, a.sym)
        best = min(best, time.perf_counter() - t0)
    print(f"ktb_mm_read: {best:.3f}s  {size / best / 1e9:.2f} GB/s  "
          f"{m.nnz() / best / 1e6:.1f} M entries/s  ({os.cpu_count()} host cores)")
    assert np.array_equal(b.col_idx, m.col_idx) and np.array_equal(b.values, m.values)
    if a.device:
        import torch

        K.load_matrix_market_device(path, a.sym)  # warm the CUDA context
        torch.cuda.synchronize()
        best_d = 1e9
        for _ in range(3):
            t0 = time.perf_counter()
            d = K.load_matrix_market_device(path, a.sym)
            torch.cuda.synchronize()
            best_d = min(best_d, time.perf_counter() - t0)
            del d
        print(f"file -> device (ktb_mm_read + ktb_csr_host_upload): {best_d:.3f}s  "
              f"{size / best_d / 1e9:.2f} GB/s of text")
    if a.ref:
        t0 = time.perf_counter()
        r = O.Ref.mm_load(path, a.sym)
        tr = time.perf_counter() - t0
        print(f"reference load_matrix_market: {tr:.3f}s  {size / tr / 1e9:.3f} GB/s  "
              f"speed-up {tr / best:.1f}x")
        assert np.array_equal(r[3], b.col_idx) and np.array_equal(r[4], b.values)
    if not a.keep:
        os.remove(path)


if __name__ == "__main__":
    main()
