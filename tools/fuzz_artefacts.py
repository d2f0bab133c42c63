"""Randomised bit-exact check of the integer plan artefacts built on the
device against the oracle (partition.hpp:28-96, bss.hpp:34-69, csr.hpp:88-123):
row partitions of both schemes for P from 1 to 5,000 (incl. P > n), reduction
regions, BSS plans for jl from 1 to 4,096 (incl. jl > nnz), expand_symmetric,
and the selector's report (every candidate that built is correct), on the
fuzz_all matrix families.

    python tools/fuzz_artefacts.py [cases] [seed]
"""
import faulthandler
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "tools"))

import numpy as np  # noqa: E402

import matgen  # noqa: E402
from fuzz_all import gen_unsym  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2405_01599_b200 import ktune as K  # noqa: E402


def main():
    faulthandler.enable()
    if os.environ.get("FUZZ_WATCHDOG"):
        faulthandler.dump_traceback_later(int(os.environ["FUZZ_WATCHDOG"]), exit=True)
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    rng = np.random.default_rng(seed)
    parts = plans = regs = exps = sels = 0
    for c in range(cases):
        n, rp, ci, v = gen_unsym(rng, c)
        a = K.CsrMatrix(n, rp, ci, v)
        for P in sorted(set([1, 2, 148] + [int(x) for x in rng.integers(1, 5001, 4)])):
            for scheme in (0, 1):
                got = K.build_row_partition(a, P, scheme).boundaries
                assert np.array_equal(got, O.build_row_partition(rp, P, scheme)), (c, n, P, scheme)
                parts += 1
        if rp[-1]:
            for jl in sorted(set([1, 8, 256] + [int(x) for x in rng.integers(1, 4097, 3)])):
                p, q = K.build_bss_plan(a, jl), O.build_bss_plan(n, rp, jl)
                assert p.jl == q.jl, (c, n, jl)
                for f in ("slice_start", "slice_len", "slice_row", "lane_slice_ptr",
                          "row_slice_ptr", "row_start_flag"):
                    assert np.array_equal(getattr(p, f), getattr(q, f)), (c, n, jl, f)
                plans += 1
        if c % 4 == 0 and rp[-1]:
            _, rep = K.select_spmv_unsym(a)
            # a candidate either never ran (refused layout: no time) or passed the check
            for cand in rep.candidates:
                assert cand.correct or cand.best_seconds == float("inf"), (c, n, cand.name, cand.jl)
            assert rep.selected_candidate().correct
            sels += 1
        # symmetric side: regions for both schemes, expand_symmetric
        ns = int(rng.choice([1, 7, 300, 5000, 30000]))
        ns, srp, sci, sv = matgen.random_csr(ns, min(0.5, float(rng.choice([2.0, 8.0])) / ns), rng,
                                             upper=True, skew=bool(rng.integers(0, 2)))
        s = K.SymCsrMatrix(ns, srp, sci, sv)
        for P in sorted(set([1, 3, 148] + [int(x) for x in rng.integers(1, 600, 2)])):
            for scheme in (0, 1):
                part = K.build_row_partition(s, P, scheme)
                assert np.array_equal(part.boundaries, O.build_row_partition(srp, P, scheme))
                r = K.build_reduction_regions(s, part)
                lo, hi = O.build_reduction_regions(ns, srp, sci, part.boundaries)
                assert np.array_equal(r.lo, lo) and np.array_equal(r.hi, hi), (c, ns, P, scheme)
                regs += 1
        if srp[-1]:
            frp, fci, fv = K.expand_symmetric(s).to_host()
            erp, eci, ev = O.expand_symmetric(ns, srp, sci, sv)
            assert np.array_equal(frp, erp) and np.array_equal(fci, eci), (c, ns)
            assert np.array_equal(fv.view(np.int64), ev.view(np.int64)), (c, ns)
            exps += 1
    print(f"fuzz_artefacts: seed {seed}: {parts} row partitions, {plans} BSS plans, {regs} reduction regions, "
          f"{exps} expand_symmetric bit-exact; {sels} selections with every built candidate correct")


if __name__ == "__main__":
    main()
