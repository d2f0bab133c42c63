"""Concurrency stress of the C ABI: T host threads, each on its own CUDA
stream, build plans of random variants on their own random matrices at the same
time (plan setup races: per-kernel attributes, lazily built caches) and apply
them repeatedly while the others do the same; every result must equal the
thread's own single-threaded oracle result (tolerance, bitwise for U1 100 /
102-106), and a symmetric matrix shared by all threads gets S1 106 / S3 plans
built concurrently (the lazily expanded matrix is shared).

    python tools/fuzz_threads.py [threads] [rounds] [seed]
"""
import faulthandler
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "tools"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import matgen  # noqa: E402
from fuzz_all import BITWISE, S, UNSYM_PLANS, gen_unsym  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2405_01599_b200 import ktune as K  # noqa: E402


def main():
    faulthandler.enable()
    if os.environ.get("FUZZ_WATCHDOG"):
        faulthandler.dump_traceback_later(int(os.environ["FUZZ_WATCHDOG"]), exit=True)
    T = int(sys.argv[1]) if len(sys.argv) > 1 else 6
    rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 6
    seed = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    shared = K.SymCsrMatrix(*matgen.stencil27_upper(24, 20, 18))
    srp, sci, sv = shared.row_ptr, shared.col_idx, shared.values
    xs = O.seeded_vector(shared.n, 2)
    erp, eci, ev = O.expand_symmetric(shared.n, srp, sci, sv)
    ys_ref = O.spmv_ref(shared.n, erp, eci, ev, xs)
    ys_abs = O.spmv_ref(shared.n, erp, eci, np.abs(ev), np.abs(xs))
    errs, counts = [], [0] * T
    start = threading.Barrier(T)

    def body(t):
        try:
            torch.cuda.set_device(0)
            rng = np.random.default_rng(1000 * seed + t)
            stream = torch.cuda.Stream()
            with torch.cuda.stream(stream):
                for rd in range(rounds):
                    n, rp, ci, v = gen_unsym(rng, int(rng.integers(0, 6)))
                    a = K.CsrMatrix(n, rp, ci, v)
                    x = O.seeded_vector(n, 5 + t)
                    yref = O.spmv_ref(n, rp, ci, v, x)
                    absax = O.spmv_ref(n, rp, ci, np.abs(v), np.abs(x))
                    xd = torch.from_numpy(x).cuda()
                    start.wait()  # every thread sets its plans up at the same time
                    plans = []
                    for i in rng.permutation(len(UNSYM_PLANS))[:8]:
                        kern, prm = UNSYM_PLANS[int(i)]
                        if kern >= 2 and rp[-1] == 0:
                            continue
                        try:
                            plans.append((kern, prm, K.DevicePlan(a, kern, prm)))
                        except K.Error:
                            pass
                    sk, sp = [(16, 106), (18, 0), (18, 512 * S), (16, 0)][int(rng.integers(0, 4))]
                    splan = K.DevicePlan(shared, sk, sp)
                    for rep in range(3):
                        for kern, prm, plan in plans:
                            yd = torch.full((n,), float("nan"), dtype=torch.float64, device="cuda")
                            plan.apply(xd, yd)
                            y = yd.cpu().numpy()
                            if kern == 0 and (prm & (S - 1)) in BITWISE:
                                assert np.array_equal(y, yref), (t, rd, n, kern, prm)
                            else:
                                assert (np.abs(y - yref) <= 1e-12 * absax).all(), (t, rd, n, kern, prm)
                            counts[t] += 1
                        ys = np.full(shared.n, np.nan)
                        splan.apply(xs, ys)
                        assert (np.abs(ys - ys_ref) <= 1e-12 * ys_abs).all(), (t, rd, "shared sym", sk, sp)
                        counts[t] += 1
        except BaseException as e:  # noqa: BLE001
            errs.append((t, e))
            import traceback

            traceback.print_exc()
            start.abort()

    ts = [threading.Thread(target=body, args=(t,)) for t in range(T)]
    for th in ts:
        th.start()
    for th in ts:
        th.join()
    assert not errs, errs[0]
    print(f"fuzz_threads: {T} threads x {rounds} rounds, seed {seed}: {sum(counts)} applies on concurrently "
          "built plans, all equal to the oracle")


if __name__ == "__main__":
    main()
