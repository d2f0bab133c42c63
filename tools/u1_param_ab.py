"""A/B of U1 variants by plan param (100 = warp-sliced, 102 = column-coded)
on configs 1, 5 and 4 (512^3), cold L2 per apply, CUDA events, alternated.

    python tools/u1_param_ab.py 100 102 [--reps 200]
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


def main():
    params = [int(a) for a in sys.argv[1:] if a.isdigit()]
    reps = 200
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    mats = [("cfg1 64^3", lambda: K.stencil7(64, 64, 64), 1),
            ("cfg5 128^3 cd", lambda: K.stencil7(128, 128, 128, c_xm=-1.3, c_xp=-0.7), 5),
            ("cfg4 512^3", lambda: K.stencil7(512, 512, 512), 4)]
    for name, mk, seed in mats:
        a = mk()
        x = torch.from_numpy(O.seeded_vector(a.n, seed)).cuda()
        nnz = a.nnz()
        B = 12 * nnz + 4 * (a.n + 1) + 16 * a.n
        r = reps if a.n < 10 ** 8 else 30
        for t in (128,):
            plans = {p: K.DevicePlan(a, K.UnsymKernel.u1_row, p | (t << 16 if p < 103 else 0))
                     for p in params}
            res, ys = {p: [] for p in params}, {}
            for _ in range(5):
                for p in params:
                    y = torch.empty_like(x)
                    avg, mn = plans[p].time(x, y, reps=max(r // 5, 2), flush_bytes=2 * l2)
                    res[p].append(avg * 1e3)
                    ys[p] = y
            torch.cuda.synchronize()
            for p in params:
                med = float(np.median(res[p]))
                same = bool(torch.equal(ys[p], ys[params[0]]))
                print(f"{name:14s} t{t:3d} param {p}: " + " ".join(f"{q:9.2f}" for q in res[p]) +
                      f"  median {med:9.2f} us = {B / med / 1e3:7.1f} GB/s (algorithmic)"
                      f"  same {same}", flush=True)
            del plans, ys
            torch.cuda.empty_cache()
        del a


if __name__ == "__main__":
    main()
