"""A/B of S3 variants on config 2 (cold L2 per apply, CUDA events):
env knobs read at plan setup, alternated to share one box's clocks.

    python tools/s3_ab.py KTB_S3_FLAGS=0 KTB_S3_FLAGS=1 [reps]
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
    variants = [a for a in sys.argv[1:] if "=" in a]
    reps = int(next((a for a in sys.argv[1:] if a.isdigit()), "200"))
    a = K.stencil27_upper(128, 128, 128)
    x = torch.from_numpy(O.seeded_vector(a.n, 2)).cuda()
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    plans, ys = {}, {}
    for v in variants:
        k, val = v.split("=")
        os.environ[k] = val
        plans[v] = K.DevicePlan(a, K.SymKernel.s3_nnz_zero_omit)
        os.environ.pop(k)
    res = {v: [] for v in variants}
    for rnd in range(5):
        for v in variants:
            y = torch.empty_like(x)
            avg, mn = plans[v].time(x, y, reps=reps // 5, flush_bytes=2 * l2)
            res[v].append(avg * 1e3)
            ys[v] = y.cpu().numpy()
    base = ys[variants[0]]
    for v in variants:
        print(f"{v:24s} us/apply per round: " + " ".join(f"{t:7.2f}" for t in res[v]) +
              f"  median {np.median(res[v]):7.2f}  bitwise-equal {np.array_equal(ys[v], base)}")


if __name__ == "__main__":
    main()
