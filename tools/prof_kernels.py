"""Run chosen SpMV kernels on a config a few times (for ncu / timing sweeps).

    python tools/prof_kernels.py --config 2 --kernels s1,s2,s3 --reps 3
Prints per-kernel CUDA-event timings (cold L2: flush before each apply).
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2405_01599_b200 import _lib  # noqa: E402
from paper_2405_01599_b200 import ktune as K  # noqa: E402

TAGS = {"u1": 0, "u2": 1, "u3": 2, "u4": 3, "s1": 16, "s2": 17, "s3": 18}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--kernels", default="s1,s2,s3")
    ap.add_argument("--params", default="")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--time-reps", type=int, default=20)
    args = ap.parse_args()
    if args.config == 2:
        a = K.stencil27_upper(128, 128, 128)
    elif args.config == 1:
        a = K.stencil7(64, 64, 64)
    elif args.config == 3:
        a = K.powerlaw()
    elif args.config == 4:
        a = K.stencil7(512, 512, 512)
    elif args.config == 5:
        a = K.stencil7(128, 128, 128, c_xm=-1.3, c_xp=-0.7)
    n, nnz = a.n, a.nnz()
    B = 12 * nnz + 4 * (n + 1) + 16 * n
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    _lib.load().ktb_seeded_vector(n, args.config, 0, x.data_ptr(), None)
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    params = [int(p) for p in args.params.split(",")] if args.params else [0]
    for kn in args.kernels.split(","):
        for prm in params:
            plan = K.DevicePlan(a, TAGS[kn], prm)
            for _ in range(args.reps):
                plan.apply(x, y)
            torch.cuda.synchronize()
            avg, mn = plan.time(x, y, reps=args.time_reps, flush_bytes=2 * l2)
            print(f"{kn} param={plan.param} ctas={plan.ctas} launches={plan.launches} "
                  f"extra_bytes={plan.extra_bytes} avg_ms={avg:.4f} min_ms={mn:.4f} "
                  f"GB/s(avg)={B / avg / 1e6:.1f}", flush=True)
            plan.close()


if __name__ == "__main__":
    main()
