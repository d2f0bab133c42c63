"""A/B of U1 warp-sliced variants (env knobs read at plan setup) on configs
1, 5 and a 256^3 stencil, cold L2 per apply, CUDA events, alternated.

    python tools/u1_ab.py KTB_U1S_XPF=0 KTB_U1S_XPF=1 [reps]
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
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    mats = {"cfg1 64^3": K.stencil7(64, 64, 64),
            "cfg5 128^3 cd": K.stencil7(128, 128, 128, c_xm=-1.3, c_xp=-0.7),
            "256^3": K.stencil7(256, 256, 256)}
    for name, a in mats.items():
        x = torch.from_numpy(O.seeded_vector(a.n, 1)).cuda()
        for t in (128, 256):
            plans, ys, res = {}, {}, {v: [] for v in variants}
            for v in variants:
                k, val = v.split("=")
                os.environ[k] = val
                plans[v] = K.DevicePlan(a, K.UnsymKernel.u1_row, 100 | (t << 16))
                os.environ.pop(k)
            for _ in range(5):
                for v in variants:
                    y = torch.empty_like(x)
                    avg, mn = plans[v].time(x, y, reps=reps // 5, flush_bytes=2 * l2)
                    res[v].append(avg * 1e3)
                    ys[v] = y.cpu().numpy()
            for v in variants:
                print(f"{name:14s} t{t:3d} {v:18s} us: " + " ".join(f"{q:8.2f}" for q in res[v]) +
                      f"  median {np.median(res[v]):8.2f} same {np.array_equal(ys[v], ys[variants[0]])}")


if __name__ == "__main__":
    main()
