"""Kernel time of the halo operator's interior kernel (U1 106) at the slab a
rank owns when config 4 is split over N = 1, 2, 4, 8 GPUs (512 x 512 x 512/N
planes), on ONE GPU: how the per-rank kernel scales with the shard size.
Not a multi-GPU measurement -- no exchange runs here; the halo message of a
rank is one 512 x 512 plane (2 MB) per neighbour.

    python tools/shard_size_probe.py
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

l2 = torch.cuda.get_device_properties(0).L2_cache_size
base = None
for N in (1, 2, 4, 8):
    a = K.stencil7(512, 512, 512 // N)
    x = torch.from_numpy(O.seeded_vector(a.n, 4)).cuda()
    y = torch.empty_like(x)
    plan = K.DevicePlan(a, K.UnsymKernel.u1_row, 106)
    ts = [plan.time(x, y, reps=20, flush_bytes=2 * l2)[0] * 1e3 for _ in range(5)]
    t = float(np.median(ts))
    base = base or t
    B = 12 * a.nnz() + 4 * (a.n + 1) + 16 * a.n
    print(f"N={N}: slab 512x512x{512 // N} ({a.n:,} rows): {t:8.1f} us per apply, "
          f"{B / t / 1e3:8.0f} GB/s of model bytes per GPU, "
          f"kernel-side speed-up {base / t:5.2f}x of {N}")
    del plan, a, x, y
    torch.cuda.empty_cache()
