"""One plan, a few applies (for an ncu capture of one kernel):
    python tools/ncu_one.py <config 1|2|3|4|5> <kernel> <param>"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2405_01599_b200 import ktune as K  # noqa: E402

MK = {1: lambda: K.stencil7(64, 64, 64), 2: lambda: K.stencil27_upper(128, 128, 128),
      3: lambda: K.powerlaw(), 4: lambda: K.stencil7(512, 512, 512),
      5: lambda: K.stencil7(128, 128, 128, c_xm=-1.3, c_xp=-0.7)}
cfg, kern, prm = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
a = MK[cfg]()
p = K.DevicePlan(a, kern, prm)
x = torch.from_numpy(O.seeded_vector(a.n, cfg)).cuda()
y = torch.empty_like(x)
l2 = torch.cuda.get_device_properties(0).L2_cache_size
p.time(x, y, reps=3, flush_bytes=2 * l2)
torch.cuda.synchronize()
print("ok", a.n, a.nnz(), p.kernel, p.param)
