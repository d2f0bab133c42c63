import sys, numpy as np, faulthandler
faulthandler.enable()
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from paper_2405_01599_b200 import ktune as K
a = K.powerlaw()
print("matrix ok", a.n, a.nnz(), flush=True)
rp, ci, v = a.to_host()
L = np.diff(rp); print("long rows", (L > 256).sum(), "max", L.max(), flush=True)
plan = K.DevicePlan(a, K.UnsymKernel.u1_row, 101)
print(" plan ok", plan.launches, flush=True)
import torch
from oracle import oracle as O
x = O.seeded_vector(a.n, 3)
xd = torch.from_numpy(x).cuda()
y = torch.full((a.n,), float("nan"), dtype=torch.float64, device="cuda")
try:
    plan.apply(xd, y); torch.cuda.synchronize()
    print("apply ok", flush=True)
except Exception as e:
    print("apply failed", e, flush=True)
