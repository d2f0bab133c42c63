"""The pipelined host call (ktb_spmv_host_pipelined) on config 1, 40 consecutive
50-step calls per plan: the first call of a process pays the one-time costs
(stream / buffer creation, module load and the host link coming up: ~0.3 s),
every later call runs at the steady 66 us per step whatever the kernel -- which
is why bench.py warms the host path for 0.5 s before timing e2e.

    python tools/host_link_probe.py
"""
import sys, time
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np, torch
from oracle import oracle as O
from paper_2405_01599_b200 import ktune as K
a = K.stencil7(64, 64, 64)
n = a.n
xh = torch.empty(n, dtype=torch.float64, pin_memory=True); xh.copy_(torch.from_numpy(O.seeded_vector(n, 1)))
yh = torch.empty(n, dtype=torch.float64, pin_memory=True)
xn, yn = xh.numpy(), yh.numpy()
for prm in (100, 106, 100, 106):
    plan = K.DevicePlan(a, K.UnsymKernel.u1_row, prm)
    torch.cuda.synchronize(); time.sleep(1.0)
    out = []
    T0 = time.perf_counter()
    for r in range(40):
        t0 = time.perf_counter(); plan.apply_host_pipelined(xn, yn, count=50); out.append(round((time.perf_counter() - t0) / 50 * 1e6))
    print("param", prm, "us/step of 40 consecutive 50-step calls:", out, "elapsed ms", round((time.perf_counter() - T0) * 1e3))
