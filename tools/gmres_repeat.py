"""Config 5 (GMRES(30), 128^3 convection-diffusion) solved 8 times on the selected
SpMV plan: iterations, wall seconds and SpMV seconds per solve (host b in, host x
out; the workspace is cached on the plan after the first solve).

    python tools/gmres_repeat.py
"""
import time, sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2405_01599_b200 import ktune as K
a = K.stencil7(128, 128, 128, c_xm=-1.3, c_xp=-0.7, device=0)
choice, rep = K.select_spmv_unsym(a)
plan = choice.plan
ones = torch.ones(a.n, dtype=torch.float64, device="cuda"); bd = torch.empty_like(ones)
plan.apply(ones, bd); torch.cuda.synchronize(); b = bd.cpu().numpy()
kcfg = K.KrylovConfig(30, 30, 1e-8, 3000)
for i in range(8):
    t0 = time.perf_counter(); r = K.gmres_m(a, b, kcfg, plan=plan); t = time.perf_counter() - t0
    print(i, r.iterations, round(t, 4), round(r.spmv_seconds, 4), flush=True)
