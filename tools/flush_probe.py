"""Does the L2 flush (a write of 2x L2 before each timed step) leave dirty
lines whose write-back lands inside the timed SpMV? Times the selected
kernel of configs 1/2/3 per step with CUDA events under three regimes:
  write      : flush buffer written (current bench.py behaviour)
  write+read : the same write, then a read pass over a second 2x L2 buffer
               (L2 cold AND clean when the timed kernel starts)
  none       : no flush (warm L2, for reference)
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2405_01599_b200 import _lib  # noqa: E402
from paper_2405_01599_b200 import ktune as K  # noqa: E402


def main():
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    wbuf = torch.empty(2 * l2, dtype=torch.uint8, device="cuda")
    rbuf = torch.ones(2 * l2 // 8, dtype=torch.float64, device="cuda")
    for cfg, mk, sym in ((1, lambda: K.stencil7(64, 64, 64), False),
                         (2, lambda: K.stencil27_upper(128, 128, 128), True),
                         (3, lambda: K.powerlaw(), False)):
        a = mk()
        choice, _ = (K.select_spmv_sym if sym else K.select_spmv_unsym)(a)
        plan = choice.plan
        x = torch.empty(a.n, dtype=torch.float64, device="cuda")
        _lib.load().ktb_seeded_vector(a.n, cfg, 0, x.data_ptr(), None)
        y = torch.empty_like(x)
        for mode in ("write", "write+read", "none"):
            ts = []
            for k in range(30):
                if mode != "none":
                    wbuf.fill_(k & 0xff)
                if mode == "write+read":
                    s = rbuf.sum()  # noqa: F841  (read pass: evicts the dirty lines)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                plan.apply(x, y)
                e1.record()
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
            ts = np.array(ts[5:])
            print(f"cfg{cfg} {K.kernel_name(plan.kernel)} {mode:11s} mean {ts.mean() * 1e3:8.1f} us"
                  f"  min {ts.min() * 1e3:8.1f} us", flush=True)


if __name__ == "__main__":
    main()
