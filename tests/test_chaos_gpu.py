"""Race evidence without compute-sanitizer (closed on this GPU pool): the
race-stress build libktb_chaos.so (KTB_CHAOS: a pseudo-random 0-2 us sleep
before every block barrier, mbarrier wait, MGS publish/poll and ILU cluster
barrier, plus device bounds checks that trap) must produce results bitwise
equal to the normal build's on every kernel with hand-written
synchronisation -- S3 (TMA/mbarrier ring, window rounds, fixup, patch pass),
the U2/U3 warp tiles in both CTA shapes, device GMRES's cross-CTA tag
exchange, the ILU(0) cluster sweep and the halo operator -- and reproduce
itself across repeated applies. A missing barrier or fence surfaces as a
differing or non-reproducible array, an out-of-bounds index as a trap."""
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHAOS = os.path.join(ROOT, "paper_2405_01599_b200", "_lib", "libktb_chaos.so")

pytestmark = pytest.mark.gpu


def _run(lib, out, reps):
    env = dict(os.environ, KTB_LIB_NAME=lib)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "chaos_cases.py"), str(out),
                        str(reps)], env=env, capture_output=True, text=True, timeout=1200)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    return np.load(out)


@pytest.mark.skipif(not os.path.exists(CHAOS), reason="libktb_chaos.so not built")
def test_race_stress_build_bitwise_equal(tmp_path):
    ref = _run("libktb.so", tmp_path / "ref.npz", 3)
    got = _run("libktb_chaos.so", tmp_path / "chaos.npz", 6)
    assert str(got["lib"]) == "libktb_chaos.so" and str(ref["lib"]) == "libktb.so"
    keys = sorted(k for k in ref.files if k != "lib")
    assert len(keys) >= 16
    for k in keys:
        assert np.array_equal(ref[k], got[k]), k
