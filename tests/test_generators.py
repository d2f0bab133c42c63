"""Config-3 generator: the native libktb host generator and the numpy
restatement in tests/matgen.py produce identical bytes (no GPU needed)."""
import numpy as np

import matgen
from oracle import oracle as O
from paper_2405_01599_b200 import ktune as K


def test_powerlaw_native_equals_numpy_small():
    for (n, tgt, seed) in ((20000, 200000, 3), (5000, 60000, 11), (1, 1, 3)):
        a = K.powerlaw_host(n, seed, tgt, 0.1, 65536)
        b = matgen.powerlaw(n, seed, tgt, 0.1, 65536)
        for u, v in zip(a[1:], b[1:]):
            assert np.array_equal(u, v)
        n, rp, ci, v = a
        assert O.validate(n, rp, ci) is None


def test_powerlaw_shape_properties():
    n, rp, ci, v = K.powerlaw_host(200000, 3, 2000000, 0.1, 65536)
    lens = np.diff(rp)
    assert abs((lens == 0).mean() - 0.1) < 0.01          # ~10% empty rows
    assert abs(rp[-1] - 2_000_000) < 0.05 * 2_000_000     # ~target nnz
    assert v.min() >= -1.0 and v.max() < 1.0
    assert lens.max() <= 65536 and lens[lens > 0].min() >= 1
