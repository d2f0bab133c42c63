"""Config-4 sharding on one GPU: the device slab generator matches the host
layout bit-exactly, and P slabs with the halo protocol (emulated by
local_exchange in one process: no ranks waiting on each other on one GPU)
reproduce the global SpMV within 1e-12 (|A||x|)_i."""
import numpy as np
import pytest

import matgen
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def test_slab_generator_bit_exact():
    from paper_2405_01599_b200 import dist as D
    from paper_2405_01599_b200 import ktune as K

    for world in (1, 2, 3):
        for r in range(world):
            L = D.slab_layout(10, 7, 9, r, world)
            dev = K.stencil7_slab(10, 7, 9, L.z0, L.z1)
            rp, ci, v = dev.to_host()
            n, rp2, ci2, v2 = D.slab_csr_numpy(L)
            assert np.array_equal(rp, rp2) and np.array_equal(ci, ci2) and np.array_equal(v, v2)


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_sharded_spmv_matches_global(world):
    import torch

    from paper_2405_01599_b200 import dist as D

    nx, ny, nz = 48, 40, 32
    shards = [D.DistSpMV(nx, ny, nz, r, world, 0) for r in range(world)]
    D.local_exchange([s.L for s in shards], [s.x for s in shards])
    y = torch.cat([s.compute_local() for s in shards]).cpu().numpy()
    n, rp, ci, v = matgen.stencil7(nx, ny, nz)
    x = O.seeded_vector(n, 4)
    yref = O.spmv_ref(n, rp, ci, v, x)
    absax = O.spmv_ref(n, rp, ci, np.abs(v), np.abs(x))
    assert (np.abs(y - yref) <= 1e-12 * absax).all()


def test_matrix_slice_rows_bytes():
    """ktb_matrix_slice: rows [r0, r1) with rebased row_ptr and the same
    columns/values, including empty and full ranges and a halo slab."""
    from paper_2405_01599_b200 import dist as D
    from paper_2405_01599_b200 import ktune as K

    n, rp, ci, v = matgen.random_csr(900, 0.01, np.random.default_rng(4), empty_frac=0.2)
    a = K.CsrMatrix(n, rp, ci, v)
    d = K.DeviceCsr.__new__(K.DeviceCsr)
    d._owner, d._dev, d._kind, d.n = a, a.dev, 0, n  # borrowed view of a's device matrix
    for r0, r1 in ((0, n), (0, 0), (17, 17), (5, 400), (899, 900), (123, 777)):
        s = d.slice_rows(r0, r1)
        srp, sci, sv = s.to_host()
        assert s.n == r1 - r0
        assert np.array_equal(srp, rp[r0:r1 + 1] - rp[r0])
        assert np.array_equal(sci, ci[rp[r0]:rp[r1]]) and np.array_equal(sv, v[rp[r0]:rp[r1]])
    L = D.slab_layout(10, 7, 9, 1, 3)
    slab = K.stencil7_slab(10, 7, 9, L.z0, L.z1)
    lo, hi = L.interior_rows()
    s = slab.slice_rows(lo, hi)
    full = slab.to_host()
    part = s.to_host()
    assert np.array_equal(part[1], full[1][full[0][lo]:full[0][hi]])
    with pytest.raises(K.Error, match="bad row range"):
        d.slice_rows(5, 3)
