"""Config-4 sharding through libktb's native data plane (ktb_comm / ktb_halo,
csrc/ktb_comm.cu) on one GPU:

* the device slab generator matches the host layout bit-exactly;
* W in-process loopback ranks (one host thread each; the native code's
  exchange is matched on the host, never ranks spinning on each other in a
  kernel) run ktb_halo_spmv -- NCCL-group offsets, peers, interior/boundary
  split and the overlap events exactly as on W GPUs -- and the concatenated y
  matches the oracle on every row: |y - y_ref| <= 1e-12 (|A||x|)_i;
* the real NCCL communicator at world 1 (ncclCommInitRank, all-reduce, the
  halo operator with no peers);
* with >= 2 GPUs, the real NCCL exchange across processes (skipped on a
  1-GPU box)."""
import os
import socket

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


def _oracle(nx, ny, nz, seed=4):
    n, rp, ci, v = matgen.stencil7(nx, ny, nz)
    x = O.seeded_vector(n, seed)
    return O.spmv_ref(n, rp, ci, v, x), O.spmv_ref(n, rp, ci, np.abs(v), np.abs(x))


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_native_halo_loopback_matches_oracle(world):
    import torch

    from paper_2405_01599_b200 import dist as D

    nx, ny, nz = 48, 40, 32
    comms = D.Comm.loopback(world)

    def rank(r):
        s = D.DistSpMV(nx, ny, nz, comms[r])
        lo, hi = s.L.interior_rows()
        assert (s.interior_begin, s.interior_end) == (lo, hi)  # native split = layout rule
        s.apply()
        s.apply()  # a second apply reuses the events/streams
        torch.cuda.current_stream().synchronize()
        return s.y.cpu().numpy()

    y = np.concatenate(D.run_ranks(world, rank))
    yref, absax = _oracle(nx, ny, nz)
    assert (np.abs(y - yref) <= 1e-12 * absax).all()


def test_native_halo_kernels_and_exchange_only():
    """Interior/boundary plans on other kernels; the exchange alone fills the
    halo planes with the neighbours' edge planes."""
    import torch

    from paper_2405_01599_b200 import dist as D

    nx, ny, nz, world = 20, 18, 12, 3
    yref, absax = _oracle(nx, ny, nz)
    for kernel, param in ((0, 0), (1, 0), (2, 8)):
        comms = D.Comm.loopback(world)

        def rank(r):
            s = D.DistSpMV(nx, ny, nz, comms[r], kernel=kernel, param=param)
            s.exchange_only()
            torch.cuda.current_stream().synchronize()
            xs = s.x.cpu().numpy()
            s.apply()
            torch.cuda.current_stream().synchronize()
            return xs, s.L, s.y.cpu().numpy()

        outs = D.run_ranks(world, rank)
        y = np.concatenate([o[2] for o in outs])
        assert (np.abs(y - yref) <= 1e-12 * absax).all(), (kernel, param)
        xg = O.seeded_vector(nx * ny * nz, 4)
        for xs, L, _ in outs:
            lo = L.row0 - L.owned_offset
            assert np.array_equal(xs, xg[lo:lo + L.x_local_len])


def test_native_general_halo_matrix():
    """ktb_halo_create_csr on a banded row block in global numbering (halo
    widths differ per rank and side; some rows touch no halo): loopback
    ranks vs the oracle on every row."""
    import ctypes as C

    import torch

    from paper_2405_01599_b200 import _lib
    from paper_2405_01599_b200 import dist as D
    from paper_2405_01599_b200 import ktune as K

    rng = np.random.default_rng(11)
    n, band = 3000, 37
    rows = [np.unique(np.clip(i + rng.integers(-band, band + 1, size=6), 0, n - 1))
            for i in range(n)]
    rp = np.zeros(n + 1, np.int64)
    rp[1:] = np.cumsum([len(c) for c in rows])
    ci = np.concatenate(rows).astype(np.int64)
    v = rng.uniform(-1, 1, len(ci))
    x = O.seeded_vector(n, 9)
    yref = O.spmv_ref(n, rp, ci, v, x)
    absax = O.spmv_ref(n, rp, ci, np.abs(v), np.abs(x))
    world, bnd = 4, [0, 500, 1400, 2100, n]
    comms = D.Comm.loopback(world)
    L = _lib.load()

    def rank(r):
        r0, r1 = bnd[r], bnd[r + 1]
        lrp = np.ascontiguousarray(rp[r0:r1 + 1] - rp[r0])
        lci = np.ascontiguousarray(ci[rp[r0]:rp[r1]])
        lv = np.ascontiguousarray(v[rp[r0]:rp[r1]])
        hh = C.c_void_p()
        K._check(L.ktb_halo_create_csr(n, r0, r1 - r0, lrp.ctypes.data, lci.ctypes.data,
                                       lv.ctypes.data, comms[r].h, 0, 100, C.byref(hh)))
        try:
            info = [C.c_int64() for _ in range(6)] + [C.c_int()]
            K._check(L.ktb_halo_info(hh, *[C.byref(q) for q in info]))
            n_loc, x_len, off = info[0].value, info[1].value, info[2].value
            lo = r0 - off
            xl = torch.zeros(x_len, dtype=torch.float64, device="cuda")
            xl[off:off + n_loc] = torch.from_numpy(x[r0:r1].copy()).cuda()
            y = torch.empty(n_loc, dtype=torch.float64, device="cuda")
            K._check(L.ktb_halo_spmv(hh, xl.data_ptr(), y.data_ptr(),
                                     torch.cuda.current_stream().cuda_stream))
            torch.cuda.current_stream().synchronize()
            assert np.array_equal(xl.cpu().numpy(), x[lo:lo + x_len])  # halos landed
            return y.cpu().numpy()
        finally:
            L.ktb_halo_destroy(hh)

    y = np.concatenate(D.run_ranks(world, rank))
    assert (np.abs(y - yref) <= 1e-12 * absax).all()


def test_nccl_world1_comm_and_halo():
    """The real NCCL communicator (ncclCommInitRank at world 1): all-reduce,
    all-gather and the halo operator over it, checked against the oracle."""
    import torch

    from paper_2405_01599_b200 import dist as D

    c = D.Comm.nccl(device=0)
    assert c.is_nccl and c.world == 1 and c.rank == 0 and c.nccl_version >= 21800
    t = torch.arange(5, dtype=torch.float64, device="cuda")
    c.allreduce(t)
    g = torch.empty(5, dtype=torch.float64, device="cuda")
    c.allgather(t, g)
    torch.cuda.synchronize()
    assert torch.equal(t.cpu(), torch.arange(5, dtype=torch.float64))
    assert torch.equal(g.cpu(), t.cpu())
    s = D.DistSpMV(24, 20, 16, c)
    s.apply()
    torch.cuda.synchronize()
    yref, absax = _oracle(24, 20, 16)
    assert (np.abs(s.y.cpu().numpy() - yref) <= 1e-12 * absax).all()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _nccl_worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist

    from paper_2405_01599_b200 import dist as D

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c = D.Comm.nccl(device=rank)
        s = D.DistSpMV(40, 36, 32, c)
        s.apply()
        torch.cuda.synchronize()
        np.save(os.path.join(out_dir, f"y{rank}.npy"), s.y.cpu().numpy())
    finally:
        dist.destroy_process_group()


def test_nccl_multi_gpu_halo(tmp_path):
    """Real NCCL P2P halo exchange across processes, one GPU each."""
    import torch
    import torch.multiprocessing as mp

    world = min(torch.cuda.device_count(), 4)
    if world < 2:
        pytest.skip("needs >= 2 GPUs (the gpurun box has one)")
    mp.spawn(_nccl_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    y = np.concatenate([np.load(tmp_path / f"y{r}.npy") for r in range(world)])
    yref, absax = _oracle(40, 36, 32)
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


@pytest.mark.parametrize("world,chunks", [(1, 1), (1, 7), (1, 16), (3, 5)])
def test_native_halo_host_path_chunked(world, chunks):
    """ktb_halo_spmv_host (host x in, host y out, copies overlapped inside
    the call in row chunks) equals the device-pointer apply bitwise."""
    import torch

    from paper_2405_01599_b200 import dist as D

    nx, ny, nz = 40, 36, 30
    comms = D.Comm.loopback(world)

    def rank(r):
        s = D.DistSpMV(nx, ny, nz, comms[r])
        xo = s.x[s.owned_offset:s.owned_offset + s.n_local].cpu().pin_memory().numpy()
        yh = torch.empty(s.n_local, dtype=torch.float64).pin_memory().numpy()
        yh[:] = np.nan
        s.apply_host(xo, yh, chunks=chunks)
        s.apply()
        torch.cuda.current_stream().synchronize()
        return yh.copy(), s.y.cpu().numpy()

    outs = D.run_ranks(world, rank)
    for yh, yd in outs:
        assert np.array_equal(yh, yd)
    yref, absax = _oracle(nx, ny, nz)
    y = np.concatenate([o[0] for o in outs])
    assert (np.abs(y - yref) <= 1e-12 * absax).all()
