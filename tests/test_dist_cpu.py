"""Multi-rank z-slab sharding (config 4 layout) on CPU with the
gloo backend: halo exchange protocol + local layouts reproduce the global
SpMV bitwise (same per-row summation order) for world sizes 2 and 3."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import matgen
from oracle import oracle as O
from paper_2405_01599_b200 import dist as D

GRID = (6, 5, 9)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nx, ny, nz = GRID
        L = D.slab_layout(nx, ny, nz, rank, world)
        xg = O.seeded_vector(nx * ny * nz, 4)
        xloc = torch.zeros(L.x_local_len, dtype=torch.float64)
        xloc[L.owned_offset:L.owned_offset + L.n_local] = torch.from_numpy(
            xg[L.row0:L.row0 + L.n_local])
        for r in D.halo_exchange(L, xloc):
            r.wait()
        n, rp, ci, v = D.slab_csr_numpy(L)
        y = O.spmv_ref(n, rp, ci, v, xloc.numpy())
        np.save(os.path.join(out_dir, f"y{rank}.npy"), y)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_halo_exchange_reproduces_global_spmv(world, tmp_path):
    port = _free_port()
    mp.spawn(_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    nx, ny, nz = GRID
    n, rp, ci, v = matgen.stencil7(nx, ny, nz)
    yg = O.spmv_ref(n, rp, ci, v, O.seeded_vector(n, 4))
    parts = [np.load(tmp_path / f"y{r}.npy") for r in range(world)]
    assert np.array_equal(np.concatenate(parts), yg)


def test_layout_invariants():
    for world in (1, 2, 4, 8):
        Ls = [D.slab_layout(512, 512, 512, r, world) for r in range(world)]
        assert sum(L.n_local for L in Ls) == 512 ** 3
        assert Ls[0].row0 == 0 and all(Ls[i].z1 == Ls[i + 1].z0 for i in range(world - 1))
        for L in Ls:
            lo, hi = L.interior_rows()
            covered = sum(b - a for a, b in L.boundary_ranges()) + (hi - lo)
            assert covered == L.n_local
            assert L.x_local_len == L.n_local + L.plane * (L.has_lo + L.has_hi)
            # each halo message is one plane = 2 MiB of fp64 at 512^2
            for _, s, r in D.halo_plan(L):
                assert (s.stop - s.start) * 8 == 2 * 1024 * 1024


def test_local_exchange_matches_protocol():
    nx, ny, nz = GRID
    world = 3
    Ls = [D.slab_layout(nx, ny, nz, r, world) for r in range(world)]
    xg = O.seeded_vector(nx * ny * nz, 4)
    xs = []
    for L in Ls:
        x = np.zeros(L.x_local_len)
        x[L.owned_offset:L.owned_offset + L.n_local] = xg[L.row0:L.row0 + L.n_local]
        xs.append(x)
    D.local_exchange(Ls, xs)
    for L, x in zip(Ls, xs):
        assert np.array_equal(x, xg[L.col_base:L.col_base + L.x_local_len])
