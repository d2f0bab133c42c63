"""Randomised check of the native multi-GPU data plane with loopback ranks on
one GPU (csrc/ktb_comm.cu: the exact exchange code of W ranks, one host thread
each): random matrices of the fuzz_all families split into W = 1..8
NNZ_BALANCED row blocks (ranks may own no rows, no ghosts, or need all of x),
A_d on a random kernel, the concatenated y against the oracle.

    python tools/fuzz_dist.py [cases] [seed]
"""
import faulthandler
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "tools"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from fuzz_all import gen_unsym  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2405_01599_b200 import dist as D  # noqa: E402


def run(n, rp, ci, v, world, kernel, x):
    b = D.nnz_balanced_boundaries(rp, world)
    comms = D.Comm.loopback(world)

    def rank(r):
        r0, r1 = int(b[r]), int(b[r + 1])
        sp = D.DistCsrSpMV(n, b, comms[r], rp[r0:r1 + 1] - rp[r0], ci[rp[r0]:rp[r1]],
                           v[rp[r0]:rp[r1]], kernel=kernel)
        xo = torch.from_numpy(x[r0:r1].copy()).cuda()
        y = torch.full((max(sp.n_local, 1),), float("nan"), dtype=torch.float64, device="cuda")
        for _ in range(2):
            sp.apply(xo, y[:sp.n_local])
        torch.cuda.current_stream().synchronize()
        return y[:sp.n_local].cpu().numpy(), sp.dc.n_ghost

    outs = D.run_ranks(world, rank)
    return np.concatenate([o[0] for o in outs]), [o[1] for o in outs], b


def run_halo(nx, ny, nz, world, param, seed, chunks):
    """The z-slab halo operator (config 4's path) on an nx x ny x nz grid."""
    comms = D.Comm.loopback(world)

    def rank(r):
        s = D.DistSpMV(nx, ny, nz, comms[r], seed=seed, param=param)
        s.apply()
        s.apply()
        torch.cuda.current_stream().synchronize()
        y = s.y.cpu().numpy()
        if chunks:  # the host-chunked call must give the same rows
            xo = s.x[s.owned_offset:s.owned_offset + s.n_local].cpu().numpy()
            yh = np.full(s.n_local, np.nan)
            s.apply_host(xo, yh, chunks=chunks)
            assert np.array_equal(yh, y), ("host-chunked", r, chunks)
        return y

    return np.concatenate(D.run_ranks(world, rank))


def main():
    faulthandler.enable()
    if os.environ.get("FUZZ_WATCHDOG"):  # dump every thread's stack and exit on a hang
        faulthandler.dump_traceback_later(int(os.environ["FUZZ_WATCHDOG"]), exit=True)
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    rng = np.random.default_rng(seed)
    done = 0
    import matgen
    halo = 0
    for c in range(max(cases // 3, 1)):
        nx, ny = int(rng.integers(1, 40)), int(rng.integers(1, 40))
        world = int(rng.choice([1, 2, 3, 4, 8]))
        nz = int(rng.integers(world, 3 * world + 12))  # every rank owns >= 1 plane
        param = int(rng.choice([106, 105, 104, 100, 0]))
        sd = 4 + c
        chunks = int(rng.choice([0, 1, 3, 16]))
        if os.environ.get("FUZZ_VERBOSE"):
            print("halo case", c, nx, ny, nz, world, param, chunks, flush=True)
        y = run_halo(nx, ny, nz, world, param, sd, chunks)
        n, rp, ci, v = matgen.stencil7(nx, ny, nz)
        x = O.seeded_vector(n, sd)
        yref = O.spmv_ref(n, rp, ci, v, x)
        if param >= 100:
            assert np.array_equal(y, yref), ("halo", c, nx, ny, nz, world, param)
        else:
            assert (np.abs(y - yref) <= 1e-12 * O.spmv_ref(n, rp, ci, np.abs(v), np.abs(x))).all(), \
                ("halo", c, nx, ny, nz, world, param)
        halo += 1
    for c in range(cases):
        n, rp, ci, v = gen_unsym(rng, c)
        if n > 100000:
            continue
        world = int(rng.choice([1, 2, 3, 4, 7, 8]))
        kernel = [0, 1, 2, None][int(rng.integers(0, 4))]
        if rp[-1] == 0:
            kernel = 0
        x = O.seeded_vector(n, 50 + c)
        y, ghosts, b = run(n, rp, ci, v, world, kernel, x)
        yref = O.spmv_ref(n, rp, ci, v, x)
        bound = 1e-12 * O.spmv_ref(n, rp, ci, np.abs(v), np.abs(x))
        bad = np.flatnonzero(~(np.abs(y - yref) <= bound))
        assert bad.size == 0, (c, n, world, kernel, bad[:5], list(b))
        done += 1
    print(f"fuzz_dist: seed {seed}: {halo} halo-operator grids (worlds 1-8, U1 106/105/104/100/lanes, bitwise for "
          f"100-106, host-chunked call equal) and {done} general splits (worlds 1-8), every y within "
          "1e-12 (|A||x|)_i of the oracle")


if __name__ == "__main__":
    main()
