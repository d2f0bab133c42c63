"""Randomised bitwise parity of the pair-coded record kernels (U1 106, S1 106)
against the oracle: tools/fuzz_u1v.py on a fixed seed (random banded
matrices, 1-32 deltas, per-block value palettes, dropped entries, empty rows,
n from 1 to 70,001; whole applies and random row sub-ranges; refused layouts
must fail with the documented message)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def test_pair_coded_records_fuzz_bitwise():
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "fuzz_u1v.py"), "160", "11"],
                       capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-3000:]
    assert "all built plans bitwise equal to the oracle" in p.stdout


def test_every_plan_variant_fuzz():
    """tools/fuzz_all.py on a fixed seed: every device plan variant (U1 lanes
    and 100-106, U2 / U3 / U4 in both CTA shapes, S1 / S2 / S3, S1 106) on
    random matrices of six families against the oracle."""
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "fuzz_all.py"), "24", "5"],
                       capture_output=True, text=True, timeout=1200)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-3000:]
    assert "all reproducible" in p.stdout


def test_multi_gpu_data_plane_fuzz():
    """tools/fuzz_dist.py on a fixed seed: the halo operator on random grids
    (worlds 1-8 incl. one-plane slabs, every U1 form, the host-chunked call)
    and the general split on random matrices (ranks without rows or ghosts),
    loopback ranks running the native exchange code, against the oracle."""
    env = dict(os.environ, FUZZ_WATCHDOG="600")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "fuzz_dist.py"), "30", "4"],
                       capture_output=True, text=True, timeout=900, env=env)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-3000:]
    assert "of the oracle" in p.stdout


def test_gmres_and_ilu0_fuzz():
    """tools/fuzz_krylov.py on a fixed seed: device GMRES(m) against the
    oracle's restatement (+-2 iterations on solves of up to 200 iterations,
    true residual < 1e-8 when converged) and ILU(0) factors and solves bitwise,
    on random dominant matrices (n from 1 to 60,001, restart lengths 1-40)."""
    env = dict(os.environ, FUZZ_WATCHDOG="600")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "fuzz_krylov.py"), "30", "6"],
                       capture_output=True, text=True, timeout=900, env=env)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-3000:]
    assert "bitwise equal" in p.stdout


def test_integer_artefacts_and_selector_fuzz():
    """tools/fuzz_artefacts.py on a fixed seed: row partitions (both schemes, P
    up to 5,000 incl. P > n), BSS plans (jl up to 4,096 incl. jl > nnz),
    reduction regions and expand_symmetric bit-exact against the oracle on
    random matrices; the selector's report never holds a built candidate that
    failed its check."""
    env = dict(os.environ, FUZZ_WATCHDOG="600")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "fuzz_artefacts.py"), "18", "7"],
                       capture_output=True, text=True, timeout=900, env=env)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-3000:]
    assert "bit-exact" in p.stdout


def test_concurrent_plan_setup_and_applies():
    """tools/fuzz_threads.py: six host threads build plans of random variants
    at the same time (on their own matrices and on one shared symmetric
    matrix) and apply them on their own streams; every result equals the
    oracle."""
    env = dict(os.environ, FUZZ_WATCHDOG="600")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "fuzz_threads.py"), "6", "3", "5"],
                       capture_output=True, text=True, timeout=900, env=env)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-3000:]
    assert "all equal to the oracle" in p.stdout


def test_lanczos_fuzz():
    """tools/fuzz_lanczos.py on a fixed seed: restarted Lanczos on an S3 plan
    against numpy's dense eigendecomposition (random stencils and random
    sparse symmetric matrices, the k largest-magnitude eigenvalues to 1e-8)."""
    env = dict(os.environ, FUZZ_WATCHDOG="600")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "fuzz_lanczos.py"), "10", "3"],
                       capture_output=True, text=True, timeout=900, env=env)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-3000:]
    assert "eigenproblems" in p.stdout
