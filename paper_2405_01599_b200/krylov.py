"""Restarted GMRES(m) over row-sharded vectors: the
reference's gmres_m (gmres.hpp:16-173) and orthogonalize (ortho.hpp:69-111)
with every global reduction a sum of local partials across the process group
(NCCL all-reduce on GPUs).

The loop is the reference's, statement for statement: the Givens rotations,
back-substitution and stopping rule run on host scalars; vectors stay on the
device and go through libktb's deterministic BLAS-1 kernels (ktb_vec_*).
Each orthogonaliser keeps its reduction structure, so its all-reduce count
per Arnoldi step is explicit:

    mgs   k+2  (one per projection, the input norm, the output norm)
    cgs   3    (all projections at once, two norms)
    dgks  4    (two classical passes)
    bcgs  ceil(k / block_len) + 2

`op` is any row-sharded operator with ``n_local`` and ``apply(x, y)``
(dist.DistCsrSpMV, or a single-rank DevicePlan wrapper); ``ops`` the local
vector kernels (DeviceVecOps here; tests drive the same loop on CPU ranks
with a stand-in); ``allreduce`` sums a tensor in place over the ranks.
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

ORTHO = ("cgs", "mgs", "dgks", "bcgs")  # ortho.hpp:12 OrthoKind


@dataclass
class DistSolverResult:  # the SolverResult fields gmres_m fills (solver_types.hpp:56-77)
    x: object = None
    iterations: int = 0
    converged: bool = False
    breakdown: bool = False
    breakdown_reason: str = ""
    recurrence_residual: float = 0.0
    true_residual: float = 0.0
    fault_convergence: bool = False
    residual_history: list = field(default_factory=list)
    restarts: list = field(default_factory=list)
    allreduces: int = 0
    elapsed_seconds: float = 0.0


class DeviceVecOps:
    """Local BLAS-1 on torch CUDA tensors through libktb (ktb_vec_*)."""

    def __init__(self, max_cols: int, device: int):
        import torch

        from . import _lib

        self._L = _lib.load()
        self.device = device
        self.launches = 0  # kernels launched (mdot = 2, the others 1)
        self.scratch = torch.empty(max(int(self._L.ktb_vec_mdot_scratch(max_cols)), 1),
                                   dtype=torch.float64, device=f"cuda:{device}")

    def _s(self):
        import torch

        return torch.cuda.current_stream(self.device).cuda_stream

    def _chk(self, rc):
        if rc != 0:
            from .ktune import _check

            _check(rc)

    def empty(self, *shape):
        import torch

        return torch.empty(*shape, dtype=torch.float64, device=f"cuda:{self.device}")

    def zeros(self, *shape):
        import torch

        return torch.zeros(*shape, dtype=torch.float64, device=f"cuda:{self.device}")

    def mdot(self, V, k, w, out):
        """out[:k] = V[:k] . w (local partials); V is (cols, n) row-major."""
        n = w.shape[0]
        self._chk(self._L.ktb_vec_mdot(n, k, V.data_ptr(), V.stride(0), w.data_ptr(),
                                       out.data_ptr(), self.scratch.data_ptr(), self._s()))
        self.launches += 2 if k else 0

    def maxpy(self, V, k, coef, alpha, w):
        """w += alpha * coef[j] * V[j], j = 0..k-1 in order."""
        n = w.shape[0]
        self._chk(self._L.ktb_vec_maxpy(n, k, V.data_ptr(), V.stride(0), coef.data_ptr(),
                                        float(alpha), w.data_ptr(), self._s()))
        self.launches += 1 if k and n else 0

    def axpby(self, a, x, b, y):
        self._chk(self._L.ktb_vec_axpby(y.shape[0], float(a), x.data_ptr(), float(b),
                                        y.data_ptr(), self._s()))
        self.launches += 1 if y.shape[0] else 0

    def scale(self, s, x, divide=False):
        self._chk(self._L.ktb_vec_scale(x.shape[0], float(s), int(divide), x.data_ptr(),
                                        self._s()))
        self.launches += 1 if x.shape[0] else 0

    def to_host(self, t):
        return t.detach().cpu().tolist()

    def from_host(self, vals, out):
        import torch

        out.copy_(torch.tensor(vals, dtype=torch.float64))

    def copy(self, src, dst):
        self.axpby(1.0, src, 0.0, dst)

    def seeded(self, seed, offset, out):
        """out[i] = detail::seeded_vector(N, seed)[offset + i] (lanczos.hpp:17-29)."""
        self._chk(self._L.ktb_seeded_vector(out.shape[0], int(seed) & (2 ** 64 - 1), int(offset),
                                            out.data_ptr(), self._s()))
        self.launches += 1 if out.shape[0] else 0


def process_group_allreduce(group=None):
    """Sum a tensor in place over the default (or given) process group; a
    no-op for a single rank."""
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return lambda t: None
    return lambda t: dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)


def comm_allreduce(comm):
    """Sum a float64 CUDA tensor in place over a native communicator
    (dist.Comm: NCCL, or the in-process loopback world)."""
    if comm.world == 1:
        return lambda t: None
    return lambda t: comm.allreduce(t)


class _Counter:
    def __init__(self, allreduce):
        self.f, self.n = allreduce, 0

    def __call__(self, t):
        self.n += 1
        self.f(t)


def _norm(ops, ar, v, buf):
    ops.mdot(v.unsqueeze(0), 1, v, buf)
    ar(buf[:1])
    return math.sqrt(ops.to_host(buf[:1])[0])


def orthogonalize(kind, V, k, w, ops, ar, bufs, block_len=4):
    """ortho.hpp:69-111 on sharded vectors: returns (h[0..k], breakdown);
    w becomes the new unit vector unless breakdown."""
    if kind not in ORTHO:
        raise ValueError(f"orthogonalize: unknown kind {kind!r}")
    if block_len < 1:
        raise ValueError("orthogonalize: block length must be >= 1")
    coef, nbuf = bufs
    input_norm = _norm(ops, ar, w, nbuf)
    h = [0.0] * (k + 1)

    def classical(first, count):  # detail::classical_pass (ortho.hpp:55-64)
        if count == 0:
            return
        ops.mdot(V[first:first + count], count, w, coef)
        ar(coef[:count])
        ops.maxpy(V[first:first + count], count, coef, -1.0, w)
        c = ops.to_host(coef[:count])
        for j in range(count):
            h[first + j] += c[j]

    if kind == "cgs":
        classical(0, k)
    elif kind == "dgks":
        classical(0, k)
        classical(0, k)
    elif kind == "mgs":
        for j in range(k):  # one projection at a time, coefficient stays on the device
            ops.mdot(V[j:j + 1], 1, w, coef[j:j + 1])
            ar(coef[j:j + 1])
            ops.maxpy(V[j:j + 1], 1, coef[j:j + 1], -1.0, w)
        c = ops.to_host(coef[:k])
        for j in range(k):
            h[j] += c[j]
    else:  # bcgs
        for b in range(0, k, block_len):
            classical(b, min(block_len, k - b))
    norm = _norm(ops, ar, w, nbuf)
    h[k] = norm
    if norm <= 1e-14 * input_norm:
        return h, True
    ops.scale(1.0 / norm, w)
    return h, False


def gmres_m_dist(op, b, m=30, tol=1e-8, max_iters=3000, ortho="mgs", block_len=4, ops=None,
                 allreduce=None, max_time=math.inf, precond=None) -> DistSolverResult:
    """gmres.hpp:16-173 (fixed restart m) with sharded vectors. b: this rank's
    slice (device tensor for DeviceVecOps). precond(r, z): the right
    preconditioner on this rank's slice (e.g. ILU(0) factors of the rank's
    diagonal block -- block Jacobi across ranks; the exact reference
    pairing on one rank)."""
    if m < 1:
        raise ValueError("gmres: need 1 <= m <= m_max")
    if tol <= 0.0:
        raise ValueError("gmres: tol must be positive")
    if b.shape[0] != op.n_local:
        raise ValueError("gmres: dimension mismatch")
    ar = _Counter(allreduce or process_group_allreduce())
    ops = ops or DeviceVecOps(m + 1, b.device.index)
    n = op.n_local
    t0 = time.perf_counter()
    res = DistSolverResult()
    coef = ops.zeros(m + 1)
    nbuf = ops.zeros(1)
    x = ops.zeros(n)
    res.x = x
    nb = _norm(ops, ar, b, nbuf)
    if nb == 0.0:
        res.converged = True
        res.allreduces = ar.n
        res.elapsed_seconds = time.perf_counter() - t0
        return res
    V = ops.zeros(m + 1, n)
    r, w = ops.zeros(n), ops.zeros(n)
    zp = ops.zeros(n) if precond is not None else None
    cs, sn = [0.0] * (m + 1), [0.0] * (m + 1)
    r_cols = [[0.0] * (m + 1) for _ in range(m)]
    rr = 1.0
    stop = False
    while not stop:
        op.apply(x, r)
        ops.axpby(1.0, b, -1.0, r)  # r = b - A x
        beta = _norm(ops, ar, r, nbuf)
        rr = beta / nb
        if rr < tol:
            res.converged = True
            break
        ops.axpby(1.0, r, 0.0, V[0])
        ops.scale(beta, V[0], divide=True)  # basis[i] = r[i] / beta
        g = [0.0] * (m + 2)
        g[0] = beta
        j = 0
        lucky = False
        while j < m:
            if res.iterations >= max_iters or time.perf_counter() - t0 > max_time:
                stop = True
                break
            if precond is not None:  # gmres.hpp:91-92
                precond(V[j], zp)
                op.apply(zp, w)
            else:
                op.apply(V[j], w)
            h, breakdown = orthogonalize(ortho, V, j + 1, w, ops, ar, (coef, nbuf), block_len)
            if breakdown:
                h[j + 1] = 0.0
                lucky = True
            else:
                ops.axpby(1.0, w, 0.0, V[j + 1])
            for i in range(j):
                t1, t2 = h[i], h[i + 1]
                h[i] = cs[i] * t1 + sn[i] * t2
                h[i + 1] = -sn[i] * t1 + cs[i] * t2
            denom = math.hypot(h[j], h[j + 1])
            if denom == 0.0:
                cs[j], sn[j] = 1.0, 0.0
            else:
                cs[j], sn[j] = h[j] / denom, h[j + 1] / denom
            h[j] = denom
            g[j + 1] = -sn[j] * g[j]
            g[j] *= cs[j]
            r_cols[j][: j + 1] = h[: j + 1]
            res.iterations += 1
            rr = abs(g[j + 1]) / nb
            res.residual_history.append(rr)
            j += 1
            if lucky or rr < tol:
                break
        if j > 0:  # back-substitute R y = g, x += Q y
            y = [0.0] * j
            for i in range(j - 1, -1, -1):
                s = g[i]
                for l in range(i + 1, j):
                    s -= r_cols[l][i] * y[l]
                rii = r_cols[i][i]
                y[i] = s / rii if rii != 0.0 else 0.0
            ops.from_host(y, coef[:j])
            ops.scale(0.0, w)
            ops.maxpy(V[:j], j, coef, 1.0, w)
            if precond is not None:
                precond(w, zp)
                ops.axpby(1.0, zp, 1.0, x)
            else:
                ops.axpby(1.0, w, 1.0, x)
        if rr < tol:
            res.converged = True
            break
        if lucky:
            res.breakdown = True
            res.breakdown_reason = "arnoldi breakdown before reaching tol"
            break
        if stop:
            break
        res.restarts.append((res.iterations, m))
    res.recurrence_residual = rr
    op.apply(x, r)
    ops.axpby(1.0, b, -1.0, r)
    res.true_residual = _norm(ops, ar, r, nbuf) / nb
    res.fault_convergence = res.converged and res.true_residual > tol
    res.allreduces = ar.n
    res.elapsed_seconds = time.perf_counter() - t0
    return res


@dataclass
class DistEigenResult:  # EigenResult (solver_types.hpp:79-100), real eigenpairs
    eigenvalues: list = field(default_factory=list)
    eigenvectors: list = field(default_factory=list)  # this rank's slices
    residuals: list = field(default_factory=list)
    max_residual: float = 0.0
    converged: bool = False
    breakdown: bool = False
    breakdown_reason: str = ""
    fault_convergence: bool = False
    iterations: int = 0
    restarts: list = field(default_factory=list)
    residual_history: list = field(default_factory=list)
    allreduces: int = 0
    elapsed_seconds: float = 0.0


def tridiag_eig(alpha, beta):
    """dense_eig.hpp:22-35 (LAPACKE_dsteqr, compz 'I'): eigenvalues ascending,
    eigenvector i = column i. dstev computes the vectors with the same dsteqr
    QL iteration. Host scalars (m <= m_max)."""
    import numpy as np
    from scipy.linalg import eigh_tridiagonal

    d = np.asarray(alpha, np.float64)
    if len(d) == 1:
        return np.array([d[0]]), np.ones((1, 1))
    return eigh_tridiagonal(d, np.asarray(beta, np.float64), lapack_driver="stev")


def lanczos_restarted_dist(op, k, m=30, m_max=None, tol=1e-8, max_iters=10000, ortho="mgs",
                           block_len=4, seed=20080517, row0=0, n_global=None, ops=None,
                           allreduce=None, max_time=math.inf) -> DistEigenResult:
    """lanczos.hpp:54-192: explicitly restarted Lanczos for the k largest-
    magnitude eigenpairs of a symmetric operator, every new basis vector fully
    re-orthogonalised (the configured variant; DGKS for seating and locking),
    on row-sharded vectors. `op` is the symmetric operator on this rank's
    rows (e.g. the S3 plan: SymEngine::op, meta.hpp:53-68); row0/n_global
    place this rank's slice of the seeded start vector."""
    n = op.n_local
    N = n if n_global is None else n_global
    m_max = m if m_max is None else m_max
    if k < 1:
        raise ValueError("lanczos: k must be >= 1")
    if k > N:
        raise ValueError("lanczos: k exceeds the matrix dimension")
    if m < k + 2:
        raise ValueError("lanczos: restart_m must be >= k+2")
    if m > m_max:
        raise ValueError("lanczos: restart_m exceeds m_max")
    ar = _Counter(allreduce or process_group_allreduce())
    ops = ops or DeviceVecOps(k + m_max + 2, op.device if hasattr(op, "device") else 0)
    t0 = time.perf_counter()
    res = DistEigenResult()
    cols = k + m_max + 2
    vecs = ops.zeros(cols, n)
    coef = ops.zeros(cols)
    nbuf = ops.zeros(1)
    bufs = (coef, nbuf)
    w = ops.zeros(n)
    start = ops.zeros(n)
    ops.seeded(seed, row0, start)
    reseed = seed
    nlocked = 0
    locked_vals = []
    msize = m
    out_of_budget = False
    while nlocked < k and not out_of_budget:
        seated = False
        for _ in range(16):  # seat the start vector orthogonal to the locked set
            ops.copy(start, w)
            _, brk = orthogonalize("dgks", vecs, nlocked, w, ops, ar, bufs, block_len)
            if not brk:
                seated = True
                break
            reseed += 1
            ops.seeded(reseed, row0, start)
        if not seated:
            res.breakdown = True
            res.breakdown_reason = "invariant subspace exhausted before k pairs"
            break
        ops.copy(w, vecs[nlocked])
        alpha, beta = [], []
        ma = 0
        for j in range(msize):
            if res.iterations >= max_iters or time.perf_counter() - t0 > max_time:
                out_of_budget = True
                break
            op.apply(vecs[nlocked + j], w)
            res.iterations += 1
            h, brk = orthogonalize(ortho, vecs, nlocked + j + 1, w, ops, ar, bufs, block_len)
            alpha.append(h[nlocked + j])
            ma = j + 1
            if brk:
                beta.append(0.0)  # the subspace closed exactly
                break
            beta.append(h[nlocked + j + 1])
            ops.copy(w, vecs[nlocked + j + 1])
        if ma == 0:
            break
        vals, Y = tridiag_eig(alpha, beta[: ma - 1])
        beta_last = beta[ma - 1]
        order = sorted(range(ma), key=lambda i: -abs(vals[i]))  # stable, as magnitude_order
        want = min(k - nlocked, ma)
        sample = 0.0
        ready, restart_dir = [], None
        for t in range(want):
            i = order[t]
            y = [float(Y[l, i]) for l in range(ma)]
            est = abs(beta_last * y[ma - 1])
            sample = max(sample, est)
            ops.scale(0.0, w)
            ops.from_host(y, coef[:ma])
            ops.maxpy(vecs[nlocked:nlocked + ma], ma, coef, 1.0, w)
            if est < tol:
                v = ops.zeros(n)
                ops.copy(w, v)
                ready.append((float(vals[i]), v))
            elif restart_dir is None:
                restart_dir = ops.zeros(n)
                ops.copy(w, restart_dir)
        for val, vec in ready:
            _, brk = orthogonalize("dgks", vecs, nlocked, vec, ops, ar, bufs, block_len)
            if brk:
                continue
            ops.copy(vec, vecs[nlocked])
            nlocked += 1
            locked_vals.append(val)
        if nlocked >= k:
            break
        if restart_dir is not None:
            start = restart_dir
        else:
            reseed += 1
            ops.seeded(reseed, row0, start)
        if not out_of_budget:
            res.restarts.append((res.iterations, msize))
            if sample > 0.0:
                res.residual_history.append(sample)
    res.converged = nlocked >= k
    r = ops.zeros(n)
    for i in sorted(range(nlocked), key=lambda i: -abs(locked_vals[i])):
        v = vecs[i]
        op.apply(v, r)  # true_residual_eigen (solver_types.hpp:113-119)
        ops.axpby(-locked_vals[i], v, 1.0, r)
        rn = _norm(ops, ar, r, nbuf)
        res.eigenvalues.append(locked_vals[i])
        res.eigenvectors.append(v)
        res.residuals.append(rn)
        res.max_residual = max(res.max_residual, rn)
    res.fault_convergence = res.converged and res.max_residual > tol
    res.allreduces = ar.n
    res.elapsed_seconds = time.perf_counter() - t0
    return res
