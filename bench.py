#!/usr/bin/env python
"""SpMV benchmark (BASELINE.json metric: "SpMV GB/s (% of HBM peak) & GFLOP/s
at 1/2/4/8 B200 vs host-CPU reference").

Default workload = BASELINE.json configs[1] (config 2): 3-D 27-point stencil
on 128^3, symmetric upper-triangle storage (n=2,097,152, nnz_s=28,920,060),
x = seeded_vector(n, 2). One step = one y = A*x through the tuned engine
(select_spmv_sym on device time -> S3 window kernel on this matrix).

GB/s uses the minimum-traffic model:
    B = 12*nnz + 4*(n+1) + 16*n      (nnz = stored nonzeros)

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
                    [--config 1|2|3|4]

N>1 (torchrun): every rank runs its own replica of the workload on its GPU
(config 2 does not shard: "replicas only", weak scaling, no collective on the
data path); ms_per_step is the max over ranks, value sums all ranks' bytes.
"""
from __future__ import annotations

import argparse
import json
import os

# the reference's OpenMP pool (CPU baseline / reference arm): one thread per
# physical core, bound close
os.environ.setdefault("OMP_PROC_BIND", "close")
os.environ.setdefault("OMP_PLACES", "cores")
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

METRIC = "SpMV GB/s (% of HBM peak) & GFLOP/s at 1/2/4/8 B200 vs host-CPU reference"

CONFIGS = {
    1: dict(workload="cfg1: 64^3 7-pt Laplacian, full CRS (n=262,144, nnz=1,810,432)",
            sym=False, seed=1,
            gpu=lambda K, dev: K.stencil7(64, 64, 64, device=dev),
            host=lambda M: M.stencil7(64, 64, 64), sample="the full matrix"),
    2: dict(workload="cfg2: 128^3 27-pt stencil, symmetric upper CRS "
                     "(n=2,097,152, nnz_s=28,920,060)", sym=True, seed=2,
            gpu=lambda K, dev: K.stencil27_upper(128, 128, 128, device=dev),
            host=lambda M: M.stencil27_upper(128, 128, 128), sample="the full matrix"),
    3: dict(workload="cfg3: power-law, n=4,000,000, 10% empty rows, Pareto(1.5) lengths <= 65,536, "
                     "nnz=39,552,727 (DESIGN.md recipe, seed 3)", sym=False, seed=3,
            gpu=lambda K, dev: K.powerlaw(device=dev),
            host=lambda M: M.powerlaw(), sample="the full matrix"),
    4: dict(workload="cfg4: 512^3 7-pt Laplacian, full CRS (n=134,217,728, nnz=937,951,232), "
                     "single GPU", sym=False, seed=4,
            gpu=lambda K, dev: K.stencil7(512, 512, 512, device=dev),
            host=lambda M: M.stencil7(512, 512, 64),
            sample="a 512x512x64 slab of the 512^3 7-pt matrix (1/8 of the rows; GB/s is "
                   "size-intensive)"),
}


class L2Flush:
    """Between timed steps: write a buffer of 2x L2 (evicts everything), then
    read a second 2x L2 buffer so the dirty flush lines are written back
    BEFORE the timed region; the timed kernel starts with a cold, clean L2."""

    def __init__(self, l2_bytes: int):
        import torch

        nb = 2 * max(l2_bytes, 64 << 20)
        self.w = torch.empty(nb, dtype=torch.uint8, device="cuda")
        self.r = torch.ones(nb // 8, dtype=torch.float64, device="cuda")
        self.sink = torch.empty((), dtype=torch.float64, device="cuda")

    def __call__(self, k: int) -> None:
        import torch

        self.w.fill_(k & 0xFF)
        torch.sum(self.r, dim=0, out=self.sink)


L2_NOTE = ("cold: before every timed step a 2x L2 buffer is written, then a second 2x L2 "
           "buffer is read (dirty lines written back outside the per-step event pairs)")


def min_bytes(n: int, nnz: int) -> int:
    return 12 * nnz + 4 * (n + 1) + 16 * n


def flops(n: int, nnz: int, sym: bool) -> int:
    return 4 * nnz - 2 * n if sym else 2 * nnz


def peak_hbm() -> tuple[float, str]:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ----------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,"
              "utilization.gpu")

    def __init__(self, gpu_id: str):
        self.gpu_id = gpu_id
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", self.gpu_id,
                                      f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def start(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        return self.summary()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no nvidia-smi samples"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for nm, val in zip(names, s[3:7]):
                if val.strip().lower() == "active":
                    reasons.add(nm)
        busy = [float(s[0]) for s in self.samples
                if len(s) > 7 and s[7].strip().isdigit() and int(s[7]) > 0 and s[0].isdigit()]
        med = float(np.median(busy if busy else sm)) if (busy or sm) else None
        return {"sm_mhz": med, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.samples)}


def gpu_uuid(dev: int) -> str:
    import torch

    try:
        u = torch.cuda.get_device_properties(dev).uuid
        s = str(u)
        return s if s.startswith("GPU-") else "GPU-" + s
    except Exception:
        return str(dev)


# ---------------------------------------------------------- CPU baseline
def cpu_reference_engine(cfg: dict):
    """The reference's own tuned CPU path (oracle/_ref = unmodified reference
    headers): select_spmv_sym/unsym + Sym/UnsymEngine::op, all host threads."""
    import matgen
    from oracle import oracle as O

    n, rp, ci, v = cfg["host"](matgen)
    cores = os.cpu_count() or 1
    eng = O.RefEngine(cfg["sym"], n, rp, ci, v, cores)
    x = O.Ref.seeded_vector(n, cfg["seed"])
    return eng, n, len(ci), x, cores


def time_cpu(eng, x, n, max_seconds=10.0, max_reps=2000, min_reps=3):
    y = np.empty(n)
    eng.apply(x, y)  # warm
    times = []
    t_end = time.perf_counter() + max_seconds
    while (len(times) < min_reps) or (time.perf_counter() < t_end and len(times) < max_reps):
        t0 = time.perf_counter()
        eng.apply(x, y)
        times.append(time.perf_counter() - t0)
    return float(np.mean(times)), len(times), y


# ------------------------------------------------------------- main arms
def run_reference(args, cfg):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    from oracle import oracle as O

    if not O.ref_available():
        print(json.dumps({"impl": "reference",
                          "unavailable": "oracle/_ref/libktune_ref.so not built"}))
        return 0
    eng, n, nnz, x, cores = cpu_reference_engine(cfg)
    B = min_bytes(n, nnz)
    y = np.empty(n)
    for _ in range(args.warmup):
        eng.apply(x, y)
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        eng.apply(x, y)
        ts.append(time.perf_counter() - t0)
    t = float(np.mean(ts))
    gbs = B / t / 1e9
    line = {
        "metric": METRIC, "value": gbs, "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (SURVEY.md §8d recipe, seeded)",
        "config": dict(config_block(cfg, f"reference {eng.selected['name']}"),
                       l2="n/a (host CPU; inputs resident in host memory)"),
        "impl": "reference",
        "gflops": flops(n, nnz, cfg["sym"]) / t / 1e9,
        "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": cores, "kind": "reference",
                         "sample": f"{args.steps} applies of {cfg['sample']} ({cfg['workload']}) through "
                                   f"the reference's tuned engine ({eng.selected['name']}, "
                                   f"{eng.selected['workers']} OpenMP workers)", **REF_BUILD},
        "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def config_block(cfg, kernel):
    return {"workload": cfg["workload"], "kernel": kernel,
            "x": f"seeded_vector(n, {cfg['seed']})",
            "l2": L2_NOTE,
            "bytes_model": "12*nnz + 4*(n+1) + 16*n (int32 idx, fp64 val, x read once, y written once)"}


def run_gpu(args, cfg):
    import torch

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2405_01599_b200 import _lib
    from paper_2405_01599_b200 import ktune as K

    a = cfg["gpu"](K, local)
    n, nnz = a.n, a.nnz()
    B = min_bytes(n, nnz)
    F = flops(n, nnz, cfg["sym"])
    stream = torch.cuda.Stream()
    if cfg["sym"]:
        choice, rep = K.select_spmv_sym(a)
    else:
        choice, rep = K.select_spmv_unsym(a)
    plan = choice.plan
    plan.set_stream(stream.cuda_stream)
    sel = rep.selected_candidate()
    kname = f"{sel.name} (param {sel.jl})"

    x = torch.empty(n, dtype=torch.float64, device="cuda")
    assert _lib.load().ktb_seeded_vector(n, cfg["seed"], 0, x.data_ptr(),
                                         stream.cuda_stream) == 0
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    l2 = torch.cuda.get_device_properties(local).L2_cache_size
    flush = L2Flush(l2)

    sampler = ClockSampler(gpu_uuid(local))
    sampler.start()
    with torch.cuda.stream(stream):
        # warm-up: >= W steps and ~1 s of load so the clocks settle
        t_warm = time.perf_counter() + args.warm_seconds
        w = 0
        while w < args.warmup or time.perf_counter() < t_warm:
            plan.apply(x, y)
            w += 1
            if w % 50 == 0:
                stream.synchronize()
        stream.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps)]
        r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        r0.record(stream)
        for k in range(args.steps):
            flush(k)
            ev[k][0].record(stream)
            plan.apply(x, y)
            ev[k][1].record(stream)
        r1.record(stream)
        stream.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
    step_ms = [e0.elapsed_time(e1) for e0, e1 in ev]
    ms = float(np.mean(step_ms))
    region_ms = r0.elapsed_time(r1)

    # e2e: public API with host buffers (pinned), H2D x + SpMV + D2H y per step
    xh = torch.empty(n, dtype=torch.float64, pin_memory=True)
    xh.copy_(x.cpu())
    yh = torch.empty(n, dtype=torch.float64, pin_memory=True)
    xn, yn = xh.numpy(), yh.numpy()
    plan.apply(xn, yn)
    e2e_ms = []
    for k in range(max(3, args.steps)):
        with torch.cuda.stream(stream):
            flush(k)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        plan.apply(xn, yn)  # copies in, runs, copies out, synchronises
        e1.record(stream)
        e1.synchronize()
        e2e_ms.append(e0.elapsed_time(e1))
    e2e_single = float(np.mean(e2e_ms))
    # pipelined: the same per-step H2D x / SpMV / D2H y through the public
    # batched host call (ktb_spmv_host_pipelined), copies of neighbouring
    # steps overlapping the SpMV; wall clock around the call (it returns
    # after the last y is on the host)
    kpipe = max(3, args.steps)
    plan.apply_host_pipelined(xn, yn, count=2)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan.apply_host_pipelined(xn, yn, count=kpipe)
    e2e = (time.perf_counter() - t0) * 1e3 / kpipe
    clocks = sampler.stop()

    if dist:
        t = torch.tensor([ms, e2e, e2e_single], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, e2e, e2e_single = float(t[0]), float(t[1]), float(t[2])

    if rank == 0:
        peak, peak_src = peak_hbm()
        achieved = B / (ms / 1e3) / 1e9
        line = {
            "metric": METRIC,
            "value": ws * B / (ms / 1e3) / 1e9,
            "unit": "GB/s",
            "n_gpus": ws,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (SURVEY.md §8d recipe, seeded; replicas per rank)",
            "config": config_block(cfg, kname),
            "gflops": ws * F / (ms / 1e3) / 1e9,
            "pct_hbm_peak": 100.0 * achieved / peak,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic_from_profile(cfg),
                         "peak_source": peak_src,
                         "kernel": f"{sel.name} apply ({plan.launches} launch{'es' if plan.launches != 1 else ''})",
                         "bytes_per_launch": B},
            "e2e": {"value": ws * B / (e2e / 1e3) / 1e9, "unit": "GB/s",
                    "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n,
                    "ms_per_step": e2e,
                    "def": "public batched host call (ktb_spmv_host_pipelined): every step "
                           "copies its x in from pinned host memory and its y out; copies "
                           "of neighbouring steps overlap the SpMV; wall clock",
                    "unpipelined": {"value": ws * B / (e2e_single / 1e3) / 1e9,
                                    "ms_per_step": e2e_single,
                                    "def": "one ktb_spmv(KTB_PTR_HOST) call per step, "
                                           "CUDA events"}},
            "gpu_launches": args.steps * plan.launches,
            "timed_region_ms": region_ms,
            "clocks": clocks,
            "selection": [{"name": c.name, "param": c.jl, "best_ms": c.best_seconds * 1e3,
                           "correct": c.correct} for c in rep.candidates],
        }
        if ws == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(cfg)
        print(json.dumps(line))
    if dist:
        dist.destroy_process_group()
    return 0


class _GeneralShard:
    """--shard: an arbitrary config matrix split by NNZ_BALANCED row blocks
    over the ranks (dist.DistCsrSpMV: native split + ghost map, NCCL ghost
    exchange overlapped with the diagonal block). Same fields as DistSpMV."""

    def __init__(self, cfg, rank, ws, local):
        import types

        import torch

        from paper_2405_01599_b200 import _lib
        from paper_2405_01599_b200 import dist as D

        if cfg["seed"] == 3:  # config 3: the native multi-threaded host generator
            from paper_2405_01599_b200 import ktune as K

            n, rp, ci, v = K.powerlaw_host()
        else:
            import matgen

            n, rp, ci, v = cfg["host"](matgen)
        self.n_glob, self.nnz_glob = n, int(rp[-1])
        b = D.nnz_balanced_boundaries(rp, ws)
        r0, r1 = int(b[rank]), int(b[rank + 1])
        self.sp = D.DistCsrSpMV(n, b, rank, ws, rp[r0:r1 + 1] - rp[r0], ci[rp[r0]:rp[r1]],
                                v[rp[r0]:rp[r1]], local)
        del rp, ci, v
        self.nnz = self.sp.A_d.nnz() + self.sp.dc.nnz_ghost
        self.kname = ("u%d" % (self.sp.plan.kernel + 1)) if self.sp.A_d.nnz() else "none"
        self.L = types.SimpleNamespace(owned_offset=0, n_local=self.sp.n_local)
        dev = f"cuda:{local}"
        self.x = torch.empty(max(self.sp.n_local, 1), dtype=torch.float64, device=dev)
        assert _lib.load().ktb_seeded_vector(self.sp.n_local, cfg["seed"], r0, self.x.data_ptr(),
                                             torch.cuda.current_stream(local).cuda_stream) == 0
        self.y = torch.empty_like(self.x)

    def apply(self):
        n = self.sp.n_local
        return self.sp.apply(self.x[:n], self.y[:n])

    def launches_per_apply(self):
        return self.sp.launches_per_apply()

    def exchange_only(self):
        n = self.sp.n_local
        self.sp.exchange_only(self.x[:n])


def run_gpu_dist(args, cfg):
    """Config 4: z-slab row-block sharding over the ranks (paper_2405_01599_b200
    .dist), NCCL P2P halo exchange overlapped with the interior rows; with
    --shard (configs 1/3): general NNZ_BALANCED row blocks with a ghost-column
    exchange. Fixed total problem: strong scaling; value = whole-matrix bytes
    / max-rank time."""
    import torch

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2405_01599_b200 import dist as D

    if args.config == 4:
        nx = ny = nz = 512
        shard = D.DistSpMV(nx, ny, nz, rank, ws, local, seed=cfg["seed"])
        n_glob = nx * ny * nz
        nnz_glob = 7 * n_glob - 6 * nx * nx  # 7-pt stencil with Dirichlet boundary
        klabel = "u1 warp-sliced (param 100) interior + boundary planes (z-slab shards, NCCL halo)"
        par = f"row-block z-slabs x{ws}, one-plane halo"
        rlabel = "u1 thread-per-row over the warp-sliced copy (rank-0 slab interior + boundary planes)"
    else:
        shard = _GeneralShard(cfg, rank, ws, local)
        n_glob, nnz_glob = shard.n_glob, shard.nnz_glob
        klabel = f"{shard.kname} on A_d + ghost accumulate (general row blocks, NCCL ghosts)"
        par = f"NNZ_BALANCED row blocks x{ws}, ghost-column exchange"
        rlabel = f"{shard.kname} (rank 0 diagonal block) + k_ghost_acc"
    B = min_bytes(n_glob, nnz_glob)
    B_local = min_bytes(shard.L.n_local, shard.nnz)
    F = flops(n_glob, nnz_glob, False)
    stream = torch.cuda.Stream()
    l2 = torch.cuda.get_device_properties(local).L2_cache_size
    flush = L2Flush(l2)
    sampler = ClockSampler(gpu_uuid(local))
    sampler.start()
    with torch.cuda.stream(stream):
        t_warm = time.perf_counter() + args.warm_seconds
        w = 0
        while w < args.warmup or time.perf_counter() < t_warm:
            shard.apply()
            w += 1
            if w % 10 == 0:
                stream.synchronize()
        stream.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps)]
        for k in range(args.steps):
            flush(k)
            if dist:  # all ranks start the step together (halo partners)
                dist.barrier()
            ev[k][0].record(stream)
            shard.apply()
            ev[k][1].record(stream)
        stream.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
    ms = float(np.mean([a.elapsed_time(b) for a, b in ev]))
    # the exchange step alone (halo planes / packed ghosts over NCCL P2P), same
    # stream and events; 0 messages at one rank
    hx = []
    with torch.cuda.stream(stream):
        for k in range(max(3, min(args.steps, 20))):
            if dist:
                dist.barrier()
            h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            h0.record(stream)
            shard.exchange_only()
            h1.record(stream)
            h1.synchronize()
            hx.append(h0.elapsed_time(h1))
    halo_ms = float(np.mean(hx))
    # e2e: owned x from pinned host, sharded apply, owned y back to host
    o0, n_loc = shard.L.owned_offset, shard.L.n_local
    xh = torch.empty(n_loc, dtype=torch.float64, pin_memory=True)
    xh.copy_(shard.x[o0:o0 + n_loc].cpu())
    yh = torch.empty(n_loc, dtype=torch.float64, pin_memory=True)
    e2e_ms = []
    with torch.cuda.stream(stream):
        for k in range(max(3, min(args.steps, 10))):
            flush(k)
            if dist:
                dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            shard.x[o0:o0 + n_loc].copy_(xh, non_blocking=True)
            shard.apply()
            yh.copy_(shard.y, non_blocking=True)
            e1.record(stream)
            e1.synchronize()
            e2e_ms.append(e0.elapsed_time(e1))
    clocks = sampler.stop()
    e2e = float(np.mean(e2e_ms))
    if dist:
        t = torch.tensor([ms, e2e, halo_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, e2e, halo_ms = float(t[0]), float(t[1]), float(t[2])
    if rank == 0:
        peak, peak_src = peak_hbm()
        achieved = B_local / (ms / 1e3) / 1e9
        line = {
            "metric": METRIC, "value": B / (ms / 1e3) / 1e9, "unit": "GB/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (SURVEY.md §8d recipe, seeded)",
            "config": dict(config_block(cfg, klabel), parallelism=par),
            "gflops": F / (ms / 1e3) / 1e9,
            "pct_hbm_peak_per_gpu": 100.0 * achieved / peak,
            "per_gpu_gbs": achieved,
            "exchange_ms": halo_ms,
            "exchange_def": "the step's x-halo / ghost exchange alone (NCCL P2P, max over "
                            "ranks); inside the step it overlaps the interior rows",
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak,
                         "traffic": traffic_from_profile(cfg) if ws == 1 and args.config == 4
                         else None,
                         "peak_source": peak_src,
                         "kernel": rlabel,
                         "bytes_per_launch": B_local,
                         "note": "peak is the measured copy (read + write) bandwidth; a "
                                 "read-dominated stream can exceed it (frac > 1); the "
                                 "warp-sliced kernel does not read row_ptr (4 B/row of the "
                                 "model)"},
            "e2e": {"value": B / (e2e / 1e3) / 1e9, "unit": "GB/s",
                    "h2d_bytes_per_step": 8 * n_glob, "d2h_bytes_per_step": 8 * n_glob,
                    "ms_per_step": e2e},
            "gpu_launches": args.steps * shard.launches_per_apply(),
            "clocks": clocks,
        }
        if ws == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(cfg)
        print(json.dumps(line))
    if dist:
        dist.destroy_process_group()
    return 0


class _TimedOp:
    """Row-sharded operator wrapper that times every apply with CUDA events
    on the current stream (SpMV device seconds inside the solve)."""

    def __init__(self, op, launches):
        self.op, self.n_local, self.launches_per = op, op.n_local, launches
        self.events, self.calls = [], 0

    def apply(self, x, y):
        import torch

        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        self.op.apply(x, y)
        e1.record()
        self.events.append((e0, e1))
        self.calls += 1

    def seconds(self):
        return sum(a.elapsed_time(b) for a, b in self.events) * 1e-3


def run_gmres(args, cfg):
    """Config 5: GMRES(30)+MGS on the 128^3 convection-diffusion matrix,
    b = A*ones (computed by our SpMV), tol 1e-8, <= 3000 iterations
    (BASELINE.json configs[4]). One step = one full solve. value = SpMV GB/s
    inside the solve (algorithmic bytes x SpMV calls / SpMV device seconds);
    e2e = the same bytes over the wall time of the public call with host b in
    and host x out. Default: the fused single-GPU solver (ktb_gmres, one
    replica per rank). --shard: krylov.gmres_m_dist over general row blocks,
    all-reduced dots (NCCL), one solve across all ranks."""
    import torch

    from paper_2405_01599_b200 import _lib
    from paper_2405_01599_b200 import ktune as K

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    a = K.stencil7(128, 128, 128, c_xm=-1.3, c_xp=-0.7, device=local)
    n, nnz = a.n, a.nnz()
    B = min_bytes(n, nnz)
    kcfg = K.KrylovConfig(30, 30, 1e-8, 3000)
    sampler = ClockSampler(gpu_uuid(local))
    if not args.shard:
        choice, rep = K.select_spmv_unsym(a)
        plan = choice.plan
        kname = f"{rep.selected_candidate().name} SpMV + cooperative MGS (ktb_gmres)"
        ones = torch.ones(n, dtype=torch.float64, device="cuda")
        bd = torch.empty_like(ones)
        plan.apply(ones, bd)  # b = A * ones on the device
        torch.cuda.synchronize()
        b_host = bd.cpu().numpy()
        for _ in range(max(1, args.warmup // 3)):
            K.gmres_m(a, b_host, kcfg, plan=plan)
        sampler.start()
        runs = []
        for _ in range(max(1, args.steps // 10)):
            t0 = time.perf_counter()
            r = K.gmres_m(a, b_host, kcfg, plan=plan)  # host b in, host x out
            runs.append((r, time.perf_counter() - t0))
        clocks = sampler.stop()
        r = runs[-1][0]
        wall = float(np.mean([t for _, t in runs]))
        spmv = float(np.mean([x.spmv_seconds for x, _ in runs]))
        calls, its, cyc = r.spmv_calls, r.iterations, r.restarts + 1
        L = plan.launches
        launches = 1 + cyc * (L + 4) + its * (L + 1) + L + 2
        info = {"iterations": its, "restarts": r.restarts, "true_residual": r.true_residual,
                "converged": r.converged, "spmv_calls": calls, "solve_seconds": wall}
        par, ranks_note = "replicas (one full solve per GPU)", ws
        value_scale = ws
    else:
        from paper_2405_01599_b200 import dist as D
        from paper_2405_01599_b200 import krylov as KR

        rp, ci, v = a.to_host()
        bnd = D.nnz_balanced_boundaries(rp, ws)
        r0, r1 = int(bnd[rank]), int(bnd[rank + 1])
        op = D.DistCsrSpMV(n, bnd, rank, ws, rp[r0:r1 + 1] - rp[r0], ci[rp[r0]:rp[r1]],
                           v[rp[r0]:rp[r1]], local)
        del rp, ci, v
        kname = f"u{op.plan.kernel + 1} on A_d + ghost acc, gmres_m_dist (MGS, NCCL all-reduce)"
        ones = torch.ones(op.n_local, dtype=torch.float64, device="cuda")
        bd = torch.empty_like(ones)
        op.apply(ones, bd)
        b_host = bd.cpu().numpy()
        ar = KR.process_group_allreduce()
        ops = KR.DeviceVecOps(31, local)
        for _ in range(max(1, args.warmup // 3)):
            KR.gmres_m_dist(op, bd, m=30, tol=1e-8, max_iters=3000, ortho="mgs", ops=ops,
                            allreduce=ar)
        if dist:
            dist.barrier()
        sampler.start()
        runs = []
        for _ in range(max(1, args.steps // 10)):
            top = _TimedOp(op, op.launches_per_apply())
            ops.launches = 0
            t0 = time.perf_counter()
            bh = torch.from_numpy(b_host).pin_memory().cuda(non_blocking=True)  # host b in
            rr = KR.gmres_m_dist(top, bh, m=30, tol=1e-8, max_iters=3000, ortho="mgs", ops=ops,
                                 allreduce=ar)
            xh = rr.x.cpu()  # host x out
            torch.cuda.synchronize()
            runs.append((rr, time.perf_counter() - t0, top.seconds(), top.calls, ops.launches,
                         top.launches_per * top.calls))
        clocks = sampler.stop()
        r = runs[-1][0]
        wall = float(np.mean([t for _, t, *_ in runs]))
        spmv = float(np.mean([s for _, _, s, *_ in runs]))
        if dist:
            t = torch.tensor([wall, spmv], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            wall, spmv = float(t[0]), float(t[1])
        calls, its = runs[-1][3], r.iterations
        launches = runs[-1][4] + runs[-1][5]
        info = {"iterations": its, "restarts": len(r.restarts), "true_residual": r.true_residual,
                "converged": r.converged, "spmv_calls": calls, "solve_seconds": wall,
                "allreduces": r.allreduces}
        par, ranks_note = f"one solve over {ws} NNZ_BALANCED row blocks", 1
        value_scale = 1
        del xh
    info.update({"spmv_seconds": spmv, "spmv_share": spmv / wall,
                 "reference_iterations_survey": 653})
    peak, peak_src = peak_hbm()
    achieved = B * calls / spmv / 1e9
    if rank == 0:
        line = {"metric": METRIC, "value": value_scale * achieved, "unit": "GB/s", "n_gpus": ws,
                "steps": len(runs), "warmup": args.warmup, "ms_per_step": wall * 1e3,
                "higher_is_better": True, "scaling": "weak" if not args.shard else "strong",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic (SURVEY.md §8d recipe)",
                "config": {"workload": "cfg5: GMRES(30)+MGS, 128^3 7-pt convection-diffusion, "
                                       "b = A*ones, tol 1e-8, max 3000 its",
                           "kernel": kname, "parallelism": par,
                           "value_def": "algorithmic SpMV bytes x SpMV calls / SpMV device "
                                        "seconds inside the solve"},
                "gmres": info,
                "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                             "frac": achieved / peak,
                             "traffic": traffic_from_profile({"workload": "cfg5:"}),
                             "peak_source": peak_src,
                             "kernel": "the SpMV applies inside the solve"},
                "e2e": {"value": value_scale * B * calls / wall / 1e9, "unit": "GB/s",
                        "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n,
                        "def": "same SpMV bytes over the wall time of the whole solve call, "
                               "host b in, host x out"},
                "gpu_launches": launches * len(runs) * ranks_note,
                "clocks": clocks}
        if ws == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = _gmres_cpu_baseline(a, B)
        print(json.dumps(line))
    if dist:
        dist.destroy_process_group()
    return 0


def _gmres_cpu_baseline(a, B):
    from oracle import oracle as O  # cpu_baseline leg only

    try:
        rp, ci, v = a.to_host()
        n = a.n
        b = O.spmv_ref(n, rp, ci, v, np.ones(n))
        its = 60  # bounded sample: two restarts of the reference solver
        _, rr = O.Ref.gmres(n, rp, ci, v, b, 30, 1e-8, its, 1, os.cpu_count() or 1)
        return {"value": B * rr["spmv_calls"] / max(rr["spmv_seconds"], 1e-12) / 1e9,
                "unit": "GB/s", "cores": os.cpu_count(), "kind": "reference",
                "sample": f"{its} iterations of ktune::gmres_m (MGS) with a U1 UnsymEngine on "
                          f"all cores: {rr['seconds']:.2f} s ({rr['seconds'] / its * 1e3:.1f} "
                          f"ms/it; 653 its extrapolate to {rr['seconds'] / its * 653:.1f} s)"}
    except Exception as e:
        return {"value": None, "sample": f"unavailable: {e}"}


def traffic_from_profile(cfg):
    """dram bytes (read+write) per launch of the dominant kernel from the
    committed ncu --set full summary, if present (profiles/traffic.json)."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(cfg["workload"].split(":")[0])
    except Exception:
        return None


REF_BUILD = {"build": "unmodified reference headers via oracle/Makefile: g++ -O2 -std=c++20 "
                      "-fopenmp -ffp-contract=off (no -march=native)",
             "binding": "OMP_PROC_BIND=%s OMP_PLACES=%s" % (os.environ.get("OMP_PROC_BIND"),
                                                          os.environ.get("OMP_PLACES"))}


def cpu_baseline(cfg):
    try:
        eng, n, nnz, x, cores = cpu_reference_engine(cfg)
        t, reps, _ = time_cpu(eng, x, n)
        return {"value": min_bytes(n, nnz) / t / 1e9, "unit": "GB/s", "cores": cores,
                "kind": "reference",
                "sample": f"{reps} applies ({reps * t:.1f} s) of {cfg['sample']} ({cfg['workload']}) "
                          f"through the reference's tuned engine ({eng.selected['name']}, "
                          f"{eng.selected['workers']} OpenMP workers)",
                "ms_per_apply": t * 1e3, **REF_BUILD}
    except Exception as e:  # report, never fail the GPU line
        return {"value": None, "unit": "GB/s", "cores": os.cpu_count(), "kind": "reference",
                "sample": f"unavailable: {e}"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2, choices=sorted(CONFIGS) + [5])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--shard", action="store_true",
                    help="configs 1/3: general row-block sharding over the ranks; config 5: "
                         "one distributed solve (default: replicas)")
    ap.add_argument("--warm-seconds", type=float, default=1.0,
                    help="keep warming up at least this long (clocks settle); 0 under ncu")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = CONFIGS.get(args.config, {"workload": "cfg5", "sym": False, "seed": 5})
    if args.impl == "reference":
        return run_reference(args, cfg)
    if args.config == 4 or (args.shard and args.config in (1, 3)):
        return run_gpu_dist(args, cfg)
    if args.config == 5:
        return run_gmres(args, cfg)
    return run_gpu(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
