#!/usr/bin/env python
"""SpMV benchmark (BASELINE.json metric: "SpMV GB/s (% of HBM peak) & GFLOP/s
at 1/2/4/8 B200 vs host-CPU reference").

Default workload = config 4 (BASELINE.json configs[3], the one quoted "at
1/2/4/8 B200" and the largest that fits one GPU): 3-D 7-point Laplacian on
512^3 (n=134,217,728, nnz=937,951,232), full CRS, row-block partitioned by
z-planes over the ranks with a one-plane x halo. One step = one y = A*x
through libktb's native halo operator (ktb_halo_spmv: NCCL group on a
high-priority stream overlapped with the interior rows, boundary planes after
an event wait; the rows by U1 param 106 -- persistent warps over pair-coded
records, falling back to 105 / 104 / 100 when a layout is refused -- bitwise
equal to the reference's spmv_ref). The same code path runs at every N.
`e2e` = the public host call (host x in, host y out, copies inside the timed
region), timed after 0.5 s of untimed calls of the same kind.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
                    [--config 1|2|3|4|5] [--shard] [--ref-build release|native|parity]

--gpus N with WORLD_SIZE unset re-launches itself under torchrun with N ranks
(127.0.0.1 rendezvous), failing loudly if fewer than N GPUs exist; under
torchrun (the driver's launch) each rank drives LOCAL_RANK's GPU. The control
plane (id hand-off, barriers, max over ranks) is torch.distributed on gloo;
the data plane is libktb's own NCCL communicator.

GB/s uses the minimum-traffic model:
    B = 12*nnz + 4*(n+1) + 16*n      (nnz = stored nonzeros)
Config 4: value = whole-matrix B / max-over-ranks step time (strong scaling).
"""
from __future__ import annotations

import argparse
import json
import os

# the reference's OpenMP pool (CPU baseline / reference arm): one thread per
# physical core, bound close
os.environ.setdefault("OMP_PROC_BIND", "close")
os.environ.setdefault("OMP_PLACES", "cores")
# the NCCL communicator init line (nranks, devices) goes to a per-process log
# that bench.py re-emits on stderr and in the JSON line
if os.environ.get("NCCL_DEBUG", "").upper() not in ("INFO", "TRACE"):
    os.environ["NCCL_DEBUG"] = "INFO"  # the image sets VERSION
os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
os.environ.setdefault("NCCL_DEBUG_FILE", f"/tmp/ktb_bench_nccl.{os.getpid()}.log")
import socket  # noqa: E402
import subprocess  # noqa: E402
import sys  # noqa: E402
import threading  # noqa: E402
import time  # noqa: E402

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

METRIC = "SpMV GB/s (% of HBM peak) & GFLOP/s at 1/2/4/8 B200 vs host-CPU reference"


def _ref_stencil(nx, ny, nz):
    def make(pool, variant):
        from oracle import oracle as O

        return O.RefEngine.stencil7(nx, ny, nz, 6.0, -1.0, pool, variant)
    return make


def _ref_host(builder, sym):
    def make(pool, variant):
        import matgen
        from oracle import oracle as O

        n, rp, ci, v = builder(matgen)
        return O.RefEngine(sym, n, rp, ci, v, pool, variant)
    return make


CONFIGS = {
    1: dict(workload="cfg1: 64^3 7-pt Laplacian, full CRS (n=262,144, nnz=1,810,432)",
            sym=False, seed=1, n=262_144, nnz=1_810_432,
            gpu=lambda K, dev: K.stencil7(64, 64, 64, device=dev),
            host=lambda M: M.stencil7(64, 64, 64), ref=_ref_stencil(64, 64, 64),
            sample="the full matrix"),
    2: dict(workload="cfg2: 128^3 27-pt stencil, symmetric upper CRS "
                     "(n=2,097,152, nnz_s=28,920,060)", sym=True, seed=2,
            gpu=lambda K, dev: K.stencil27_upper(128, 128, 128, device=dev),
            host=lambda M: M.stencil27_upper(128, 128, 128),
            ref=_ref_host(lambda M: M.stencil27_upper(128, 128, 128), True),
            sample="the full matrix"),
    3: dict(workload="cfg3: power-law, n=4,000,000, 10% empty rows, Pareto(1.5) lengths <= 65,536, "
                     "nnz=39,552,727 (DESIGN.md recipe, seed 3)", sym=False, seed=3,
            gpu=lambda K, dev: K.powerlaw(device=dev),
            host=lambda M: M.powerlaw(), ref=_ref_host(lambda M: M.powerlaw(), False),
            sample="the full matrix"),
    4: dict(workload="cfg4: 512^3 7-pt Laplacian, full CRS (n=134,217,728, nnz=937,951,232), "
                     "z-plane row blocks over the ranks, one-plane x halo",
            sym=False, seed=4, n=134_217_728, nnz=937_951_232,
            ref=_ref_stencil(512, 512, 512), sample="the full 512^3 matrix"),
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
# the same string in both arms' `config` (so the two lines name one config)
L2_BOTH = ("GPU arm: " + L2_NOTE + "; CPU reference arm: n/a (inputs resident in host memory)")


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


def physical_cores() -> int:
    """Physical cores (distinct (physical id, core id) pairs, i.e. lscpu
    sockets x cores per socket), bounded by the CPU affinity this process
    started with (read at import, before CUDA/NCCL touch any thread mask)."""
    return _PHYS_CORES


def _physical_cores() -> int:
    try:
        pairs, cur = set(), {}
        with open("/proc/cpuinfo") as f:
            for line in f:
                if not line.strip():
                    if "core id" in cur:
                        pairs.add((cur.get("physical id", "0"), cur["core id"]))
                    cur = {}
                    continue
                k, _, v = line.partition(":")
                cur[k.strip()] = v.strip()
        if "core id" in cur:
            pairs.add((cur.get("physical id", "0"), cur["core id"]))
        n = len(pairs) or (os.cpu_count() or 1)
    except OSError:
        n = os.cpu_count() or 1
    return max(1, min(n, len(os.sched_getaffinity(0))))


_PHYS_CORES = _physical_cores()
# the CPU set this process started with: NCCL narrows a communicator-creating
# thread's affinity, and a child would inherit the narrowed mask
_AFFINITY0 = set(os.sched_getaffinity(0))


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def self_launch(args):
    """--gpus N > 1 without a torchrun environment: exec N ranks under
    torch.distributed.run on this node (127.0.0.1 rendezvous)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    if not args.launch_probe:
        import torch

        have = torch.cuda.device_count()
        if have < args.gpus:
            print(json.dumps({"error": f"--gpus {args.gpus} but only {have} CUDA device(s)"}),
                  file=sys.stderr)
            return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


class Control:
    """The host control plane across ranks (torch.distributed on gloo):
    barriers, max over ranks, gathering small objects. Not on the data path."""

    def __init__(self, ws: int):
        self.ws = ws
        self.dist = None
        if ws > 1:
            import torch.distributed as dist

            dist.init_process_group("gloo")
            self.dist = dist

    def barrier(self):
        if self.dist:
            self.dist.barrier()

    def max(self, vals):
        if not self.dist:
            return list(vals)
        import torch

        t = torch.tensor(list(vals), dtype=torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return [float(v) for v in t]

    def min(self, vals):
        return [-v for v in self.max([-v for v in vals])]

    def gather(self, obj):
        if not self.dist:
            return [obj]
        out = [None] * self.ws
        self.dist.all_gather_object(out, obj)
        return out

    def close(self):
        if self.dist:
            self.dist.destroy_process_group()


def nccl_init_lines() -> list[str]:
    """This process's NCCL communicator-init lines (NCCL_DEBUG=INFO, INIT)."""
    import ctypes

    ctypes.CDLL(None).fflush(None)  # NCCL's debug FILE is buffered
    path = os.environ.get("NCCL_DEBUG_FILE", "")
    path = path.replace("%h", socket.gethostname().split(".")[0]).replace("%p", str(os.getpid()))
    try:
        with open(path) as f:
            lines = [ln.strip() for ln in f if "Init COMPLETE" in ln or " nRanks " in ln]
    except OSError:
        lines = []
    if not lines:
        print(f"[bench] no NCCL init line in NCCL_DEBUG_FILE={path!r} (exists "
              f"{os.path.exists(path)}); NCCL_DEBUG={os.environ.get('NCCL_DEBUG')!r} "
              f"SUBSYS={os.environ.get('NCCL_DEBUG_SUBSYS')!r}", file=sys.stderr)
    return lines


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
REF_BINDING = "OMP_PROC_BIND=%s OMP_PLACES=%s" % (os.environ.get("OMP_PROC_BIND"),
                                                 os.environ.get("OMP_PLACES"))


def reference_engine(cfg: dict, variant: str):
    """The reference's own tuned CPU path (oracle/_ref: the unmodified
    reference headers): select_spmv_sym/unsym + Sym/UnsymEngine::op on a
    WorkerPool of every physical core."""
    cores = physical_cores()
    eng = cfg["ref"](cores, variant)
    from oracle import oracle as O

    x = O.Ref.seeded_vector(eng.n, cfg["seed"])
    return eng, x, cores


def _engine_desc(eng) -> dict:
    cands, sel = eng.report()
    return {"selected": f"{eng.selected['name']} (jl {eng.selected['jl']}, "
                        f"{eng.selected['workers']} workers)",
            "selection_seconds": eng.select_seconds,
            "candidates": [{"name": c["name"], "jl": c["jl"], "best_ms": c["best_seconds"] * 1e3,
                            "correct": c["correct"]} for c in cands]}


def cpu_baseline(args, seconds=10.0):
    """The reference arm (`--impl reference`) in a FRESH process: no CUDA or
    NCCL state (NCCL pins the calling thread's CPU affinity during
    communicator init, which would squeeze the OpenMP pool onto one core),
    timing as many applies as fit in `seconds` on every physical core."""
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "LOCAL_WORLD_SIZE", "GROUP_RANK",
                        "MASTER_ADDR", "MASTER_PORT", "TORCHELASTIC_RUN_ID", "OMP_NUM_THREADS")}
    cmd = [sys.executable, os.path.abspath(__file__), "--impl", "reference",
           "--config", str(args.config), "--steps", "3", "--warmup", "1",
           "--ref-build", args.ref_build, "--ref-seconds", str(seconds)]
    try:
        out = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=900,
                             preexec_fn=lambda: os.sched_setaffinity(0, _AFFINITY0))
        line = next(json.loads(ln) for ln in reversed(out.stdout.splitlines())
                    if ln.startswith("{"))
        cb = dict(line["cpu_baseline"])
        cb["ms_per_apply"] = line["ms_per_step"]
        cb["sample"] = cb["sample"].replace("rank 0 only", "a fresh process")
        return cb
    except Exception as e:  # report, never fail the GPU line
        return {"value": None, "unit": "GB/s", "cores": physical_cores(), "kind": "reference",
                "sample": f"unavailable: {e}"}


def config_block(cfg):
    """The workload, identical in both arms' lines; what an arm ran it with
    (kernel, partitioning) goes into its `run` key."""
    return {"workload": cfg["workload"],
            "x": f"seeded_vector(n, {cfg['seed']})",
            "l2": L2_BOTH,
            "bytes_model": "12*nnz + 4*(n+1) + 16*n (int32 idx, fp64 val, x read once, y written once)"}


# ------------------------------------------------------------- reference arm
def run_reference(args, cfg):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    from oracle import oracle as O

    if args.config == 5:
        print(json.dumps({"impl": "reference", "unavailable": "config 5 reference arm: see "
                          "cpu_baseline of `bench.py --config 5`"}))
        return 0
    if not O.ref_available(args.ref_build):
        print(json.dumps({"impl": "reference",
                          "unavailable": f"oracle/_ref ({args.ref_build} build) not built"}))
        return 0
    eng, x, cores = reference_engine(cfg, args.ref_build)
    n = eng.n
    nnz = cfg.get("nnz") or eng.nnz
    B = min_bytes(n, nnz)
    y = np.empty(n)
    for _ in range(args.warmup):
        eng.apply(x, y)
    ts = []
    t_end = time.perf_counter() + (args.ref_seconds or 0.0)
    while len(ts) < args.steps or (args.ref_seconds and time.perf_counter() < t_end):
        t0 = time.perf_counter()
        eng.apply(x, y)
        ts.append(time.perf_counter() - t0)
    t = float(np.mean(ts))
    gbs = B / t / 1e9
    line = {
        "metric": METRIC, "value": gbs, "unit": "GB/s", "n_gpus": ws,
        "steps": len(ts), "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "strong" if args.config == 4 else "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (SURVEY.md §8d recipe, seeded)",
        "config": config_block(cfg),
        "run": {"kernel": f"reference {eng.selected['name']}",
                "parallelism": f"{eng.selected['workers']} OpenMP workers, one host"},
        "impl": "reference",
        "gflops": flops(n, nnz, cfg["sym"]) / t / 1e9,
        "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": cores, "kind": "reference",
                         "sample": f"{len(ts)} applies of {cfg['sample']} ({cfg['workload']}) "
                                   f"through the reference's tuned engine "
                                   f"({eng.selected['name']}, {eng.selected['workers']} OpenMP "
                                   f"workers); rank 0 only",
                         "build": O.REF_FLAGS[args.ref_build], "binding": REF_BINDING,
                         **_engine_desc(eng)},
        "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# -------------------------------------------------- single-GPU plan (1, 2, 3)
def measure_plan(cfg, local, steps, warmup, warm_seconds, sampler=None):
    """select_spmv_* on device time, then `steps` cold-L2 applies; returns a
    dict of the numbers (device ms per apply, e2e host-call ms, selection)."""
    import torch

    from paper_2405_01599_b200 import _lib
    from paper_2405_01599_b200 import ktune as K

    t0 = time.perf_counter()
    a = cfg["gpu"](K, local)
    torch.cuda.synchronize()
    t_build = time.perf_counter() - t0
    n, nnz = a.n, a.nnz()
    stream = torch.cuda.Stream()
    t0 = time.perf_counter()
    choice, rep = (K.select_spmv_sym if cfg["sym"] else K.select_spmv_unsym)(a)
    t_select = time.perf_counter() - t0
    plan = choice.plan
    plan.set_stream(stream.cuda_stream)
    sel = rep.selected_candidate()
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    assert _lib.load().ktb_seeded_vector(n, cfg["seed"], 0, x.data_ptr(), stream.cuda_stream) == 0
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    flush = L2Flush(torch.cuda.get_device_properties(local).L2_cache_size)
    if sampler:
        sampler.start()
    with torch.cuda.stream(stream):
        t_warm = time.perf_counter() + warm_seconds
        w = 0
        while w < warmup or time.perf_counter() < t_warm:
            plan.apply(x, y)
            w += 1
            if w % 50 == 0:
                stream.synchronize()
        stream.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(steps)]
        for k in range(steps):
            flush(k)
            ev[k][0].record(stream)
            plan.apply(x, y)
            ev[k][1].record(stream)
        stream.synchronize()
    ms = float(np.mean([e0.elapsed_time(e1) for e0, e1 in ev]))
    graph_us = None
    if n <= (1 << 20):
        # small matrices: launch + ramp dominate a cold single apply; the
        # same applies captured back to back in one CUDA graph (warm L2: the
        # whole matrix fits in it) show the amortised per-apply time
        reps = 50
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(reps):
                plan.apply(x, y)
        plan.set_stream(stream.cuda_stream)
        g.replay()
        torch.cuda.synchronize()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record()
        for _ in range(5):
            g.replay()
        g1.record()
        torch.cuda.synchronize()
        graph_us = g0.elapsed_time(g1) * 1e3 / (5 * reps)
        del g
    # e2e: the public host call, pipelined over steps (ktb_spmv_host_pipelined)
    xh = torch.empty(n, dtype=torch.float64, pin_memory=True)
    xh.copy_(x.cpu())
    yh = torch.empty(n, dtype=torch.float64, pin_memory=True)
    xn, yn = xh.numpy(), yh.numpy()
    kpipe = max(3, steps)
    # warm-up: untimed batches of the same call for 0.5 s. The first ~0.3 s of
    # host-link traffic in a process (stream / staging-buffer creation, the link
    # coming out of its idle state) runs at less than half the steady rate
    # (tools/host_link_probe.py: 66 us per step from the second call on, config 1)
    t_w = time.perf_counter()
    while time.perf_counter() - t_w < 0.5:
        plan.apply_host_pipelined(xn, yn, count=kpipe)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan.apply_host_pipelined(xn, yn, count=kpipe)
    e2e = (time.perf_counter() - t0) * 1e3 / kpipe
    clocks = sampler.stop() if sampler else None
    return dict(n=n, nnz=nnz, ms=ms, e2e_ms=e2e, plan=plan, sel=sel, rep=rep, clocks=clocks,
                build_s=t_build, select_s=t_select, graph_us=graph_us)


def run_gpu(args, cfg):
    """Configs 1-3: the tuned plan on each rank's GPU (replicas only: these
    matrices are not sharded by default; weak scaling, no collective)."""
    import torch

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    ctl = Control(ws)
    ctl.barrier()
    r = measure_plan(cfg, local, args.steps, args.warmup, args.warm_seconds,
                     ClockSampler(gpu_uuid(local)))
    ms, e2e = ctl.max([r["ms"], r["e2e_ms"]])
    n, nnz, plan, sel = r["n"], r["nnz"], r["plan"], r["sel"]
    B, F = min_bytes(n, nnz), flops(n, nnz, cfg["sym"])
    if rank == 0:
        peak, peak_src = peak_hbm()
        achieved = B / (ms / 1e3) / 1e9
        line = {
            "metric": METRIC, "value": ws * achieved, "unit": "GB/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (SURVEY.md §8d recipe, seeded; replicas per rank)",
            "config": config_block(cfg),
            "run": {"kernel": f"{sel.name} (param {sel.jl})", "parallelism": f"replicas x{ws}"},
            "gflops": ws * F / (ms / 1e3) / 1e9,
            "pct_hbm_peak": 100.0 * achieved / peak,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic_from_profile(cfg),
                         "peak_source": peak_src,
                         "kernel": f"{sel.name} apply ({plan.launches} launch"
                                   f"{'es' if plan.launches != 1 else ''})",
                         "bytes_per_launch": B},
            "e2e": {"value": ws * B / (e2e / 1e3) / 1e9, "unit": "GB/s",
                    "h2d_bytes_per_step": ws * 8 * n, "d2h_bytes_per_step": ws * 8 * n,
                    "ms_per_step": e2e,
                    "def": "public batched host call (ktb_spmv_host_pipelined): every step "
                           "copies its x in from pinned host memory and its y out; copies "
                           "of neighbouring steps overlap the SpMV; wall clock of one "
                           "batch of max(3, steps) steps after 0.5 s of untimed batches "
                           "of the same call"},
            "gpu_launches": ws * args.steps * plan.launches,
            "clocks": r["clocks"],
            "setup_seconds": {"matrix": r["build_s"], "selection": r["select_s"]},
            "selection": [{"name": c.name, "param": c.jl, "cta_threads": c.cta_threads,
                           "best_ms": c.best_seconds * 1e3, "setup_s": c.setup_seconds,
                           "correct": c.correct} for c in r["rep"].candidates],
        }
        if r["graph_us"] is not None:
            line["graph_amortised"] = {
                "us_per_apply": r["graph_us"], "gbs": B / (r["graph_us"] * 1e-6) / 1e9,
                "def": "50 applies captured back to back in one CUDA graph, replayed 5 times, "
                       "warm L2 (the matrix fits in it): the amortised per-apply time next to "
                       "the single cold-L2 apply of ms_per_step"}
        if ws == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(args)
        print(json.dumps(line))
    ctl.close()
    return 0


# ---------------------------------------------------- config 4: halo shards
def run_halo(args, cfg):
    """Config 4 over the ranks: z-slab row blocks, native halo operator over
    libktb's NCCL communicator, the same code path at every N (at N=1 the
    interior is every row and there is no message)."""
    import torch

    from paper_2405_01599_b200 import dist as D

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    ctl = Control(ws)
    t0 = time.perf_counter()
    comm = D.Comm.nccl(device=local)
    t_comm = time.perf_counter() - t0
    nccl_lines = ctl.gather(nccl_init_lines())
    if rank == 0:
        for r, lines in enumerate(nccl_lines):
            for ln in lines:
                print(f"[rank {r}] {ln}", file=sys.stderr)
    t0 = time.perf_counter()
    shard = D.DistSpMV(512, 512, 512, comm, seed=cfg["seed"], param=args.u1_param)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0
    shard.set_timing(True)
    n_glob, nnz_glob = cfg["n"], cfg["nnz"]
    B, F = min_bytes(n_glob, nnz_glob), flops(n_glob, nnz_glob, False)
    ir, inz, br, bnz = shard.parts()
    u1p = shard.plan_params()[0]
    B_int = min_bytes(ir, inz)
    stream = torch.cuda.Stream()
    flush = L2Flush(torch.cuda.get_device_properties(local).L2_cache_size)
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
        ctl.barrier()
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps)]
        kern = []
        for k in range(args.steps):
            flush(k)
            stream.synchronize()
            ctl.barrier()  # halo partners start the step together
            ev[k][0].record(stream)
            shard.apply()
            ev[k][1].record(stream)
            stream.synchronize()
            kern.append(shard.last_times())
        ctl.barrier()
        torch.cuda.synchronize()
    ms = float(np.mean([a.elapsed_time(b) for a, b in ev]))
    int_ms = float(np.mean([a for a, _ in kern]))
    bnd_ms = float(np.mean([b for _, b in kern]))
    # the exchange step alone (one NCCL group), same stream and events
    hx = []
    with torch.cuda.stream(stream):
        for k in range(max(3, min(args.steps, 20))):
            ctl.barrier()
            h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            h0.record(stream)
            shard.exchange_only()
            h1.record(stream)
            h1.synchronize()
            hx.append(h0.elapsed_time(h1))
    halo_ms = float(np.mean(hx))
    # e2e: the public host call (ktb_halo_spmv_host): owned x from pinned host
    # memory in, owned y out, copies overlapped with the rows inside the call
    xo = shard.x[shard.owned_offset:shard.owned_offset + shard.n_local].cpu().pin_memory()
    yh = torch.empty(shard.n_local, dtype=torch.float64).pin_memory()
    xn, yn = xo.numpy(), yh.numpy()
    e2e = {}
    t_w = time.perf_counter()
    while time.perf_counter() - t_w < 0.5:  # host path warm (as for configs 1-3)
        shard.apply_host(xn, yn, chunks=16)
    for chunks in (64, 32, 16, 1):
        shard.apply_host(xn, yn, chunks=chunks)  # warm
        ts = []
        for k in range(max(3, min(args.steps, 10))):
            with torch.cuda.stream(stream):
                flush(k)
            stream.synchronize()
            ctl.barrier()
            t0 = time.perf_counter()
            shard.apply_host(xn, yn, chunks=chunks)
            ts.append((time.perf_counter() - t0) * 1e3)
        e2e[chunks] = float(np.mean(ts))
    clocks = sampler.stop()
    ach_rank = B_int / (int_ms / 1e3) / 1e9 if int_ms > 0 else 0.0
    ms, e2e64, e2e32, e2e16, e2e1, halo_max, int_max, bnd_max = ctl.max(
        [ms, e2e[64], e2e[32], e2e[16], e2e[1], halo_ms, int_ms, bnd_ms])
    by_chunks = {64: e2e64, 32: e2e32, 16: e2e16}
    e2e_chunks = min(by_chunks, key=by_chunks.get)  # the chunk count a caller would pick
    e2e_best = by_chunks[e2e_chunks]
    ach_min, = ctl.min([ach_rank])
    if rank == 0:
        peak, peak_src = peak_hbm()
        line = {
            "metric": METRIC, "value": B / (ms / 1e3) / 1e9, "unit": "GB/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (SURVEY.md §8d recipe, seeded)",
            "config": config_block(cfg),
            "run": {"kernel": f"{U1_DESC.get(u1p, 'u1')} (param {u1p}), ktb_halo_spmv",
                    "parallelism": f"row-block z-slabs x{ws}, one-plane halo, NCCL P2P"},
            "gflops": F / (ms / 1e3) / 1e9,
            "per_gpu_gbs": B / ws / (ms / 1e3) / 1e9,
            "pct_hbm_peak_per_gpu": 100.0 * B / ws / (ms / 1e3) / 1e9 / peak,
            "exchange_ms": halo_max,
            "exchange_def": "the step's halo exchange alone (one NCCL group, max over ranks); "
                            "inside the step it overlaps the interior rows",
            "kernel_ms": {"interior": int_max, "boundary": bnd_max,
                          "def": "CUDA events on the compute stream around the interior / "
                                 "boundary rows of each timed step, mean, max over ranks"},
            "roofline": {"bound": "hbm", "achieved": ach_min, "peak": peak, "unit": "GB/s",
                         "frac": ach_min / peak,
                         "traffic": traffic_from_profile(cfg) if ws == 1 else None,
                         "peak_source": peak_src,
                         "kernel": f"{U1_KERNEL.get(u1p, 'u1')} over the interior rows "
                                   "(1 launch per step)",
                         "bytes_per_launch": B_int,
                         "stream_bytes_per_launch": u1_stream_bytes(u1p, ir, inz),
                         "note": "achieved = the minimum-traffic model's bytes (12 B/nnz) over "
                                 "the kernel time, min over ranks; the kernel moves fewer bytes "
                                 "than the model (" + U1_BYTES.get(u1p, "") + "), so frac can "
                                 "exceed 1; stream_bytes_per_launch = the bytes of its own "
                                 "layout + x + y; traffic = its measured DRAM bytes per launch "
                                 "(ncu)"},
            "e2e": {"value": B / (e2e_best / 1e3) / 1e9, "unit": "GB/s",
                    "h2d_bytes_per_step": 8 * n_glob, "d2h_bytes_per_step": 8 * n_glob,
                    "ms_per_step": e2e_best, "chunks": e2e_chunks,
                    "def": "ktb_halo_spmv_host on every rank: owned x from pinned host memory "
                           "in, owned y out, copies overlapped with the row chunks inside the "
                           "call (16, 32 and 64 chunks timed, the fastest reported); wall "
                           "clock, max over ranks",
                    "ms_by_chunks": {str(k): v for k, v in by_chunks.items()},
                    "unchunked": {"value": B / (e2e1 / 1e3) / 1e9, "ms_per_step": e2e1}},
            "gpu_launches": args.steps * shard.launches_per_apply() * ws,
            "clocks": clocks,
            "nccl": {"version": comm.nccl_version, "world": comm.world,
                     "comm_init": [ln for lines in nccl_lines for ln in lines
                                   if "Init COMPLETE" in ln]},
            "setup_seconds": {"comm": t_comm, "matrix_and_plans": t_setup},
        }
        if ws == 1:
            if not args.no_secondary:
                line["secondary"] = secondary_cfg2(local, args)
            if not args.no_cpu_baseline:
                line["cpu_baseline"] = cpu_baseline(args)
        print(json.dumps(line))
    shard.close()
    comm.close()
    ctl.close()
    return 0


def secondary_cfg2(local, args):
    """Config 2 (S3, symmetric upper) at one GPU, GPU side only: kept in the
    headline line as an extra key (row a11's driver-timed evidence)."""
    try:
        r = measure_plan(CONFIGS[2], local, max(10, min(args.steps, 50)), args.warmup, 0.5)
        B = min_bytes(r["n"], r["nnz"])
        peak, _ = peak_hbm()
        a = B / (r["ms"] / 1e3) / 1e9
        s3 = [c.best_seconds * 1e3 for c in r["rep"].candidates
              if c.name == "s3" and c.correct and c.best_seconds < float("inf")]
        return {"cfg2_sym": {"workload": CONFIGS[2]["workload"],
                            "kernel": f"{r['sel'].name} (param {r['sel'].jl})",
                            "s3_ms_in_selection": min(s3) if s3 else None,
                            "ms_per_step": r["ms"], "value": a, "unit": "GB/s",
                            "frac": a / peak, "launches": r["plan"].launches,
                            "gflops": flops(r["n"], r["nnz"], True) / (r["ms"] / 1e3) / 1e9,
                            "e2e_gbs": B / (r["e2e_ms"] / 1e3) / 1e9,
                            "setup_seconds": {"matrix": r["build_s"], "selection": r["select_s"]},
                            "l2": L2_NOTE}}
    except Exception as e:
        return {"cfg2_sym": {"unavailable": str(e)}}


# ------------------------------------- configs 1/3 --shard: general row blocks
def run_general_shard(args, cfg):
    """--shard (configs 1/3): NNZ_BALANCED row blocks over the ranks, native
    ghost exchange (ktb_dist_spmv over libktb's NCCL communicator)."""
    import torch

    from paper_2405_01599_b200 import _lib
    from paper_2405_01599_b200 import dist as D

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    ctl = Control(ws)
    comm = D.Comm.nccl(device=local)
    if cfg["seed"] == 3:
        from paper_2405_01599_b200 import ktune as K

        n, rp, ci, v = K.powerlaw_host()
    else:
        import matgen

        n, rp, ci, v = cfg["host"](matgen)
    nnz_glob = int(rp[-1])
    b = D.nnz_balanced_boundaries(rp, ws)
    r0, r1 = int(b[rank]), int(b[rank + 1])
    sp = D.DistCsrSpMV(n, b, comm, rp[r0:r1 + 1] - rp[r0], ci[rp[r0]:rp[r1]], v[rp[r0]:rp[r1]])
    del rp, ci, v
    x = torch.empty(max(sp.n_local, 1), dtype=torch.float64, device="cuda")
    assert _lib.load().ktb_seeded_vector(sp.n_local, cfg["seed"], r0, x.data_ptr(),
                                         torch.cuda.current_stream().cuda_stream) == 0
    y = torch.empty_like(x)
    B, F = min_bytes(n, nnz_glob), flops(n, nnz_glob, False)
    stream = torch.cuda.Stream()
    flush = L2Flush(torch.cuda.get_device_properties(local).L2_cache_size)
    sampler = ClockSampler(gpu_uuid(local))
    sampler.start()
    with torch.cuda.stream(stream):
        for _ in range(max(args.warmup, 3)):
            sp.apply(x[:sp.n_local], y[:sp.n_local])
        stream.synchronize()
        ctl.barrier()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps)]
        for k in range(args.steps):
            flush(k)
            stream.synchronize()
            ctl.barrier()
            ev[k][0].record(stream)
            sp.apply(x[:sp.n_local], y[:sp.n_local])
            ev[k][1].record(stream)
        stream.synchronize()
        hx = []
        for k in range(max(3, min(args.steps, 20))):
            ctl.barrier()
            h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            h0.record(stream)
            sp.exchange_only(x[:sp.n_local])
            h1.record(stream)
            h1.synchronize()
            hx.append(h0.elapsed_time(h1))
    clocks = sampler.stop()
    ms, halo = ctl.max([float(np.mean([a.elapsed_time(b) for a, b in ev])), float(np.mean(hx))])
    if rank == 0:
        peak, peak_src = peak_hbm()
        line = {"metric": METRIC, "value": B / (ms / 1e3) / 1e9, "unit": "GB/s", "n_gpus": ws,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic (SURVEY.md §8d recipe, seeded)",
                "config": config_block(cfg),
                "run": {"kernel": f"{sp.kernel_name()} on A_d + k_ghost_acc (ktb_dist_spmv)",
                        "parallelism": f"NNZ_BALANCED row blocks x{ws}, ghost exchange"},
                "gflops": F / (ms / 1e3) / 1e9, "exchange_ms": halo,
                "roofline": {"bound": "hbm", "achieved": B / ws / (ms / 1e3) / 1e9,
                             "peak": peak, "unit": "GB/s",
                             "frac": B / ws / (ms / 1e3) / 1e9 / peak, "traffic": None,
                             "peak_source": peak_src, "kernel": "the sharded apply per rank"},
                "gpu_launches": args.steps * sp.launches_per_apply() * ws, "clocks": clocks}
        print(json.dumps(line))
    ctl.close()
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
    ctl = Control(ws)
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
        comm = D.Comm.nccl(device=local)
        op = D.DistCsrSpMV(n, bnd, comm, rp[r0:r1 + 1] - rp[r0], ci[rp[r0]:rp[r1]],
                           v[rp[r0]:rp[r1]])
        del rp, ci, v
        kname = f"{op.kernel_name()} on A_d + ghost acc, gmres_m_dist (MGS, NCCL all-reduce)"
        ones = torch.ones(op.n_local, dtype=torch.float64, device="cuda")
        bd = torch.empty_like(ones)
        op.apply(ones, bd)
        b_host = bd.cpu().numpy()
        ar = KR.comm_allreduce(comm)
        ops = KR.DeviceVecOps(31, local)
        for _ in range(max(1, args.warmup // 3)):
            KR.gmres_m_dist(op, bd, m=30, tol=1e-8, max_iters=3000, ortho="mgs", ops=ops,
                            allreduce=ar)
        ctl.barrier()
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
        wall, spmv = ctl.max([wall, spmv])
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
                           "value_def": "algorithmic SpMV bytes x SpMV calls / SpMV device "
                                        "seconds inside the solve"},
                "run": {"kernel": kname, "parallelism": par},
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
            line["cpu_baseline"] = _gmres_cpu_baseline(a, B, args.gmres_full_reference)
        print(json.dumps(line))
    ctl.close()
    return 0


def _gmres_cpu_baseline(a, B, full=False):
    """The reference's gmres_m (MGS) with a U1 UnsymEngine on every physical
    core: a 60-iteration sample by default, the whole 653-iteration solve with
    --gmres-full-reference (about a minute on 16 cores)."""
    from oracle import oracle as O  # cpu_baseline leg only

    try:
        rp, ci, v = a.to_host()
        n = a.n
        b = O.spmv_ref(n, rp, ci, v, np.ones(n))
        its = 3000 if full else 60
        cores = physical_cores()
        _, rr = O.Ref.gmres(n, rp, ci, v, b, 30, 1e-8, its, 1, cores)
        done = rr["iterations"]
        what = (f"the whole solve: {done} iterations, {rr['seconds']:.2f} s, true residual "
                f"{rr['true_residual']:.3e}" if full else
                f"{its} iterations (two restarts): {rr['seconds']:.2f} s "
                f"({rr['seconds'] / its * 1e3:.1f} ms/it)")
        return {"value": B * rr["spmv_calls"] / max(rr["spmv_seconds"], 1e-12) / 1e9,
                "unit": "GB/s", "cores": cores, "kind": "reference",
                "solve_seconds": rr["seconds"], "iterations": done,
                "spmv_share": rr["spmv_seconds"] / max(rr["seconds"], 1e-12),
                "sample": f"ktune::gmres_m (MGS) with a U1 UnsymEngine on all physical cores, "
                          + what, "build": O.REF_FLAGS["parity"]}
    except Exception as e:
        return {"value": None, "sample": f"unavailable: {e}"}



U1_DESC = {
    106: "u1 persistent warp slices, coded (column delta, value) pairs, bulk-copy staged",
    105: "u1 persistent warp slices, coded columns, bulk-copy staged",
    104: "u1 persistent pipelined warp slices, coded columns",
    100: "u1 warp slices",
}
U1_KERNEL = {106: "k_u1v", 105: "k_u1t", 104: "k_u1p<coded>", 100: "k_u1s"}
U1_BYTES = {
    106: "one 640-byte record per 64 rows: a dictionary of the record's (column delta, fp64 "
         "value) pairs and one 8-bit pair code per slot; no row_ptr",
    105: "8 B value + 0.5 B column code per slot, no row_ptr",
    104: "8 B value + 0.5 B column code per slot, no row_ptr",
    100: "no row_ptr",
}


def u1_stream_bytes(param, rows, nnz, width=7):
    """Bytes the U1 variant's own layout streams per launch (+ x and y once)."""
    slices = (rows + 31) // 32
    xy = 16 * rows
    if param == 106:
        return (rows + 63) // 64 * (16 * (width + 1) + 256 * ((width + 3) // 4)) + xy
    if param in (104, 105):
        return slices * (32 * width * 8 + 16 * width + 64) + xy
    if param == 100:
        return slices * 32 * width * 12 + xy
    return None


def traffic_from_profile(cfg):
    """dram bytes (read+write) per launch of the dominant kernel from the
    committed ncu --set full summary, if present (profiles/traffic.json)."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(cfg["workload"].split(":")[0])
    except Exception:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4, choices=sorted(CONFIGS) + [5])
    ap.add_argument("--ref-build", default="release", choices=["release", "native", "parity"],
                    help="reference build for the reference arm / cpu_baseline "
                         "(oracle/Makefile): the reference's CMake Release (default), "
                         "+ -march=native, or the -ffp-contract=off parity build")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--u1-param", type=int, default=106,
                    help="config 4: the halo operator's U1 variant (106 = coded columns and "
                         "values, falls back to 105 = coded columns, 104, 100)")
    ap.add_argument("--ref-seconds", type=float, default=0.0,
                    help=argparse.SUPPRESS)  # cpu_baseline: time applies for this long
    ap.add_argument("--no-secondary", action="store_true",
                    help="config 4: skip the config-2 S3 extra key")
    ap.add_argument("--shard", action="store_true",
                    help="configs 1/3: general row-block sharding over the ranks; config 5: "
                         "one distributed solve (default: replicas)")
    ap.add_argument("--gmres-full-reference", action="store_true",
                    help="config 5: time the reference's whole 653-iteration solve")
    ap.add_argument("--warm-seconds", type=float, default=1.0,
                    help="keep warming up at least this long (clocks settle); 0 under ncu")
    ap.add_argument("--launch-probe", action="store_true",
                    help="print each rank's launch environment and exit (CPU test of the "
                         "--gpus self-launch)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    rc = self_launch(args)
    if rc is not None:
        return rc
    if args.launch_probe:
        ws, rank, local = dist_env()
        print(json.dumps({"launch_probe": True, "rank": rank, "world": ws, "local_rank": local,
                          "master_addr": os.environ.get("MASTER_ADDR")}), flush=True)
        return 0
    cfg = CONFIGS.get(args.config, {"workload": "cfg5", "sym": False, "seed": 5})
    if args.impl == "reference":
        return run_reference(args, cfg)
    if args.config == 4:
        return run_halo(args, cfg)
    if args.shard and args.config in (1, 3):
        return run_general_shard(args, cfg)
    if args.config == 5:
        return run_gmres(args, cfg)
    return run_gpu(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
