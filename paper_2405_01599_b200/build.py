"""Build libktb.so in-tree for sm_100a (nvcc, no JIT cache).

    python -m paper_2405_01599_b200.build        # or __graft_entry__.build()
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "_lib")
LIB = os.path.join(LIBDIR, os.environ.get("KTB_LIB_NAME", "libktb.so"))
# race-stress variant (KTB_CHAOS: random sleeps at every barrier / publish,
# device bounds checks), loaded only by tests/test_chaos_gpu.py
CHAOS_LIB = os.path.join(LIBDIR, "libktb_chaos.so")
SOURCES = ["ktb_api.cu", "ktb_build.cu", "ktb_unsym.cu", "ktb_sym.cu", "ktb_gen.cu", "ktb_gmres.cu",
           "ktb_mm.cu", "ktb_dist.cu", "ktb_comm.cu", "ktb_vec.cu",
           "ktb_ilu.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# NCCL for the native halo / ghost exchange (ktb_comm.cu): the system headers
# for the types; libnccl.so.2 itself is dlopen'ed at the first communicator
# call (the copy torch already loaded, else the system library).
NCCL_INC = os.environ.get("KTB_NCCL_INC", "/usr/include")


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "ktb.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, chaos: bool = False) -> str:
    lib = CHAOS_LIB if chaos else LIB
    if not force and not _stale(lib):
        return lib
    os.makedirs(LIBDIR, exist_ok=True)
    cmds, objs = [], []
    for src in SOURCES:
        path = os.path.join(CSRC, src)
        if not os.path.exists(path):
            continue
        obj = os.path.join(LIBDIR, os.path.basename(lib) + "." + src.replace(".cu", ".o"))
        extra = os.environ.get("KTB_EXTRA_FLAGS", "").split() + (["-DKTB_CHAOS"] if chaos else [])
        cmds.append([nvcc(), *ARCH, "-O3", *extra, "-lineinfo", "-std=c++17", "-Xcompiler",
                     "-fPIC", "--expt-relaxed-constexpr", "-Xptxas", "-v" if verbose else "-O3",
                     "-I", NCCL_INC, "-c", path, "-o", obj])
        objs.append(obj)
    # translation units are independent: compile them concurrently
    with ThreadPoolExecutor(max_workers=min(len(cmds), os.cpu_count() or 1)) as ex:
        for f in [ex.submit(subprocess.run, c, check=True) for c in cmds]:
            f.result()
    tmp = lib + ".tmp"
    subprocess.run([nvcc(), *ARCH, "-shared", "-o", tmp, *objs, "-lcudart", "-ldl"], check=True)
    os.replace(tmp, lib)
    for o in objs:
        os.remove(o)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, chaos="--chaos" in sys.argv))
