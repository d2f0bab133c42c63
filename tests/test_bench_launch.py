"""bench.py's multi-rank launch contract on CPU: `--gpus N` with no torchrun
environment re-launches itself under torch.distributed.run with N ranks on
127.0.0.1 (each rank sees WORLD_SIZE=N and its own RANK/LOCAL_RANK); the
probe flag stops each rank before any device work."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_gpus_2_spawns_two_ranks():
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                          "--launch-probe"], capture_output=True, text=True, env=env,
                         timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(ln) for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert sorted(ln["rank"] for ln in lines) == [0, 1]
    assert all(ln["world"] == 2 and ln["master_addr"] == "127.0.0.1" for ln in lines)
    assert sorted(ln["local_rank"] for ln in lines) == [0, 1]


def test_gpus_more_than_present_fails_loudly():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "8"],
                         capture_output=True, text=True, env=env, timeout=300, cwd=ROOT)
    assert out.returncode != 0
    assert "--gpus 8 but only" in out.stderr
