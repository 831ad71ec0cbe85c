"""bench.py plumbing on CPU: `--gpus N` without a torchrun environment re-launches the
script under torch.distributed.run with N ranks (one process per GPU), each seeing the
rank environment the driver's own torchrun launch provides."""
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_gpus_flag_spawns_ranks():
    env = {k: v for k, v in os.environ.items()
           if k not in ("RANK", "LOCAL_RANK", "WORLD_SIZE", "MASTER_ADDR", "MASTER_PORT")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                          "--dry-run-ranks"], capture_output=True, text=True, env=env,
                         timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    # the two ranks print concurrently: their lines may interleave, so parse objects
    lines = [json.loads(m) for m in re.findall(r"\{[^{}]*\}", out.stdout)]
    assert sorted(int(d["RANK"]) for d in lines) == [0, 1]
    assert sorted(int(d["LOCAL_RANK"]) for d in lines) == [0, 1]
    assert all(d["WORLD_SIZE"] == "2" and d["MASTER_ADDR"] == "127.0.0.1" for d in lines)
    assert len({d["MASTER_PORT"] for d in lines}) == 1


def test_bench_single_gpu_runs_in_process():
    env = {k: v for k, v in os.environ.items() if k != "WORLD_SIZE"}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--dry-run-ranks"],
                         capture_output=True, text=True, env=env, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    lines = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1 and lines[0]["WORLD_SIZE"] is None
