"""bench.py's multi-GPU launch contract, checked on CPU (`python bench.py --gpus N`
must never silently time one GPU): with WORLD_SIZE unset it starts N ranks itself through
torch.distributed.run on 127.0.0.1, rank 0 alone prints one JSON line carrying n_gpus = N and the
max-over-ranks reduction; a WORLD_SIZE / --gpus mismatch and too few visible GPUs fail loudly."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(ROOT, "bench.py")


def _run(args, env_extra=None, timeout=240):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_PORT")}
    env.update(env_extra or {})
    return subprocess.run([sys.executable, BENCH, *args], capture_output=True, text=True, env=env, timeout=timeout)


def test_self_launch_world2_dry_run():
    r = _run(["--gpus", "2", "--dry-run"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, r.stdout  # rank 0 only
    d = json.loads(lines[0])
    assert d["dry_run"] and d["n_gpus"] == 2 and d["max_over_ranks"] == 2.0 and d["local_rank"] == 0
    assert "torch.distributed.run" in r.stderr and "--nproc-per-node=2" in r.stderr


def test_world_size_mismatch_fails():
    r = _run(["--gpus", "4", "--steps", "1", "--warmup", "3"], env_extra={"WORLD_SIZE": "2", "RANK": "0"})
    assert r.returncode == 2 and "refusing" in r.stderr
    assert not r.stdout.strip()


def test_too_few_gpus_fails_loudly():
    import torch
    if torch.cuda.is_available() and torch.cuda.device_count() >= 8:
        return  # a real 8-GPU node: the launch would run
    r = _run(["--gpus", "8", "--steps", "1", "--warmup", "3"])
    assert r.returncode == 2 and "CUDA device(s) visible" in r.stderr
    assert not r.stdout.strip()


def test_launcher_command_shape():
    sys.path.insert(0, ROOT)
    import bench
    cmd = bench.launcher_cmd(8, ["--gpus", "8", "--steps", "5"], 29500)
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=8" in cmd and "127.0.0.1" in cmd and cmd[-3:] == ["--gpus", "8", "--steps", "5"][-3:]
