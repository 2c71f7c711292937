"""bench.py refuses to measure something other than what it was asked for (no GPU needed)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args, env=None):
    e = dict(os.environ)
    for k in ("RANK", "LOCAL_RANK", "WORLD_SIZE"):
        e.pop(k, None)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          env=e, timeout=300)


def test_gpus_without_launcher_fails_loudly():
    r = _run("--gpus", "2")
    assert r.returncode == 2 and "WORLD_SIZE=1" in r.stderr and "torch.distributed.run" in r.stderr


def test_world_size_mismatch_fails():
    r = _run("--gpus", "4", env={"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode == 2


def test_no_gpu_no_cpu_path():
    import torch
    if torch.cuda.is_available():
        import pytest
        pytest.skip("a GPU is present")
    r = _run("--steps", "1", "--warmup", "3")
    assert r.returncode == 3 and "no CPU path" in r.stderr
