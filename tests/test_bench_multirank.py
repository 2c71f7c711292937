"""The N > 1 path of bench.py (one canonical batch sharded r mod N, results gathered to rank 0 inside the
e2e timing, max over ranks) run as two ranks on the single GPU of a gpurun box (gloo for the host
collectives: NCCL refuses two ranks on one device).  Functional only: such a run measures nothing about
two GPUs."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.gpu
def test_two_ranks_one_canonical_batch():
    env = dict(os.environ, FASTGED_BENCH_SHARE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "3", "--npairs", "2000", "--cpu-seconds", "3"]
    r = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["pairs_total"] == 4000 and d["config"]["pairs_per_gpu"] == 2000
    assert d["scaling"] == "weak" and "gather" in d["e2e"]["includes"]
    # rank 0 gathered every pair: its first 4000 pairs are the golden cfg3 pairs, all bit-exact
    assert d["parity"]["golden"]["checked"] == 4000 and d["parity"]["golden"]["mismatches"] == 0
    assert d["parity"]["oracle_live"]["mismatches"] == 0
