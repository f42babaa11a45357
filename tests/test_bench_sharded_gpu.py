"""bench.py's N > 1 line through the library's C++ orchestration
(ctd_gpu_ctd_s_sharded): two ranks sharing one B200 (CTD_BENCH_SAME_GPU=1,
gloo host callbacks; a one-GPU box cannot run two NCCL ranks), weak-scaled C2.
The replicated kept set must equal the single-rank C2 run's size class and the
line must report both ranks."""
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
def test_bench_two_ranks_native_orchestration():
    env = dict(os.environ, CTD_BENCH_SAME_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "1", "--warmup", "3", "--no-e2e"]
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0
    assert d["orchestration"].startswith("C++")
    assert d["result"]["nnz_global"] > 1.9e7
    assert 0 < d["result"]["kept"] <= d["result"]["unique_sampled"] <= 2000
    assert 0.0 < d["result"]["relative_error"] < 1.0
