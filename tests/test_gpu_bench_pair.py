"""bench.py's N > 1 path end to end on a one-GPU box (MPC_BENCH_ONE_GPU=1): two torchrun ranks
form one party pair on cuda:0 (gloo for the host collectives, cudaIpc for the exchange memory),
run the cfg2 softmax in MPC_MODE_PAIR through the same code the multi-GPU driver runs, and rank 0
prints the JSON line.  The parties' kernels time-slice on one GPU, so only the plumbing and the
line's structure are checked, not the throughput."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_two_ranks_one_gpu():
    env = dict(os.environ, MPC_BENCH_ONE_GPU="1", MASTER_ADDR="127.0.0.1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29533", os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--no-per-op", "--no-cpu-baseline"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["config"]["parallelism"] == "pairs1"
    assert "PAIR" in d["config"]["mode"] and d["roofline"]["nvlink"]["payload_bytes_per_party_per_step"] > 0
    assert d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
    # party 1 is fed by the trusted dealer's offline stream, its context has no K_0
    assert d["roofline"]["dealer"]["party1_stream_bytes_per_step"] > 0
    assert d["parity_ok"] is True
