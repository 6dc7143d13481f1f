"""The multi-rank bench path run for real: two ranks under
torch.distributed.run on the box's one GPU, over gloo (the driver's
multi-GPU runs use NCCL, one rank per GPU).  Both ranks run the C1 shard
with the per-step size-table all-gather and the sharded whole-checkpoint
line (planner.encode_sharded + decode_chain per rank); the ranks' kernels
never wait on each other (only the host all-gathers do)."""

import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_bench_two_ranks_gloo(dev):
    env = dict(os.environ, BSNP_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py",
           "--gpus", "2", "--steps", "2", "--warmup", "1", "--log2n", "24",
           "--ckpt-config", "C0", "--no-e2e", "--no-cpu", "--no-c2", "--no-sweep"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]          # rank 0 prints ONE line
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["scaling"] == "weak"
    assert line["config"]["n_c"] > 0
    assert line["dist"]["world"] == 2 and [r["rank"] for r in line["dist"]["ranks"]] == [0, 1]
    assert "2 ranks joined" in out.stderr
    c = line["c0_sharded"]
    assert c["ranks"] == 2 and c["restored_bit_exact"] is True
    assert c["raw_bytes"] == 1244398080
    assert 2.5 < c["compression_ratio"] < 3.2


def test_bench_nccl_process_group_one_rank(dev):
    """The NCCL path on the box's one GPU: the bench under
    torch.distributed.run with an NCCL process group (one rank): the
    planner's size-table all_gather_into_tensor runs over NCCL on device
    tensors (NCCL_DEBUG shows the communicator)."""
    env = dict(os.environ, BSNP_FORCE_PG="1", NCCL_DEBUG="INFO")
    env.pop("BSNP_DIST_BACKEND", None)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py",
           "--gpus", "1", "--steps", "2", "--warmup", "1", "--log2n", "24",
           "--ckpt-config", "C0", "--no-e2e", "--no-cpu", "--no-c2", "--no-sweep", "--no-c0"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    assert "NCCL INFO" in out.stdout + out.stderr
    line = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][0])
    c = line["c0_sharded"]
    assert c["ranks"] == 1 and c["restored_bit_exact"] is True
