"""bench.py's multi-rank path on one GPU: torchrun ranks (gloo for the host
collectives, all on cuda:0 -- their kernels never wait on each other) render
their interleaved bins and either pack tiles for a gather to rank 0 ('nccl'
path, through host memory under gloo) or write their pixels straight into
rank 0's framebuffer through CUDA IPC ('peer' path, NVLink peer memory on a
multi-GPU node); rank 0's frame must equal the unsharded render byte for
byte."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.gpu
@pytest.mark.parametrize("world,workload,gather", [(2, "boxes1080", "nccl"), (3, "stack64k", "nccl"),
                                                   (2, "boxes1080", "peer"), (3, "stack64k", "peer"),
                                                   (2, "tiny4m", "peer")])
def test_bench_multirank_frame_identical(world, workload, gather):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr", "127.0.0.1",
           "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", str(world), "--steps", "3", "--warmup", "3", "--workload", workload,
           "--dist-backend", "gloo", "--single-device", "--check-frame", "--no-cpu-baseline",
           "--gather", gather]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    line = [l for l in out.stdout.splitlines() if l.startswith("{")][-1]
    res = json.loads(line)
    assert res["n_gpus"] == world
    assert res["frame_check"]["identical"], res["frame_check"]
    if gather == "peer":  # CUDA IPC between processes on one device works as across NVLink
        assert "peer-memory" in res["parallelism"], res["parallelism"]
    assert res["value"] > 0 and res["e2e"]["value"] > 0
