"""Multi-GPU dispatch/combine parity over CUDA-IPC peer memory (NVLink):
runs tests/mgpu_worker.py under torchrun on every visible GPU (>= 2)."""

import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_multi_gpu_parity():
    n = torch.cuda.device_count()
    n = 8 if n >= 8 else (4 if n >= 4 else 2)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    worker = Path(__file__).resolve().parent / "mgpu_worker.py"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(worker)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600,
                       env={**os.environ, "OMP_NUM_THREADS": "1"})
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "MULTI-GPU PARITY OK" in r.stdout
