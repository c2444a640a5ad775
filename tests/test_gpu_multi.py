"""Multi-GPU SUMMA path on real GPUs (skipped unless >= 2 devices are visible):
runs tools/multi_gpu_check.py under torchrun on 2 (and 4) GPUs -- maps identical
to the 1-GPU run, C bitwise identical to the 1-GPU C, received bytes equal to the
closed form; with GMP_FLAG_SENDER_SIDE (hybrid conversion, NEXT-2)
the same bitwise C with fewer bytes on NVLink; with --balance (NEXT-3) the rank owners come from
gemm_mp_balance and C is still bitwise the 1-GPU C."""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


# grids 1x4 / 4x1: a 4-member row (column) communicator, as in the 2x4 grid of 8 GPUs
@pytest.mark.parametrize("G,sender,cfg,grid,balance,nccl", [
    (2, False, "small", None, False, False), (2, True, "small", None, False, False),
    (4, False, "small", None, False, False), (4, True, "small", None, False, False),
    (2, False, "uneven", None, False, False), (4, True, "uneven", None, False, False),
    (4, False, "small", "1x4", False, False), (4, True, "uneven", "4x1", False, False),
    (2, False, "small", None, True, False), (4, True, "small", None, True, False),
    (4, False, "uneven", None, True, False),
    # the NCCL-broadcast transport (GMP_FLAG_NCCL_BCAST)
    (2, False, "small", None, False, True), (4, True, "uneven", None, False, True),
    (4, False, "small", "1x4", True, True)])
def test_summa_bitwise_vs_single_gpu(G, sender, cfg, grid, balance, nccl):
    if torch.cuda.device_count() < G:
        pytest.skip(f"needs {G} GPUs")
    for attempt in range(3):   # a free port can be taken between probing and binding: retry
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={G}",
               "--master-addr", "127.0.0.1", "--master-port", str(_port()),
               os.path.join(ROOT, "tools", "multi_gpu_check.py"), "--cfg", cfg] + (["--sender"] if sender else []) + \
            (["--grid", grid] if grid else []) + (["--balance"] if balance else []) + (["--nccl"] if nccl else [])
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
        if r.returncode == 0 or "EADDRINUSE" not in r.stderr:
            break
    assert r.returncode == 0, r.stderr[-2000:]
    line = [l for l in r.stdout.splitlines() if l.startswith("{")][-1]
    res = json.loads(line)
    assert res["ok"], res["msgs"]
    if sender and cfg == "small":   # the FP8-enabled random workload has panel tiles sent cheaper than stored
        assert res["recv_bytes_all"] < res["stored_bytes_all"], res
