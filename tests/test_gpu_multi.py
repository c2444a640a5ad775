"""Multi-GPU SUMMA path on real GPUs (skipped unless >= 2 devices are visible):
runs tools/multi_gpu_check.py under torchrun on 2 (and 4) GPUs -- maps identical
to the 1-GPU run, C bitwise identical to the 1-GPU C, received bytes equal to the
closed form; with GMP_FLAG_SENDER_SIDE (hybrid conversion, NEXT-2)
the same bitwise C with fewer bytes on NVLink."""
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


@pytest.mark.parametrize("G,sender,cfg", [(2, False, "small"), (2, True, "small"), (4, False, "small"),
                                          (4, True, "small"), (2, False, "uneven"), (4, True, "uneven")])
def test_summa_bitwise_vs_single_gpu(G, sender, cfg):
    if torch.cuda.device_count() < G:
        pytest.skip(f"needs {G} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={G}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tools", "multi_gpu_check.py"), "--cfg", cfg] + (["--sender"] if sender else [])
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = [l for l in r.stdout.splitlines() if l.startswith("{")][-1]
    res = json.loads(line)
    assert res["ok"], res["msgs"]
    if sender and cfg == "small":   # the FP8-enabled random workload has panel tiles sent cheaper than stored
        assert res["recv_bytes_all"] < res["stored_bytes_all"], res
