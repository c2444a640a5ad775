"""A/B of the 16-bit tensor class kernels under the board power cap: one all-BF16
(explicit maps) GEMM executed back to back for a few seconds per variant, TF/s,
median SM clock and board power (NVML), next to cuBLAS BF16 on random data.
Prints one JSON line per run.  Usage: python tools/power_ab.py [N] [variants...]
variants: default, pair, mcast, fused  (GMP_FLAG_TC_PAIR / _MCAST / _FUSED)"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import gmp_inputs  # noqa: E402
from paper_2508_14848_b200 import api  # noqa: E402
from paper_2508_14848_b200 import binding as B  # noqa: E402


def timed(fn, seconds, flops):
    fn()
    torch.cuda.synchronize()
    clk = bench.Clocks(0)
    clk.start()
    n, t0 = 0, time.time()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    while time.time() - t0 < seconds:
        fn()
        n += 1
        if n % 2 == 0:
            torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    c = clk.stop()
    tf = flops * n / (ms * 1e-3) / 1e12
    return dict(tflops=round(tf, 1), runs=n, sm_mhz=c["sm_mhz"], power_w=c["power_w_median"], reasons=c["reasons"],
                pj_per_flop=round(c["power_w_median"] / (tf * 1e12) * 1e12, 4) if c["power_w_median"] else None)


FLAGS = {"default": 0, "single": B.GMP_FLAG_TC_SINGLE, "pair": B.GMP_FLAG_TC_PAIR}


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
    variants = sys.argv[2:] or ["default"]
    secs = float(os.environ.get("SECS", "5"))
    for m in ((8192, 16384) if not os.environ.get("NO_CUBLAS") else ()):
        a = torch.randn(m, m, dtype=torch.bfloat16, device="cuda")
        b = torch.randn(m, m, dtype=torch.bfloat16, device="cuda")
        c = torch.empty(m, m, dtype=torch.bfloat16, device="cuda")
        r = timed(lambda: torch.matmul(a, b, out=c), secs, 2.0 * m ** 3)
        print(json.dumps(dict(run=f"cublas_bf16_{m}", **r)), flush=True)
        del a, b, c
    torch.cuda.empty_cache()
    nb = 2048
    w = gmp_inputs.small_workload(n, n, n, nb, 1e-4, mode="random", E=32, beta=0.0, seed=3000)
    A = api.synth(w.M, w.K, w.nb, w.a)
    Bm = api.synth(w.K, w.N, w.nb, w.b)
    t = n // nb
    amap = np.full((t, t), 3, np.uint8)
    out = torch.empty(w.M, w.N, dtype=torch.float64, device="cuda")
    for v in variants:
        cls, zero = 3, False
        if v.endswith("_zero"):
            zero, v = True, v[:-5]
        if v.endswith("_fp16"):
            cls, v = 2, v[:-5]
        if zero:
            A.zero_()
            Bm.zero_()
        amap[:] = cls
        desc = B.make_desc(w.M, w.N, w.K, w.nb, w.tol, w.alpha, w.beta, 0b01111, FLAGS[v], a_map=amap, b_map=amap)
        g = api.GemmMP(desc, A, Bm, None)
        g.convert()
        r = timed(lambda: g.execute(out), secs, w.flops)
        tag = os.environ.get("TAG", "")
        print(json.dumps(dict(run=f"gemm_mp_all_{'BF16' if cls == 3 else 'FP16'}_{n}_{v}{'_zero' if zero else ''}{tag}",
                              **r)), flush=True)
        g.close()
        del g
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
