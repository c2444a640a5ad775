"""Clock / power / throughput of a long tensor-pipe run: cuBLAS BF16 GEMM
(torch.matmul) vs this library's FP16 class (cfg5 uniform tol 1e-2, all FP16),
each for a few seconds, clocks and board power sampled by NVML (bench.Clocks)."""
import os
import sys
import json
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import gmp_inputs  # noqa: E402
from paper_2508_14848_b200 import api  # noqa: E402
from paper_2508_14848_b200 import binding as B  # noqa: E402


def timed(fn, seconds, flops):
    fn(); torch.cuda.synchronize()
    clk = bench.Clocks(0); clk.start()
    n, t0 = 0, time.time()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    while time.time() - t0 < seconds:
        fn(); n += 1
        if n % 4 == 0:
            torch.cuda.synchronize()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    return dict(tflops=flops * n / (ms * 1e-3) / 1e12, runs=n, clocks=clk.stop())


def main():
    n = 16384
    a = torch.randn(n, n, dtype=torch.bfloat16, device="cuda")
    b = torch.randn(n, n, dtype=torch.bfloat16, device="cuda")
    c = torch.empty(n, n, dtype=torch.bfloat16, device="cuda")
    r = timed(lambda: torch.matmul(a, b, out=c), 4.0, 2.0 * n ** 3)
    print(json.dumps(dict(run="cublas_bf16_16384", **r)), flush=True)
    del a, b, c
    torch.cuda.empty_cache()
    w = gmp_inputs.workload(5, "uniform_1e-2")
    A = api.synth(w.M, w.K, w.nb, w.a)
    Bm = api.synth(w.K, w.N, w.nb, w.b)
    desc = B.make_desc(w.M, w.N, w.K, w.nb, w.tol, w.alpha, w.beta, w.class_mask)
    g = api.GemmMP(desc, A, Bm, None)
    g.convert()
    out = torch.empty(w.M, w.N, dtype=torch.float64, device="cuda")
    r = timed(lambda: g.execute(out), 4.0, w.flops)
    print(json.dumps(dict(run="gemm_mp_cfg5_uniform_1e-2_all_FP16", **r)), flush=True)


if __name__ == "__main__":
    main()
