"""Measure per-class library GEMM peaks on one B200 (roofline denominators).

Same method as the driver's MEASURED_PEAKS.json: library GEMM 8192^3, best of
n_burst with CUDA events (burst), plus a back-to-back loop of `sustain_s`
seconds (sustained, i.e. under the board power cap).
FP64: cuBLAS DGEMM.  FP32: cuBLAS SGEMM with TF32 disabled (CUBLAS_COMPUTE_32F, no
emulation).  FP16/BF16: cuBLASLt, FP32 accumulate.  E4M3: torch._scaled_mm (cuBLASLt,
FP32 accumulate).  bench.py imports measure(); run as a script it prints JSON.
"""
import json
import time

import torch


def _bench(fn, flops, n_burst=10, sustain_s=3.0):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(n_burst):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = max(1, int(sustain_s / best))
    s.record()
    for _ in range(n):
        fn()
    e.record()
    e.synchronize()
    sus = s.elapsed_time(e) / 1e3 / n
    return flops / best / 1e12, flops / sus / 1e12


def measure(sustain_s=2.0, N=8192, dev="cuda", hbm=False):
    """{class}_tflops (burst) and {class}_tflops_sustained for fp64, fp32, fp16, bf16, e4m3"""
    old = (torch.backends.cuda.matmul.allow_tf32,
           torch.backends.cuda.matmul.allow_fp16_reduced_precision_reduction,
           torch.backends.cuda.matmul.allow_bf16_reduced_precision_reduction)
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cuda.matmul.allow_fp16_reduced_precision_reduction = False
    torch.backends.cuda.matmul.allow_bf16_reduced_precision_reduction = False
    fl = 2.0 * N ** 3
    out = {"method": f"library GEMM {N}^3: best of 10 (burst) and back to back for {sustain_s} s (sustained); "
                     "fp64 cuBLAS DGEMM, fp32 cuBLAS SGEMM (TF32 off), fp16/bf16 cuBLASLt, "
                     "e4m3 torch._scaled_mm (cuBLASLt), FP32 accumulate"}
    try:
        for name, dt in [("fp64", torch.float64), ("fp32", torch.float32), ("fp16", torch.float16),
                         ("bf16", torch.bfloat16)]:
            a = torch.randn(N, N, device=dev, dtype=torch.float32).to(dt)
            b = torch.randn(N, N, device=dev, dtype=torch.float32).to(dt)
            c = torch.empty(N, N, device=dev, dtype=dt)
            burst, sus = _bench(lambda: torch.matmul(a, b, out=c), fl, sustain_s=sustain_s)
            out[name + "_tflops"] = round(burst, 1)
            out[name + "_tflops_sustained"] = round(sus, 1)
            del a, b, c
        try:
            a = torch.randn(N, N, device=dev).to(torch.float8_e4m3fn)
            b = torch.randn(N, N, device=dev).to(torch.float8_e4m3fn).t()
            one = torch.ones((), device=dev)
            burst, sus = _bench(lambda: torch._scaled_mm(a, b, scale_a=one, scale_b=one, out_dtype=torch.bfloat16),
                                fl, sustain_s=sustain_s)
            out["e4m3_tflops"] = round(burst, 1)
            out["e4m3_tflops_sustained"] = round(sus, 1)
            del a, b
        except Exception as ex:  # noqa
            out["e4m3_error"] = repr(ex)[:200]
        try:   # MXFP4 (E2M1 x E2M1, E8M0 scale per 32 K) through torch._scaled_mm (cuBLASLt block scaling)
            a = torch.randint(0, 256, (N, N // 2), device=dev, dtype=torch.uint8).view(torch.float4_e2m1fn_x2)
            b = torch.randint(0, 256, (N, N // 2), device=dev, dtype=torch.uint8).view(torch.float4_e2m1fn_x2)
            sa = torch.full((N, N // 32), 127, device=dev, dtype=torch.uint8).view(torch.float8_e8m0fnu)
            sb = torch.full((N, N // 32), 127, device=dev, dtype=torch.uint8).view(torch.float8_e8m0fnu)
            burst, sus = _bench(lambda: torch._scaled_mm(a, b.t(), scale_a=sa, scale_b=sb, out_dtype=torch.bfloat16),
                                fl, sustain_s=sustain_s)
            out["mxfp4_tflops"] = round(burst, 1)
            out["mxfp4_tflops_sustained"] = round(sus, 1)
            del a, b, sa, sb
        except Exception as ex:  # noqa
            out["mxfp4_error"] = repr(ex)[:200]
        if hbm:
            x = torch.empty(1 << 30, device=dev, dtype=torch.bfloat16)
            y = torch.empty_like(x)
            burst, _ = _bench(lambda: y.copy_(x), 2.0 * x.numel() * 2, sustain_s=0.5)
            out["hbm_copy_gbs"] = round(burst * 1e3, 1)
            del x, y
    finally:
        (torch.backends.cuda.matmul.allow_tf32,
         torch.backends.cuda.matmul.allow_fp16_reduced_precision_reduction,
         torch.backends.cuda.matmul.allow_bf16_reduced_precision_reduction) = old
        torch.cuda.empty_cache()
    out["device"] = torch.cuda.get_device_name()
    out["when"] = time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())
    return out


if __name__ == "__main__":
    print(json.dumps(measure(sustain_s=3.0, hbm=True)))
