"""Measure per-class library GEMM peaks on one B200 (roofline denominators).

Same method as the driver's MEASURED_PEAKS.json: library GEMM 8192^3, best of
10 with CUDA events (burst), plus a ~3 s back-to-back loop (sustained).
FP64: cuBLAS DGEMM. FP32: cuBLAS SGEMM with TF32 disabled. FP16/BF16: cuBLASLt.
E4M3: torch._scaled_mm (cuBLASLt, FP32 accumulate). Writes JSON to stdout.
"""
import json, time, sys
import torch

def bench(fn, flops, n_burst=10, sustain_s=3.0):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(n_burst):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); e.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    # sustained
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = max(1, int(sustain_s / best))
    s.record()
    for _ in range(n):
        fn()
    e.record(); e.synchronize()
    sus = s.elapsed_time(e) / 1e3 / n
    return flops / best / 1e12, flops / sus / 1e12

def main():
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cuda.matmul.allow_fp16_reduced_precision_reduction = False
    torch.backends.cuda.matmul.allow_bf16_reduced_precision_reduction = False
    N = 8192
    fl = 2.0 * N ** 3
    out = {}
    dev = "cuda"
    for name, dt in [("fp64", torch.float64), ("fp32", torch.float32), ("fp16", torch.float16), ("bf16", torch.bfloat16)]:
        a = torch.randn(N, N, device=dev, dtype=torch.float32).to(dt)
        b = torch.randn(N, N, device=dev, dtype=torch.float32).to(dt)
        c = torch.empty(N, N, device=dev, dtype=dt)
        burst, sus = bench(lambda: torch.matmul(a, b, out=c), fl, sustain_s=3.0 if name not in ("fp64", "fp32") else 2.0)
        out[name + "_tflops"] = round(burst, 1)
        out[name + "_tflops_sustained"] = round(sus, 1)
        del a, b, c
    try:
        a = torch.randn(N, N, device=dev).to(torch.float8_e4m3fn)
        b = torch.randn(N, N, device=dev).to(torch.float8_e4m3fn).t()
        one = torch.ones((), device=dev)
        burst, sus = bench(lambda: torch._scaled_mm(a, b, scale_a=one, scale_b=one, out_dtype=torch.bfloat16), fl)
        out["e4m3_tflops"] = round(burst, 1)
        out["e4m3_tflops_sustained"] = round(sus, 1)
    except Exception as ex:  # noqa
        out["e4m3_error"] = repr(ex)[:200]
    # HBM copy
    x = torch.empty(1 << 30, device=dev, dtype=torch.bfloat16)
    y = torch.empty_like(x)
    burst, _ = bench(lambda: y.copy_(x), 2.0 * x.numel() * 2 / 1e3 * 1e3, sustain_s=0.5)
    out["hbm_copy_gbs"] = round(burst * 1e3, 1)
    out["device"] = torch.cuda.get_device_name()
    out["when"] = time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())
    print(json.dumps(out))

if __name__ == "__main__":
    main()
