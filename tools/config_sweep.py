"""BASELINE.json config sweep on ONE B200 (dev/evidence tool, not the bench).

For each BASELINE config (and SURVEY 8(d)'s comparison runs) it synthesises the
workload on the GPU, runs plan + convert + execute through the C ABI, repeats
execute, and prints one JSON line per run with the realised mix, the
per-class device times and the precision-mix roofline
    T_roof = sum_c F_c / Peak_c      (Peak from MEASURED_PEAKS.json, bf16 burst;
                                      FP64 = DMMA 37.2, FP32 class = BF16 / 6)
Comparison runs:
  cfg2 all-FP64 (class_mask = FP64)            -- the paper's 100D:0S baseline
  cfg2 cuBLAS DGEMM (torch.matmul float64)     -- the library FP64 GEMM
  cfg4 explicit all-FP16 maps                  -- "pure FP16" of SURVEY 8(d)
usage: python tools/config_sweep.py [--only NAME] [--reps 3] > out.jsonl
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402  (Clocks sampler)
import gmp_inputs  # noqa: E402
from paper_2508_14848_b200 import api  # noqa: E402
from paper_2508_14848_b200 import binding as B  # noqa: E402

NAMES = ["FP64", "FP32", "FP16", "BF16", "E4M3", "E5M2", "MX4"]


def peaks():
    try:
        p = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        p = {"bf16_tflops": 1590.0}
    bf16 = p.get("bf16_tflops", 1590.0)
    # FP32 class: BF16x6 on tcgen05 (R32); MXFP4: 2 x E4M3 (nominal)
    return [37.22496, bf16 / 6.0, bf16, bf16, 2 * bf16, 2 * bf16, 4 * bf16]


def run(w, reps, mask=None, flags=0, explicit=None, label=None):
    dev = torch.device("cuda:0")
    A = api.synth(w.M, w.K, w.nb, w.a)
    Bm = api.synth(w.K, w.N, w.nb, w.b)
    C = api.synth(w.M, w.N, w.nb, w.c) if w.beta != 0 else None
    mt, nt, kt = w.M // w.nb, w.N // w.nb, w.K // w.nb
    maps = {}
    if explicit is not None:
        maps = dict(a_map=np.full((mt, kt), explicit, np.uint8), b_map=np.full((kt, nt), explicit, np.uint8),
                    c_map=np.full((mt, nt), explicit, np.uint8))
    desc = B.make_desc(w.M, w.N, w.K, w.nb, w.tol, w.alpha, w.beta,
                       w.class_mask if mask is None else mask, flags | B.GMP_FLAG_TIMING, **maps)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record()
    g = api.GemmMP(desc, A, Bm, C)
    ev[1].record()
    g.convert()
    ev[2].record()
    out = torch.empty(w.M, w.N, dtype=torch.float64, device=dev)
    g.execute(out)
    ev[3].record()
    torch.cuda.synchronize()
    times, cms = [], []
    clk = bench.Clocks(torch.cuda.current_device())
    clk.start()
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); g.execute(out); e.record(); e.synchronize()
        times.append(s.elapsed_time(e))
        cms.append(g.stats()["class_ms"])
    clocks = clk.stop()
    st = g.stats()
    best = min(times)
    pk = peaks()
    t_roof = sum(st["flops"][c] / (pk[c] * 1e12) for c in range(len(NAMES))) * 1e3
    cls_ms = [min(x[c] for x in cms) for c in range(len(NAMES))]
    res = dict(run=label or w.name, M=w.M, N=w.N, K=w.K, nb=w.nb, tol=w.tol,
               plan_ms=ev[0].elapsed_time(ev[1]), convert_ms=ev[1].elapsed_time(ev[2]),
               exec_ms_best=best, exec_ms=times, tflops_exec=w.flops / best / 1e9,
               tflops_step=w.flops / (best + ev[0].elapsed_time(ev[2])) / 1e9,
               pairs={NAMES[c]: st["pairs"][c] for c in range(len(NAMES))},
               tiles_a={NAMES[c]: st["tiles_a"][c] for c in range(len(NAMES))},
               tiles_c={NAMES[c]: st["tiles_c"][c] for c in range(len(NAMES))},
               class_ms={NAMES[c]: round(cls_ms[c], 3) for c in range(len(NAMES)) if st["pairs"][c]},
               class_tflops={NAMES[c]: round(st["flops"][c] / (cls_ms[c] * 1e-3) / 1e12, 1)
                             for c in range(len(NAMES)) if st["pairs"][c] and cls_ms[c] > 0},
               t_roof_ms=t_roof, roof_frac_exec=t_roof / best,
               peaks_tflops={NAMES[c]: round(pk[c], 1) for c in range(len(NAMES))}, clocks=clocks)
    g.close()
    del A, Bm, C, out
    torch.cuda.empty_cache()
    return res


def cublas_dgemm(n, reps):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    c = a @ b
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); torch.matmul(a, b, out=c); e.record(); e.synchronize()
        ts.append(s.elapsed_time(e))
    best = min(ts)
    del a, b, c
    torch.cuda.empty_cache()
    return dict(run=f"cublas_dgemm_{n}", exec_ms_best=best, exec_ms=ts, tflops_exec=2.0 * n ** 3 / best / 1e9)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default=None)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    W = gmp_inputs.workload
    plan = [
        ("cfg1", lambda: run(W(1), a.reps)),
        ("cfg2", lambda: run(W(2), a.reps)),
        ("cfg2_allfp64", lambda: run(W(2), a.reps, mask=1, label="cfg2_all_FP64 (class_mask=FP64)")),
        ("cfg2_cublas", lambda: cublas_dgemm(16384, a.reps)),
        ("cfg3", lambda: run(W(3), a.reps)),
        ("cfg4", lambda: run(W(4), a.reps)),
        ("cfg4_allfp16", lambda: run(W(4), a.reps, explicit=2, label="cfg4_explicit_all_FP16")),
        ("cfg4_mx4", lambda: run(W(4, "mx4"), a.reps)),
        ("cfg5_uniform", lambda: run(W(5, "uniform"), a.reps)),
        ("cfg5_uniform_1e-2", lambda: run(W(5, "uniform_1e-2"), a.reps)),
        ("cfg5_E8", lambda: run(W(5, "E8"), a.reps)),
        ("cfg5_E16", lambda: run(W(5, "E16"), a.reps)),
        ("cfg5_E32", lambda: run(W(5, "E32"), a.reps)),
        ("cfg5_E48", lambda: run(W(5, "E48"), a.reps)),
    ]
    for name, fn in plan:
        if a.only and not name.startswith(a.only):
            continue
        t = time.time()
        try:
            r = fn()
        except Exception as e:  # report and continue with the next config
            r = dict(run=name, error=str(e)[:300])
        r["wall_s"] = round(time.time() - t, 1)
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
