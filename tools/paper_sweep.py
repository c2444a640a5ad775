"""The paper's own experiment on B200: random exact-count
aD:bS FP64/FP32 maps, the Fig. 3 heatmaps
and the Fig. 4 methodology -- TFLOP/s per ratio and speedup relative to
100D:0S -- through the C ABI with explicit maps.

usage: python tools/paper_sweep.py [--n 16384] [--nb 1024] [--out gpurun_out/paper_sweep]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import gmp_inputs  # noqa: E402
from gmp_inputs import paper_maps as pm  # noqa: E402
from paper_2508_14848_b200 import api  # noqa: E402
from paper_2508_14848_b200 import binding as B  # noqa: E402

RATIOS = [100, 80, 50, 20, 0]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--nb", type=int, default=1024)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "paper_sweep"))
    a = ap.parse_args()
    os.makedirs(a.out, exist_ok=True)
    # Fig. 3 heatmaps: 102,400^2 matrix, nb = 1,024 -> 100 x 100 tiles
    for d in (80, 50, 20):
        m = pm.ratio_map(100, 100, d, 1000 + d)
        open(os.path.join(a.out, f"fig3_{d}D{100 - d}S.pgm"), "w").write(pm.heatmap_pgm(m))
        open(os.path.join(a.out, f"fig3_{d}D{100 - d}S.csv"), "w").write(pm.heatmap_csv(m))
    n, nb = a.n, a.nb
    w = gmp_inputs.small_workload(n, n, n, nb, 1e-6, mode="uniform", E=0, beta=1.0, seed=2000)
    dev = torch.device("cuda:0")
    A = api.synth(n, n, nb, w.a)
    Bm = api.synth(n, n, nb, w.b)
    C = api.synth(n, n, nb, w.c)
    out = torch.empty(n, n, dtype=torch.float64, device=dev)
    t = n // nb
    res = {}
    for flags, tag in [(0, "fp32_tensor_bf16x6"), (B.GMP_FLAG_FP32_X9, "fp32_tensor_bf16x9"),
                       (B.GMP_FLAG_FP32_FFMA, "fp32_ffma2")]:
        rows = []
        for d in RATIOS:
            maps = pm.paper_maps(t, t, t, d, 5000 + d)
            desc = B.make_desc(n, n, n, nb, 1e-6, 1.0, 1.0, 0b00011, flags | B.GMP_FLAG_TIMING,
                               a_map=maps[0], b_map=maps[1], c_map=maps[2])
            g = api.GemmMP(desc, A, Bm, C)
            g.convert()
            g.execute(out)
            torch.cuda.synchronize()
            best = 1e30
            for _ in range(a.reps):
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record(); g.execute(out); e.record(); e.synchronize()
                best = min(best, s.elapsed_time(e))
            st = g.stats()
            g.close()
            rows.append({"ratio": f"{d}D:{100 - d}S", "ms": best, "tflops": w.flops / best / 1e9,
                         "pairs": st["pairs"][:2], "class_ms": st["class_ms"][:2]})
        base = rows[0]["tflops"]
        for r in rows:
            r["speedup_vs_100D"] = r["tflops"] / base
        res[tag] = rows
    res["config"] = {"n": n, "nb": nb, "maps": "exact-count Fisher-Yates (SPEC.md:169-177)",
                     "note": "FP64/FP32 classes only, as in the paper (PAPER.md:148)"}
    txt = json.dumps(res, indent=1)
    open(os.path.join(a.out, "paper_sweep.json"), "w").write(txt)
    print(txt)


if __name__ == "__main__":
    main()
