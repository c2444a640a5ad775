"""Quick device timing of plan / convert / execute on one config (dev tool)."""
import argparse
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json
import time

import torch

import gmp_inputs
from paper_2508_14848_b200 import api
from paper_2508_14848_b200 import binding as B


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, default=2)
    ap.add_argument("--variant", default=None)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--flags", type=int, default=0)
    ap.add_argument("--mask", type=int, default=None)
    ap.add_argument("--size", type=int, default=0, help="override M=N=K (keeps the config's recipe)")
    a = ap.parse_args()
    w = gmp_inputs.workload(a.cfg, a.variant)
    if a.size:
        import dataclasses
        w = dataclasses.replace(w, M=a.size, N=a.size, K=a.size, name=w.name + f"_size{a.size}")
    dev = torch.device("cuda:0")
    t0 = time.time()
    A = api.synth(w.M, w.K, w.nb, w.a)
    Bm = api.synth(w.K, w.N, w.nb, w.b)
    C = api.synth(w.M, w.N, w.nb, w.c) if w.beta != 0 else None
    torch.cuda.synchronize()
    mask = w.class_mask if a.mask is None else a.mask
    desc = B.make_desc(w.M, w.N, w.K, w.nb, w.tol, w.alpha, w.beta, mask, a.flags | B.GMP_FLAG_TIMING)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    ev[0].record()
    g = api.GemmMP(desc, A, Bm, C)
    ev[1].record()
    g.convert()
    ev[2].record()
    out = torch.empty(w.M, w.N, dtype=torch.float64, device=dev)
    g.execute(out)
    ev[3].record()
    torch.cuda.synchronize()
    times = []
    for _ in range(a.reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); g.execute(out); e.record(); e.synchronize()
        times.append(s.elapsed_time(e))
    st = g.stats()
    best = min(times) if times else ev[2].elapsed_time(ev[3])
    print(json.dumps(dict(cfg=w.name, plan_ms=ev[0].elapsed_time(ev[1]), convert_ms=ev[1].elapsed_time(ev[2]),
                          first_exec_ms=ev[2].elapsed_time(ev[3]), exec_ms=times, tflops=w.flops / best / 1e9,
                          tiles_a=st["tiles_a"], tiles_b=st["tiles_b"], tiles_c=st["tiles_c"],
                          pairs=st["pairs"], launches=st["launches_execute"], ws_gb=st["workspace_bytes"] / 1e9,
                          class_ms=[round(x, 3) for x in st["class_ms"]],
                          class_tflops=[round(st["flops"][c] / (st["class_ms"][c] * 1e-3) / 1e12, 1) if st["class_ms"][c] else 0
                                        for c in range(len(st["class_ms"]))])))


if __name__ == "__main__":
    main()
