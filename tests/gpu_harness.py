"""Shared helpers for the -m gpu tests: run the CUDA path through the C ABI
and the oracle on the SAME seeded inputs (gmp_inputs), never feeding one from
the other."""
import numpy as np
import torch

import oracle
from paper_2508_14848_b200 import api
from paper_2508_14848_b200 import binding as B


def run_gpu(A, Bm, C, nb, tol, alpha, beta, mask, flags=0, maps=(None, None, None), reps=1):
    dev = torch.device("cuda:0")
    tA = torch.from_numpy(A).to(dev)
    tB = torch.from_numpy(Bm).to(dev)
    tC = torch.from_numpy(C).to(dev) if C is not None else None
    M, K = A.shape
    N = Bm.shape[1]
    desc = B.make_desc(M, N, K, nb, tol, alpha, beta, mask, flags, a_map=maps[0], b_map=maps[1], c_map=maps[2])
    g = api.GemmMP(desc, tA, tB, tC if beta != 0.0 else None)
    g.convert()
    outs = []
    for _ in range(reps):
        out = torch.full((M, N), np.nan, dtype=torch.float64, device=dev)
        g.execute(out)
        g.sync()
        outs.append(out.cpu().numpy())
    return g, outs


def run_oracle(A, Bm, C, nb, tol, alpha, beta, mask, maps=(None, None, None), ctiles=None):
    return oracle.gemm_mp(A, Bm, C, nb, tol, alpha, beta, mask, ctiles=ctiles, a_map=maps[0],
                          b_map=maps[1], c_map=maps[2])


def tol_metric(Cmp, A, Bm, C, alpha, beta):
    """||C - C_fp64||_F / (|a| ||A|| ||B|| + |b| ||C||), C_fp64 by cuBLAS DGEMM on the GPU."""
    dev = torch.device("cuda:0")
    ref = alpha * (torch.from_numpy(A).to(dev) @ torch.from_numpy(Bm).to(dev))
    if beta != 0.0:
        ref = ref + beta * torch.from_numpy(C).to(dev)
    num = torch.linalg.norm(torch.from_numpy(Cmp).to(dev) - ref).item()
    den = abs(alpha) * np.linalg.norm(A) * np.linalg.norm(Bm) + (abs(beta) * np.linalg.norm(C) if beta else 0.0)
    return num / den
