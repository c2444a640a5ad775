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


U_CLASS = [2.0 ** -53, 2.0 ** -24, 2.0 ** -11, 2.0 ** -8, 2.0 ** -4, 2.0 ** -3]
ETA_CLASS = [2.0 ** -1074, 2.0 ** -149, 2.0 ** -24, 2.0 ** -133, 2.0 ** -9, 2.0 ** -16]


def c_parity(Cg, Co, ccode, cscale, nb, K, allfp64):
    """DESIGN.md section 4 / SURVEY C6: W-level agreement within 1e-13 (all-FP64) or
    4 u32 sqrt(K) (relative Frobenius) on tiles stored in FP64/FP32; tiles stored
    below FP32 may in addition differ by the final rounding into C's class: at most
    one step of that class's grid per element.  Returns (ok, worst relative error)."""
    bound = 1e-13 if allfp64 else 4 * 2.0 ** -24 * np.sqrt(K)
    mt, nt = ccode.shape
    num = den = 0.0
    ok = True
    for i in range(mt):
        for j in range(nt):
            sl = (slice(i * nb, (i + 1) * nb), slice(j * nb, (j + 1) * nb))
            g, o = Cg[sl], Co[sl]
            c = int(ccode[i, j])
            if c <= 1:
                num += float(((g - o) ** 2).sum())
                den += float((o ** 2).sum())
            else:
                # one class step at this magnitude + the W-level tolerance
                step = 2 * U_CLASS[c] * np.maximum(np.abs(g), np.abs(o)) + ETA_CLASS[c] * 2.0 ** (-int(cscale[i, j]))
                w_tol = bound * np.linalg.norm(o) + 1e-300
                excess = np.maximum(np.abs(g - o) - step, 0.0)
                if np.linalg.norm(excess) > w_tol:
                    ok = False
    rel = np.sqrt(num / den) if den > 0 else 0.0
    return ok and rel <= bound, rel
