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
U32 = 2.0 ** -24
# a sub-FP32 C element may differ from the oracle's only where W_gpu and W_oracle straddle a
# rounding boundary of C's class; expected rate ~ |dW| / spacing <~ 0.5 % for FP16
MAX_FLIP_RATE = 0.02


def tile_bound(o, i, j, K):
    """SURVEY C6 / DESIGN.md 4: 1e-13 when the C tile and every pair folded into it are FP64,
    else 4 u32 sqrt(K) (relative Frobenius, per C tile)"""
    allfp64 = o["ccode"][i, j] == 0 and (o["acode"][i, :] == 0).all() and (o["bcode"][:, j] == 0).all()
    return 1e-13 if allfp64 else 4 * U32 * np.sqrt(K)


def gpu_w_tile(g, i, j, code, nb):
    raw, _ = g.tile("W", i, j, code)
    return raw.view(np.float64 if code == 0 else np.float32).astype(np.float64).reshape(nb, nb)


def w_and_finalize_parity(g, o, Cg, nb, K, bitwise=False):
    """Per C tile: (1) the GPU's W accumulator vs the oracle's exported W -- bitwise on the
    SIMT path, else within tile_bound; (2) the GPU's packed C_out, its scale and the user C
    tile are EXACTLY the oracle's finalize (O9) of the GPU's own W.  Returns the worst
    relative W error."""
    worst = 0.0
    mt, nt = o["ccode"].shape
    for i in range(mt):
        for j in range(nt):
            code = int(o["ccode"][i, j])
            sl = (slice(i * nb, (i + 1) * nb), slice(j * nb, (j + 1) * nb))
            Wg, Wo = gpu_w_tile(g, i, j, code, nb), o["W"][sl]
            if bitwise:
                assert np.array_equal(Wg, Wo), ("W", i, j)
            else:
                den = np.linalg.norm(Wo)
                rel = np.linalg.norm(Wg - Wo) / den if den > 0 else float(np.abs(Wg).max())
                assert rel <= tile_bound(o, i, j, K), ("W", i, j, code, rel)
                worst = max(worst, rel)
            pay, user, e = oracle.finalize(Wg, code)
            got, sc = g.tile("C", i, j, code)
            assert sc == e, ("C scale", i, j, sc, e)
            assert np.array_equal(got, pay.view(np.uint8)), ("C_out bytes", i, j)
            assert np.array_equal(Cg[sl], user), ("user C", i, j)
    return worst


def c_parity(Cg, Co, ccode, cscale, nb, K, allfp64):
    """User C vs the oracle's C per tile (DESIGN.md 4 / SURVEY C6).  Tiles stored in FP64 /
    FP32: relative Frobenius error <= 1e-13 (all-FP64 runs) or 4 u32 sqrt(K), per tile.
    Tiles stored below FP32 (class c, scale e): C = RN_c(W 2^e) 2^-e on both sides, so
    ||C_g - C_o|| <= ||C_g - W_g|| + ||W_g - W_o|| + ||W_o - C_o||
                 <= (4 u32 sqrt(K) + 2 u_c) ||C_o|| + nb eta_c 2^-e   (per tile),
    and the final RN may flip at most MAX_FLIP_RATE of the tile's elements.  (SURVEY C6's
    "<= 1 ulp of C's class per element" does not hold for an element whose W cancels to
    far below the tile's magnitude: there |dW| alone exceeds that element's ulp; DESIGN.md
    reading R29.  Each GPU C element is checked exactly against the finalize of the GPU's
    own W in w_and_finalize_parity.)
    Returns (ok, worst relative error of the FP64/FP32 tiles)."""
    bound = 1e-13 if allfp64 else 4 * U32 * np.sqrt(K)
    mt, nt = ccode.shape
    ok, worst = True, 0.0
    for i in range(mt):
        for j in range(nt):
            sl = (slice(i * nb, (i + 1) * nb), slice(j * nb, (j + 1) * nb))
            g, o = Cg[sl], Co[sl]
            c = int(ccode[i, j])
            den = np.linalg.norm(o)
            err = np.linalg.norm(g - o)
            if c <= 1:
                rel = err / den if den > 0 else float(np.abs(g).max())
                worst = max(worst, rel)
                ok = ok and rel <= bound
            else:
                if (g != o).mean() > MAX_FLIP_RATE:
                    ok = False
                lim = (bound + 2 * U_CLASS[c]) * (1 + 2 * U_CLASS[c]) * den + nb * ETA_CLASS[c] * 2.0 ** (-int(cscale[i, j]))
                if err > lim:
                    ok = False
    return ok, worst
