"""Per-tile diagnostic of the product-path C vs the oracle (cfg1): W error, C error, flips."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "..", "tests"))
import numpy as np
import gmp_inputs
from gpu_harness import run_gpu, run_oracle, gpu_w_tile, U_CLASS, ETA_CLASS

w = gmp_inputs.workload(1)
A, Bm, C = w.matrices()
o = run_oracle(A, Bm, C, w.nb, w.tol, w.alpha, w.beta, w.class_mask)
g, (Cg,) = run_gpu(A, Bm, C, w.nb, w.tol, w.alpha, w.beta, w.class_mask)
nb = w.nb
mt, nt = o["ccode"].shape
for i in range(mt):
    for j in range(nt):
        c = int(o["ccode"][i, j]); e = int(o["cscale"][i, j])
        sl = (slice(i * nb, (i + 1) * nb), slice(j * nb, (j + 1) * nb))
        Wg, Wo = gpu_w_tile(g, i, j, c, nb), o["W"][sl]
        wrel = np.linalg.norm(Wg - Wo) / np.linalg.norm(Wo)
        cg, co = Cg[sl], o["C"][sl]
        crel = np.linalg.norm(cg - co) / np.linalg.norm(co)
        diff = cg != co
        step = 2 * U_CLASS[c] * np.maximum(np.abs(cg), np.abs(co)) + ETA_CLASS[c] * 2.0 ** (-e)
        big = (np.abs(cg - co)[diff] > step[diff]).sum()
        _, sg = g.tile("C", i, j, c)
        print(f"tile {i},{j} code {c} scale o={e} g={sg} Wrel {wrel:.3e} Crel {crel:.3e} flips {diff.mean():.4f} beyond-step {big}")
