"""Randomised parity sweep (48 fixed seeds, plus 24 with MXFP4 enabled): shapes of 1..6 tiles per dimension, nb in
{128, 256, 384, 512}, tolerances from 1e-12 to 0.5, every class mask with FP8 on or
off, alpha/beta signs and zeros, graded / random / uniform inputs.  Each case runs
the CUDA path twice through the C ABI -- the product kernels and the SIMT (bitwise)
kernels -- and the oracle once on the same seeded inputs: maps bit-exact, SIMT C
bit-exact, product C within the parity bound, tolerance met, and repeated
executes bitwise identical."""
import numpy as np
import pytest

import gmp_inputs
from gpu_harness import c_parity, run_gpu, run_oracle, tol_metric, w_and_finalize_parity
from paper_2508_14848_b200 import binding as B

pytestmark = pytest.mark.gpu


def _case(seed, masks=(0b000001, 0b000011, 0b001111, 0b011111, 0b111111, 0b101111, 0b000111), rng_base=1000):
    r = np.random.default_rng(rng_base + seed)
    nb = int(r.choice([128, 256, 384, 512]))
    mt, nt, kt = (int(x) for x in r.integers(1, 5 if nb >= 384 else 7, size=3))
    tol = float(10.0 ** r.uniform(-10, np.log10(0.5)))
    mask = int(r.choice(list(masks)))
    mode = str(r.choice(["graded", "random", "uniform"]))
    E = int(r.integers(0, 48))
    alpha = float(r.choice([1.0, -0.75, 2.0 ** -20, 3.0]))
    beta = float(r.choice([0.0, 1.0, -0.5, 0.0]))
    w = gmp_inputs.small_workload(mt * nb, nt * nb, kt * nb, nb, tol, mode=mode, E=E, alpha=alpha, beta=beta,
                                  class_mask=mask, seed=50 + seed)
    return w


# MXFP4 enabled (class 6, NEXT-4): its own 24 seeds (tolerances up to 0.5 put many tiles there)
MX_MASKS = (0b1111111, 0b1011111, 0b1000001, 0b1001111, 0b1000011)


@pytest.mark.parametrize("seed", list(range(48)) + [f"mx{k}" for k in range(24)])
def test_fuzz_parity(seed):
    w = _case(int(seed[2:]), MX_MASKS, 5000) if isinstance(seed, str) else _case(seed)
    A, Bm, C = w.matrices()
    Cin = C if w.beta != 0.0 else None
    o = run_oracle(A, Bm, Cin, w.nb, w.tol, w.alpha, w.beta, w.class_mask)
    assert o["rc"] == 0
    g, (Cg, Cg2) = run_gpu(A, Bm, Cin, w.nb, w.tol, w.alpha, w.beta, w.class_mask, reps=2)
    gs, (Cs,) = run_gpu(A, Bm, Cin, w.nb, w.tol, w.alpha, w.beta, w.class_mask, flags=B.GMP_FLAG_SIMT_ONLY)
    m = g.maps()
    for k in ("acode", "bcode", "ccode"):
        assert np.array_equal(m[k], o[k]), (seed, k)
    assert np.array_equal(Cs, o["C"]), seed
    assert np.array_equal(Cg, Cg2), seed
    allfp64 = (o["acode"] == 0).all() and (o["bcode"] == 0).all() and (o["ccode"] == 0).all()
    ok, rel = c_parity(Cg, o["C"], o["ccode"], o["cscale"], w.nb, w.K, allfp64)
    assert ok, (seed, rel)
    assert tol_metric(Cg, A, Bm, Cin, w.alpha, w.beta) <= w.tol, seed
    # S1 export bitwise (CNORM order), W per tile and the exact finalize of the GPU's W
    for which, So in (("A", o["SA"]), ("B", o["SB"])):
        S, _, _ = g.tile_stats(which)
        assert np.array_equal(S.view(np.uint64), So.view(np.uint64)), (seed, which)
    w_and_finalize_parity(g, o, Cg, w.nb, w.K)
    w_and_finalize_parity(gs, o, Cs, w.nb, w.K, bitwise=True)
