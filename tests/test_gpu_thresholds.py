"""Near-threshold map fuzz on RANDOM (non-constant) tiles ("fuzzing
near thresholds"; VERDICT r1 "Next round" item 1).

For a chosen tile t and class k the tolerance is solved so that the criterion of O5,
    (delta_k (x) sqrt(S_t)) (+) nb eta_k 2^(-e-1)  <=  ((tol/4) (x) ||X||_F) / NT,
holds with the smallest binary64 tol (tol*), evaluated in the oracle's operation
order with Python's binary64 arithmetic; the maps are then computed at tol*, at the
binary64 predecessor of tol* (where t must fall back to a higher-precision class)
and at the successor.  The GPU's maps (and its exported per-tile S) must equal the
oracle's at all three.  Random tiles make S depend on the summation order, so a
GPU that summed in any other order than CNORM (O4) would show up here -- unlike
constant tiles, whose S is the same in every order."""
import math

import numpy as np
import pytest
import torch

import gmp_inputs
import oracle
from paper_2508_14848_b200 import api
from paper_2508_14848_b200 import binding as B

pytestmark = pytest.mark.gpu

ETA = [2.0 ** -1074, 2.0 ** -149, 2.0 ** -24, 2.0 ** -133, 2.0 ** -9, 2.0 ** -16]


def _lhs(k, S, mx, nb):
    e = oracle.scale_exp(mx, k)
    return oracle.delta(k, nb) * math.sqrt(S) + nb * math.ldexp(ETA[k], -e - 1)


def _rhs(tol, SX, ntiles):
    return ((tol / 4.0) * math.sqrt(SX)) / math.sqrt(ntiles)


def _solve_tol(lhs, SX, ntiles):
    """smallest binary64 tol with lhs <= rhs(tol)"""
    t = 4.0 * lhs * math.sqrt(ntiles) / math.sqrt(SX)
    while _rhs(t, SX, ntiles) < lhs:
        t = np.nextafter(t, np.inf)
    while _rhs(np.nextafter(t, 0.0), SX, ntiles) >= lhs:
        t = np.nextafter(t, 0.0)
    return float(t)


def _gpu_maps(A, Bm, nb, tol, mask):
    dev = torch.device("cuda:0")
    M, K = A.shape
    N = Bm.shape[1]
    desc = B.make_desc(M, N, K, nb, tol, 1.0, 0.0, mask)
    g = api.GemmMP(desc, torch.from_numpy(A).to(dev), torch.from_numpy(Bm).to(dev), None)
    m = g.maps()
    S, _, _ = g.tile_stats("A")
    g.close()
    return m, S


CASES = [(128, 1, 0), (128, 2, 1), (128, 3, 2), (128, 4, 3), (1024, 1, 4), (1024, 2, 5), (1024, 3, 6),
         (2048, 1, 7), (2048, 3, 8), (2048, 4, 9)]


@pytest.mark.parametrize("nb,k,seed", CASES)
def test_map_at_random_tile_threshold(nb, k, seed):
    mask = 0b011111
    w = gmp_inputs.small_workload(3 * nb, nb, 2 * nb, nb, 1e-3, mode="random", E=6, beta=0.0,
                                  class_mask=mask, seed=300 + seed)
    A, Bm, _ = w.matrices()
    S, Mx, _ = oracle.tile_stats(A, nb)
    Sf = S.ravel()
    SX = 0.0
    for v in Sf:                      # O5: sequential row-major sum
        SX = SX + float(v)
    t = int(np.random.default_rng(seed).integers(Sf.size))
    lhs = _lhs(k, float(Sf[t]), float(Mx.ravel()[t]), nb)
    tstar = _solve_tol(lhs, SX, Sf.size)
    seen = set()
    for tol in (tstar, float(np.nextafter(tstar, 0.0)), float(np.nextafter(tstar, np.inf))):
        o = oracle.gemm_mp(A, Bm, None, nb, tol, 1.0, 0.0, mask, ctiles=[], want_w=False)
        m, Sg = _gpu_maps(A, Bm, nb, tol, mask)
        assert np.array_equal(Sg.view(np.uint64), S.view(np.uint64))
        for key in ("acode", "bcode", "ccode"):
            assert np.array_equal(m[key], o[key]), (nb, k, tol, key)
        seen.add(int(o["acode"].ravel()[t]))
    # the chosen tile really sits on the threshold: class k at tol*, a higher-precision one just below
    o_at = oracle.gemm_mp(A, Bm, None, nb, tstar, 1.0, 0.0, mask, ctiles=[], want_w=False)
    o_below = oracle.gemm_mp(A, Bm, None, nb, float(np.nextafter(tstar, 0.0)), 1.0, 0.0, mask, ctiles=[],
                             want_w=False)
    assert o_at["acode"].ravel()[t] == k, (o_at["acode"], k)
    assert o_below["acode"].ravel()[t] < k
    assert len(seen) == 2
