"""The oracle's streaming driver (oracle.gemm_mp_synth: inputs generated tile by tile by
the O1 recipe, never materialised -- what makes full-size N = 65536 parity samples
possible) against the in-memory driver (oracle.gemm_mp on the materialised matrices of
the same recipe): maps, scales, tile statistics, the listed C tiles and their W
accumulators are bit-identical.  Both run the same O1-O9 code on the same binary64
tile values; the streaming form only changes where tiles are read from and computes
the independent tile-GEMMs of one C tile concurrently (folds stay in O9 order)."""
import numpy as np
import pytest

import gmp_inputs
import oracle


def _gen(r):
    return (r.seed, r.mode, r.E, r.s, r.tau)


@pytest.mark.parametrize("shape,nb,beta,mode,E,mask,seed", [
    ((384, 512, 640), 128, 0.0, "random", 30, 0b0011111, 5),
    ((512, 256, 1152), 128, 0.75, "graded", 18, 0b0001111, 6),
    ((256, 384, 2304), 128, 1.0, "random", 40, 0b1111111, 7),   # 18 K tiles: 3 SUMMA steps, MXFP4 on
])
def test_streaming_driver_matches_in_memory(shape, nb, beta, mode, E, mask, seed):
    M, N, K = shape
    w = gmp_inputs.small_workload(M, N, K, nb, 1e-3, mode=mode, E=E, beta=beta, class_mask=mask, seed=seed)
    A, Bm, C = w.matrices()
    mt, nt = M // nb, N // nb
    tiles = sorted({0, mt * nt - 1, (mt // 2) * nt + nt // 3})
    o = oracle.gemm_mp(A, Bm, C, nb, w.tol, w.alpha, w.beta, w.class_mask, ctiles=tiles)
    s = oracle.gemm_mp_synth(M, N, K, nb, w.tol, _gen(w.a), _gen(w.b), _gen(w.c), tiles,
                             alpha=w.alpha, beta=w.beta, class_mask=w.class_mask)
    assert o["rc"] == 0 and s["rc"] == 0
    for k in ("acode", "bcode", "ccode", "ascale5", "bscale5"):
        assert np.array_equal(o[k], s[k]), k
    for k in ("SA", "MA", "SB", "MB", "SC", "MC"):
        assert np.array_equal(o[k].view(np.uint64), s[k].view(np.uint64)), k
    for q, t in enumerate(tiles):
        i, j = divmod(t, nt)
        sl = (slice(i * nb, (i + 1) * nb), slice(j * nb, (j + 1) * nb))
        assert np.array_equal(o["C"][sl], s["C"][q]), ("C", t)
        assert np.array_equal(o["W"][sl], s["W"][q]), ("W", t)
        assert o["cscale"][i, j] == s["cscale"][i, j] and o["cin_scale"][i, j] == s["cin_scale"][i, j]
