"""Full-size parity at the bench workload (BASELINE configs[1] = cfg2, N=16384,
nb=1024, tol 1e-8), in the launch configuration bench.py times: the GPU path
runs the whole GEMM; the oracle recomputes the complete maps (all tiles of A,
B, C) and a sample of C tiles one by one.  Maps bit-exact, sampled packed
tiles bit-exact, sampled C tiles within the parity bound, tolerance met on the
sampled tiles against a binary64 reference computed on the host."""
import numpy as np
import pytest
import torch

import gmp_inputs
import oracle
from gpu_harness import gpu_w_tile, tile_bound
from paper_2508_14848_b200 import api
from paper_2508_14848_b200 import binding as B

pytestmark = pytest.mark.gpu

U32 = 2.0 ** -24


def test_cfg2_fullsize_sampled():
    w = gmp_inputs.workload(2)
    nb = w.nb
    mt, nt, kt = w.M // nb, w.N // nb, w.K // nb
    dev = torch.device("cuda:0")
    A = api.synth(w.M, w.K, nb, w.a, device=dev)
    Bm = api.synth(w.K, w.N, nb, w.b, device=dev)
    C = api.synth(w.M, w.N, nb, w.c, device=dev)
    desc = B.make_desc(w.M, w.N, w.K, nb, w.tol, w.alpha, w.beta, w.class_mask)
    g = api.GemmMP(desc, A, Bm, C)
    g.convert()
    out = torch.empty(w.M, w.N, dtype=torch.float64, device=dev)
    g.execute(out)
    g.sync()
    gm = g.maps()
    # oracle inputs come from the oracle's own generator (never from the GPU)
    Ah = oracle.synth_block(w.M, w.K, nb, w.a.seed, 2, w.a.E, w.a.s, w.a.tau)
    Bh = oracle.synth_block(w.K, w.N, nb, w.b.seed, 2, w.b.E, w.b.s, w.b.tau)
    Ch = oracle.synth_block(w.M, w.N, nb, w.c.seed, 2, w.c.E, w.c.s, w.c.tau)
    rng = np.random.default_rng(2)
    sample = sorted(set(int(x) for x in rng.choice(mt * nt, size=4, replace=False)) | {0, mt * nt - 1})
    o = oracle.gemm_mp(Ah, Bh, Ch, nb, w.tol, w.alpha, w.beta, w.class_mask, ctiles=sample)
    assert o["rc"] == 0
    for k in ["acode", "bcode", "ccode"]:
        assert np.array_equal(gm[k], o[k]), k
    # S1 export: the canonical sums of squares of ALL tiles of A, B and C, bitwise
    for which, So, Mo in (("A", o["SA"], o["MA"]), ("B", o["SB"], o["MB"]), ("C", o["SC"], o["MC"])):
        S, M, F = g.tile_stats(which)
        assert np.array_equal(S.view(np.uint64), So.view(np.uint64)), which
        assert np.array_equal(M, Mo) and F.all(), which
    # packed bytes of a few stored and shadow tiles
    for (ti, tj) in [(0, 0), (3, 7), (mt - 1, kt - 1)]:
        code = int(o["acode"][ti, tj])
        got, sc = g.tile("A", ti, tj, code)
        ref = oracle.pack_tile(Ah[ti * nb:(ti + 1) * nb, tj * nb:(tj + 1) * nb], code,
                               int(o["ascale5"][ti, tj, code]), role="A")
        assert sc == o["ascale5"][ti, tj, code]
        assert np.array_equal(got, ref.view(np.uint8))
    Cg = out.cpu().numpy()
    for t in sample:
        i, j = divmod(t, nt)
        sl = (slice(i * nb, (i + 1) * nb), slice(j * nb, (j + 1) * nb))
        co, cg = o["C"][sl], Cg[sl]
        rel = np.linalg.norm(cg - co) / np.linalg.norm(co)
        assert rel <= tile_bound(o, i, j, w.K), (t, rel)
        # W accumulator per sampled tile, and C_out = the exact finalize of the GPU's W
        code = int(o["ccode"][i, j])
        Wg = gpu_w_tile(g, i, j, code, nb)
        relw = np.linalg.norm(Wg - o["W"][sl]) / np.linalg.norm(o["W"][sl])
        assert relw <= tile_bound(o, i, j, w.K), (t, relw)
        pay, user, e = oracle.finalize(Wg, code)
        got, sc = g.tile("C", i, j, code)
        assert sc == e and np.array_equal(got, pay.view(np.uint8)) and np.array_equal(cg, user), t
        ref = w.alpha * (Ah[sl[0], :] @ Bh[:, sl[1]]) + w.beta * Ch[sl]
        # per-tile tolerance check against the global normaliser (sampled form of the tol metric)
        den = abs(w.alpha) * np.linalg.norm(Ah) * np.linalg.norm(Bh) + abs(w.beta) * np.linalg.norm(Ch)
        assert np.linalg.norm(cg - ref) / den <= w.tol
    g.close()


@pytest.mark.parametrize("cfg", [3, 4])
def test_n65536_fullsize_properties(cfg):
    """BASELINE configs[2]/[3] (N=65536, nb=2048) at full size on one GPU, as bench.py
    --config 3/4 runs them.  The oracle cannot redo a 65536^3 GEMM, so properties
    that hold at any size are checked: (1) every stored scale is the oracle's scale
    definition (O3) of the tile's maxabs; (2) sampled tiles satisfy the criterion for
    their class and fail it for the next-lower-precision enabled class (O5, norms in
    binary64 by torch, a 1e-9 band around the threshold is skipped); (3) two sampled
    row panels of C meet the tolerance against a cuBLAS DGEMM of those panels, with
    the global normaliser; (4) repeated executes are bitwise identical; (5) the
    oracle's streaming driver (inputs generated tile by tile, oracle.gemm_mp_synth)
    computes the maps of all 2048 A/B tiles and one whole C tile (32 tile-GEMMs of
    2048^3 in its emulated class arithmetic, O9 fold order): maps and scales bitwise,
    the GPU's W and C tiles within the parity bound, C_out = the exact finalize of the
    GPU's W."""
    w = gmp_inputs.workload(cfg)
    nb = w.nb
    mt, nt, kt = w.M // nb, w.N // nb, w.K // nb
    dev = torch.device("cuda:0")
    torch.cuda.empty_cache()
    A = api.synth(w.M, w.K, nb, w.a, device=dev)
    Bm = api.synth(w.K, w.N, nb, w.b, device=dev)
    desc = B.make_desc(w.M, w.N, w.K, nb, w.tol, w.alpha, w.beta, w.class_mask)
    g = api.GemmMP(desc, A, Bm, None)
    g.convert()
    out = torch.empty(w.M, w.N, dtype=torch.float64, device=dev)
    g.execute(out)
    g.sync()
    m = g.maps()
    st = g.stats()
    assert sum(st["pairs"]) == mt * nt * kt
    enabled = {c for c in range(7) if (w.class_mask | 1) >> c & 1}
    assert set(np.unique(m["acode"])) <= enabled and set(np.unique(m["bcode"])) <= enabled
    rng = np.random.default_rng(cfg)
    tiles = [(int(rng.integers(mt)), int(rng.integers(kt))) for _ in range(12)]
    def sumsq(X):   # chunked: no full-size temporaries next to a 150 GB working set
        return sum(float((X[r:r + nb] * X[r:r + nb]).sum()) for r in range(0, X.shape[0], nb))

    SX = sumsq(A)
    rhs = (w.tol / 4.0) * np.sqrt(SX) / np.sqrt(mt * kt)
    u = [2.0 ** -53, 2.0 ** -24, 2.0 ** -11, 2.0 ** -8, 2.0 ** -4, 2.0 ** -3]
    eta = [2.0 ** -1074, 2.0 ** -149, 2.0 ** -24, 2.0 ** -133, 2.0 ** -9, 2.0 ** -16]
    ladder = [c for c in (5, 4, 3, 2, 1) if c in enabled]

    def lhs(k, S, mx):
        e = oracle.scale_exp(mx, k)
        return (u[k] + np.sqrt(nb) * 2.0 ** -24) * np.sqrt(S) + nb * np.ldexp(eta[k], -e - 1)

    SA_gpu, MA_gpu, _ = g.tile_stats("A")
    for (ti, tl) in tiles[:4]:   # S1 at nb = 2048: CNORM of the oracle's own copy of the tile, bitwise
        th = oracle.synth_block(w.M, w.K, nb, w.a.seed, 2, w.a.E, w.a.s, w.a.tau, ti * nb, nb, tl * nb, nb)
        assert oracle.cnorm(th) == SA_gpu[ti, tl] and np.abs(th).max() == MA_gpu[ti, tl], (ti, tl)
    for (ti, tl) in tiles:
        t = A[ti * nb:(ti + 1) * nb, tl * nb:(tl + 1) * nb]
        mx = float(t.abs().max())
        S = float((t * t).sum())
        code = int(m["acode"][ti, tl])
        assert int(m["ascale"][ti, tl]) == oracle.scale_exp(mx, code)          # (1)
        if code != 0:                                                           # (2) eligible
            assert lhs(code, S, mx) <= rhs * (1 + 1e-9)
        for k in ladder:                                                        # lower classes rejected
            if k == code:
                break
            assert lhs(k, S, mx) >= rhs * (1 - 1e-9), (ti, tl, k, code)
    nA = np.sqrt(SX)
    nB = np.sqrt(sumsq(Bm))
    den = abs(w.alpha) * nA * nB
    for i in (0, mt - 1):                                                       # (3)
        rows = slice(i * nb, (i + 1) * nb)
        ref = w.alpha * (A[rows, :] @ Bm)
        err = float(torch.linalg.norm(out[rows, :] - ref))
        assert err / den <= w.tol, (i, err / den)
        del ref
    _oracle_tile_parity(g, w, out, mt, nt, cfg)   # (5) full-size parity against the oracle, one C tile
    panels = [slice(0, nb), slice((mt // 2) * nb, (mt // 2 + 1) * nb), slice((mt - 1) * nb, mt * nb)]
    first = [out[p].clone() for p in panels]
    g.execute(out)                                                              # (4)
    g.sync()
    assert all(torch.equal(f, out[p]) for f, p in zip(first, panels))
    g.close()
    del A, Bm, out, first
    torch.cuda.empty_cache()


def _oracle_tile_parity(g, w, out, mt, nt, cfg):
    from gpu_harness import gpu_w_tile, tile_bound
    nb = w.nb
    gen = lambda r: (r.seed, r.mode, r.E, r.s, r.tau)   # noqa: E731
    i, j = (mt - 2, 5) if cfg == 3 else (3, nt - 7)
    o = oracle.gemm_mp_synth(w.M, w.N, w.K, nb, w.tol, gen(w.a), gen(w.b), gen(w.c), [i * nt + j],
                             alpha=w.alpha, beta=w.beta, class_mask=w.class_mask)
    assert o["rc"] == 0
    gm = g.maps()
    for k in ("acode", "bcode", "ccode"):
        assert np.array_equal(gm[k], o[k]), k
    kt = o["acode"].shape[1]
    assert np.array_equal(gm["ascale"], o["ascale5"][np.arange(mt)[:, None], np.arange(kt)[None, :], o["acode"]])
    assert np.array_equal(gm["bscale"], o["bscale5"][np.arange(kt)[:, None], np.arange(nt)[None, :], o["bcode"]])
    code = int(o["ccode"][i, j])
    Wg = gpu_w_tile(g, i, j, code, nb)
    Wo = o["W"][0]
    bound = tile_bound(o, i, j, w.K)
    relw = np.linalg.norm(Wg - Wo) / np.linalg.norm(Wo)
    assert relw <= bound, relw
    cg = out[i * nb:(i + 1) * nb, j * nb:(j + 1) * nb].cpu().numpy()
    rel = np.linalg.norm(cg - o["C"][0]) / np.linalg.norm(o["C"][0])
    assert rel <= bound, rel
    pay, user, e = oracle.finalize(Wg, code)
    got, sc = g.tile("C", i, j, code)
    assert sc == e and np.array_equal(got, pay.view(np.uint8)) and np.array_equal(cg, user)
