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
        allfp64 = (o["acode"][i, :] == 0).all() and (o["bcode"][:, j] == 0).all() and o["ccode"][i, j] == 0
        assert rel <= (1e-13 if allfp64 else 4 * U32 * np.sqrt(w.K)), (t, rel)
        ref = w.alpha * (Ah[sl[0], :] @ Bh[:, sl[1]]) + w.beta * Ch[sl]
        # per-tile tolerance check against the global normaliser (sampled form of the tol metric)
        den = abs(w.alpha) * np.linalg.norm(Ah) * np.linalg.norm(Bh) + abs(w.beta) * np.linalg.norm(Ch)
        assert np.linalg.norm(cg - ref) / den <= w.tol
    g.close()
