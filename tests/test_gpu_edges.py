"""Edge cases and error paths of the CUDA path (through the C ABI)."""
import numpy as np
import pytest
import torch

import gmp_inputs
import oracle
from gpu_harness import c_parity, run_gpu, run_oracle
from paper_2508_14848_b200 import api
from paper_2508_14848_b200 import binding as B

pytestmark = pytest.mark.gpu


def test_generator_bitwise_vs_numpy():
    for (rows, cols, nb, P, Q, p, q, mode) in [(512, 384, 128, 1, 1, 0, 0, "graded"),
                                               (1024, 768, 128, 2, 3, 1, 2, "random"),
                                               (640, 640, 128, 2, 2, 0, 1, "uniform")]:
        rec = gmp_inputs.MatrixRecipe(99, mode, 17, -2)
        t = api.synth(rows, cols, nb, rec, P, Q, p, q).cpu().numpy()
        full = gmp_inputs.synth_block(rows, cols, nb, rec.seed, mode, rec.E, rec.s, rec.tau)
        ti = np.arange(p, rows // nb, P)
        tj = np.arange(q, cols // nb, Q)
        rr = (ti[:, None] * nb + np.arange(nb)[None, :]).ravel()
        cc = (tj[:, None] * nb + np.arange(nb)[None, :]).ravel()
        assert np.array_equal(t, full[np.ix_(rr, cc)])


def test_nonfinite_input_is_an_error():
    A = np.ones((256, 256)); A[3, 200] = np.inf
    with pytest.raises(B.GmpError) as e:
        run_gpu(A, np.ones((256, 256)), None, 128, 1e-6, 1.0, 0.0, 0b01111)
    assert "NONFINITE" in str(e.value)


def test_nan_in_c_only_matters_if_beta_nonzero():
    A = np.ones((256, 256)); Bm = np.ones((256, 256)); C = np.zeros((256, 256)); C[0, 0] = np.nan
    g, (out,) = run_gpu(A, Bm, C, 128, 1e-6, 1.0, 0.0, 0b01111)
    assert np.array_equal(out, np.full((256, 256), 256.0))
    with pytest.raises(B.GmpError):
        run_gpu(A, Bm, C, 128, 1e-6, 1.0, 1.0, 0b01111)


def test_all_zero_inputs():
    z = np.zeros((256, 256))
    g, (out,) = run_gpu(z, z, z, 128, 1e-8, 1.0, 1.0, 0b01111)
    assert np.array_equal(out, z)
    m = g.maps()
    assert (m["acode"] == 3).all()  # first enabled ladder class (BF16), scale 0


def test_alpha_zero_beta_one_keeps_c():
    rng = np.random.default_rng(1)
    A, Bm, C = rng.standard_normal((3, 256, 256))
    g, (out,) = run_gpu(A, Bm, C, 128, 1e-6, 0.0, 1.0, 0b00001)
    assert np.array_equal(out, C)


def test_explicit_maps_match_oracle():
    w = gmp_inputs.small_workload(512, 512, 512, 128, 1e-6, beta=1.0, seed=3)
    A, Bm, C = w.matrices()
    rng = np.random.default_rng(0)
    maps = tuple(rng.integers(0, 2, (4, 4)).astype(np.uint8) for _ in range(3))
    o = run_oracle(A, Bm, C, 128, 1e-6, 1.0, 1.0, 0b00011, maps=maps)
    # FP32 class on the FP32 pipe (FFMA2): bitwise the oracle (FP64 class on DMMA: 1e-13)
    g, (out,) = run_gpu(A, Bm, C, 128, 1e-6, 1.0, 1.0, 0b00011, flags=B.GMP_FLAG_FP32_FFMA, maps=maps)
    m = g.maps()
    assert np.array_equal(m["acode"], maps[0]) and np.array_equal(m["ccode"], maps[2])
    assert np.linalg.norm(out - o["C"]) / np.linalg.norm(o["C"]) <= 1e-13
    g2, (out2,) = run_gpu(A, Bm, C, 128, 1e-6, 1.0, 1.0, 0b00011, flags=B.GMP_FLAG_SIMT_ONLY, maps=maps)
    assert np.array_equal(out2, o["C"])  # FP64 DFMA + FP32 FFMA2: bitwise
    # default: FP32 class on the tensor pipe (exact BF16x3 split, FP32 accumulation)
    g3, (out3,) = run_gpu(A, Bm, C, 128, 1e-6, 1.0, 1.0, 0b00011, maps=maps)
    assert np.linalg.norm(out3 - o["C"]) / np.linalg.norm(o["C"]) <= 4 * 2.0 ** -24 * np.sqrt(512)


@pytest.mark.parametrize("flags", [0, B.GMP_FLAG_SIMT_ONLY], ids=["tcgen05", "simt"])
def test_explicit_all_mxfp4_operands(flags):
    """NEXT-4: every A and B tile forced to MXFP4 (explicit maps, R19), C in FP32 / FP64:
    stored MXFP4 bytes (nibbles + block scales) bitwise, C bitwise vs the oracle on the SIMT
    kernel and within 4 u32 sqrt(K) on tcgen05 kind::mxf4.block_scale (3 x 2 x 4 tiles of 256,
    several K blocks, both W precisions)"""
    nb = 256
    w = gmp_inputs.small_workload(3 * nb, 2 * nb, 4 * nb, nb, 1e-2, mode="random", E=20, beta=0.5,
                                  class_mask=0b1111111, seed=61)
    A, Bm, C = w.matrices()
    maps = (np.full((3, 4), 6, np.uint8), np.full((4, 2), 6, np.uint8),
            np.array([[1, 0], [0, 1], [1, 1]], np.uint8))
    o = run_oracle(A, Bm, C, nb, w.tol, w.alpha, w.beta, w.class_mask, maps=maps)
    assert o["rc"] == 0 and (o["acode"] == 6).all() and (o["bcode"] == 6).all()
    g, (out,) = run_gpu(A, Bm, C, nb, w.tol, w.alpha, w.beta, w.class_mask, flags=flags, maps=maps)
    for which, X, codes, s5 in (("A", A, o["acode"], o["ascale5"]), ("B", Bm, o["bcode"], o["bscale5"])):
        for ti in range(codes.shape[0]):
            for tj in range(codes.shape[1]):
                tile = X[ti * nb:(ti + 1) * nb, tj * nb:(tj + 1) * nb]
                want = oracle.pack_tile(tile, 6, int(s5[ti, tj, 6]), role=which)
                got, sc = g.tile(which, ti, tj, 6)
                assert sc == s5[ti, tj, 6] and np.array_equal(got, want), (which, ti, tj)
    if flags & B.GMP_FLAG_SIMT_ONLY:
        assert np.array_equal(out, o["C"])
    else:
        ok, rel = c_parity(out, o["C"], o["ccode"], o["cscale"], nb, w.K, False)
        assert ok, rel


@pytest.mark.parametrize("nb,beta,seed", [(256, 0.0, 42), (128, 0.5, 44), (512, 1.0, 44)])
def test_merged_16bit_launch_bitwise_vs_per_class(nb, beta, seed):
    """the default plan runs the FP16 pairs of a step on the BF16 launch (per item BF16 then FP16,
    the O9 fold order); GMP_FLAG_SPLIT16 runs one launch per class: same pairs, same arithmetic,
    same order -> C bit-identical, fewer launches, and C within the parity bound of the oracle"""
    w = gmp_inputs.small_workload(3 * nb, 2 * nb, 4 * nb, nb, 1e-4, mode="random", E=28, beta=beta, seed=seed)
    A, Bm, C = w.matrices()
    g, (out,) = run_gpu(A, Bm, C, nb, w.tol, w.alpha, w.beta, w.class_mask)
    g2, (out2,) = run_gpu(A, Bm, C, nb, w.tol, w.alpha, w.beta, w.class_mask, flags=B.GMP_FLAG_SPLIT16)
    st, st2 = g.stats(), g2.stats()
    assert st["pairs"][2] > 0 and st["pairs"][3] > 0
    assert st["launches_execute"] < st2["launches_execute"]
    assert np.array_equal(out, out2)
    o = run_oracle(A, Bm, C, nb, w.tol, w.alpha, w.beta, w.class_mask)
    ok, rel = c_parity(out, o["C"], o["ccode"], o["cscale"], nb, w.K, False)
    assert ok, rel


def test_cnorm_sentinels_gpu_bitwise():
    """the O4 reduction order on the GPU map kernel: sentinel tiles whose sum of squares
    depends on the order (tests/test_oracle_map.py) give the oracle's S bit for bit"""
    from test_oracle_map import _cnorm_order, _sentinels
    for t in _sentinels(128):
        A = np.ascontiguousarray(t)
        g, _ = run_gpu(A, np.ones((128, 128)), None, 128, 1e-6, 1.0, 0.0, 0b01111)
        S, M, F = g.tile_stats("A")
        assert S[0, 0] == oracle.cnorm(A) == _cnorm_order(A)


def test_fp32_split_parts_are_exact():
    """The tensor-pipe FP32 class consumes x = x0 + x1 + x2 (three BF16 parts,
    K-major): the parts must reproduce every FP32 operand value exactly."""
    w = gmp_inputs.small_workload(512, 512, 512, 128, 1e-5, mode="random", E=10, beta=0.0, seed=21)
    A, Bm, C = w.matrices()
    g, _ = run_gpu(A, Bm, None, 128, w.tol, 1.0, 0.0, w.class_mask)
    o = run_oracle(A, Bm, None, 128, w.tol, 1.0, 0.0, w.class_mask)
    nb = 128
    checked = 0
    for which, X, codes, s5 in [("A", A, o["acode"], o["ascale5"]), ("B", Bm, o["bcode"], o["bscale5"])]:
        for ti in range(codes.shape[0]):
            for tj in range(codes.shape[1]):
                try:
                    parts, sc = g.tile(which, ti, tj, B.TILE_SPLIT)
                except B.GmpError:
                    continue
                code = int(codes[ti, tj])
                tile = X[ti * nb:(ti + 1) * nb, tj * nb:(tj + 1) * nb]
                stored = oracle.pack_tile(tile, code, int(s5[ti, tj, code]), role=which)
                f32 = stored if code == 1 else oracle.shadow_tile(stored, nb, code, int(s5[ti, tj, code]), 1, role=which)[0]
                v = oracle.payload_values(f32, 1).reshape(nb, nb)     # MN-major payload
                want = v.T                                            # K-major view
                pv = [oracle.decode(parts.view(np.uint16)[k * nb * nb:(k + 1) * nb * nb].astype(np.uint32), 3)
                      .reshape(nb, nb) for k in range(3)]
                assert np.array_equal(pv[0] + pv[1] + pv[2], want)
                assert np.all(np.abs(pv[1]) <= np.abs(pv[0]) * 2.0 ** -8 + 1e-300)
                checked += 1
    assert checked > 0


def test_fp32_split_wide_dynamic_range_limit():
    """The exactness limit of the BF16x3 split (FP32 class): BF16 has
    FP32's exponent range, so x2 = x - x0 - x1 is representable only down to the BF16
    subnormal quantum 2^-133.  With FP32 tiles scaled to max <= 1 (R10), elements with
    |x| >= 2^-110 split EXACTLY; below that the parts differ from x by at most 2^-134
    (half the BF16 subnormal quantum).  Checked on tiles whose elements span 2^0 .. 2^-140."""
    nb = 128
    rng = np.random.default_rng(5)
    A = rng.uniform(0.5, 1.0, (256, 256)) * rng.choice([-1, 1], (256, 256)) * \
        2.0 ** -rng.integers(0, 141, (256, 256)).astype(np.float64)
    A[0, 0] = 1.0   # tile max 1: scale 0 (the payload IS x)
    Bm = A.T.copy()
    fp32 = (np.ones((2, 2), np.uint8), np.ones((2, 2), np.uint8), np.zeros((2, 2), np.uint8))
    g, _ = run_gpu(A, Bm, None, nb, 1e-6, 1.0, 0.0, 0b00011, maps=fp32)
    small = exact = 0
    for which, X in (("A", A), ("B", Bm)):
        for ti in range(2):
            for tj in range(2):
                parts, sc = g.tile(which, ti, tj, B.TILE_SPLIT)
                stored, sc32 = g.tile(which, ti, tj, 1)
                v = oracle.payload_values(stored.view(np.uint32), 1).reshape(nb, nb)   # MN-major payload
                want = v.T
                pv = [oracle.decode(parts.view(np.uint16)[k * nb * nb:(k + 1) * nb * nb].astype(np.uint32), 3)
                      .reshape(nb, nb) for k in range(3)]
                got = pv[0] + pv[1] + pv[2]            # exact in binary64 (disjoint bit ranges)
                big = np.abs(want) >= 2.0 ** -110
                assert np.array_equal(got[big], want[big])
                assert np.all(np.abs(got[~big] - want[~big]) <= 2.0 ** -134)
                exact += int(big.sum())
                small += int((~big & (want != 0)).sum())
    assert small > 1000 and exact > 1000, (small, exact)


def test_rectangular_many_tiles_sampled_vs_oracle():
    """cfg5-shaped (K >> M, N) at reduced size: sampled C tiles vs the oracle"""
    w = gmp_inputs.small_workload(512, 512, 4096, 128, 1e-4, mode="random", E=16, beta=0.0, seed=7)
    A, Bm, C = w.matrices()
    g, (out,) = run_gpu(A, Bm, C, w.nb, w.tol, w.alpha, w.beta, w.class_mask, flags=B.GMP_FLAG_SIMT_ONLY)
    o = run_oracle(A, Bm, C, w.nb, w.tol, w.alpha, w.beta, w.class_mask, ctiles=[0, 6, 15])
    for t in [0, 6, 15]:
        i, j = divmod(t, 4)
        sl = (slice(i * 128, (i + 1) * 128), slice(j * 128, (j + 1) * 128))
        assert np.array_equal(out[sl], o["C"][sl])


def test_fp64_digit_planes_reconstruct():
    """FP64 class on the (experimental, opt-in) INT8 tensor pipe: the seven int8 digit planes of every
    sliced operand satisfy x = 2^e_r (sum_i q_i 2^-7i + rho), |rho| < 2^-49, |q| <= 127
    (checked against the oracle-packed binary64 payload, K-major view)."""
    w = gmp_inputs.small_workload(512, 512, 512, 128, 1e-12, mode="random", E=12, beta=0.0,
                                  class_mask=0b00001, seed=31)
    A, Bm, C = w.matrices()
    g, (out,) = run_gpu(A, Bm, None, 128, w.tol, 1.0, 0.0, w.class_mask, flags=B.GMP_FLAG_FP64_INT8)
    nb = 128
    checked = 0
    for which, X in [("A", A), ("B", Bm)]:
        for ti in range(4):
            for tj in range(4):
                planes, _ = g.tile(which, ti, tj, B.TILE_DIGITS)
                q = planes.view(np.int8).reshape(7, nb, nb).astype(np.float64)
                tile = X[ti * nb:(ti + 1) * nb, tj * nb:(tj + 1) * nb]
                kmaj = tile if which == "A" else tile.T          # rows = output rows / cols, K contiguous
                rowmax = np.abs(kmaj).max(axis=1)
                _, e = np.frexp(rowmax)
                rec = sum(q[i] * 2.0 ** (-7 * (i + 1)) for i in range(7))
                rec = np.ldexp(rec, e[:, None])
                assert np.all(np.abs(q) <= 127)
                assert np.all(np.abs(rec - kmaj) <= np.ldexp(1.0, e - 49)[:, None])
                checked += 1
    assert checked == 32
    o = run_oracle(A, Bm, None, 128, w.tol, 1.0, 0.0, w.class_mask)
    assert np.linalg.norm(out - o["C"]) / np.linalg.norm(o["C"]) <= 1e-13


@pytest.mark.parametrize("nb,mask,tol", [(128, 0b01111, 1e-6), (256, 0b11111, 1e-1), (128, 0b00001, 1e-12),
                                         (256, 0b111111, 0.5)])
def test_single_tile(nb, mask, tol):
    """degenerate grid: M = N = K = nb (one tile each, one SUMMA step, one pair)"""
    w = gmp_inputs.small_workload(nb, nb, nb, nb, tol, mode="uniform", E=0, beta=0.25, class_mask=mask, seed=61)
    A, Bm, C = w.matrices()
    o = run_oracle(A, Bm, C, nb, tol, 1.0, 0.25, mask)
    g, (out,) = run_gpu(A, Bm, C, nb, tol, 1.0, 0.25, mask)
    m = g.maps()
    assert np.array_equal(m["acode"], o["acode"]) and np.array_equal(m["ccode"], o["ccode"])
    gs, (outs,) = run_gpu(A, Bm, C, nb, tol, 1.0, 0.25, mask, flags=B.GMP_FLAG_SIMT_ONLY)
    assert np.array_equal(outs, o["C"])
    ok, rel = c_parity(out, o["C"], o["ccode"], o["cscale"], nb, nb, mask == 1)
    assert ok, rel


@pytest.mark.parametrize("k,mask", [(1, 0b000011), (2, 0b000111), (3, 0b001111), (4, 0b011111), (5, 0b111111)])
def test_c_map_at_the_threshold_matches_oracle(k, mask):
    """Equal constant tiles put every C tile exactly at its class threshold
    (d_k = tol / 2, tests/test_oracle_gemm.py::test_c_map_closed_form_equal_tiles);
    at the threshold and 1e-6 either side the GPU's C map is the oracle's, bit for bit
    (same evaluation order of the criterion)."""
    nb = 128
    u = [2.0 ** -53, 2.0 ** -24, 2.0 ** -11, 2.0 ** -8, 2.0 ** -4, 2.0 ** -3][k]
    eta = [0, 2.0 ** -149, 2.0 ** -24, 2.0 ** -133, 2.0 ** -9, 2.0 ** -16][k]
    omega = [0, 1.0, 65504.0, 1.0, 448.0, 57344.0][k]
    dk = u + 2.0 * 2.0 ** -24 + nb * eta / omega
    A = np.full((4 * nb, 4 * nb), 0.75)
    Bm = np.full((4 * nb, 4 * nb), -1.25)
    amap = np.zeros((4, 4), np.uint8)
    for tol in (2 * dk * (1 + 1e-6), 2 * dk, 2 * dk * (1 - 1e-6)):
        o = run_oracle(A, Bm, None, nb, tol, 1.0, 0.0, mask, maps=(amap, amap, None), ctiles=[])
        g, _ = run_gpu(A, Bm, None, nb, tol, 1.0, 0.0, mask, maps=(amap, amap, None))
        assert np.array_equal(g.maps()["ccode"], o["ccode"]), (k, tol)
        g.close()


@pytest.mark.parametrize("k,mask", [(1, 0b000011), (2, 0b000111), (3, 0b001111), (4, 0b011111), (5, 0b111111)])
def test_ab_map_at_the_threshold_matches_oracle(k, mask):
    """Equal constant tiles: ||X_ij|| / ||X|| = 1/NT, so an A/B tile takes class k iff
    delta_k (+ its underflow term) <= tol / 4.  At tol = 4 delta_k and 1e-6 either
    side the GPU's A and B maps are the oracle's, bit for bit."""
    nb = 128
    u = [2.0 ** -53, 2.0 ** -24, 2.0 ** -11, 2.0 ** -8, 2.0 ** -4, 2.0 ** -3][k]
    dk = u + np.sqrt(nb) * 2.0 ** -24
    A = np.full((3 * nb, 4 * nb), 0.75)
    Bm = np.full((4 * nb, 2 * nb), -1.25)
    for tol in (4 * dk * (1 + 1e-6), 4 * dk, 4 * dk * (1 - 1e-6)):
        o = run_oracle(A, Bm, None, nb, tol, 1.0, 0.0, mask, ctiles=[])
        g, _ = run_gpu(A, Bm, None, nb, tol, 1.0, 0.0, mask)
        m = g.maps()
        assert np.array_equal(m["acode"], o["acode"]) and np.array_equal(m["bcode"], o["bcode"]), (k, tol)
        assert np.array_equal(m["ccode"], o["ccode"]), (k, tol)
        g.close()


def test_extreme_exponents_match_oracle():
    """A's sum of squares overflows binary64 (|a| ~ 2^520: S_A = inf, every A tile FP64 by
    O5's rule), B's entries are tiny (~2^-520, per-tile scales far from 0) and their
    product is O(1): maps and scales equal the oracle's bit for bit, C meets the parity
    bound against the oracle"""
    rng = np.random.default_rng(5)
    nb = 128
    A = np.ldexp(rng.uniform(-1, 1, (256, 384)), 520)
    Bm = np.ldexp(rng.uniform(-1, 1, (384, 256)), -520)
    Bm[:128, :128] = np.ldexp(Bm[:128, :128], -30)        # a wider spread of tile norms in B
    C = rng.uniform(-1, 1, (256, 256))
    tol, alpha, beta, mask = 1e-6, 1.0, 0.5, 0b01111
    assert np.isinf((A * A).sum())
    o = run_oracle(A, Bm, C, nb, tol, alpha, beta, mask)
    assert o["rc"] == 0 and (o["acode"] == 0).all()
    g, (out,) = run_gpu(A, Bm, C, nb, tol, alpha, beta, mask)
    m = g.maps()
    for k in ("acode", "bcode", "ccode"):
        assert np.array_equal(m[k], o[k]), k
    assert np.array_equal(m["bscale"], np.take_along_axis(o["bscale5"], o["bcode"][..., None].astype(np.int64),
                                                          axis=2)[..., 0])
    allfp64 = (o["bcode"] == 0).all() and (o["ccode"] == 0).all()
    ok, rel = c_parity(out, o["C"], o["ccode"], o["cscale"], nb, 384, allfp64)
    assert ok, rel


def test_explicit_fp32_c_map_at_extreme_scales():
    """an explicit FP32 c_map on outputs beyond 2^100 (R23) is demoted to FP64
    on the GPU exactly as in the oracle -- no binary32 overflow in the epilogue"""
    nb = 128
    A = np.full((256, 256), 2.0 ** 60); Bm = np.full((256, 256), 2.0 ** 60)
    maps = (None, None, np.ones((2, 2), np.uint8))
    o = run_oracle(A, Bm, None, nb, 1e-2, 1.0, 0.0, 0b01111, maps=maps)
    g, (out,) = run_gpu(A, Bm, None, nb, 1e-2, 1.0, 0.0, 0b01111, maps=maps)
    assert (o["ccode"] == 0).all() and np.array_equal(g.maps()["ccode"], o["ccode"])
    assert np.isfinite(out).all()
    assert np.linalg.norm(out - o["C"]) / np.linalg.norm(o["C"]) <= 1e-13


@pytest.mark.parametrize("nb,beta,seed,mask", [(256, 0.5, 42, 0b1111111), (128, 1.0, 45, 0b0111111),
                                               (256, 0.0, 46, 0b0011111)])
def test_fused_maxabs_bitwise_vs_separate(nb, beta, seed, mask):
    """S7 pass 1: max|W| of a binary32-W C tile is emitted by its last tcgen05 launch (atomicMax
    on the register copy of W); GMP_FLAG_SEPARATE_MAXABS re-reads W in k_c_maxabs.  The max is
    independent of the order, so C (and its scales) are bit-identical; one launch fewer"""
    w = gmp_inputs.small_workload(3 * nb, 2 * nb, 4 * nb, nb, 1e-3, mode="random", E=36, beta=beta,
                                  class_mask=mask, seed=seed)
    A, Bm, C = w.matrices()
    g, (out,) = run_gpu(A, Bm, C, nb, w.tol, w.alpha, w.beta, w.class_mask)
    g2, (out2,) = run_gpu(A, Bm, C, nb, w.tol, w.alpha, w.beta, w.class_mask, flags=B.GMP_FLAG_SEPARATE_MAXABS)
    assert np.array_equal(out, out2)
    assert g.stats()["launches_execute"] <= g2.stats()["launches_execute"]
    o = run_oracle(A, Bm, C, nb, w.tol, w.alpha, w.beta, w.class_mask)
    ok, rel = c_parity(out, o["C"], o["ccode"], o["cscale"], nb, w.K, False)
    assert ok, rel
