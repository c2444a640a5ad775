"""GPU parity: the CUDA path (through the C ABI) against the oracle on the same
seeded inputs.  Maps, scales, packed payload bytes (stored and shadow) must be
bit-exact; C must match the oracle's emulated result to 1e-13 (all-FP64) or
4 u32 sqrt(K) (mixed; relative Frobenius), bitwise when every class runs on the
SIMT kernels, and meet the user tolerance against cuBLAS DGEMM."""
import numpy as np
import pytest

import gmp_inputs
import oracle
from gpu_harness import c_parity, run_gpu, run_oracle, tol_metric, w_and_finalize_parity
from paper_2508_14848_b200 import binding as B

pytestmark = pytest.mark.gpu

U32 = 2.0 ** -24


def _cases():
    w1 = gmp_inputs.workload(1)
    w1b = gmp_inputs.workload(1, "beta0")
    return [
        ("cfg1", w1),
        ("cfg1_beta0", w1b),
        ("e4m3_mix", gmp_inputs.small_workload(512, 384, 640, 128, 1e-2, mode="random", E=40, beta=0.5,
                                               class_mask=0b11111, seed=41)),
        ("bf16_mix", gmp_inputs.small_workload(768, 512, 512, 256, 1e-4, mode="random", E=32, beta=0.0, seed=42)),
        ("nb384_graded", gmp_inputs.small_workload(768, 1152, 384, 384, 1e-6, mode="graded", E=20, beta=-1.5,
                                                   seed=43)),
        ("fp64_only", gmp_inputs.small_workload(512, 512, 512, 128, 1e-12, mode="random", E=10, beta=1.0,
                                                class_mask=0b00001, seed=44)),
        # E5M2 enabled: E5M2 tiles, E5M2 shadows of every class, E5M2 pairs on
        # tcgen05 kind::f8f6f4, E5M2 C tiles
        ("e5m2_mix", gmp_inputs.small_workload(512, 384, 640, 128, 1e-1, mode="random", E=48, beta=0.5,
                                               class_mask=0b111111, seed=46)),
        ("e5m2_nb256", gmp_inputs.small_workload(768, 512, 1024, 256, 2e-2, mode="random", E=40, beta=0.0,
                                                 class_mask=0b111111, seed=47)),
        # nb = 512 with GMP_FLAG_TC_PAIR: 2 x 2 sub-tiles of 256 x 256 per C tile on the SM-pair
        # kernel (k_tc2_class), rastered by C tile row bands; the plain nb = 512 run covers the 1-SM kernel
        ("pairs_nb512", gmp_inputs.small_workload(1024, 1536, 1536, 512, 1e-2, mode="random", E=24, beta=0.75,
                                                  class_mask=0b11111, seed=45), B.GMP_FLAG_TC_PAIR),
        ("nb512", gmp_inputs.small_workload(1024, 1536, 1536, 512, 1e-2, mode="random", E=24, beta=0.75,
                                            class_mask=0b11111, seed=45)),
        # GMP_FLAG_TC_SINGLE (explicit 1-SM choice) with the raster of the 1-SM launches (GMP_RASTER=1
        # is process-wide, so here the flag only pins the default)
        ("single_nb512", gmp_inputs.small_workload(1024, 1536, 1536, 512, 1e-2, mode="random", E=24, beta=0.75,
                                                   class_mask=0b11111, seed=45), B.GMP_FLAG_TC_SINGLE),
        ("pairs_e5m2_nb512", gmp_inputs.small_workload(1024, 1024, 1536, 512, 5e-2, mode="random", E=32,
                                                       beta=0.0, class_mask=0b111111, seed=48),
         B.GMP_FLAG_TC_PAIR),
        # MXFP4 enabled (NEXT-4, R31): MXFP4 tiles (E2M1 nibbles + E8M0 block scales),
        # MXFP4 shadows of every other class (k_mx), MXFP4 pairs on tcgen05 kind::mxf4.block_scale
        ("mx4_mix", gmp_inputs.small_workload(512, 384, 640, 128, 1e-2, mode="random", E=40, beta=0.5,
                                              class_mask=0b1111111, seed=41)),
        ("mx4_nb256", gmp_inputs.small_workload(768, 512, 1024, 256, 2e-2, mode="random", E=40, beta=0.0,
                                                class_mask=0b1111111, seed=50)),
        ("mx4_fine", gmp_inputs.small_workload(512, 384, 640, 128, 1e-3, mode="random", E=40, beta=-0.75,
                                               class_mask=0b1111111, seed=52)),
    ]


CASES = _cases()


@pytest.fixture(scope="module", params=CASES, ids=[c[0] for c in CASES])
def case(request):
    name, w = request.param[:2]
    flags = request.param[2] if len(request.param) > 2 else 0
    A, Bm, C = w.matrices()
    orc = run_oracle(A, Bm, C, w.nb, w.tol, w.alpha, w.beta, w.class_mask)
    assert orc["rc"] == 0
    g, (Cg, Cg2) = run_gpu(A, Bm, C, w.nb, w.tol, w.alpha, w.beta, w.class_mask, flags=flags, reps=2)
    gs, (Cs,) = run_gpu(A, Bm, C, w.nb, w.tol, w.alpha, w.beta, w.class_mask, flags=B.GMP_FLAG_SIMT_ONLY)
    gp, (Cp,) = run_gpu(A, Bm, C, w.nb, w.tol, w.alpha, w.beta, w.class_mask,
                        flags=flags | B.GMP_FLAG_SPLIT16)
    return dict(name=name, w=w, A=A, B=Bm, C=C, orc=orc, g=g, Cg=Cg, Cg2=Cg2, gs=gs, Cs=Cs, gp=gp, Cp=Cp)


def test_maps_bitwise(case):
    m = case["g"].maps()
    o = case["orc"]
    assert np.array_equal(m["acode"], o["acode"])
    assert np.array_equal(m["bcode"], o["bcode"])
    assert np.array_equal(m["ccode"], o["ccode"])
    amask = o["acode"][..., None] == np.arange(B.NCLS)
    bmask = o["bcode"][..., None] == np.arange(B.NCLS)
    assert np.array_equal(m["ascale"], (o["ascale5"] * amask).sum(-1))
    assert np.array_equal(m["bscale"], (o["bscale5"] * bmask).sum(-1))


def test_packed_bytes_bitwise(case):
    """every stored and every materialised shadow payload, byte for byte"""
    w, o, g = case["w"], case["orc"], case["g"]
    nb = w.nb
    checked = 0
    for which, X, codes, s5, kmaj in [("A", case["A"], o["acode"], o["ascale5"], False),
                                      ("B", case["B"], o["bcode"], o["bscale5"], True)]:
        rows, cols = codes.shape
        for ti in range(rows):
            for tj in range(cols):
                code = int(codes[ti, tj])
                tile = X[ti * nb:(ti + 1) * nb, tj * nb:(tj + 1) * nb]
                stored = oracle.pack_tile(tile, code, int(s5[ti, tj, code]), role=which)
                got, sc = g.tile(which, ti, tj, code)
                assert sc == s5[ti, tj, code]
                assert np.array_equal(got, stored.view(np.uint8)), (which, ti, tj, code)
                checked += 1
                for c in range(code + 1, B.NCLS):
                    try:
                        got, sc = g.tile(which, ti, tj, c)
                    except B.GmpError:
                        continue  # not needed by any local tile-GEMM
                    sh, e = oracle.shadow_tile(stored, nb, code, int(s5[ti, tj, code]), c, role=which)
                    assert sc == e == s5[ti, tj, c]
                    assert np.array_equal(got, sh.view(np.uint8)), (which, ti, tj, code, c)
                    checked += 1
    assert checked > 0


def test_tile_stats_bitwise(case):
    """S1 debug export: every tile's canonical sum of squares (CNORM, O4), maxabs and
    finite flag as the GPU map kernel computed them == the oracle's, bitwise"""
    o, g, w = case["orc"], case["g"], case["w"]
    for which, So, Mo in (("A", o["SA"], o["MA"]), ("B", o["SB"], o["MB"]), ("C", o["SC"], o["MC"])):
        S, M, F = g.tile_stats(which)
        if which == "C" and w.beta == 0.0:
            assert not S.any() and not M.any()
            continue
        assert np.array_equal(S.view(np.uint64), So.view(np.uint64)), which
        assert np.array_equal(M, Mo), which
        assert F.all(), which


def test_w_and_finalize_product_path(case):
    """per C tile: GPU W accumulator within the parity bound of the oracle's W, and packed
    C_out / scale / user C exactly the oracle finalize of the GPU's W"""
    o, w = case["orc"], case["w"]
    w_and_finalize_parity(case["g"], o, case["Cg"], w.nb, w.K)


def test_w_and_finalize_simt_path_bitwise(case):
    """SIMT kernels (per-thread sequential k): W is the oracle's, bit for bit"""
    o, w = case["orc"], case["w"]
    w_and_finalize_parity(case["gs"], o, case["Cs"], w.nb, w.K, bitwise=True)


def test_c_bitwise_on_simt_path(case):
    """all classes on per-thread sequential-k kernels: C is the oracle's, bit for bit"""
    assert np.array_equal(case["Cs"], case["orc"]["C"])


def test_c_parity_product_path(case):
    o, w = case["orc"], case["w"]
    allfp64 = (o["acode"] == 0).all() and (o["bcode"] == 0).all() and (o["ccode"] == 0).all()
    ok, rel = c_parity(case["Cg"], o["C"], o["ccode"], o["cscale"], w.nb, w.K, allfp64)
    assert ok, rel


def test_merged_16bit_launch_equals_per_class_launches(case):
    """the default merged FP16 + BF16 launch (R33) runs the same pairs with the same
    arithmetic in the same fold order as one launch per class (GMP_FLAG_SPLIT16): C is
    bit-identical"""
    assert np.array_equal(case["Cg"], case["Cp"])


def test_c_meets_tolerance(case):
    w = case["w"]
    assert tol_metric(case["Cg"], case["A"], case["B"], case["C"], w.alpha, w.beta) <= w.tol


def test_repeat_execute_bitwise(case):
    assert np.array_equal(case["Cg"], case["Cg2"])


def test_packed_c_matches_oracle_finalize(case):
    """packed C_out of each local tile = oracle finalize of the oracle's C (SIMT path)"""
    o, w, gs = case["orc"], case["w"], case["gs"]
    nb = w.nb
    maps = gs.maps()
    for ti in range(o["ccode"].shape[0]):
        for tj in range(o["ccode"].shape[1]):
            code = int(o["ccode"][ti, tj])
            got, sc = gs.tile("C", ti, tj, code)
            assert sc == o["cscale"][ti, tj] == maps["cscale"][ti, tj]
            dec = oracle.payload_values(got.view(oracle.PAYLOAD_DTYPE[code]), code)
            want = o["C"][ti * nb:(ti + 1) * nb, tj * nb:(tj + 1) * nb].ravel()
            assert np.array_equal(np.ldexp(dec, -sc) if code else dec, want)


def test_mixes_are_mixed():
    """the synthetic recipes really produce the class mixes the configs name"""
    w = gmp_inputs.workload(1)
    A, Bm, C = w.matrices()
    g, _ = run_gpu(A, Bm, C, w.nb, w.tol, w.alpha, w.beta, w.class_mask)
    st = g.stats()
    assert st["tiles_a"][0] > 0 and st["tiles_a"][1] > 0 and st["tiles_a"][2] > 0
