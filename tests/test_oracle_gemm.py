"""Pins for the oracle's tile-GEMM emulation, fold, finalize and whole-method
driver (O8-O9): step-by-step Fraction emulation (bitwise), the
gamma_n bound against the exact product, exact rational GEMM for all-FP64,
SPEC.md scalar examples, and the end-to-end tolerance bound
||C - C_fp64||_F / (|a| ||A|| ||B|| + |b| ||C||) <= tol."""
from fractions import Fraction

import numpy as np
import pytest

import gmp_inputs
import oracle
import gmp_refs as refs

FP64, FP32, FP16, BF16, E4M3, E5M2 = range(6)


def _payload(vals, cls, kmajor=False):
    """A operand (kmajor=False) or B operand (kmajor=True) payload in the O6 layout"""
    return oracle.pack_tile(vals, cls, 0, role="B" if kmajor else "A")


def _values(payload, cls, role, nb):
    v = oracle.payload_values(payload, cls).reshape(nb, nb)
    return v.T if oracle.layout_transposed(role, cls) else v


def _fraction_tile_gemm(a, b, cls):
    """step-by-step emulation with exact rationals, rounding after every op"""
    nb = a.shape[0]
    P = np.zeros((nb, nb))
    for r in range(nb):
        for c in range(nb):
            acc = Fraction(0)
            for p in range(nb):
                prod = Fraction(float(a[r, p])) * Fraction(float(b[p, c]))
                if cls == FP64:
                    acc = Fraction(refs.rn64(prod + acc))           # fma: one rounding
                elif cls == FP32:
                    acc = Fraction(float(refs.rn32(prod + acc)))    # fmaf: one rounding
                else:
                    pr = Fraction(float(refs.rn32(prod)))          # exact for 16/8-bit inputs
                    assert pr == prod
                    acc = Fraction(float(refs.rn32(acc + pr)))
            P[r, c] = float(acc)
    return P


@pytest.mark.parametrize("cls", [FP64, FP32, FP16, BF16, E4M3, E5M2])
def test_tile_gemm_bitwise_vs_fraction_emulation(cls):
    nb = 8
    rng = np.random.default_rng(10 + cls)
    a = rng.standard_normal((nb, nb)) * 3
    b = rng.standard_normal((nb, nb)) * 3
    # make the operands exactly representable in the class first
    pa, pb = _payload(a, cls), _payload(b, cls, kmajor=True)
    av = _values(pa, cls, "A", nb)
    bv = _values(pb, cls, "B", nb)
    got = oracle.tile_gemm(cls, pa, pb, nb)
    want = _fraction_tile_gemm(av, bv, cls)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("cls,u", [(FP64, 2.0 ** -53), (FP32, 2.0 ** -24), (FP16, 2.0 ** -24),
                                   (BF16, 2.0 ** -24), (E4M3, 2.0 ** -24), (E5M2, 2.0 ** -24)])
def test_tile_gemm_gamma_bound(cls, u):
    nb = 64
    rng = np.random.default_rng(20 + cls)
    scale = {FP16: 100.0, E4M3: 10.0, E5M2: 100.0}.get(cls, 1.0)
    pa = _payload(rng.standard_normal((nb, nb)) * scale, cls)
    pb = _payload(rng.standard_normal((nb, nb)) * scale, cls, kmajor=True)
    av = _values(pa, cls, "A", nb)
    bv = _values(pb, cls, "B", nb)
    got = oracle.tile_gemm(cls, pa, pb, nb)
    exact = [[sum(Fraction(float(av[r, p])) * Fraction(float(bv[p, c])) for p in range(nb))
              for c in range(0, nb, 7)] for r in range(0, nb, 5)]
    absprod = np.abs(av) @ np.abs(bv)
    g = refs.gamma(nb, u)
    for ri, r in enumerate(range(0, nb, 5)):
        for ci, c in enumerate(range(0, nb, 7)):
            assert abs(Fraction(float(got[r, c])) - exact[ri][ci]) <= Fraction(g * absprod[r, c] * (1 + 1e-12))


def _identity_blocks(n, v):
    return np.eye(n) * v


@pytest.mark.parametrize("alpha,beta,a,b,c,want", [
    (1.0, 1.0, 2.0, 3.0, 1.0, 7.0),      # SPEC.md:265-267 nb=1 example, block-diagonal form
    (2.0, 3.0, 1.0, 4.0, 5.0, 23.0),
    (0.0, 1.0, 2.0, 3.0, 1.0, 1.0),      # alpha=0, beta=1 -> C unchanged
])
@pytest.mark.parametrize("mask", [0b00001, 0b01111])
def test_spec_scalar_examples(alpha, beta, a, b, c, want, mask):
    n, nb = 64, 32
    A, B, C = _identity_blocks(n, a), _identity_blocks(n, b), _identity_blocks(n, c)
    o = oracle.gemm_mp(A, B, C, nb, 1e-6, alpha, beta, class_mask=mask)
    assert o["rc"] == 0
    assert np.array_equal(o["C"], _identity_blocks(n, want))


def test_identity_a_gives_b():
    n, nb = 64, 32
    B = np.random.default_rng(3).standard_normal((n, n))
    o = oracle.gemm_mp(np.eye(n), B, None, nb, 1e-12, 1.0, 0.0, class_mask=0b00001)
    assert np.array_equal(o["C"], B)


def test_all_fp64_vs_exact_rational():
    M = N = K = 64
    nb = 32
    rng = np.random.default_rng(7)
    A = rng.standard_normal((M, K)); B = rng.standard_normal((K, N)); C = rng.standard_normal((M, N))
    alpha, beta = 1.25, -0.5
    o = oracle.gemm_mp(A, B, C, nb, 1e-6, alpha, beta, class_mask=0b00001)
    assert (o["acode"] == 0).all() and (o["bcode"] == 0).all() and (o["ccode"] == 0).all()
    u = 2.0 ** -53
    absref = abs(alpha) * np.abs(A) @ np.abs(B) + abs(beta) * np.abs(C)
    for (r, c) in [(0, 0), (5, 17), (33, 40), (63, 63), (31, 32)]:
        ex = Fraction(alpha) * sum(Fraction(float(A[r, p])) * Fraction(float(B[p, c])) for p in range(K)) \
            + Fraction(beta) * Fraction(float(C[r, c]))
        assert abs(Fraction(float(o["C"][r, c])) - ex) <= Fraction(refs.gamma(K + 2, u) * absref[r, c])
    ref = alpha * A @ B + beta * C
    assert np.linalg.norm(o["C"] - ref) / np.linalg.norm(ref) <= 1e-13


def _tol_metric(Cmp, A, B, C, alpha, beta):
    ref = alpha * (A @ B) + beta * C
    den = abs(alpha) * np.linalg.norm(A) * np.linalg.norm(B) + abs(beta) * np.linalg.norm(C)
    return np.linalg.norm(Cmp - ref) / den


@pytest.mark.parametrize("variant", [None, "beta0"])
def test_cfg1_meets_tolerance_and_mixes_classes(variant):
    w = gmp_inputs.workload(1, variant)
    A, B, C = w.matrices()
    o = oracle.gemm_mp(A, B, C, w.nb, w.tol, w.alpha, w.beta, w.class_mask)
    assert o["rc"] == 0
    assert _tol_metric(o["C"], A, B, C, w.alpha, w.beta) <= w.tol
    codes = set(np.unique(o["acode"])) | set(np.unique(o["bcode"]))
    assert {FP64, FP32, FP16} <= codes


@pytest.mark.parametrize("tol,mask,E", [(1e-3, 0b11111, 30), (1e-2, 0b11111, 40), (1e-5, 0b01111, 22),
                                        (1e-9, 0b01111, 22), (1e-2, 0b111111, 40), (0.1, 0b111111, 48)])
def test_small_workloads_meet_tolerance(tol, mask, E):
    w = gmp_inputs.small_workload(256, 192, 320, 64, tol, mode="random", E=E, beta=0.5,
                                  class_mask=mask, seed=E)
    A, B, C = w.matrices()
    o = oracle.gemm_mp(A, B, C, w.nb, w.tol, w.alpha, w.beta, w.class_mask)
    assert o["rc"] == 0
    assert _tol_metric(o["C"], A, B, C, w.alpha, w.beta) <= tol


def test_sampled_tiles_equal_full_run():
    w = gmp_inputs.small_workload(256, 256, 256, 64, 1e-4, mode="random", E=20, beta=1.0, seed=5)
    A, B, C = w.matrices()
    full = oracle.gemm_mp(A, B, C, w.nb, w.tol, w.alpha, w.beta, w.class_mask)
    part = oracle.gemm_mp(A, B, C, w.nb, w.tol, w.alpha, w.beta, w.class_mask, ctiles=[0, 5, 15])
    for t in [0, 5, 15]:
        i, j = divmod(t, 4)
        sl = (slice(i * 64, i * 64 + 64), slice(j * 64, j * 64 + 64))
        assert np.array_equal(full["C"][sl], part["C"][sl])
    assert np.array_equal(full["ccode"], part["ccode"])


def test_c_map_fp64_guard_for_huge_outputs():
    """R23: a C tile whose estimate exceeds 2^100 is kept in FP64 (W = binary64)."""
    nb = 32
    A = np.full((64, 64), 2.0 ** 60); B = np.full((64, 64), 2.0 ** 60)
    o = oracle.gemm_mp(A, B, None, nb, 1e-2, 1.0, 0.0, class_mask=0b01111)
    assert (o["ccode"] == 0).all()
    ref = A @ B
    assert np.linalg.norm(o["C"] - ref) / np.linalg.norm(ref) <= 1e-2


def test_explicit_maps_paper_mode():
    """aD:bS explicit maps: codes honoured, scales by rule."""
    w = gmp_inputs.small_workload(128, 128, 128, 32, 1e-6, beta=1.0)
    A, B, C = w.matrices()
    amap = np.array([[0, 1, 1, 0]] * 4, np.uint8)
    bmap = np.array([[1, 0, 0, 1]] * 4, np.uint8)
    cmap = np.array([[0, 1, 0, 1]] * 4, np.uint8)
    o = oracle.gemm_mp(A, B, C, 32, 1e-6, 1.0, 1.0, 0b00011, a_map=amap, b_map=bmap, c_map=cmap)
    assert np.array_equal(o["acode"], amap) and np.array_equal(o["ccode"], cmap)
    assert _tol_metric(o["C"], A, B, C, 1.0, 1.0) < 1e-6


@pytest.mark.parametrize("cls", [FP64, FP32, FP16, BF16, E4M3, E5M2])
def test_every_pair_class_contributes(cls):
    """All tiles of A, B, C mapped to one class (explicit maps), non-negative data
    (no cancellation, so ||A B|| ~ ||A|| ||B||): C must match alpha A B + beta C
    relative to itself within that class's storage + accumulation error -- a class
    that the fold skipped leaves C = beta C_in (relative error ~1) -- and, for the
    16/8-bit classes, show that class's rounding (the class path really ran)."""
    nb = 32
    w = gmp_inputs.small_workload(96, 64, 128, nb, 1e-6, mode="uniform", E=0, beta=0.5, seed=11)
    A, B, C = (np.abs(x) for x in w.matrices())
    mt, nt, kt = 3, 2, 4
    maps = dict(a_map=np.full((mt, kt), cls, np.uint8), b_map=np.full((kt, nt), cls, np.uint8),
                c_map=np.full((mt, nt), cls, np.uint8))
    o = oracle.gemm_mp(A, B, C, nb, 1e-6, 1.0, 0.5, 0b111111, **maps)
    assert o["rc"] == 0 and (o["acode"] == cls).all() and (o["ccode"] == cls).all()
    ref = A @ B + 0.5 * C
    err = np.linalg.norm(o["C"] - ref) / np.linalg.norm(ref)
    u = [2.0 ** -53, 2.0 ** -24, 2.0 ** -11, 2.0 ** -8, 2.0 ** -4, 2.0 ** -3][cls]
    # storage of A, B, C_in and the final C each <= u relative (no cancellation), accumulation <= K u32
    assert err <= 4 * u + 128 * 2.0 ** -24 + 1e-15, err
    if cls >= FP16:
        assert err > 1e-2 * u   # the class's rounding is visible: the class path really ran


@pytest.mark.parametrize("k,mask", [(1, 0b000011), (2, 0b000111), (3, 0b001111), (4, 0b011111), (5, 0b111111)])
def test_c_map_closed_form_equal_tiles(k, mask):
    """O7 on equal constant tiles (mt = nt = kt = 4, beta = 0): R_i = 2a, Q_j = 2b, so
    n_hat = 4ab for every C tile while N_hat = 16ab and NT_C = 4 -- the C tile takes
    class k iff d_k = u_k + sqrt(kt) u32 + nb eta_k / Omega'_k <= tol / 2.  Just above
    the threshold of the lowest enabled class the map is that class; just below, the
    next class up (FP64 below FP32's)."""
    nb = 32
    u = [2.0 ** -53, 2.0 ** -24, 2.0 ** -11, 2.0 ** -8, 2.0 ** -4, 2.0 ** -3][k]
    eta = [0, 2.0 ** -149, 2.0 ** -24, 2.0 ** -133, 2.0 ** -9, 2.0 ** -16][k]
    omega = [0, 1.0, 65504.0, 1.0, 448.0, 57344.0][k]
    dk = u + 2.0 * 2.0 ** -24 + nb * eta / omega
    A = np.full((4 * nb, 4 * nb), 0.75)
    Bm = np.full((4 * nb, 4 * nb), -1.25)
    # A/B maps forced to FP64 so only the C criterion is exercised
    amap = np.zeros((4, 4), np.uint8)
    for tol, want_k in [(2 * dk * (1 + 1e-6), True), (2 * dk * (1 - 1e-6), False)]:
        o = oracle.gemm_mp(A, Bm, None, nb, tol, 1.0, 0.0, mask, a_map=amap, b_map=amap, ctiles=[])
        assert o["rc"] == 0
        if want_k:
            assert (o["ccode"] == k).all(), (k, tol, o["ccode"])
        else:
            assert (o["ccode"] < k).all(), (k, tol, o["ccode"])


def test_w_export_consistent_with_finalize():
    """The W debug export is the accumulator the finalize consumed:
    re-finalizing each exported tile reproduces the oracle's C tile and scale bitwise,
    W of a binary32-accumulated tile holds binary32 values, and W of an FP64 C tile is C."""
    w = gmp_inputs.small_workload(192, 256, 320, 64, 1e-3, mode="random", E=30, beta=0.5,
                                  class_mask=0b111111, seed=21)
    A, B, C = w.matrices()
    o = oracle.gemm_mp(A, B, C, w.nb, w.tol, w.alpha, w.beta, w.class_mask)
    nb = w.nb
    assert len(set(np.unique(o["ccode"]))) >= 2
    for i in range(o["ccode"].shape[0]):
        for j in range(o["ccode"].shape[1]):
            code = int(o["ccode"][i, j])
            sl = (slice(i * nb, (i + 1) * nb), slice(j * nb, (j + 1) * nb))
            Wt = o["W"][sl]
            _, user, e = oracle.finalize(Wt, code)
            assert e == o["cscale"][i, j]
            assert np.array_equal(user, o["C"][sl])
            if code == 0:
                assert np.array_equal(Wt, o["C"][sl])
            else:
                assert np.array_equal(Wt.astype(np.float32).astype(np.float64), Wt)


@pytest.mark.parametrize("cls", [FP64, FP32, FP16, BF16, E4M3, E5M2])
def test_w_export_vs_exact_product(cls):
    """W (before the final rounding into C's class) of one-class explicit maps on
    non-negative data is alpha A B + beta C within the storage error of A, B, C_in
    (<= u_cls each) plus binary32 (or binary64) accumulation over K -- independent of
    the oracle: the reference is numpy's binary64 GEMM."""
    nb = 32
    w = gmp_inputs.small_workload(96, 64, 128, nb, 1e-6, mode="uniform", E=0, beta=0.5, seed=12)
    A, B, C = (np.abs(x) for x in w.matrices())
    mt, nt, kt = 3, 2, 4
    maps = dict(a_map=np.full((mt, kt), cls, np.uint8), b_map=np.full((kt, nt), cls, np.uint8),
                c_map=np.full((mt, nt), cls, np.uint8))
    o = oracle.gemm_mp(A, B, C, nb, 1e-6, 1.0, 0.5, 0b111111, **maps)
    ref = A @ B + 0.5 * C
    u = [2.0 ** -53, 2.0 ** -24, 2.0 ** -11, 2.0 ** -8, 2.0 ** -4, 2.0 ** -3][cls]
    uacc = 2.0 ** -53 if cls == FP64 else 2.0 ** -24
    err = np.abs(o["W"] - ref) / ref
    assert err.max() <= 3 * u + 130 * uacc, err.max()


def test_explicit_c_map_keeps_r23_guard():
    """R23 holds for explicit C codes too: an explicit FP32 c_map on a tile
    whose output estimate exceeds 2^100 is demoted to FP64 (W = binary64), so the
    result is not a binary32 overflow"""
    nb = 32
    A = np.full((64, 64), 2.0 ** 60); B = np.full((64, 64), 2.0 ** 60)
    cmap = np.ones((2, 2), np.uint8)
    o = oracle.gemm_mp(A, B, None, nb, 1e-2, 1.0, 0.0, 0b01111, c_map=cmap)
    assert (o["ccode"] == 0).all()
    assert np.isfinite(o["C"]).all()
    ref = A @ B
    assert np.linalg.norm(o["C"] - ref) / np.linalg.norm(ref) <= 1e-2
    # an ordinary explicit FP32 c_map is honoured
    o2 = oracle.gemm_mp(A / 2.0 ** 60, B / 2.0 ** 60, None, nb, 1e-2, 1.0, 0.0, 0b01111, c_map=cmap)
    assert (o2["ccode"] == 1).all()
