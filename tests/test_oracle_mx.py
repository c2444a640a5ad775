"""Pins of the oracle's MXFP4 class (class 6; O2/O3/O5/O6/O8,
reading R31) against definitions written out independently here:

* E2M1 (OCP MX v1.0 element): the 16 codes decode to +-{0, 0.5, 1, 1.5, 2, 3, 4, 6};
  encode is round-to-nearest on that grid with ties to the even code (mantissa bit 0),
  saturating at 6 -- checked against a brute-force nearest-even search over the enumerated
  value set on a dense grid that contains every midpoint and its neighbours;
* the E8M0 block scale: the smallest s >= -127 with max|y| <= 6 * 2^s (exact rationals);
* block encoding: every element is the nearest-even E2M1 value of y / 2^s_b; the layout is
  element 2i in the low nibble of byte i, scales after the nibbles;
* the storage bound the O5 criterion uses: ||dec(pack(X)) - X||_F <= u_6 ||X||_F +
  nb * 0.25 * 2^(s_max - e) on tiles with intra-tile dynamic range;
* the MXFP4 tile-GEMM (binary32 acc + RN32(a b), sequential k) vs an exact Fraction emulation;
* the criterion on equal constant tiles (closed form), MXFP4 never chosen for C, and
  the whole method meeting the tolerance with MXFP4 enabled."""
from fractions import Fraction

import numpy as np
import pytest

import gmp_inputs
import oracle

MX = 6
GRID = [0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0]


def test_e2m1_decode_exhaustive():
    got = oracle.decode(np.arange(16, dtype=np.uint32), MX)
    want = GRID + [-v for v in GRID]
    assert [float(x) for x in got] == want
    assert np.signbit(got[8])   # code 8 is -0


def _nearest_even(x):
    """brute force over the enumerated E2M1 set: nearest value, ties to the even code"""
    a = abs(x)
    if a > 6.0:
        a = 6.0
    best = min(range(8), key=lambda q: (abs(GRID[q] - a), q & 1))
    return (best | (8 if x < 0 or (x == 0 and np.signbit(x)) else 0))


def test_e2m1_encode_nearest_even_dense():
    mids = [(GRID[i] + GRID[i + 1]) / 2 for i in range(7)]
    pts = set()
    for v in GRID + mids + [6.5, 7.0, 100.0, 1e-300]:
        for d in (-1e-12, 0.0, 1e-12):
            pts.add(v + d)
            pts.add(np.nextafter(v, np.inf))
            pts.add(np.nextafter(v, -np.inf))
    pts |= set(np.linspace(0, 7, 7001).tolist())
    xs = np.array(sorted(p for p in pts if p >= 0))
    xs = np.concatenate([xs, -xs])
    got = oracle.encode(xs, MX)
    want = np.array([_nearest_even(float(x)) for x in xs], np.uint32)
    bad = np.nonzero(got != want)[0]
    assert bad.size == 0, [(xs[i], got[i], want[i]) for i in bad[:5]]
    # ties: 0.25 -> 0, 0.75 -> 1.0 (code 2, even), 1.25 -> 1.0, 1.75 -> 2.0, 2.5 -> 2.0,
    # 3.5 -> 4.0, 5.0 -> 4.0 (code 6 even; 6.0 is code 7)
    ties = oracle.decode(oracle.encode(np.array([0.25, 0.75, 1.25, 1.75, 2.5, 3.5, 5.0]), MX), MX)
    assert list(ties) == [0.0, 1.0, 1.0, 2.0, 2.0, 4.0, 4.0]


def _block_exp_def(amax):
    """smallest s >= -127 with amax <= 6 * 2^s, in exact rationals"""
    if amax == 0:
        return -127
    a = Fraction(amax)
    s = -127
    while a > 6 * Fraction(2) ** s:
        s += 1
    return s


@pytest.mark.parametrize("k", [-130, -127, -126, -40, -3, -2, 0, 5, 60])
def test_block_exp_closed_form(k):
    six = 6.0 * 2.0 ** k
    for amax in (six, np.nextafter(six, 0), np.nextafter(six, np.inf), 0.75 * 2.0 ** (k + 3),
                 np.nextafter(0.75 * 2.0 ** (k + 3), np.inf), 2.0 ** k):
        assert oracle.mx_block_exp(amax) == _block_exp_def(amax), amax
    assert oracle.mx_block_exp(0.0) == -127


def _unpack(payload, nb):
    n = nb * nb
    q = np.empty(n, np.uint32)
    q[0::2] = payload[:n // 2] & 15
    q[1::2] = payload[:n // 2] >> 4
    s = payload[n // 2:n // 2 + n // 32].astype(np.int64) - 127
    return q, s


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_block_encode_nearest_even_per_element(seed):
    nb = 64
    rng = np.random.default_rng(seed)
    y = rng.standard_normal(nb * nb) * 2.0 ** rng.integers(-20, 1, nb * nb).astype(float)
    y[:32] = 0.0                               # an all-zero block
    y[32:64] = 2.0 ** -140                     # a block clamped at s = -127
    pay = oracle.mx_encode(y, nb)
    assert pay.size == nb * nb // 2 + nb * nb // 32
    q, s = _unpack(pay, nb)
    for b in range(nb * nb // 32):
        blk = y[32 * b:32 * (b + 1)]
        assert s[b] == _block_exp_def(float(np.abs(blk).max())), b
        for v in range(32):
            x = blk[v] * 2.0 ** -int(s[b])
            assert q[32 * b + v] == _nearest_even(x) or (x == 0 and q[32 * b + v] in (0, 8)), (b, v)
    vals = oracle.payload_values(pay, MX, nb)
    assert np.array_equal(vals, oracle.decode(q, MX) * 2.0 ** np.repeat(s, 32))


def test_pack_layout_k_major():
    """A tiles: payload row = tile row; B tiles: payload row = tile column (K-major, as the
    tensor cores read them); element (m, k) is nibble m*nb + k"""
    nb = 64
    rng = np.random.default_rng(4)
    t = rng.uniform(-1, 1, (nb, nb))
    e = oracle.scale_exp(np.abs(t).max(), MX)
    pa = oracle.pack_tile(t, MX, e, role="A")
    pb = oracle.pack_tile(t, MX, e, role="B")
    assert np.array_equal(pa, oracle.mx_encode((t * 2.0 ** e).ravel(), nb))
    assert np.array_equal(pb, oracle.mx_encode((t.T * 2.0 ** e).ravel(), nb))


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_storage_bound_with_intra_tile_range(seed):
    """the bound the O5 criterion charges for MXFP4: ||dec(pack(X)) - X||_F <=
    u_6 ||X||_F + nb * (eta_6 / 2) * 2^(s_max - e)"""
    nb = 128
    rng = np.random.default_rng(seed)
    X = rng.uniform(-1, 1, (nb, nb)) * 2.0 ** rng.integers(0, 30, (nb, nb)).astype(float) * 1e3
    m = np.abs(X).max()
    e = oracle.scale_exp(m, MX)
    assert m * 2.0 ** e <= 1.0 < m * 2.0 ** (e + 1)
    pay = oracle.pack_tile(X, MX, e, role="A")
    dec = oracle.payload_values(pay, MX, nb).reshape(nb, nb) * 2.0 ** -e
    smax = oracle.mx_block_exp(m * 2.0 ** e)
    bound = 2.0 ** -2 * np.linalg.norm(X) + nb * 0.25 * 2.0 ** (smax - e)
    assert np.linalg.norm(dec - X) <= bound
    # and per element: |err| <= u |x| + 0.25 * 2^(s_b - e)
    q, s = _unpack(pay, nb)
    err = np.abs(dec - X).ravel()
    assert np.all(err <= 2.0 ** -2 * np.abs(X).ravel() + 0.25 * 2.0 ** (np.repeat(s, 32) - e))


def test_tile_gemm_vs_fraction_emulation():
    """O8 for MXFP4: P = sum_p RN32(a_p b_p) accumulated in binary32, sequential p from +0,
    emulated exactly with Fractions (nb = 32, random blocks incl. tiny scales whose
    products are inexact in binary32)"""
    from gmp_refs import rn32
    nb = 32
    rng = np.random.default_rng(7)
    A = rng.uniform(-1, 1, (nb, nb)) * 2.0 ** rng.integers(0, 12, (nb, 1)).astype(float)
    Bm = rng.uniform(-1, 1, (nb, nb))
    A[3] *= 2.0 ** -130                          # rows whose products underflow binary32
    pa = oracle.pack_tile(A, MX, 0, role="A")
    pb = oracle.pack_tile(Bm, MX, 0, role="B")
    P = oracle.tile_gemm(MX, pa, pb, nb)
    av = oracle.payload_values(pa, MX, nb).reshape(nb, nb)          # [r][k]
    bv = oracle.payload_values(pb, MX, nb).reshape(nb, nb)          # [col][k]
    for r in range(nb):
        for c in range(nb):
            acc = Fraction(0)
            for k in range(nb):
                prod = Fraction(float(rn32(Fraction(av[r, k]) * Fraction(bv[c, k]))))
                acc = Fraction(float(rn32(acc + prod)))
            assert P[r, c] == float(acc), (r, c)


def test_criterion_closed_form_constant_tiles():
    """equal constant tiles c: S = nb^2 c^2, so the MXFP4 test is
    delta_6 nb c + nb (eta_6/2) 2^(s_max - e) <= (tol/4) nb c, with e = scale_exp(c),
    s_max = block_exp(c 2^e): MXFP4 iff tol >= 4 (delta_6 + 2^(s_max-e-1) eta_6 / c)"""
    nb = 128
    for c in (0.3, 1.0, 5.0e-3, 7.7e9):
        e = oracle.scale_exp(c, MX)
        smax = oracle.mx_block_exp(c * 2.0 ** e)
        d6 = oracle.delta(MX, nb)
        thr = 4 * (d6 + 0.5 * 2.0 ** (smax - e - 1) / c)
        S = np.full((2, 2), nb * nb * c * c)
        M = np.full((2, 2), c)
        for tol, want in ((thr * (1 + 1e-9), MX), (thr * (1 - 1e-9), None)):
            rc, code, scale = oracle.map_input(S, M, nb, tol, 0b1111111)
            assert rc == 0
            if want == MX:
                assert (code == MX).all(), (c, tol)
            else:
                assert (code != MX).all(), (c, tol)


def test_mx_never_a_c_class():
    w = gmp_inputs.small_workload(256, 256, 256, 128, 0.5, mode="random", E=40, beta=0.5,
                                  class_mask=0b1111111, seed=3)
    A, Bm, C = w.matrices()
    o = oracle.gemm_mp(A, Bm, C, w.nb, w.tol, w.alpha, w.beta, w.class_mask,
                       c_map=np.full((2, 2), MX, np.uint8))
    assert o["rc"] == 0 and (o["ccode"] == 0).all()          # explicit MXFP4 C codes -> FP64
    o = oracle.gemm_mp(A, Bm, C, w.nb, w.tol, w.alpha, w.beta, w.class_mask)
    assert (o["ccode"] != MX).all() and (o["acode"] == MX).any()


@pytest.mark.parametrize("seed,tol", [(49, 5e-2), (41, 1e-2), (52, 1e-3)])
def test_method_meets_tolerance_with_mxfp4(seed, tol):
    w = gmp_inputs.small_workload(512, 384, 640, 128, tol, mode="random", E=40, beta=0.5,
                                  class_mask=0b1111111, seed=seed)
    A, Bm, C = w.matrices()
    o = oracle.gemm_mp(A, Bm, C, w.nb, w.tol, w.alpha, w.beta, w.class_mask)
    assert o["rc"] == 0
    pc = np.maximum(o["acode"][:, :, None], o["bcode"][None, :, :])
    assert (pc == MX).any()
    ref = w.alpha * A @ Bm + w.beta * C
    den = abs(w.alpha) * np.linalg.norm(A) * np.linalg.norm(Bm) + abs(w.beta) * np.linalg.norm(C)
    assert np.linalg.norm(o["C"] - ref) / den <= tol
