"""Pins for CNORM, the tile-norm criterion and packing (O4-O7).

Pins are: exact sums for constant power-of-two tiles, the rational-sum error
bound, hand-derived maps for grids of constant tiles, monotonicity in tol,
invariance under 2^s scaling, and the Higham-Mary style storage bound
||decode(pack(X)) - X||_F <= (tol/4) ||X||_F that the criterion is built to
guarantee."""
from fractions import Fraction

import numpy as np
import pytest

import gmp_inputs
import oracle

FP64, FP32, FP16, BF16, E4M3, E5M2 = range(6)
ALL = 0b11111
NOE4 = 0b01111
ALL6 = 0b111111   # with E5M2


@pytest.mark.parametrize("nb,k", [(32, 0), (128, -3), (64, 5), (256, -40)])
def test_cnorm_constant_power_of_two_exact(nb, k):
    t = np.full((nb, nb), 2.0 ** k)
    assert oracle.cnorm(t) == nb * nb * 4.0 ** k


@pytest.mark.parametrize("nb", [32, 64, 128])
def test_cnorm_within_rational_bound(nb):
    rng = np.random.default_rng(nb)
    t = rng.standard_normal((nb, nb)) * np.exp2(rng.integers(-20, 20, (nb, nb)))
    exact = sum(Fraction(float(x)) ** 2 for x in t.ravel())
    got = Fraction(oracle.cnorm(t))
    assert abs(got - exact) <= Fraction(nb * nb) * Fraction(2.0 ** -53) * exact


def _rn(x: Fraction) -> float:
    return float(x)          # Fraction -> float rounds to nearest, ties to even


def _cnorm_order(tile, order="O4"):
    """DESIGN.md O4 written out with exact rationals and one rounding per operation:
    256 lanes x 2 slots, lane t slot s runs an fma chain over q = 2t + s + 512w (w = 0, 1, ...);
    t = a0 + a1; butterfly t <- t + t[lane ^ off] inside each 32-lane warp for off = 16, 8, 4, 2, 1;
    S = ((w0 + w1) + ...) + w7.  `order` selects a plausible wrong variant (to show the
    sentinel tiles below can tell them apart): "slot256" (q = t + 256 s + 512 w), "bfly1"
    (offsets 1, 2, 4, 8, 16), "warptree" (pairwise sum of the warp results)."""
    x = [Fraction(float(v)) for v in np.asarray(tile, np.float64).ravel()]
    n = len(x)
    acc = [[Fraction(0), Fraction(0)] for _ in range(256)]
    for base in range(0, n, 512):
        for t in range(256):
            for sl in range(2):
                q = base + (t + 256 * sl if order == "slot256" else 2 * t + sl)
                acc[t][sl] = Fraction(_rn(x[q] * x[q] + acc[t][sl]))
    lane = [Fraction(_rn(a[0] + a[1])) for a in acc]
    offs = (1, 2, 4, 8, 16) if order == "bfly1" else (16, 8, 4, 2, 1)
    for off in offs:
        lane = [Fraction(_rn(lane[t] + lane[t ^ off])) for t in range(256)]
    w = [lane[32 * k] for k in range(8)]
    if order == "warptree":
        while len(w) > 1:
            w = [Fraction(_rn(w[2 * i] + w[2 * i + 1])) for i in range(len(w) // 2)]
        return float(w[0])
    S = w[0]
    for k in range(1, 8):
        S = Fraction(_rn(S + w[k]))
    return float(S)


def _sentinels(nb=64):
    """tiles whose CNORM depends on the reduction order: a big element and tiny ones whose
    squares (each below half an ulp of the big square) survive only if they meet each other
    before they meet the big one"""
    out = []
    tiny = 2.0 ** -27 * 0.75 ** 0.5   # tiny^2 = 0.75 * 2^-54
    for big_q, tiny_qs in [(0, [1, 513, 1025]),            # slot 1 of lane 0 vs slot 0
                           (0, [2, 64, 514]),             # lanes 1 and 32 (another warp)
                           (0, [32, 256 + 32, 96]),       # lane 16 / 48 (butterfly offset 16)
                           (0, [64 * 2 * 8, 130, 258]),   # warps 4, lane 65, lane 129
                           (512, [0, 2, 4])]:             # the big one later in a chain
        t = np.zeros(nb * nb)
        t[big_q] = 1.0
        for q in tiny_qs:
            t[q] = tiny
        out.append(t.reshape(nb, nb))
    return out


def test_cnorm_order_written_out():
    """O4's reduction order, pinned: the oracle's CNORM equals the order written out above
    on sentinel tiles (where plausible other orders give other results) and on tiles with
    a wide dynamic range"""
    tiles = _sentinels()
    rng = np.random.default_rng(11)
    for nb in (32, 64):
        tiles.append(rng.standard_normal((nb, nb)) * np.exp2(rng.integers(-30, 30, (nb, nb))))
    for t in tiles:
        assert oracle.cnorm(t) == _cnorm_order(t)
    # the sentinels really separate the plausible variants from O4
    for variant in ("slot256", "bfly1", "warptree"):
        assert any(_cnorm_order(t, variant) != _cnorm_order(t) for t in tiles), variant


def test_cnorm_reads_ld_not_contiguity():
    rng = np.random.default_rng(5)
    big = rng.standard_normal((64, 96))
    S, M, F = oracle.tile_stats(big[:, :64].copy(), 32)
    S2, M2, F2 = oracle.tile_stats(big, 32)
    assert np.array_equal(S, S2[:, :2]) and np.array_equal(M, M2[:, :2])


def test_tile_stats_flags_nonfinite():
    X = np.ones((64, 64))
    X[40, 3] = np.nan
    S, M, F = oracle.tile_stats(X, 32)
    assert F.tolist() == [[1, 1], [0, 1]]
    rc, code, scale = oracle.map_input(S, M, 32, 1e-3, NOE4, F)
    assert rc == 1


def _const_grid(vals, nb):
    vals = np.asarray(vals, dtype=np.float64)
    return np.kron(vals, np.ones((nb, nb)))


# Equal constant tiles: S_ij = nb^2 4^k exactly, ||X|| = NT nb 2^k exactly, so a
# tile is eligible for class k iff delta_k <= tol/4 (underflow term ~2^-18 smaller).
# delta_k (nb=128): FP32 7.34e-7, FP16 4.89e-4, BF16 3.907e-3, E4M3 6.25e-2.
@pytest.mark.parametrize("tol,mask,want", [
    (1e-6, NOE4, FP64),     # eps 2.5e-7 < delta_FP32
    (1e-5, NOE4, FP32),     # eps 2.5e-6
    (1e-2, NOE4, FP16),     # eps 2.5e-3 < delta_BF16
    (2e-2, NOE4, BF16),     # eps 5e-3 >= delta_BF16
    (2e-2, ALL, BF16),      # E4M3 needs eps >= 6.25e-2
    (0.3, ALL, E4M3),
    (0.3, 0b00111, FP16),   # BF16/E4M3 disabled
    (0.3, 0b00011, FP32),
    (0.3, 0b00001, FP64),
    # delta_E5M2 (nb=128) = 2^-3 + sqrt(128) 2^-24 = 0.1250007: eligible iff tol/4 >= it
    (0.3, ALL6, E4M3),      # eps 0.075 < delta_E5M2
    (0.6, ALL6, E5M2),      # eps 0.15
    (0.6, 0b101111, E5M2),  # E4M3 off, E5M2 on
])
def test_map_equal_constant_tiles_closed_form(tol, mask, want):
    nb = 128
    X = _const_grid(np.full((4, 4), 0.75), nb)  # 0.75 is not a power of two: S exact still
    S, M, F = oracle.tile_stats(X, nb)
    rc, code, scale = oracle.map_input(S, M, nb, tol, mask, F)
    assert rc == 0 and (code == want).all()


def test_map_hand_built_grid():
    """4x4 grid, nb=32, one big tile and tiles 2^-5, 2^-9, 2^-20 times smaller.
    ||X||^2 = nb^2 (1 + 5*4^-5 + 5*4^-10 + 5*4^-20) ~ nb^2 (1.0049), NT = 4,
    tol = 1e-3 -> eps = 2.5e-4; a tile of relative size r = ||Xij||/||X|| is
    eligible for k iff r <= eps/(NT delta_k) (+ tiny underflow term):
      FP32: delta 1.86e-7 -> r <= 336;  FP16: delta 4.89e-4 -> r <= 0.1277;
      BF16: delta 3.906e-3 -> r <= 0.016;  E4M3 (enabled): delta 6.25e-2 -> r <= 1.0e-3.
    r: big 0.998 -> FP32; 2^-5 = 0.0311 -> FP16; 2^-9 = 1.95e-3 -> BF16; 2^-20 -> E4M3.
    Zero tile -> first enabled ladder class (E4M3), scale 0."""
    v = np.array([[1.0, 2 ** -5, 2 ** -5, 2 ** -9],
                  [2 ** -5, 2 ** -9, 2 ** -20, 2 ** -20],
                  [2 ** -5, 2 ** -9, 2 ** -20, 2 ** -9],
                  [2 ** -20, 2 ** -20, 2 ** -9, 0.0]])
    # cnt: 1 big, 4 of 2^-5, 5 of 2^-9, 5 of 2^-20, 1 zero (norm estimate above uses 5/5/5)
    nb = 32
    X = _const_grid(v, nb)
    S, M, F = oracle.tile_stats(X, nb)
    rc, code, scale = oracle.map_input(S, M, nb, 1e-3, ALL, F)
    want = np.array([[FP32, FP16, FP16, BF16],
                     [FP16, BF16, E4M3, E4M3],
                     [FP16, BF16, E4M3, BF16],
                     [E4M3, E4M3, BF16, E4M3]])
    assert rc == 0
    assert np.array_equal(code, want), code
    # stored scales: FP32/BF16 target 1.0 (value 2^-k -> e = k), FP16 65504 -> 2^15 * 2^-k scale,
    # E4M3 448 -> 2^8 * 2^-k scale
    assert scale[0, 0] == 0 and scale[0, 1] == 5 + 15 and scale[0, 3] == 9
    assert scale[1, 2] == 20 + 8 and scale[3, 3] == 0


def test_map_hand_built_grid_with_e5m2():
    """The grid above with E5M2 enabled: delta_E5M2 = 2^-3 + sqrt(32) 2^-24 -> r <= 2.5e-4 /
    (4 * 0.125) = 5.0e-4.  Only the 2^-20 tiles (r ~ 9.5e-7) and the zero tile (first enabled
    ladder class) move from E4M3 to E5M2; their E5M2 scale targets 57344 = 0.875 2^16
    (value 2^-20 -> e = 20 + 15)."""
    v = np.array([[1.0, 2 ** -5, 2 ** -5, 2 ** -9],
                  [2 ** -5, 2 ** -9, 2 ** -20, 2 ** -20],
                  [2 ** -5, 2 ** -9, 2 ** -20, 2 ** -9],
                  [2 ** -20, 2 ** -20, 2 ** -9, 0.0]])
    nb = 32
    X = _const_grid(v, nb)
    S, M, F = oracle.tile_stats(X, nb)
    rc, code, scale = oracle.map_input(S, M, nb, 1e-3, ALL6, F)
    want = np.array([[FP32, FP16, FP16, BF16],
                     [FP16, BF16, E5M2, E5M2],
                     [FP16, BF16, E5M2, BF16],
                     [E5M2, E5M2, BF16, E5M2]])
    assert rc == 0
    assert np.array_equal(code, want), code
    assert scale[1, 2] == 20 + 15 and scale[3, 3] == 0


def test_map_all_zero_matrix():
    X = np.zeros((64, 64))
    S, M, F = oracle.tile_stats(X, 32)
    rc, code, scale = oracle.map_input(S, M, 32, 1e-8, NOE4, F)
    assert (code == BF16).all() and (scale == 0).all()


def _rand_matrix(nb=64, mt=4, nt=4, E=24, seed=3):
    return gmp_inputs.synth_block(mt * nb, nt * nb, nb, seed, "random", E, 0, seed + 100)


@pytest.mark.parametrize("mask", [NOE4, ALL])
def test_map_monotone_in_tol(mask):
    X = _rand_matrix()
    S, M, F = oracle.tile_stats(X, 64)
    prev = None
    for tol in [1e-12, 1e-9, 1e-7, 1e-6, 1e-5, 1e-4, 1e-3, 1e-2, 3e-2, 0.1, 0.5]:
        rc, code, _ = oracle.map_input(S, M, 64, tol, mask, F)
        if prev is not None:
            assert (code >= prev).all()
        prev = code


@pytest.mark.parametrize("s", [-300, -17, 5, 200])
def test_map_invariant_under_power_of_two_scaling(s):
    X = _rand_matrix(seed=9)
    S, M, F = oracle.tile_stats(X, 64)
    S2, M2, F2 = oracle.tile_stats(np.ldexp(X, s), 64)
    for tol, mask in [(1e-6, NOE4), (1e-3, ALL), (1e-2, ALL)]:
        rc, c1, e1 = oracle.map_input(S, M, 64, tol, mask, F)
        rc2, c2, e2 = oracle.map_input(S2, M2, 64, tol, mask, F2)
        assert np.array_equal(c1, c2)
        sub = c1 > 0
        assert np.array_equal(e2[sub], e1[sub] - s)


def _storage_error(X, nb, code, scale):
    mt, nt = code.shape
    err2 = 0.0
    for i in range(mt):
        for j in range(nt):
            t = X[i * nb:(i + 1) * nb, j * nb:(j + 1) * nb]
            c, e = int(code[i, j]), int(scale[i, j])
            pay = oracle.pack_tile(t, c, e)
            back = np.ldexp(oracle.payload_values(pay, c), -e).reshape(nb, nb)
            err2 += float(((back - t) ** 2).sum())
    return np.sqrt(err2)


@pytest.mark.parametrize("tol,mask,E", [(1e-6, NOE4, 14), (1e-8, NOE4, 22), (1e-4, NOE4, 32),
                                        (1e-2, ALL, 40), (1e-1, ALL, 8)])
def test_storage_error_bound(tol, mask, E):
    """C2.8: the criterion guarantees ||decode(pack(X)) - X||_F <= (tol/4)||X||_F."""
    nb = 64
    X = _rand_matrix(nb=nb, mt=4, nt=6, E=E, seed=int(E))
    S, M, F = oracle.tile_stats(X, nb)
    rc, code, scale = oracle.map_input(S, M, nb, tol, mask, F)
    err = _storage_error(X, nb, code, scale)
    assert err <= (tol / 4) * np.linalg.norm(X) * (1 + 1e-12)
    assert len(np.unique(code)) >= 2  # the recipe really mixes classes


def test_pack_layouts():
    """O6: FP64/FP32 operands MN-major (A column-major, B row-major), FP16/BF16/E4M3
    operands K-major (A row-major, B column-major), C row-major."""
    rng = np.random.default_rng(4)
    t = rng.standard_normal((32, 32))
    plain = oracle.pack_tile(t, FP32, 0, transpose=False).reshape(32, 32)
    trans = oracle.pack_tile(t, FP32, 0, transpose=True).reshape(32, 32)
    assert np.array_equal(plain.T, trans)
    assert np.array_equal(plain.view(np.float32), t.astype(np.float32))
    assert np.array_equal(oracle.pack_tile(t, FP32, 0, role="A").reshape(32, 32), trans)
    assert np.array_equal(oracle.pack_tile(t, FP32, 0, role="B").reshape(32, 32), plain)
    assert np.array_equal(oracle.pack_tile(t, FP64, 0, role="A").reshape(32, 32), oracle.pack_tile(t, FP64, 0).reshape(32, 32).T)
    for c in (FP16, BF16, E4M3):
        p = oracle.pack_tile(t, c, 0).reshape(32, 32)
        assert np.array_equal(oracle.pack_tile(t, c, 0, role="A").reshape(32, 32), p)
        assert np.array_equal(oracle.pack_tile(t, c, 0, role="B").reshape(32, 32), p.T)
    assert not oracle.layout_transposed("C", FP64) and not oracle.layout_transposed("C", FP16)


def test_pack_fp64_is_copy():
    t = np.random.default_rng(6).standard_normal((32, 32))
    p = oracle.pack_tile(t, FP64, 0)
    assert np.array_equal(p.view(np.float64).reshape(32, 32), t)


@pytest.mark.parametrize("role", ["A", "B"])
@pytest.mark.parametrize("frm,to", [(0, 1), (0, 2), (0, 4), (1, 2), (1, 3), (2, 3), (2, 4), (3, 4), (1, 4),
                                    (0, 5), (1, 5), (2, 5), (3, 5), (4, 5)])
def test_shadow_is_receiver_side_rounding_of_stored(frm, to, role):
    """Shadow = RN_to(decoded stored tile) with the scale chosen for the decoded
    tile (R7), in the target class's layout: check against the pinned encoder
    applied to the decoded tile and the scale definition."""
    nb = 32
    rng = np.random.default_rng(frm * 5 + to)
    t = rng.standard_normal((nb, nb)) * 2.0 ** -7
    e_from = oracle.scale_exp(np.abs(t).max(), frm)
    stored = oracle.pack_tile(t, frm, e_from, role=role)
    vals = oracle.payload_values(stored, frm).reshape(nb, nb)
    if oracle.layout_transposed(role, frm):
        vals = vals.T
    dec = np.ldexp(vals, -e_from)                                         # decoded tile (r, c)
    sh, e_to = oracle.shadow_tile(stored, nb, frm, e_from, to, role=role)
    assert e_to == oracle.scale_exp(np.abs(dec).max(), to)
    want = oracle.encode(np.ldexp(dec, e_to), to)
    if oracle.layout_transposed(role, to):
        want = want.T
    assert np.array_equal(sh.astype(np.uint32).reshape(nb, nb), want)
