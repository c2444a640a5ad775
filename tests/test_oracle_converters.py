"""Pins for the oracle's RNE converters (O2): exhaustive over every
16-bit / 8-bit pattern, their midpoints and midpoint +-1 ulp64, against
(a) numpy's IEEE binary16 (correct RNE from binary64),
(b) a nearest-even search over the enumerated representable set (tests/refs.py),
(c) the hardware binary64->binary32 cast.  Not a re-typing of the oracle."""
from fractions import Fraction

import numpy as np
import pytest

import oracle
import gmp_refs as refs

FP32, FP16, BF16, E4M3, E5M2 = 1, 2, 3, 4, 5


def _midpoint_probe(vals):
    """finite non-negative representables, midpoints, midpoints +- 1 ulp64"""
    v = np.unique(vals[np.isfinite(vals) & (vals >= 0)])
    mids = (v[:-1] + v[1:]) / 2.0           # exact in binary64 for these formats
    probe = np.concatenate([v, mids, np.nextafter(mids, np.inf), np.nextafter(mids, -np.inf)])
    return np.concatenate([probe, -probe])


def test_fp16_decode_exhaustive():
    bits, vals = refs.fp16_values()
    got = oracle.decode(bits.astype(np.uint32), FP16)
    assert np.array_equal(np.isnan(got), np.isnan(vals))
    ok = ~np.isnan(vals)
    assert np.array_equal(got[ok], vals[ok])
    assert np.array_equal(np.signbit(got[ok]), np.signbit(vals[ok]))


def test_fp16_encode_exhaustive_vs_numpy():
    _, vals = refs.fp16_values()
    x = _midpoint_probe(vals)
    x = np.concatenate([x, [65519.99, 65520.0, 65536.0, 1e6, 2.0 ** -25, 2.0 ** -26, 3 * 2.0 ** -26]])
    want = x.astype(np.float16).view(np.uint16).astype(np.uint32)
    got = oracle.encode(x, FP16)
    assert np.array_equal(got, want)


def test_bf16_decode_exhaustive():
    bits, vals = refs.bf16_values()
    got = oracle.decode(bits, BF16)
    ok = ~np.isnan(vals)
    assert np.array_equal(np.isnan(got), np.isnan(vals))
    assert np.array_equal(got[ok], vals[ok])


def _check_nearest_even(cls, bits, vals, x, sat):
    ne = refs.NearestEven(bits, vals, None)
    got = oracle.encode(x, cls)
    sign_shift = {BF16: 15, E4M3: 7, E5M2: 7}[cls]
    for xi, gi in zip(x, got):
        r = ne.round_abs(Fraction(abs(float(xi))))
        if r is None:
            assert sat, (xi, gi)
            r = (ne.vals[-1], ne.bits[-1])
        want = r[1] | ((1 << sign_shift) if np.signbit(xi) else 0)
        assert int(gi) == want, (cls, float(xi), hex(int(gi)), hex(want))


def test_bf16_encode_exhaustive_nearest_even():
    """EVERY finite non-negative bfloat16 value, every midpoint and midpoint +- 1 ulp64,
    both signs (~260k probes), against the vectorised nearest-even search over the
    enumerated value set (gmp_refs.nearest_even_vec; itself cross-checked against the
    scalar rational search below and shown to reject truncation)"""
    bits, vals = refs.bf16_values()
    x = _midpoint_probe(vals)
    x = np.concatenate([x, [1 + 2 ** -8 + 2 ** -40, 2.0 ** -133, 2.0 ** -134, 3 * 2.0 ** -135,
                            2.0 ** -126 * (1 - 2 ** -9)]])
    want, _ = refs.nearest_even_vec(bits, vals, x)
    want = want | np.where(np.signbit(x), 1 << 15, 0)
    got = oracle.encode(x, BF16).astype(np.int64)
    assert np.array_equal(got, want), np.nonzero(got != want)[0][:10]
    # the vectorised reference agrees with the scalar exact-rational one on a sample ...
    pick = np.random.default_rng(0).choice(x.size, size=2000, replace=False)
    _check_nearest_even(BF16, bits, vals, x[pick], sat=False)
    # ... and would catch round-toward-zero (the top 16 bits of the binary32 cast)
    trunc = (x.astype(np.float32).view(np.uint32) >> 16).astype(np.int64)
    assert not np.array_equal(trunc, want)


def test_bf16_double_rounding_vector():
    # 1 + 2^-8 + 2^-40: direct RNE gives 1.0078125; via FP32 it would tie to 1.0
    b = oracle.encode(np.array([1 + 2 ** -8 + 2 ** -40]), BF16)[0]
    assert oracle.decode(np.array([b]), BF16)[0] == 1.0078125


def test_fp16_double_rounding_vector():
    assert oracle.encode(np.array([1 + 2 ** -11 + 2 ** -40]), FP16)[0] == 0x3C01


def test_e4m3_decode_all_256():
    bits, vals = refs.e4m3_values()
    got = oracle.decode(bits, E4M3)
    assert np.array_equal(np.isnan(got), np.isnan(vals))
    ok = ~np.isnan(vals)
    assert np.array_equal(got[ok], vals[ok])
    assert np.nanmax(got) == 448.0 and got[0x01] == 2.0 ** -9


def test_e4m3_encode_exhaustive_nearest_even_satfinite():
    bits, vals = refs.e4m3_values()
    x = _midpoint_probe(vals)
    x = np.concatenate([x, [448.0, 460.0, 464.0, np.nextafter(464.0, 0), np.nextafter(464.0, 1e9),
                            480.0, 1e4, 2.0 ** -10, np.nextafter(2.0 ** -10, 1), 2.0 ** -11]])
    _check_nearest_even(E4M3, bits, vals, x, sat=True)
    # the CUDA satfinite threshold (cuda_fp8.hpp:143-144): 464 -> 448, everything above -> 448
    assert oracle.encode(np.array([464.0]), E4M3)[0] == 0x7E
    assert oracle.encode(np.array([-1e30]), E4M3)[0] == 0xFE


def test_e5m2_decode_all_256_vs_torch_float8():
    """E5M2: every pattern against torch.float8_e5m2 (a library
    decoder) and against the enumeration of the OCP format in tests/gmp_refs.py"""
    import torch
    bits, vals = refs.e5m2_values()
    lib = torch.arange(256, dtype=torch.int32).to(torch.uint8).view(torch.float8_e5m2).to(torch.float64).numpy()
    got = oracle.decode(bits, E5M2)
    for ref in (vals, lib):
        assert np.array_equal(np.isnan(got), np.isnan(ref))
        ok = ~np.isnan(ref)
        assert np.array_equal(got[ok], ref[ok])
    assert np.nanmax(got[np.isfinite(got)]) == 57344.0 and got[0x01] == 2.0 ** -16 and got[0x7C] == np.inf


def test_e5m2_encode_exhaustive_nearest_even():
    bits, vals = refs.e5m2_values()
    fin = np.isfinite(vals)
    x = _midpoint_probe(vals[fin])
    x = np.concatenate([x, [2.0 ** -17, np.nextafter(2.0 ** -17, 1), 3 * 2.0 ** -18, 1 + 2 ** -3 + 2 ** -40]])
    _check_nearest_even(E5M2, bits[fin], vals[fin], x, sat=False)


def test_e5m2_encode_vs_torch_float8():
    """float32-representable probes (random, midpoints, midpoints +- 1 ulp32) against
    torch's float32 -> float8_e5m2 conversion (round to nearest even)"""
    import torch
    _, vals = refs.e5m2_values()
    v = np.unique(vals[np.isfinite(vals) & (vals >= 0)]).astype(np.float32)
    mids = ((v[:-1].astype(np.float64) + v[1:]) / 2).astype(np.float32)    # exact in binary32
    rng = np.random.default_rng(5)
    rnd = (rng.standard_normal(20000) * np.exp2(rng.integers(-18, 16, 20000))).astype(np.float32)
    x = np.concatenate([v, mids, np.nextafter(mids, np.float32(np.inf)), np.nextafter(mids, np.float32(0)), rnd])
    x = np.concatenate([x, -x])
    x = x[np.abs(x) <= 57344.0]
    want = torch.from_numpy(x).to(torch.float8_e5m2).view(torch.uint8).numpy().astype(np.uint32)
    got = oracle.encode(x.astype(np.float64), E5M2)
    assert np.array_equal(got, want)


def test_e5m2_overflow_is_infinity():
    # IEEE-like: RN beyond 57344 (ties at 61440 go to the even 2^16) is +-inf
    got = oracle.encode(np.array([57344.0, 61439.99, 61440.0, 1e9, -1e9]), E5M2)
    assert list(got) == [0x7B, 0x7B, 0x7C, 0x7C, 0xFC]


def test_fp32_encode_vs_hardware_cast():
    rng = np.random.default_rng(1)
    x = np.concatenate([
        rng.standard_normal(100000) * np.exp2(rng.integers(-160, 130, 100000)),
        # exact midpoints between neighbouring floats and +-1ulp64
        *(lambda f: [(f.astype(np.float64) + np.nextafter(f, np.float32(np.inf)).astype(np.float64)) / 2])(
            rng.standard_normal(50000).astype(np.float32)),
        [1 + 2 ** -30, 2.0 ** -149, 2.0 ** -150, 3 * 2.0 ** -151, 2.0 ** 128, 3.4028235677973366e38],
    ])
    x = x[np.isfinite(x)]
    with np.errstate(over="ignore"):
        want = x.astype(np.float32).view(np.uint32)
    got = oracle.encode(x, FP32)
    assert np.array_equal(got, want)
    # 1 + 2^-30 -> 1.0f
    assert oracle.decode(oracle.encode(np.array([1 + 2 ** -30]), FP32), FP32)[0] == 1.0


def test_fp32_roundtrip_identity():
    rng = np.random.default_rng(2)
    f = rng.integers(0, 2 ** 32, 200000, dtype=np.uint64).astype(np.uint32)
    v = f.view(np.float32)
    f = f[np.isfinite(v)]
    back = oracle.encode(oracle.decode(f, FP32), FP32)
    assert np.array_equal(back, f)


@pytest.mark.parametrize("cls,omega", [(FP32, 1.0), (FP16, 65504.0), (BF16, 1.0), (E4M3, 448.0), (E5M2, 57344.0)])
def test_scale_exp_definition(cls, omega):
    """e = largest integer with maxabs*2^e <= Omega' (checked from the definition
    with exact power-of-two scaling), on edges, subnormals and random values."""
    rng = np.random.default_rng(cls)
    ms = list(np.exp2(rng.uniform(-1070, 1020, 3000)))
    ms += [omega, np.nextafter(omega, 0), np.nextafter(omega, np.inf), 0.5, 1.0, 2.0 ** -1074,
           2.0 ** -1022, 1.7976931348623157e308, 0.875, 0.99951171875, 0.9995117187500001]
    for m in ms:
        e = oracle.scale_exp(m, cls)
        assert Fraction(m) * Fraction(2) ** e <= omega
        assert Fraction(m) * Fraction(2) ** (e + 1) > omega
    assert oracle.scale_exp(0.0, cls) == 0


def test_scale_exp_closed_forms():
    # SURVEY 8(c) C2.5 closed forms via frexp(maxabs) = m 2^E
    for x in [0.3, 1.0, 0.5, 65504.0, 700.0, 2.0 ** -30, 0.99951171875 * 8, 0.9995117187500001 * 8]:
        m, E = np.frexp(x)
        assert oracle.scale_exp(x, FP16) == (16 - E if m <= 0.99951171875 else 15 - E)
        assert oracle.scale_exp(x, E4M3) == (9 - E if m <= 0.875 else 8 - E)
        assert oracle.scale_exp(x, E5M2) == (16 - E if m <= 0.875 else 15 - E)   # 57344 = 0.875 2^16
        assert oracle.scale_exp(x, FP32) == (1 - E if m == 0.5 else -E)
