"""Independent references used to PIN the oracle (tests only).

Nothing here re-types an oracle formula: rounding is done by nearest-neighbour
search over the enumerated set of representable values (built from the format
definitions, IEEE-754 / OCP FP8), exact arithmetic uses fractions.Fraction, and
binary32/binary64 rounding of rationals is chosen among hardware neighbours by
exact distance.
"""
import bisect
from fractions import Fraction

import numpy as np

# ---- enumerated value sets, straight from the format definitions -------------


def fp16_values():
    """all 2^16 patterns -> value via numpy's IEEE binary16 (hardware/library)."""
    bits = np.arange(1 << 16, dtype=np.uint16)
    return bits, bits.view(np.float16).astype(np.float64)


def bf16_values():
    """bfloat16 = top half of binary32: value of pattern b is float32(b << 16)."""
    bits = np.arange(1 << 16, dtype=np.uint32)
    return bits, (bits << np.uint32(16)).view(np.float32).astype(np.float64)


def e4m3_values():
    """OCP FP8 E4M3 ("FN"): bias 7, no infinities, S.1111.111 = NaN, max 448."""
    vals = []
    for b in range(256):
        s = -1.0 if b & 0x80 else 1.0
        e = (b >> 3) & 0xF
        m = b & 7
        if e == 15 and m == 7:
            vals.append(np.nan)
        elif e == 0:
            vals.append(s * m * 2.0 ** -9)
        else:
            vals.append(s * (1 + m / 8) * 2.0 ** (e - 7))
    return np.arange(256, dtype=np.uint32), np.array(vals)


def e5m2_values():
    """OCP FP8 E5M2: bias 15, IEEE-like (S.11111.00 = inf, S.11111.xx = NaN), max 57344."""
    vals = []
    for b in range(256):
        s = -1.0 if b & 0x80 else 1.0
        e = (b >> 2) & 0x1F
        m = b & 3
        if e == 31:
            vals.append(s * np.inf if m == 0 else np.nan)
        elif e == 0:
            vals.append(s * m * 2.0 ** -16)
        else:
            vals.append(s * (1 + m / 4) * 2.0 ** (e - 15))
    return np.arange(256, dtype=np.uint32), np.array(vals)


class NearestEven:
    """Round-to-nearest, ties to the pattern with even last bit, over a value set."""

    def __init__(self, bits, vals, overflow):
        fin = np.isfinite(vals) & (vals >= 0)
        pos = sorted(set((float(v), int(b)) for b, v in zip(bits[fin], vals[fin])), key=lambda t: t[0])
        # drop -0/+0 duplicates: keep the +0 pattern
        seen = {}
        for v, b in pos:
            if v not in seen or b < seen[v]:
                seen[v] = b
        self.vals = sorted(seen)
        self.bits = [seen[v] for v in self.vals]
        self.fr = [Fraction(v) for v in self.vals]
        self.overflow = overflow  # callable(sign) -> bits, used above max + half ulp
        self.sign_bit = None

    def round_abs(self, a: Fraction):
        """returns (value, bits) of RN(a) for a >= 0, or None on overflow"""
        i = bisect.bisect_left(self.fr, a)
        if i < len(self.fr) and self.fr[i] == a:
            return self.vals[i], self.bits[i]
        if i == len(self.fr):
            # above max: compare with the virtual next value (max + ulp)
            top, prev = self.fr[-1], self.fr[-2]
            nxt = top + (top - prev)
            if a - top < nxt - a:
                return self.vals[-1], self.bits[-1]
            if a - top == nxt - a and self.bits[-1] % 2 == 0:
                return self.vals[-1], self.bits[-1]
            return None
        lo, hi = self.fr[i - 1], self.fr[i]
        if a - lo < hi - a:
            return self.vals[i - 1], self.bits[i - 1]
        if hi - a < a - lo:
            return self.vals[i], self.bits[i]
        j = i - 1 if self.bits[i - 1] % 2 == 0 else i
        return self.vals[j], self.bits[j]


# ---- rounding of rationals to binary32 / binary64 ---------------------------


def rn64(x: Fraction) -> float:
    return float(x)  # Python's Fraction.__float__ is correctly rounded (RNE)


def rn32(x: Fraction) -> np.float32:
    """RNE to binary32: nearest among the hardware neighbours of a first guess."""
    f = np.float32(float(x))
    cands = {f, np.nextafter(f, np.float32(np.inf)), np.nextafter(f, np.float32(-np.inf))}
    best = None
    for c in cands:
        if not np.isfinite(c):
            continue
        dist = abs(Fraction(float(c)) - x)
        key = (dist, int(np.array(c, dtype=np.float32).view(np.uint32)) & 1)
        if best is None or key < best[0]:
            best = (key, c)
    return np.float32(best[1])


def gamma(n, u):
    return n * u / (1 - n * u)


def nearest_even_vec(bits, vals, x):
    """Vectorised round-to-nearest-even of the binary64 probes x (finite, |x| <= max
    representable) over the enumerated value set: the same rule as NearestEven, fast
    enough for an exhaustive probe set.  The neighbours lo <= |x| <= hi come from a
    binary search; the distances |x| - lo and hi - |x| are exact in binary64 wherever
    Sterbenz's lemma applies (lo <= |x| <= 2 lo, |x| <= hi <= 2|x|) -- every probe
    near a tie; the others are decided by a margin far above rounding error and, if
    not, by exact rationals.  Returns the bit patterns with the sign bit of x at
    `sign_shift`."""
    fin = np.isfinite(vals) & (vals >= 0)
    v, b = vals[fin], bits[fin].astype(np.int64)
    order = np.lexsort((b, v))             # ascending value, then the smaller pattern (+0 before -0)
    v, b = v[order], b[order]
    keep = np.concatenate([[True], v[1:] != v[:-1]])
    v, b = v[keep], b[keep]
    a = np.abs(x)
    i = np.searchsorted(v, a, side="left")
    exact_hit = (i < v.size) & (v[np.minimum(i, v.size - 1)] == a)
    i = np.clip(i, 1, v.size - 1)
    lo, hi = v[i - 1], v[i]
    d1, d2 = a - lo, hi - a
    sterbenz = ((lo == 0) | (a <= 2 * lo)) & (hi <= 2 * a)
    far = (np.maximum(d1, d2) > 1.01 * np.minimum(d1, d2))
    pick_hi = (d2 < d1) | ((d1 == d2) & (b[i - 1] % 2 == 1))
    out = np.where(pick_hi, b[i], b[i - 1])
    out = np.where(exact_hit, b[np.searchsorted(v, a, side="left").clip(0, v.size - 1)], out)
    slow = ~exact_hit & ~sterbenz & ~far
    for k in np.nonzero(slow)[0]:            # exact rationals (rare)
        fa, flo, fhi = Fraction(float(a[k])), Fraction(float(lo[k])), Fraction(float(hi[k]))
        if fa - flo < fhi - fa or (fa - flo == fhi - fa and b[i[k] - 1] % 2 == 0):
            out[k] = b[i[k] - 1]
        else:
            out[k] = b[i[k]]
    return out, int(slow.sum())
