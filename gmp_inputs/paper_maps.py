"""The paper's own experiment mode: random "aD:bS" tile
precision maps (Fig. 3) and heatmap export.

Exact-count maps (SPEC.md:169-177 reading): round(a/100 * mt*nt) tiles are FP64
(round half away from zero), chosen by a Fisher-Yates shuffle driven by the
sequential SplitMix64 stream of `seed` (swap j = next() mod (i+1), i from last
down to 1); the first nD shuffled indices are FP64, the rest FP32.  Per-matrix
seeds base+1 (A), base+2 (B), base+3 (C).  No arithmetic of the method here: the
maps are INPUTS passed to gemm_mp_plan as explicit a_map / b_map / c_map.
"""
import math

import numpy as np

_M64 = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15


class SplitMix64:
    def __init__(self, seed):
        self.state = seed & _M64

    def next(self):
        self.state = (self.state + GAMMA) & _M64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
        return z ^ (z >> 31)


def n_fp64(d_percent, ntiles):
    x = d_percent / 100.0 * ntiles
    return int(math.floor(x + 0.5)) if x >= 0 else -int(math.floor(-x + 0.5))


def ratio_map(mt, nt, d_percent, seed):
    """uint8 code grid (0 = FP64, 1 = FP32) with exactly n_fp64 FP64 tiles."""
    n = mt * nt
    idx = list(range(n))
    rng = SplitMix64(seed)
    for i in range(n - 1, 0, -1):
        j = rng.next() % (i + 1)
        idx[i], idx[j] = idx[j], idx[i]
    m = np.ones(n, dtype=np.uint8)
    m[idx[:n_fp64(d_percent, n)]] = 0
    return m.reshape(mt, nt)


def paper_maps(mt, nt, kt, d_percent, base_seed):
    """(a_map, b_map, c_map) for A (mt x kt), B (kt x nt), C (mt x nt)."""
    return (ratio_map(mt, kt, d_percent, base_seed + 1), ratio_map(kt, nt, d_percent, base_seed + 2),
            ratio_map(mt, nt, d_percent, base_seed + 3))


def serialize(m):
    """SPEC.md text format: 'mt nt' then rows of D/S (FP64 / FP32 only)."""
    rows = ["".join("D" if c == 0 else "S" for c in r) for r in m]
    return f"{m.shape[0]} {m.shape[1]}\n" + "\n".join(rows) + "\n"


def parse(text):
    lines = text.split("\n")
    mt, nt = (int(x) for x in lines[0].split())
    rows = lines[1:1 + mt]
    if len(rows) != mt or any(len(r) != nt for r in rows):
        raise ValueError("bad map shape")
    if any(ch not in "DS" for r in rows for ch in r):
        raise ValueError("illegal character")
    return np.array([[0 if ch == "D" else 1 for ch in r] for r in rows], dtype=np.uint8)


def heatmap_csv(m):
    """Fig. 3 heatmap as CSV: 64 for FP64 tiles, 32 for FP32 (16 FP16/BF16, 8 E4M3)."""
    val = {0: 64, 1: 32, 2: 16, 3: 16, 4: 8}
    return "".join(",".join(str(val[int(c)]) for c in r) + "\n" for r in m)


def heatmap_pgm(m):
    """Fig. 3 heatmap as plain PGM (P2): FP64 dark (0) ... lowest class light (255)."""
    val = {0: 0, 1: 255, 2: 255, 3: 255, 4: 255}
    body = "".join(" ".join(str(val[int(c)]) for c in r) + "\n" for r in m)
    return f"P2\n{m.shape[1]} {m.shape[0]}\n255\n" + body
