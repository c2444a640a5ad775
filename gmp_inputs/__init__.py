"""Seeded synthetic inputs shared by the tests, the oracle side and the GPU side.

Holds NO arithmetic of the method (no norms, no rounding to a class, no GEMM):
only the counter-based SplitMix64 recipe that produces binary64 matrices with a
controlled per-tile norm spread, and the workload
table of BASELINE.json's five configs.  The CUDA generator kernel and the C
oracle each implement the same recipe independently; tests check all three
agree bit for bit.

x(r,c) = v(r,c) * 2^(s - e(r//nb, c//nb))
v(r,c) = ((mix(seed + (r*cols + c + 1)*GAMMA) >> 11) * 2^-53) * 2 - 1
e      = 0 (uniform) | floor((ti+tj)*E / max(1, mt+nt-2)) (graded)
         | mix(tau + (ti*nt + tj + 1)*GAMMA) mod (E+1) (random)
"""
import dataclasses

import numpy as np

GAMMA = 0x9E3779B97F4A7C15
MODES = {"uniform": 0, "graded": 1, "random": 2}
_M64 = (1 << 64) - 1


def mix64(z):
    """SplitMix64 finaliser on a numpy uint64 array (wraps mod 2^64)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def splitmix_outputs(seed, idx):
    """Outputs number idx (>= 1) of the SplitMix64 stream seeded with `seed`."""
    idx = np.asarray(idx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        st = np.uint64(seed & _M64) + idx * np.uint64(GAMMA)
    return mix64(st)


def uniform_from_u64(u):
    return ((u >> np.uint64(11)).astype(np.float64) * 2.0 ** -53) * 2.0 - 1.0


def tile_exponents(mt, nt, mode, E, tau):
    ti, tj = np.meshgrid(np.arange(mt, dtype=np.int64), np.arange(nt, dtype=np.int64), indexing="ij")
    m = MODES[mode] if isinstance(mode, str) else mode
    if m == 0:
        return np.zeros((mt, nt), dtype=np.int64)
    if m == 1:
        den = max(1, mt + nt - 2)
        return ((ti + tj) * E) // den
    u = splitmix_outputs(tau, (ti * nt + tj + 1).astype(np.uint64))
    return (u % np.uint64(E + 1)).astype(np.int64)


def synth_block(rows, cols, nb, seed, mode, E, s, tau, r0=0, nr=None, c0=0, nc=None):
    """Rows [r0, r0+nr) x cols [c0, c0+nc) of the synthetic rows x cols matrix."""
    nr = rows if nr is None else nr
    nc = cols if nc is None else nc
    r = np.arange(r0, r0 + nr, dtype=np.uint64)[:, None]
    c = np.arange(c0, c0 + nc, dtype=np.uint64)[None, :]
    with np.errstate(over="ignore"):
        idx = r * np.uint64(cols) + c + np.uint64(1)
    v = uniform_from_u64(splitmix_outputs(seed, idx))
    ex = tile_exponents(rows // nb, cols // nb, mode, E, tau)
    e = ex[(np.arange(r0, r0 + nr) // nb)[:, None], (np.arange(c0, c0 + nc) // nb)[None, :]]
    return np.ldexp(v, (s - e).astype(np.int32))


@dataclasses.dataclass(frozen=True)
class MatrixRecipe:
    seed: int
    mode: str
    E: int
    s: int

    @property
    def tau(self):
        return self.seed + 100


@dataclasses.dataclass(frozen=True)
class Workload:
    """One BASELINE.json config: shapes, tile, tolerance, scalars, class mask, recipes."""
    name: str
    M: int
    N: int
    K: int
    nb: int
    tol: float
    alpha: float
    beta: float
    class_mask: int
    a: MatrixRecipe
    b: MatrixRecipe
    c: MatrixRecipe

    def matrices(self):
        A = synth_block(self.M, self.K, self.nb, self.a.seed, self.a.mode, self.a.E, self.a.s, self.a.tau)
        B = synth_block(self.K, self.N, self.nb, self.b.seed, self.b.mode, self.b.E, self.b.s, self.b.tau)
        C = synth_block(self.M, self.N, self.nb, self.c.seed, self.c.mode, self.c.E, self.c.s, self.c.tau)
        return A, B, C

    @property
    def flops(self):
        return 2.0 * self.M * self.N * self.K


NO_E4M3 = 0b01111
WITH_E4M3 = 0b11111
WITH_MX4 = 0b1000000   # class 6, MXFP4 (R31)


def _rec(cfg, k, mode, E, s=0):
    return MatrixRecipe(1000 * cfg + k, mode, E, s)


def workload(cfg, variant=None):
    """BASELINE.json configs[cfg-1]."""
    if cfg == 1:
        return Workload("cfg1_N512_nb128_tol1e-6", 512, 512, 512, 128, 1e-6, 1.0,
                        0.0 if variant == "beta0" else 1.0, NO_E4M3,
                        _rec(1, 1, "graded", 14), _rec(1, 2, "graded", 14), _rec(1, 3, "graded", 14))
    if cfg == 2:
        return Workload("cfg2_N16384_nb1024_tol1e-8", 16384, 16384, 16384, 1024, 1e-8, 1.0, 1.0, NO_E4M3,
                        _rec(2, 1, "random", 22), _rec(2, 2, "random", 22), _rec(2, 3, "random", 22))
    if cfg == 3:
        return Workload("cfg3_N65536_nb2048_tol1e-4", 65536, 65536, 65536, 2048, 1e-4, 1.0, 0.0, NO_E4M3,
                        _rec(3, 1, "random", 32), _rec(3, 2, "random", 32), _rec(3, 3, "random", 32))
    if cfg == 4:
        # variant "mx4": the same data with MXFP4 (class 6, NEXT-4) enabled as well
        mx = variant == "mx4"
        return Workload("cfg4_N65536_nb2048_tol1e-2_e4m3" + ("_mx4" if mx else ""), 65536, 65536, 65536, 2048,
                        1e-2, 1.0, 0.0, WITH_E4M3 | (WITH_MX4 if mx else 0),
                        _rec(4, 1, "random", 40), _rec(4, 2, "random", 40), _rec(4, 3, "random", 40))
    if cfg == 5:
        E = 0 if variant in (None, "uniform", "uniform_1e-2") else int(variant[1:])
        mode = "uniform" if E == 0 else "random"
        tol = 1e-2 if variant == "uniform_1e-2" else 1e-4
        return Workload(f"cfg5_32768x32768x131072_nb2048_{variant or 'uniform'}", 32768, 32768, 131072, 2048,
                        tol, 1.0, 0.0, NO_E4M3, _rec(5, 1, mode, E), _rec(5, 2, mode, E), _rec(5, 3, mode, E))
    raise ValueError(cfg)


def small_workload(M, N, K, nb, tol, mode="graded", E=14, alpha=1.0, beta=1.0,
                   class_mask=NO_E4M3, seed=77, s=0):
    """Scaled-down workload with the same recipe (parity tests)."""
    return Workload(f"small_{M}x{N}x{K}_nb{nb}", M, N, K, nb, tol, alpha, beta, class_mask,
                    MatrixRecipe(seed + 1, mode, E, s), MatrixRecipe(seed + 2, mode, E, s),
                    MatrixRecipe(seed + 3, mode, E, s))
