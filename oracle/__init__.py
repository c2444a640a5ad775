"""CPU oracle for the tile-centric mixed-precision GEMM (arxiv 2508.14848).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py.  The product package
(paper_2508_14848_b200) never imports it.  The arithmetic lives in
gemm_mp_oracle.c (plain C, -ffp-contract=off); this file only marshals numpy
arrays through ctypes.  Every definition is in DESIGN.md "Oracle definitions".
"""
import ctypes as ct
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gemm_mp_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-shared", "-fPIC"]


def build(force=False):
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", *CFLAGS, "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ct.CDLL(_LIB)
        u64, i64, i32, dbl, vp = ct.c_uint64, ct.c_int64, ct.c_int32, ct.c_double, ct.c_void_p
        L.orc_mix64.restype = u64; L.orc_mix64.argtypes = [u64]
        L.orc_splitmix_output.restype = u64; L.orc_splitmix_output.argtypes = [u64, u64]
        L.orc_uniform.restype = dbl; L.orc_uniform.argtypes = [u64]
        L.orc_synth_block.restype = None
        L.orc_synth_block.argtypes = [i64, i64, i32, u64, ct.c_int, ct.c_int, ct.c_int, u64,
                                      i64, i64, i64, i64, vp, i64]
        L.orc_encode.restype = ct.c_uint32; L.orc_encode.argtypes = [dbl, ct.c_int]
        L.orc_decode.restype = dbl; L.orc_decode.argtypes = [ct.c_uint32, ct.c_int]
        L.orc_encode_array.argtypes = [vp, i64, ct.c_int, vp]
        L.orc_decode_array.argtypes = [vp, i64, ct.c_int, vp]
        L.orc_scale_exp.restype = ct.c_int; L.orc_scale_exp.argtypes = [dbl, ct.c_int]
        L.orc_cnorm.restype = dbl; L.orc_cnorm.argtypes = [vp, i64, i32]
        L.orc_tile_stats.argtypes = [vp, i64, i64, i64, i32, vp, vp, vp]
        L.orc_delta.restype = dbl; L.orc_delta.argtypes = [ct.c_int, i32]
        L.orc_map_input.restype = ct.c_int
        L.orc_map_input.argtypes = [i64, i64, i32, dbl, ct.c_uint32, vp, vp, vp, vp, vp]
        L.orc_pack_tile.argtypes = [vp, i64, i32, ct.c_int, ct.c_int, ct.c_int, vp]
        L.orc_shadow_tile.restype = ct.c_int
        L.orc_shadow_tile.argtypes = [vp, i32, ct.c_int, ct.c_int, ct.c_int, ct.c_int, vp]
        L.orc_layout_transposed.restype = ct.c_int
        L.orc_layout_transposed.argtypes = [ct.c_int, ct.c_int]
        L.orc_tile_gemm.argtypes = [ct.c_int, vp, vp, i32, vp]
        L.orc_acc_init.argtypes = [i32, ct.c_int, dbl, vp, ct.c_int, vp]
        L.orc_fold.argtypes = [i32, ct.c_int, dbl, ct.c_int, ct.c_int, vp, vp]
        L.orc_finalize.restype = ct.c_int
        L.orc_finalize.argtypes = [i32, ct.c_int, vp, vp, vp, i64]
        L.orc_gemm_mp.restype = ct.c_int
        L.orc_gemm_mp.argtypes = [vp, vp, i64, vp, i64, vp, i64, vp, i64, vp, i64, vp]
        L.orc_gemm_mp_synth.restype = ct.c_int
        L.orc_gemm_mp_synth.argtypes = [vp, vp, vp, vp, vp, vp, i64, vp]
        L.orc_max_threads.restype = ct.c_int
        L.orc_class_bytes.restype = ct.c_int; L.orc_class_bytes.argtypes = [ct.c_int]
        L.orc_payload_bytes.restype = i64; L.orc_payload_bytes.argtypes = [ct.c_int, i32]
        L.orc_mx_block_exp.restype = ct.c_int; L.orc_mx_block_exp.argtypes = [dbl]
        L.orc_mx_encode.argtypes = [vp, i32, vp]
        L.orc_payload_value.restype = dbl; L.orc_payload_value.argtypes = [vp, i32, i64, ct.c_int]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ct.c_void_p) if a is not None else None


PAYLOAD_DTYPE = {0: np.uint64, 1: np.uint32, 2: np.uint16, 3: np.uint16, 4: np.uint8, 5: np.uint8, 6: np.uint8}
CLASS_NAMES = ["FP64", "FP32", "FP16", "BF16", "E4M3", "E5M2", "MX4"]
NCLS = len(CLASS_NAMES)
MX = 6   # MXFP4: E2M1 elements + one E8M0 scale per 32 K-elements (R31)


def payload_len(cls, nb):
    """elements of the payload array (PAYLOAD_DTYPE[cls]) of one nb x nb tile"""
    return int(lib().orc_payload_bytes(cls, nb)) if cls == MX else nb * nb


# ---- O1 generator -----------------------------------------------------------
def splitmix_output(seed, i):
    return int(lib().orc_splitmix_output(seed, i))


def synth_block(rows, cols, nb, seed, mode, E, s, tau, r0=0, nr=None, c0=0, nc=None):
    nr = rows if nr is None else nr
    nc = cols if nc is None else nc
    out = np.empty((nr, nc), dtype=np.float64)
    lib().orc_synth_block(rows, cols, nb, seed, mode, E, s, tau, r0, nr, c0, nc, _p(out), nc)
    return out


# ---- O2 converters ----------------------------------------------------------
def encode(x, cls):
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty(x.shape, dtype=np.uint32)
    lib().orc_encode_array(_p(x), x.size, cls, _p(out))
    return out


def decode(bits, cls):
    b = np.ascontiguousarray(bits, dtype=np.uint32)
    out = np.empty(b.shape, dtype=np.float64)
    lib().orc_decode_array(_p(b), b.size, cls, _p(out))
    return out


def scale_exp(maxabs, cls):
    return int(lib().orc_scale_exp(float(maxabs), cls))


def delta(cls, nb):
    return float(lib().orc_delta(cls, nb))


# ---- O4 norms / stats -------------------------------------------------------
def cnorm(tile):
    t = np.ascontiguousarray(tile, dtype=np.float64)
    return float(lib().orc_cnorm(_p(t), t.shape[1], t.shape[0]))


def tile_stats(X, nb):
    X = np.ascontiguousarray(X, dtype=np.float64)
    mt, nt = X.shape[0] // nb, X.shape[1] // nb
    S = np.empty(mt * nt); M = np.empty(mt * nt); F = np.empty(mt * nt, dtype=np.uint8)
    lib().orc_tile_stats(_p(X), X.shape[1], mt, nt, nb, _p(S), _p(M), _p(F))
    return S.reshape(mt, nt), M.reshape(mt, nt), F.reshape(mt, nt)


# ---- O5 map of an input matrix --------------------------------------------
def map_input(S, M, nb, tol, class_mask, finite=None):
    S = np.ascontiguousarray(S, dtype=np.float64); M = np.ascontiguousarray(M, dtype=np.float64)
    F = np.ones(S.shape, np.uint8) if finite is None else np.ascontiguousarray(finite, np.uint8)
    code = np.empty(S.shape, np.uint8); scale = np.empty(S.shape, np.int16)
    rc = lib().orc_map_input(S.shape[0], S.shape[1], nb, tol, class_mask, _p(S), _p(M), _p(F),
                             _p(code), _p(scale))
    return rc, code, scale


# ---- O6 packing / shadows -------------------------------------------------
ROLE = {"A": 0, "B": 1, "C": 2}


def layout_transposed(role, cls):
    """payload layout of a tile of matrix role ('A', 'B', 'C') at class cls (O6)"""
    return bool(lib().orc_layout_transposed(ROLE.get(role, role), cls))


def pack_tile(tile, cls, scale, transpose=False, role=None):
    """payload of one tile; pass role='A'/'B'/'C' to use the library layout of O6"""
    t = np.ascontiguousarray(tile, dtype=np.float64)
    nb = t.shape[0]
    if role is not None:
        transpose = layout_transposed(role, cls)
    out = np.empty(payload_len(cls, nb), dtype=PAYLOAD_DTYPE[cls])
    lib().orc_pack_tile(_p(t), nb, nb, cls, scale, int(transpose), _p(out))
    return out


def shadow_tile(payload, nb, frm, frm_scale, to, role="A"):
    out = np.empty(payload_len(to, nb), dtype=PAYLOAD_DTYPE[to])
    p = np.ascontiguousarray(payload)
    e = lib().orc_shadow_tile(_p(p), nb, ROLE.get(role, role), frm, frm_scale, to, _p(out))
    return out, int(e)


def payload_values(payload, cls, nb=None):
    """exact values (scaled units) in payload-index order; MXFP4 needs nb"""
    if cls == 0:
        return np.ascontiguousarray(payload).view(np.float64).copy()
    if cls == MX:
        p = np.ascontiguousarray(payload, np.uint8)
        n = nb * nb
        q = np.empty(n, np.uint32)
        q[0::2] = p[:n // 2] & 15
        q[1::2] = p[:n // 2] >> 4
        s = p[n // 2:n // 2 + n // 32].astype(np.int64) - 127
        return decode(q, MX) * np.ldexp(1.0, np.repeat(s, 32))
    return decode(payload.astype(np.uint32), cls)


def mx_block_exp(amax):
    return int(lib().orc_mx_block_exp(float(amax)))


def mx_encode(y, nb):
    """O6 MXFP4 block encoding of values y (scaled units, payload-index order)"""
    y = np.ascontiguousarray(y, np.float64).ravel()
    out = np.empty(payload_len(MX, nb), np.uint8)
    lib().orc_mx_encode(_p(y), nb, _p(out))
    return out


# ---- O8 / O9 ----------------------------------------------------------------
def tile_gemm(cls, a_payload, b_payload, nb):
    P = np.empty(nb * nb, dtype=np.float64)
    lib().orc_tile_gemm(cls, _p(np.ascontiguousarray(a_payload)),
                        _p(np.ascontiguousarray(b_payload)), nb, _p(P))
    return P.reshape(nb, nb)


class _Desc(ct.Structure):
    _fields_ = [("M", ct.c_int64), ("N", ct.c_int64), ("K", ct.c_int64), ("nb", ct.c_int32),
                ("tol", ct.c_double), ("alpha", ct.c_double), ("beta", ct.c_double),
                ("class_mask", ct.c_uint32),
                ("a_map", ct.c_void_p), ("b_map", ct.c_void_p), ("c_map", ct.c_void_p)]


class _Out(ct.Structure):
    _fields_ = [("acode", ct.c_void_p), ("bcode", ct.c_void_p), ("ccode", ct.c_void_p),
                ("ascale5", ct.c_void_p), ("bscale5", ct.c_void_p), ("cscale", ct.c_void_p),
                ("cin_scale", ct.c_void_p),
                ("SA", ct.c_void_p), ("MA", ct.c_void_p), ("SB", ct.c_void_p),
                ("MB", ct.c_void_p), ("SC", ct.c_void_p), ("MC", ct.c_void_p),
                ("threads", ct.c_int), ("W", ct.c_void_p), ("ldw", ct.c_int64)]


def gemm_mp(A, B, C, nb, tol, alpha=1.0, beta=0.0, class_mask=0b01111, ctiles=None,
            a_map=None, b_map=None, c_map=None, Cout=None, want_w=True):
    """Run the whole method (O1-O9).  Returns a dict with maps, scales and C, and
    (want_w) "W": the final W accumulator of every computed C tile (binary64 array
    holding the exact binary64 / binary32 W values, SURVEY 8(c) C6 debug export).

    ctiles: optional list of C tile indices i*nt+j to compute (sampled runs);
    tiles not listed are left as in `Cout` (default: zeros)."""
    A = np.ascontiguousarray(A, np.float64); B = np.ascontiguousarray(B, np.float64)
    M, K = A.shape; K2, N = B.shape
    assert K == K2
    C = np.zeros((M, N)) if C is None else np.ascontiguousarray(C, np.float64)
    mt, nt, kt = M // nb, N // nb, K // nb
    maps = [None if m is None else np.ascontiguousarray(m, np.uint8) for m in (a_map, b_map, c_map)]
    d = _Desc(M, N, K, nb, tol, alpha, beta, class_mask, *[_p(m) for m in maps])
    o = dict(acode=np.zeros((mt, kt), np.uint8), bcode=np.zeros((kt, nt), np.uint8),
             ccode=np.zeros((mt, nt), np.uint8), ascale5=np.zeros((mt, kt, NCLS), np.int16),
             bscale5=np.zeros((kt, nt, NCLS), np.int16), cscale=np.zeros((mt, nt), np.int16),
             cin_scale=np.zeros((mt, nt), np.int16),
             SA=np.zeros((mt, kt)), MA=np.zeros((mt, kt)), SB=np.zeros((kt, nt)),
             MB=np.zeros((kt, nt)), SC=np.zeros((mt, nt)), MC=np.zeros((mt, nt)))
    W = np.zeros((M, N)) if want_w else None
    out = _Out(*[_p(o[k]) for k in ["acode", "bcode", "ccode", "ascale5", "bscale5", "cscale",
                                     "cin_scale", "SA", "MA", "SB", "MB", "SC", "MC"]], 0, _p(W), N)
    Cout = np.zeros((M, N)) if Cout is None else Cout
    tl = None if ctiles is None else np.ascontiguousarray(ctiles, np.int64)
    rc = lib().orc_gemm_mp(ct.byref(d), _p(A), K, _p(B), N, _p(C), N, _p(Cout), N, _p(tl),
                           0 if tl is None else tl.size, ct.byref(out))
    o["rc"] = rc
    o["C"] = Cout
    o["W"] = W
    o["threads"] = out.threads
    return o


class _Synth(ct.Structure):
    _fields_ = [("seed", ct.c_uint64), ("tau", ct.c_uint64), ("mode", ct.c_int), ("E", ct.c_int), ("s", ct.c_int)]


_MODES = {"uniform": 0, "graded": 1, "random": 2}


def gemm_mp_synth(M, N, K, nb, tol, gen_a, gen_b, gen_c, ctiles, alpha=1.0, beta=0.0, class_mask=0b01111,
                  want_w=True):
    """The whole method (O1-O9) on the synthetic workload, generated tile by tile (the
    inputs are never materialised: N = 65536 fits).  gen_x: (seed, mode, E, s, tau) of the
    O1 recipe (mode 'uniform' / 'graded' / 'random' or 0/1/2).  Returns the maps, scales
    and stats of every tile as gemm_mp does, and the listed C tiles (and their final W)
    as arrays of shape (len(ctiles), nb, nb) in list order."""
    mt, nt, kt = M // nb, N // nb, K // nb

    def syn(g):
        seed, mode, E, s_, tau = g
        return _Synth(seed, tau, _MODES.get(mode, mode), E, s_)

    d = _Desc(M, N, K, nb, tol, alpha, beta, class_mask, None, None, None)
    o = dict(acode=np.zeros((mt, kt), np.uint8), bcode=np.zeros((kt, nt), np.uint8),
             ccode=np.zeros((mt, nt), np.uint8), ascale5=np.zeros((mt, kt, NCLS), np.int16),
             bscale5=np.zeros((kt, nt, NCLS), np.int16), cscale=np.zeros((mt, nt), np.int16),
             cin_scale=np.zeros((mt, nt), np.int16),
             SA=np.zeros((mt, kt)), MA=np.zeros((mt, kt)), SB=np.zeros((kt, nt)),
             MB=np.zeros((kt, nt)), SC=np.zeros((mt, nt)), MC=np.zeros((mt, nt)))
    tl = np.ascontiguousarray(ctiles, np.int64)
    Ct = np.zeros((tl.size, nb, nb))
    W = np.zeros((tl.size, nb, nb)) if want_w else None
    out = _Out(*[_p(o[k]) for k in ["acode", "bcode", "ccode", "ascale5", "bscale5", "cscale",
                                     "cin_scale", "SA", "MA", "SB", "MB", "SC", "MC"]], 0, _p(W), nb)
    ga, gb, gc = syn(gen_a), syn(gen_b), syn(gen_c)
    o["rc"] = lib().orc_gemm_mp_synth(ct.byref(d), ct.byref(ga), ct.byref(gb), ct.byref(gc), _p(Ct), _p(tl),
                                      tl.size, ct.byref(out))
    o["C"], o["W"], o["threads"] = Ct, W, out.threads
    return o


def max_threads():
    return int(lib().orc_max_threads())


def finalize(acc, code):
    """O9 finalize of one C tile's W accumulator (binary64 array of exact W values):
    returns (packed payload, user binary64 tile, scale)."""
    a = np.ascontiguousarray(acc, dtype=np.float64)
    nb = a.shape[0]
    pay = np.empty(nb * nb, dtype=PAYLOAD_DTYPE[code])
    user = np.empty((nb, nb), dtype=np.float64)
    e = lib().orc_finalize(nb, code, _p(a), _p(pay), _p(user), nb)
    return pay, user, int(e)
