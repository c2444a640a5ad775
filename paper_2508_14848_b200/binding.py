"""Thin ctypes binding of include/gemm_mp.h -- argument marshalling only.

Same names as the C ABI.  Every step of the method runs in libgemm_mp.so's CUDA
kernels; there is no CPU or PyTorch fallback: if the library cannot be loaded
the import fails loudly.  PyTorch is used by callers for device memory and
streams only (pointers are passed as integers)."""
import ctypes as ct
import os
import re

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GMP_LIB_PATH") or os.path.join(_HERE, "libgemm_mp.so")   # override: A/B builds
HEADER = os.path.join(os.path.dirname(_HERE), "include", "gemm_mp.h")

GMP_FP64, GMP_FP32, GMP_FP16, GMP_BF16, GMP_E4M3, GMP_E5M2, GMP_MXFP4 = range(7)
CLASS_NAMES = ["FP64", "FP32", "FP16", "BF16", "E4M3", "E5M2", "MX4"]
NCLS = len(CLASS_NAMES)
TILE_SPLIT, TILE_DIGITS = NCLS, NCLS + 1   # gemm_mp_get_tile cls of the FP32 splits / FP64 digit planes
CLASS_BYTES = [8, 4, 2, 2, 1, 1]


def slot_bytes(cls, nb):
    """bytes of one nb x nb payload slot (MXFP4: nb^2/2 element bytes + nb^2/32 scale bytes)"""
    return nb * nb // 2 + nb * nb // 32 if cls == GMP_MXFP4 else nb * nb * CLASS_BYTES[cls]
GMP_FLAG_SIMT_ONLY = 1
GMP_FLAG_TIMING = 2
GMP_FLAG_FP32_FFMA = 4
GMP_FLAG_FP64_INT8 = 8
GMP_FLAG_SENDER_SIDE = 16
GMP_FLAG_TC_PAIR = 32
GMP_FLAG_LOOPBACK = 256
GMP_FLAG_TC_SINGLE = 512
GMP_FLAG_FP32_X9 = 1024
GMP_FLAG_SPLIT16 = 2048
GMP_FLAG_NCCL_BCAST = 4096
GMP_FLAG_DYN_SCHED = 8192
GMP_FLAG_SPLIT_BN128 = 16384
GMP_FLAG_SEPARATE_MAXABS = 32768
STATUS = ["GMP_OK", "GMP_ERR_ARG", "GMP_ERR_NOT_DIVISIBLE", "GMP_ERR_MAP_SHAPE", "GMP_ERR_NONFINITE",
          "GMP_ERR_GRID", "GMP_ERR_WORKSPACE", "GMP_ERR_STATE", "GMP_ERR_CUDA", "GMP_ERR_NCCL",
          "GMP_ERR_UNSUPPORTED"]


class GmpError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS[code] if 0 <= code < len(STATUS) else code}: {msg}")
        self.code = code


class gmp_desc_t(ct.Structure):
    _fields_ = [("M", ct.c_int64), ("N", ct.c_int64), ("K", ct.c_int64), ("nb", ct.c_int32),
                ("tol", ct.c_double), ("alpha", ct.c_double), ("beta", ct.c_double),
                ("class_mask", ct.c_uint32), ("flags", ct.c_uint32),
                ("P", ct.c_int32), ("Q", ct.c_int32), ("rank", ct.c_int32),
                ("a_map", ct.c_void_p), ("b_map", ct.c_void_p), ("c_map", ct.c_void_p),
                ("row_owner", ct.c_void_p), ("col_owner", ct.c_void_p)]


class gmp_stats_t(ct.Structure):
    _fields_ = [("tiles_a", ct.c_int64 * 7), ("tiles_b", ct.c_int64 * 7), ("tiles_c", ct.c_int64 * 7),
                ("pairs", ct.c_int64 * 7), ("flops", ct.c_double * 7), ("pairs_local", ct.c_int64 * 7),
                ("shadows_local", ct.c_int64 * 7), ("packed_bytes_local", ct.c_int64),
                ("recv_bytes_local", ct.c_int64), ("workspace_bytes", ct.c_int64),
                ("steps", ct.c_int32), ("launches_execute", ct.c_int32),
                ("launches_plan", ct.c_int32), ("launches_convert", ct.c_int32),
                ("class_ms", ct.c_double * 7), ("class_launches", ct.c_int32 * 7),
                ("exec_other_ms", ct.c_double * 3), ("convert_ms", ct.c_double * 4)]

    def as_dict(self):
        d = {}
        for name, _ in self._fields_:
            v = getattr(self, name)
            d[name] = list(v) if hasattr(v, "__len__") else v
        return d


_lib = None


def lib():
    """Loads libgemm_mp.so (raises if it is missing: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                              "(the CUDA path has no fallback)")
        L = ct.CDLL(LIB_PATH)
        vp, i64, i32, u64, st = ct.c_void_p, ct.c_int64, ct.c_int32, ct.c_uint64, ct.c_int
        sig = {
            "gemm_mp_scratch_size": [ct.POINTER(gmp_desc_t), ct.POINTER(ct.c_size_t)],
            "gemm_mp_plan": [ct.POINTER(gmp_desc_t), vp, i64, vp, i64, vp, i64, vp, ct.c_size_t, vp, vp,
                             ct.POINTER(vp)],
            "gemm_mp_workspace_size": [vp, ct.POINTER(ct.c_size_t)],
            "gemm_mp_convert": [vp, vp, ct.c_size_t, vp],
            "gemm_mp_execute": [vp, vp, i64, vp],
            "gemm_mp_execute_after": [vp, vp, i64, vp, vp],
            "gemm_mp_sync": [vp],
            "gemm_mp_get_maps": [vp, vp, vp, vp, vp, vp, vp],
            "gemm_mp_get_tile": [vp, ct.c_char, i64, i64, i32, vp, ct.POINTER(ct.c_size_t),
                                 ct.POINTER(ct.c_int16)],
            "gemm_mp_get_stats": [vp, ct.POINTER(gmp_stats_t)],
            "gemm_mp_get_tile_stats": [vp, ct.c_char, vp, vp, vp],
            "gemm_mp_nccl_unique_id": [vp],
            "gemm_mp_nccl_comm_create": [vp, ct.c_int, ct.c_int, ct.POINTER(vp)],
            "gemm_mp_nccl_comm_destroy": [vp],
            "gemm_mp_loopback_create": [ct.c_int, ct.POINTER(vp)],
            "gemm_mp_loopback_destroy": [vp],
            "gemm_mp_synth": [vp, i64, i64, i64, i32, i32, i32, i32, i32, u64, u64, i32, i32, i32, vp],
            "gemm_mp_synth_tiles": [vp, i64, i64, i64, i32, vp, i64, vp, i64, u64, u64, i32, i32, i32, vp],
            "gemm_mp_balance": [ct.POINTER(gmp_desc_t), vp, vp, vp, vp, vp, vp],
            "gemm_mp_plan_host": [ct.POINTER(gmp_desc_t), vp, vp, vp, vp, vp, vp, ct.POINTER(vp)],
            "gemm_mp_get_schedule": [vp, i32, vp, i64, ct.POINTER(i64)],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = st
        L.gemm_mp_destroy.argtypes = [vp]
        L.gemm_mp_destroy.restype = None
        L.gemm_mp_last_error.argtypes = []
        L.gemm_mp_last_error.restype = ct.c_char_p
        _lib = L
    return _lib


def header_symbols():
    """Entry points declared in include/gemm_mp.h."""
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(gemm_mp_\w+)\s*\(", txt)))


def _check(rc):
    if rc != 0:
        raise GmpError(rc, lib().gemm_mp_last_error().decode())


def _ptr(x):
    if x is None:
        return None
    if isinstance(x, int):
        return x
    return x.data_ptr()


def _stream(s):
    if s is None:
        return None
    if isinstance(s, int):
        return s
    return s.cuda_stream


def make_desc(M, N, K, nb, tol, alpha=1.0, beta=0.0, class_mask=0b01111, flags=0, P=1, Q=1, rank=0,
              a_map=None, b_map=None, c_map=None, row_owner=None, col_owner=None):
    """gmp_desc_t; explicit maps (uint8) and owners (int32) are numpy arrays kept alive on
    the struct."""
    import numpy as np
    maps = [None if m is None else np.ascontiguousarray(m, dtype=np.uint8) for m in (a_map, b_map, c_map)]
    owners = [None if o is None else np.ascontiguousarray(o, dtype=np.int32) for o in (row_owner, col_owner)]
    d = gmp_desc_t(M, N, K, nb, tol, alpha, beta, class_mask, flags, P, Q, rank,
                   *[None if m is None else m.ctypes.data for m in maps + owners])
    d._keep = maps + owners
    return d


def gemm_mp_scratch_size(desc):
    n = ct.c_size_t()
    _check(lib().gemm_mp_scratch_size(ct.byref(desc), ct.byref(n)))
    return n.value


def gemm_mp_plan(desc, A, lda, B, ldb, C, ldc, scratch, scratch_bytes, nccl_comm=None, stream=None):
    h = ct.c_void_p()
    _check(lib().gemm_mp_plan(ct.byref(desc), _ptr(A), lda, _ptr(B), ldb, _ptr(C), ldc, _ptr(scratch),
                              scratch_bytes, nccl_comm, _stream(stream), ct.byref(h)))
    return h.value


def gemm_mp_workspace_size(plan):
    n = ct.c_size_t()
    _check(lib().gemm_mp_workspace_size(plan, ct.byref(n)))
    return n.value


def gemm_mp_convert(plan, ws, ws_bytes, stream=None):
    _check(lib().gemm_mp_convert(plan, _ptr(ws), ws_bytes, _stream(stream)))


def gemm_mp_execute(plan, C, ldc, stream=None):
    _check(lib().gemm_mp_execute(plan, _ptr(C), ldc, _stream(stream)))


def gemm_mp_execute_after(plan, C, ldc, stream=None, c_free_event=None):
    """c_free_event: a torch.cuda.Event (or raw cudaEvent_t int) the C-finalize waits for"""
    ev = c_free_event
    if ev is not None and not isinstance(ev, int):
        ev = ev.cuda_event
    _check(lib().gemm_mp_execute_after(plan, _ptr(C), ldc, _stream(stream), ev or None))


def gemm_mp_sync(plan):
    _check(lib().gemm_mp_sync(plan))


def gemm_mp_get_maps(plan, mt, nt, kt):
    import numpy as np
    a = np.zeros((mt, kt), np.uint8); b = np.zeros((kt, nt), np.uint8); c = np.zeros((mt, nt), np.uint8)
    as_ = np.zeros((mt, kt), np.int16); bs = np.zeros((kt, nt), np.int16); cs = np.zeros((mt, nt), np.int16)
    _check(lib().gemm_mp_get_maps(plan, *[x.ctypes.data for x in (a, b, c, as_, bs, cs)]))
    return dict(acode=a, bcode=b, ccode=c, ascale=as_, bscale=bs, cscale=cs)


def gemm_mp_get_tile(plan, which, ti, tj, cls, nb):
    import numpy as np
    cap = nb * nb * 8
    buf = np.empty(cap, np.uint8)
    n = ct.c_size_t(cap)
    sc = ct.c_int16()
    _check(lib().gemm_mp_get_tile(plan, which.encode() if isinstance(which, str) else which, ti, tj, cls,
                                  buf.ctypes.data, ct.byref(n), ct.byref(sc)))
    return buf[:n.value].copy(), sc.value


def gemm_mp_get_tile_stats(plan, which, rows, cols):
    """global per-tile (S, maxabs, finite) of 'A' / 'B' / 'C' as rows x cols grids"""
    import numpy as np
    S = np.zeros((rows, cols)); M = np.zeros((rows, cols)); F = np.zeros((rows, cols), np.uint8)
    _check(lib().gemm_mp_get_tile_stats(plan, which.encode() if isinstance(which, str) else which,
                                        S.ctypes.data, M.ctypes.data, F.ctypes.data))
    return S, M, F


def gemm_mp_get_stats(plan):
    s = gmp_stats_t()
    _check(lib().gemm_mp_get_stats(plan, ct.byref(s)))
    return s.as_dict()


def gemm_mp_nccl_unique_id():
    buf = (ct.c_char * 128)()
    _check(lib().gemm_mp_nccl_unique_id(buf))
    return bytes(buf)


def gemm_mp_nccl_comm_create(uid, nranks, rank):
    h = ct.c_void_p()
    b = (ct.c_char * 128).from_buffer_copy(uid)
    _check(lib().gemm_mp_nccl_comm_create(b, nranks, rank, ct.byref(h)))
    return h.value


def gemm_mp_nccl_comm_destroy(comm):
    _check(lib().gemm_mp_nccl_comm_destroy(comm))


def gemm_mp_loopback_create(nranks):
    out = ct.c_void_p()
    _check(lib().gemm_mp_loopback_create(nranks, ct.byref(out)))
    return out.value


def gemm_mp_loopback_destroy(comm):
    _check(lib().gemm_mp_loopback_destroy(comm))


def gemm_mp_synth(out, ld, rows, cols, nb, P, Q, p, q, seed, tau, mode, E, s, stream=None):
    _check(lib().gemm_mp_synth(_ptr(out), ld, rows, cols, nb, P, Q, p, q, seed, tau, mode, E, s,
                               _stream(stream)))


def gemm_mp_synth_tiles(out, ld, rows, cols, nb, row_tiles, col_tiles, seed, tau, mode, E, s, stream=None):
    import numpy as np
    rt = np.ascontiguousarray(row_tiles, np.int32)
    ctl = np.ascontiguousarray(col_tiles, np.int32)
    _check(lib().gemm_mp_synth_tiles(_ptr(out), ld, rows, cols, nb, rt.ctypes.data, rt.size, ctl.ctypes.data,
                                     ctl.size, seed, tau, mode, E, s, _stream(stream)))


def gemm_mp_balance(desc, acode, bcode, cost=None):
    """-> (row_owner int32[mt], col_owner int32[nt], (imbalance block-cyclic, balanced))"""
    import numpy as np
    a = np.ascontiguousarray(acode, np.uint8)
    b = np.ascontiguousarray(bcode, np.uint8)
    mt, nt = desc.M // desc.nb, desc.N // desc.nb
    if a.size != mt * (desc.K // desc.nb) or b.size != (desc.K // desc.nb) * nt:
        raise ValueError("acode / bcode shapes do not match desc")
    c = None if cost is None else np.ascontiguousarray(cost, np.float64)
    if c is not None and c.size != NCLS + 1:
        raise ValueError(f"cost must hold {NCLS + 1} doubles")
    ro = np.zeros(mt, np.int32); co = np.zeros(nt, np.int32); imb = np.zeros(2)
    _check(lib().gemm_mp_balance(ct.byref(desc), a.ctypes.data, b.ctypes.data,
                                 None if c is None else c.ctypes.data, ro.ctypes.data, co.ctypes.data,
                                 imb.ctypes.data))
    return ro, co, (float(imb[0]), float(imb[1]))


def gemm_mp_plan_host(desc, acode, bcode, ccode, ascale5, bscale5, cin_scale=None):
    import numpy as np
    arrs = [np.ascontiguousarray(acode, np.uint8), np.ascontiguousarray(bcode, np.uint8),
            np.ascontiguousarray(ccode, np.uint8), np.ascontiguousarray(ascale5, np.int16),
            np.ascontiguousarray(bscale5, np.int16),
            None if cin_scale is None else np.ascontiguousarray(cin_scale, np.int16)]
    # the library reads NCLS scales per tile and one C_in scale per C tile
    for codes, sc, name in ((arrs[0], arrs[3], "ascale5"), (arrs[1], arrs[4], "bscale5")):
        if sc.size != codes.size * NCLS:
            raise ValueError(f"{name} must hold {NCLS} int16 per tile ({codes.size * NCLS}), got {sc.size}")
    if arrs[5] is not None and arrs[5].size != arrs[2].size:
        raise ValueError("cin_scale must hold one int16 per C tile")
    h = ct.c_void_p()
    _check(lib().gemm_mp_plan_host(ct.byref(desc), *[None if a is None else a.ctypes.data for a in arrs],
                                   ct.byref(h)))
    return h.value


def gemm_mp_get_schedule(plan, step):
    import numpy as np
    n = ct.c_int64()
    _check(lib().gemm_mp_get_schedule(plan, step, None, 0, ct.byref(n)))
    out = np.zeros((n.value, 5), np.int64)
    if n.value:
        _check(lib().gemm_mp_get_schedule(plan, step, out.ctypes.data, n.value, ct.byref(n)))
    return out


def gemm_mp_destroy(plan):
    if plan:
        lib().gemm_mp_destroy(plan)


def gemm_mp_last_error():
    return lib().gemm_mp_last_error().decode()
