"""CPU-side checks of the C-ABI library: it loads, exports every entry point the
header declares, and validates arguments without touching a GPU."""
import ctypes as ct

import pytest

from paper_2508_14848_b200 import binding as B


def test_library_exports_every_header_symbol():
    L = B.lib()
    syms = B.header_symbols()
    assert len(syms) >= 14
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing


@pytest.mark.parametrize("kw,code", [
    (dict(M=1000, N=1024, K=1024, nb=128), "GMP_ERR_NOT_DIVISIBLE"),
    (dict(M=1024, N=1024, K=1024, nb=96), "GMP_ERR_NOT_DIVISIBLE"),
    (dict(M=1024, N=1024, K=1024, nb=128, tol=0.0), "GMP_ERR_ARG"),
    (dict(M=1024, N=1024, K=1024, nb=128, tol=float("inf")), "GMP_ERR_ARG"),
    (dict(M=1024, N=1024, K=1024, nb=128, P=2, Q=2, rank=4), "GMP_ERR_GRID"),
])
def test_scratch_size_validates(kw, code):
    args = dict(tol=1e-6)
    args.update(kw)
    d = B.make_desc(**args)
    with pytest.raises(B.GmpError) as e:
        B.gemm_mp_scratch_size(d)
    assert code in str(e.value)


def test_scratch_size_is_small():
    d = B.make_desc(65536, 65536, 65536, 2048, 1e-4)
    n = B.gemm_mp_scratch_size(d)
    assert 0 < n < 1 << 20


def test_null_plan_is_rejected():
    with pytest.raises(B.GmpError):
        B.gemm_mp_workspace_size(None)
    B.gemm_mp_destroy(None)  # NULL-safe


@pytest.mark.parametrize("kw", [dict(M=0, N=128, K=128), dict(M=128, N=-128, K=128), dict(M=128, N=128, K=0)])
def test_empty_or_negative_shapes_rejected(kw):
    d = B.make_desc(nb=128, tol=1e-6, **kw)
    with pytest.raises(B.GmpError) as e:
        B.gemm_mp_scratch_size(d)
    assert "GMP_ERR_ARG" in str(e.value)


def test_host_plan_rejects_bad_codes():
    import numpy as np
    d = B.make_desc(256, 256, 256, 128, 1e-6)
    bad = np.full((2, 2), 7, np.uint8)   # code 7: beyond MXFP4 (6)
    z = np.zeros((2, 2, B.NCLS), np.int16)
    with pytest.raises(B.GmpError) as e:
        B.gemm_mp_plan_host(d, bad, bad, bad, z, z)
    assert "GMP_ERR_MAP_SHAPE" in str(e.value)


def test_host_plan_checks_scale_array_sizes():
    """the binding refuses scale arrays shorter than NCLS entries per tile (the library
    would read past them)"""
    import numpy as np
    d = B.make_desc(256, 256, 256, 128, 1e-6)
    c = np.zeros((2, 2), np.uint8)
    with pytest.raises(ValueError):
        B.gemm_mp_plan_host(d, c, c, c, np.zeros((2, 2, B.NCLS - 1), np.int16), np.zeros((2, 2, B.NCLS), np.int16))
    pl = B.gemm_mp_plan_host(d, c, c, c, np.zeros((2, 2, B.NCLS), np.int16), np.zeros((2, 2, B.NCLS), np.int16))
    B.gemm_mp_destroy(pl)


def test_merged_16bit_launch_plan():
    """host plan only: with FP16 and BF16 pairs in each SUMMA step the default plan runs them
    in one k_tc_class<3> launch (R33); GMP_FLAG_SPLIT16 keeps one launch per class; the
    per-class launch counts still name every class present"""
    import numpy as np
    nb, t = 128, 4
    d0 = B.make_desc(t * nb, t * nb, t * nb, nb, 1e-6, 1.0, 0.0, 0b01111, B.GMP_FLAG_SPLIT16)   # one launch per class
    d1 = B.make_desc(t * nb, t * nb, t * nb, nb, 1e-6, 1.0, 0.0, 0b01111)
    ac = np.array([[0, 1, 2, 3]] * t, np.uint8)     # per l: FP64, FP32, FP16, BF16 pairs
    bc = np.zeros((t, t), np.uint8)
    cc = np.ones((t, t), np.uint8)
    z = np.zeros((t, t, B.NCLS), np.int16)
    st = []
    for d in (d0, d1):
        pl = B.gemm_mp_plan_host(d, ac, bc, cc, z, z)
        st.append(B.gemm_mp_get_stats(pl))
        B.gemm_mp_destroy(pl)
    sep, mer = st
    assert sep["pairs"][:4] == mer["pairs"][:4] == [t * t] * 4
    assert mer["launches_execute"] == sep["launches_execute"] - 1          # one step: FP16 rides on BF16
    assert list(mer["class_launches"][:4]) == list(sep["class_launches"][:4]) == [1, 1, 1, 1]


def test_host_plan_cannot_convert_or_execute():
    """a gemm_mp_plan_host plan holds no operands / statistics / communicators: convert,
    execute and the statistics export fail with GMP_ERR_STATE before touching a device
    (also on a P*Q > 1 grid, where convert would otherwise reach NCCL)"""
    import numpy as np
    for P, Q in ((1, 1), (2, 2)):
        d = B.make_desc(512, 512, 512, 128, 1e-6, P=P, Q=Q, rank=0)
        c = np.zeros((4, 4), np.uint8)
        z = np.zeros((4, 4, B.NCLS), np.int16)
        pl = B.gemm_mp_plan_host(d, c, c, c, z, z)
        try:
            for call in (lambda: B.gemm_mp_convert(pl, 1024, 1 << 40, None),
                         lambda: B.gemm_mp_execute(pl, 1024, 512, None),
                         lambda: B.gemm_mp_get_tile_stats(pl, "A", 4, 4)):
                with pytest.raises(B.GmpError) as e:
                    call()
                assert "GMP_ERR_STATE" in str(e.value)
        finally:
            B.gemm_mp_destroy(pl)
