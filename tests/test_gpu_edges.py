"""Edge cases and error paths of the CUDA path (through the C ABI)."""
import numpy as np
import pytest
import torch

import gmp_inputs
import oracle
from gpu_harness import run_gpu, run_oracle
from paper_2508_14848_b200 import api
from paper_2508_14848_b200 import binding as B

pytestmark = pytest.mark.gpu


def test_generator_bitwise_vs_numpy():
    for (rows, cols, nb, P, Q, p, q, mode) in [(512, 384, 128, 1, 1, 0, 0, "graded"),
                                               (1024, 768, 128, 2, 3, 1, 2, "random"),
                                               (640, 640, 128, 2, 2, 0, 1, "uniform")]:
        rec = gmp_inputs.MatrixRecipe(99, mode, 17, -2)
        t = api.synth(rows, cols, nb, rec, P, Q, p, q).cpu().numpy()
        full = gmp_inputs.synth_block(rows, cols, nb, rec.seed, mode, rec.E, rec.s, rec.tau)
        ti = np.arange(p, rows // nb, P)
        tj = np.arange(q, cols // nb, Q)
        rr = (ti[:, None] * nb + np.arange(nb)[None, :]).ravel()
        cc = (tj[:, None] * nb + np.arange(nb)[None, :]).ravel()
        assert np.array_equal(t, full[np.ix_(rr, cc)])


def test_nonfinite_input_is_an_error():
    A = np.ones((256, 256)); A[3, 200] = np.inf
    with pytest.raises(B.GmpError) as e:
        run_gpu(A, np.ones((256, 256)), None, 128, 1e-6, 1.0, 0.0, 0b01111)
    assert "NONFINITE" in str(e.value)


def test_nan_in_c_only_matters_if_beta_nonzero():
    A = np.ones((256, 256)); Bm = np.ones((256, 256)); C = np.zeros((256, 256)); C[0, 0] = np.nan
    g, (out,) = run_gpu(A, Bm, C, 128, 1e-6, 1.0, 0.0, 0b01111)
    assert np.array_equal(out, np.full((256, 256), 256.0))
    with pytest.raises(B.GmpError):
        run_gpu(A, Bm, C, 128, 1e-6, 1.0, 1.0, 0b01111)


def test_all_zero_inputs():
    z = np.zeros((256, 256))
    g, (out,) = run_gpu(z, z, z, 128, 1e-8, 1.0, 1.0, 0b01111)
    assert np.array_equal(out, z)
    m = g.maps()
    assert (m["acode"] == 3).all()  # first enabled ladder class (BF16), scale 0


def test_alpha_zero_beta_one_keeps_c():
    rng = np.random.default_rng(1)
    A, Bm, C = rng.standard_normal((3, 256, 256))
    g, (out,) = run_gpu(A, Bm, C, 128, 1e-6, 0.0, 1.0, 0b00001)
    assert np.array_equal(out, C)


def test_explicit_maps_match_oracle():
    w = gmp_inputs.small_workload(512, 512, 512, 128, 1e-6, beta=1.0, seed=3)
    A, Bm, C = w.matrices()
    rng = np.random.default_rng(0)
    maps = tuple(rng.integers(0, 2, (4, 4)).astype(np.uint8) for _ in range(3))
    o = run_oracle(A, Bm, C, 128, 1e-6, 1.0, 1.0, 0b00011, maps=maps)
    g, (out,) = run_gpu(A, Bm, C, 128, 1e-6, 1.0, 1.0, 0b00011, maps=maps)
    m = g.maps()
    assert np.array_equal(m["acode"], maps[0]) and np.array_equal(m["ccode"], maps[2])
    assert np.array_equal(out, o["C"])  # FP64/FP32 classes run on sequential-k kernels: bitwise


def test_rectangular_many_tiles_sampled_vs_oracle():
    """cfg5-shaped (K >> M, N) at reduced size: sampled C tiles vs the oracle"""
    w = gmp_inputs.small_workload(512, 512, 4096, 128, 1e-4, mode="random", E=16, beta=0.0, seed=7)
    A, Bm, C = w.matrices()
    g, (out,) = run_gpu(A, Bm, C, w.nb, w.tol, w.alpha, w.beta, w.class_mask, flags=B.GMP_FLAG_SIMT_ONLY)
    o = run_oracle(A, Bm, C, w.nb, w.tol, w.alpha, w.beta, w.class_mask, ctiles=[0, 6, 15])
    for t in [0, 6, 15]:
        i, j = divmod(t, 4)
        sl = (slice(i * 128, (i + 1) * 128), slice(j * 128, (j + 1) * 128))
        assert np.array_equal(out[sl], o["C"][sl])
