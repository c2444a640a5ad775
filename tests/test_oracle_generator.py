"""Pins for the counter-based SplitMix64 input recipe (O1)."""
import numpy as np

import gmp_inputs
import oracle


def test_splitmix_published_sequence():
    # seed 0 -> 0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4
    assert oracle.splitmix_output(0, 1) == 0xE220A8397B1DCDAF
    assert oracle.splitmix_output(0, 2) == 0x6E789E6AA1B965F4
    assert int(gmp_inputs.splitmix_outputs(0, [1])[0]) == 0xE220A8397B1DCDAF


def test_splitmix_counter_form_equals_recurrence():
    state, seq = 12345, []
    for _ in range(50):
        state = (state + gmp_inputs.GAMMA) % 2 ** 64
        seq.append(int(gmp_inputs.mix64(np.uint64(state))))
    got = gmp_inputs.splitmix_outputs(12345, np.arange(1, 51, dtype=np.uint64))
    assert [int(x) for x in got] == seq


def test_uniform_edges():
    # SPEC.md:86-88
    assert gmp_inputs.uniform_from_u64(np.array([0], np.uint64))[0] == -1.0
    assert gmp_inputs.uniform_from_u64(np.array([2 ** 64 - 1], np.uint64))[0] == 1 - 2.0 ** -52


def test_numpy_and_c_generators_agree():
    for mode, m in [("uniform", 0), ("graded", 1), ("random", 2)]:
        a = gmp_inputs.synth_block(384, 256, 128, 4242, mode, 17, -3, 4342)
        b = oracle.synth_block(384, 256, 128, 4242, m, 17, -3, 4342)
        assert np.array_equal(a, b)
    a = gmp_inputs.synth_block(1024, 2048, 128, 7, "random", 9, 2, 107, r0=256, nr=128, c0=1024, nc=256)
    b = oracle.synth_block(1024, 2048, 128, 7, 2, 9, 2, 107, r0=256, nr=128, c0=1024, nc=256)
    assert np.array_equal(a, b)


def test_graded_exponents():
    e = gmp_inputs.tile_exponents(4, 4, "graded", 14, 0)
    assert e[0, 0] == 0 and e[3, 3] == 14 and e[1, 2] == (3 * 14) // 6
