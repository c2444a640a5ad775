"""The paper's aD:bS experiment mode."""
import numpy as np
import pytest

from gmp_inputs import paper_maps as pm


@pytest.mark.parametrize("d,want", [(80, 8000), (50, 5000), (20, 2000), (100, 10000), (0, 0)])
def test_fig3_exact_counts(d, want):
    """Fig. 3: 102,400^2 matrix, nb = 1,024 -> 100 x 100 tiles; 80D:20S = exactly 8,000 FP64."""
    m = pm.ratio_map(100, 100, d, 7)
    assert int((m == 0).sum()) == want


def test_determinism_and_seed_dependence():
    a = pm.ratio_map(16, 16, 50, 3)
    assert np.array_equal(a, pm.ratio_map(16, 16, 50, 3))
    assert not np.array_equal(a, pm.ratio_map(16, 16, 50, 4))


def test_rounding_half_away_from_zero():
    assert pm.n_fp64(50, 3) == 2      # 1.5 -> 2
    assert pm.n_fp64(25, 2) == 1      # 0.5 -> 1


def test_serialize_roundtrip_and_errors():
    m = pm.ratio_map(5, 7, 40, 1)
    assert np.array_equal(pm.parse(pm.serialize(m)), m)
    assert pm.serialize(np.array([[0, 1], [1, 0]], np.uint8)) == "2 2\nDS\nSD\n"
    with pytest.raises(ValueError):
        pm.parse("2 2\nDX\nSD\n")


def test_heatmaps():
    m = np.array([[0, 1]], np.uint8)
    assert pm.heatmap_csv(m) == "64,32\n"
    assert pm.heatmap_pgm(m) == "P2\n2 1\n255\n0 255\n"
    big = pm.ratio_map(100, 100, 50, 9)
    body = pm.heatmap_pgm(big).split("\n", 3)[3].split()
    assert body.count("0") == 5000 and body.count("255") == 5000


def test_splitmix_sequence():
    r = pm.SplitMix64(0)
    assert r.next() == 0xE220A8397B1DCDAF and r.next() == 0x6E789E6AA1B965F4
