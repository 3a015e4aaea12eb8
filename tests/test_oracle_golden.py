"""Pin the CPU oracle (oracle/) against the reference's own outputs.

The golden fixtures were produced by running the reference package
(tests/golden/make_golden.py); these tests need no /root/reference.
"""
import numpy as np
import pytest

from oracle import (PATTERNS, TestImageSpec, banded_oracle, compare_images, generate,
                    oracle_median_filter_c, oracle_median_filter_np)
from golden_util import GOLDEN, digest, load, spec_of


def test_generator_matches_reference_inputs():
    seen = set()
    for cell in load("matrix.json") + load("sweep.json")["square"]:
        key = (cell["pattern"], cell["width"], cell["height"], cell["depth"], cell["seed"])
        if key in seen:
            continue
        seen.add(key)
        assert digest(generate(spec_of(cell))) == cell["input"], key


@pytest.mark.parametrize("impl", ["c", "np"])
def test_oracle_matrix(impl):
    """The 264-cell oracle-equivalence matrix (report.py:104-153)."""
    fn = oracle_median_filter_c if impl == "c" else oracle_median_filter_np
    cache = {}
    for cell in load("matrix.json"):
        key = (cell["pattern"], cell["width"], cell["height"], cell["depth"], cell["k"])
        if key not in cache:
            cache[key] = digest(fn(generate(spec_of(cell)), cell["k"]))
        assert cache[key] == cell["output"], cell


def test_oracle_sweep_all_k():
    for cell in load("sweep.json")["square"]:
        out = oracle_median_filter_c(generate(spec_of(cell)), cell["k"])
        assert digest(out) == cell["output"], (cell["depth"], cell["pattern"], cell["k"])


def test_oracle_rect():
    from paper_2507_19926_b200.geometry import KernelSpec
    for cell in load("sweep.json")["rect"]:
        if cell["output"].startswith("ValueError"):
            continue
        out = oracle_median_filter_c(generate(spec_of(cell)), KernelSpec(cell["k_w"], cell["k_h"]))
        assert digest(out) == cell["output"], cell


def test_c1_full_golden():
    z = np.load(f"{GOLDEN}/c1_u8_512_k3.npz")
    img = generate(TestImageSpec("random", 512, 512, 8, seed=42))
    assert np.array_equal(img, z["input"])
    assert np.array_equal(oracle_median_filter_c(img, 3), z["output"])


def test_banded_oracle_is_exact():
    img = generate(TestImageSpec("random", 70, 53, 16, seed=5))
    full = oracle_median_filter_c(img, 9)
    for y0, y1 in ((0, 7), (7, 30), (30, 53), (52, 53)):
        assert np.array_equal(banded_oracle(img, 9, y0, y1), full[y0:y1])


def test_oracle_thread_invariance():
    img = generate(TestImageSpec("impulse", 61, 45, 8, seed=1))
    a = oracle_median_filter_c(img, 7, threads=1)
    b = oracle_median_filter_c(img, 7, threads=8)
    assert np.array_equal(a, b)


def test_known_answers():
    # border replication (test_reference.py:51-58)
    img = np.zeros((5, 5), dtype=np.uint8)
    img[:, 0] = 200
    out = oracle_median_filter_c(img, 3)
    assert np.all(out[:, 0] == 200) and np.all(out[:, 1] == 0)
    # isolated impulse removal (test_reference.py:60-64)
    img = np.zeros((7, 7), dtype=np.uint8)
    img[3, 3] = 255
    assert oracle_median_filter_c(img, 3).max() == 0
    # constant is a fixed point
    img = np.full((10, 7), 99, dtype=np.uint8)
    assert np.array_equal(oracle_median_filter_c(img, 5), img)


def test_compare_images():
    a = np.zeros((4, 4), dtype=np.uint8)
    b = a.copy()
    b[2, 1] = 9
    b[3, 3] = 200
    r = compare_images(a, b)
    assert not r and r.mismatches == 2 and r.max_abs_diff == 200 and r.first_diff == (2, 1)
    with pytest.raises(ValueError):
        compare_images(np.zeros((2, 2)), np.zeros((3, 2)))


def test_generator_validation():
    with pytest.raises(ValueError):
        TestImageSpec("plaid", 4, 4)
    with pytest.raises(ValueError):
        TestImageSpec("random", 4, 4, depth=12)
    assert set(PATTERNS) == {"constant", "gradient", "random", "impulse"}
