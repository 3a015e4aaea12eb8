"""Python boundary: reference signature, variants and error behaviour (no GPU needed).

Mirrors the reference's test_engine.py:12-55 rejection cases; every error
here is raised before any device work.
"""
import numpy as np
import pytest

import paper_2507_19926_b200 as tmb
from paper_2507_19926_b200 import ComparisonCounter, KernelSpec, filter_image, filter_planes, pick_variant


def test_variants_and_crossover():
    assert tmb.VARIANTS == ("auto", "oblivious", "aware", "oracle")
    assert tmb.AUTO_CROSSOVER == 23
    assert all(pick_variant(k) == "oblivious" for k in range(3, 22, 2))
    assert all(pick_variant(k) == "aware" for k in (23, 25, 49, 101))
    assert pick_variant(KernelSpec(31, 25)) == "oblivious"


def test_rejections_match_reference_messages():
    img = np.zeros((30, 30), dtype=np.uint8)
    with pytest.raises(ValueError, match="oblivious"):
        filter_image(img, 7, "aware")
    with pytest.raises(ValueError, match="variant"):
        filter_image(img, 9, "fastest")
    with pytest.raises(ValueError, match="rectangular"):
        filter_image(img, KernelSpec(9, 11), "aware")
    with pytest.raises(ValueError, match="odd and >= 3, got 4x4"):
        filter_image(img, 4)
    with pytest.raises(ValueError, match="odd and >= 3, got 1x1"):
        filter_image(img, 1, "oracle")


def test_root_validation_like_reference():
    img = np.zeros((20, 20), dtype=np.uint8)
    with pytest.raises(ValueError, match="power of two in \\[2, 9\\], got 1"):
        filter_image(img, 9, "aware", root=1)
    with pytest.raises(ValueError, match="powers of two, got 3x3"):
        filter_image(img, 9, "oblivious", root=3)
    with pytest.raises(ValueError, match="tile 16x16 larger than kernel 9x9"):
        filter_image(img, 9, "oblivious", root=16)
    with pytest.raises(ValueError, match="exceeds 256 outputs"):
        filter_image(img, 9, "oblivious", root=32)
    with pytest.raises(ValueError, match="larger than kernel 3x9"):
        filter_image(img, KernelSpec(3, 9), "oblivious")


def test_shape_rejections_like_reference():
    with pytest.raises(ValueError, match="expected a 2-D image"):
        filter_image(np.zeros((4, 4, 3), np.uint8), 9, "oracle")
    with pytest.raises(ValueError, match="expected a 2-D image"):
        filter_image(np.zeros((4, 4, 3), np.uint8), 9, "oblivious")
    with pytest.raises(ValueError, match="non-empty 2-D"):
        filter_image(np.zeros((4, 4, 3), np.uint8), 9, "aware")
    with pytest.raises(ValueError, match="image dims must be positive, got 5x0"):
        filter_image(np.zeros((0, 5), np.uint8), 3)
    with pytest.raises(ValueError, match="can't extend empty axis 1"):
        filter_image(np.zeros((5, 0), np.uint8), 3, "oracle")
    with pytest.raises(ValueError):
        filter_planes(np.zeros((2, 2, 3, 1), dtype=np.uint8), 3)


def test_unsupported_dtype_is_type_error():
    with pytest.raises(TypeError, match="uint8"):
        filter_image(np.zeros((8, 8), np.float32), 3)
    with pytest.raises(TypeError):
        filter_image(np.zeros((8, 8), np.int64), 3, "oracle")


def test_counter_model_ticks_without_pixels():
    c = ComparisonCounter()
    from paper_2507_19926_b200.model import aware_counts
    aware_counts(48, 48, 23, counter=c)
    assert c.total > 0
