"""Helpers shared by the golden-fixture tests."""
import hashlib
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def digest(a) -> str:
    """Same digest as tests/golden/make_golden.py."""
    a = np.ascontiguousarray(a)
    h = hashlib.blake2b(digest_size=16)
    h.update(str(a.dtype).encode())
    h.update(repr(a.shape).encode())
    h.update(a.tobytes())
    return h.hexdigest()


def load(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def spec_of(cell):
    from oracle import TestImageSpec
    return TestImageSpec(cell["pattern"], cell["width"], cell["height"], cell["depth"],
                         seed=cell["seed"], density=cell["density"])
