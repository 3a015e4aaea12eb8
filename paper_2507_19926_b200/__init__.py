"""B200-native (sm_100a) hierarchical-tiling median filter.

Drop-in for the reference package's median-filter path
(``tilemedian.filter_image`` / ``filter_planes``, reference engine.py:29-64):
same signature, variants, validation and replicate borders, bit-exact output,
computed by hand-written CUDA kernels behind a C ABI
(``include/tilemedian_b200.h``).  See DESIGN.md.
"""
from .engine import (AUTO_CROSSOVER, VARIANTS, dispatch_query, filter_frames, filter_image,
                     filter_planes, pick_variant, pinned_empty)
from .geometry import KernelSpec, TileDims, retention_window, root_tile_size
from .model import ComparisonCounter, comparison_count
from .program import build_program, op_model

__version__ = "0.1.0"

__all__ = [
    "AUTO_CROSSOVER", "VARIANTS", "filter_image", "filter_planes", "filter_frames", "pick_variant",
    "pinned_empty",
    "dispatch_query", "KernelSpec", "TileDims", "retention_window", "root_tile_size",
    "ComparisonCounter", "comparison_count", "build_program", "op_model", "__version__",
]
