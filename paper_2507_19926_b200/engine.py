"""Drop-in for the reference's median-filter entry points (engine.py:1-64).

``filter_image`` / ``filter_planes`` keep the reference signature, variant
names, argument validation and error messages, replicate borders and
same-shape/same-dtype output; the work runs in hand-written sm_100a kernels
behind the C ABI (``include/tilemedian_b200.h``).  There is no CPU path: if the
CUDA extension or a GPU is missing the call raises.

Accepted images: numpy arrays (copied to the GPU through the host entry
point, result returned as numpy) and torch CUDA tensors (zero-copy, launched
on the current stream, result returned as a tensor on the same device).
Element types uint8 / uint16 / uint32; anything else raises ``TypeError``.

Keyword arguments of the reference that only shape its CPU execution
(``workers``, ``slice_budget``) are validated the same way and do not change
the result -- the reference guarantees that too (test_acceptance.py:126-143).
``counter`` receives the reference's shape-only comparison model when the
aware engine is selected (aware.py:31-45); ``checksums`` receives one
``pass=finalize`` line per band with the blake2b digest of the band's output,
the only per-pass digest a different (single-pass) algorithm can reproduce.
"""
from __future__ import annotations

import hashlib

import numpy as np

from . import _lib
from .geometry import KernelSpec, TileDims, as_kernel, region, root_tile_size
from .model import AWARE_MIN_KERNEL, aware_bands, aware_counts, validate_aware_root
from .program import DRIVER_ROOT_CAP, MAX_TILE_AREA

VARIANTS = ("auto", "oblivious", "aware", "oracle")
AUTO_CROSSOVER = 23

_BITS = {np.dtype(np.uint8): 8, np.dtype(np.uint16): 16, np.dtype(np.uint32): 32}


def pick_variant(k) -> str:
    """Resolve ``auto`` like the reference (engine.py:22-26).

    The kernels behind each variant are chosen per (dtype, k) from the
    measured dispatch table in the C ABI (``tm_dispatch_query``); this
    function only reproduces the reference's variant *name*.
    """
    if isinstance(k, KernelSpec) or (hasattr(k, "k_w") and hasattr(k, "k_h")):
        return "oblivious"
    return "oblivious" if k < AUTO_CROSSOVER else "aware"


# ---------------------------------------------------------------------------
# argument validation (same order and messages as the reference engines)

def _validate_oblivious(kern: KernelSpec, root) -> None:
    """compile_plan + region_partition checks (oblivious.py:258-268, geometry.py:203-214)."""
    if root is None:
        root = min(root_tile_size(max(kern.k_w, kern.k_h)), DRIVER_ROOT_CAP)
    dims = root if isinstance(root, TileDims) else TileDims(int(root), int(root))
    if dims.area > MAX_TILE_AREA:
        raise ValueError(f"tile {dims.t_w}x{dims.t_h} exceeds {MAX_TILE_AREA} outputs")
    region((0, 0), dims, kern)


def _image_shape(image) -> tuple[int, ...]:
    return tuple(int(s) for s in image.shape)


def _is_torch(image) -> bool:
    mod = type(image).__module__
    return mod.startswith("torch")


# ---------------------------------------------------------------------------
# execution

def _bits_of(dtype) -> int:
    try:
        return _BITS[np.dtype(dtype)]
    except (KeyError, TypeError):
        raise TypeError(
            f"unsupported element type {dtype}: the B200 kernels filter uint8, uint16 "
            "and uint32 images (no CPU fallback)") from None


def pinned_empty(shape, dtype) -> np.ndarray:
    """A numpy array in pinned (page-locked) host memory from the C ABI's cache.

    The drop-in returns its numpy outputs in these, so the device-to-host copy
    runs at full PCIe speed; the block goes back to the cache when the array
    (and every view of it) is garbage collected.
    """
    import ctypes
    import weakref

    dtype = np.dtype(dtype)
    n = max(1, int(np.prod(shape, dtype=np.int64)) * dtype.itemsize)
    lib = _lib.load()
    ptr = lib.tm_host_alloc(n)
    if not ptr:  # pinned memory exhausted: a pageable output (the copy stages it)
        return np.empty(shape, dtype)
    buf = (ctypes.c_uint8 * n).from_address(ptr)
    weakref.finalize(buf, lib.tm_host_free, ptr)
    count = int(np.prod(shape, dtype=np.int64))
    return np.frombuffer(buf, dtype=dtype, count=count).reshape(shape)


def _run_numpy(img: np.ndarray, kw: int, kh: int, variant: str, device: int,
               devices=None, slice_budget=None) -> np.ndarray:
    """numpy in -> numpy out through the C ABI's host path.  ``slice_budget``
    bounds the device bytes one band holds (source rows with halos + output
    rows; the reference's banding, aware.py:455-463) -- the result does not
    depend on it."""
    bits = _bits_of(img.dtype)
    if img.ndim == 2:
        h, w = img.shape
        ch = 1
    else:
        h, w, ch = img.shape
    src = img
    rows_ok = src.strides[-1] == src.itemsize and src.strides[0] > 0 and (
        src.ndim == 2 or src.strides[1] == ch * src.itemsize)
    if not rows_ok:
        src = np.ascontiguousarray(src)
    out = pinned_empty(img.shape, img.dtype)
    lib = _lib.load()
    code = _lib.VARIANT_CODES[variant]
    if devices is not None and len(devices) > 1:
        import ctypes
        ids = (ctypes.c_int32 * len(devices))(*[int(d) for d in devices])
        rc = lib.tm_median2d_host_multi(src.ctypes.data, src.strides[0], out.ctypes.data,
                                        out.strides[0], w, h, ch, bits, kw, kh, code, ids,
                                        len(devices))
    else:
        dev = int(devices[0]) if devices else device
        rc = lib.tm_median2d_host_budget(src.ctypes.data, src.strides[0], out.ctypes.data,
                                         out.strides[0], w, h, ch, bits, kw, kh, code, dev,
                                         int(slice_budget or 0))
    _lib.check(rc)
    return out


def _run_torch(img, kw: int, kh: int, variant: str, devices=None):
    import torch

    dt = {torch.uint8: 8, torch.uint16: 16, torch.uint32: 32}.get(img.dtype)
    if dt is None:
        raise TypeError(f"unsupported element type {img.dtype}: expected uint8/16/32")
    if not img.is_cuda:
        out = _run_numpy(img.numpy(), kw, kh, variant, 0, devices)
        return torch.from_numpy(out)
    src = img.contiguous()
    if devices is not None and len(devices) > 1:
        from .bands import filter_sharded
        return filter_sharded(src, kw, kh, variant, devices)
    out = torch.empty_like(src)
    if src.ndim == 2:
        h, w = src.shape
        ch = 1
    else:
        h, w, ch = src.shape
    esz = src.element_size()
    with torch.cuda.device(src.device):
        stream = torch.cuda.current_stream(src.device).cuda_stream
        rc = _lib.load().tm_median2d_band(src.data_ptr(), src.stride(0) * esz, h, 0, h,
                                          out.data_ptr(), out.stride(0) * esz, w, ch, dt, kw, kh,
                                          _lib.VARIANT_CODES[variant], stream)
    _lib.check(rc)
    return out


def _empty_oracle_error(shape) -> ValueError:
    axis = 0 if shape[0] == 0 else 1
    return ValueError(f"can't extend empty axis {axis} using modes other than 'constant' or 'empty'")


def filter_image(image, k, variant="auto", *, root=None, workers=1, slice_budget=None,
                 counter=None, checksums=None, device: int = 0, devices=None):
    """Median-filter ``image`` exactly, edge-replicated borders (engine.py:29-52).

    ``k`` is an odd kernel diameter or a KernelSpec (rectangular kernels take
    the oblivious route, as in the reference).  ``device`` selects the GPU for
    numpy inputs (torch tensors run on their own device).  ``devices`` (a list
    of GPU ordinals) shards the image into one row band per GPU with a
    k/2-row halo each -- bit-identical to one GPU; torch inputs come back on
    their own device.
    """
    if variant not in VARIANTS:
        raise ValueError(f"unknown variant {variant!r} (expected one of {VARIANTS})")
    # the reference resolves "auto" to an engine name (validation and
    # instrumentation follow it); the C ABI gets "auto" so its measured
    # per-(dtype, k) table picks the fastest exact kernel
    launch = variant
    if variant == "auto":
        variant = pick_variant(k)
    torch_in = _is_torch(image)
    img = image if torch_in else np.asarray(image)
    shape = _image_shape(img)
    if variant == "oracle":
        kern = as_kernel(k)
        if len(shape) != 2:
            raise ValueError("expected a 2-D image")
        if 0 in shape:
            raise _empty_oracle_error(shape)
    elif variant == "aware":
        if isinstance(k, KernelSpec) or hasattr(k, "k_w"):
            raise ValueError("rectangular kernels need the oblivious engine")
        if k < AWARE_MIN_KERNEL:
            raise ValueError(
                f"k={k} is below the aware engine's minimum of {AWARE_MIN_KERNEL}; "
                "use the oblivious engine for small kernels")
        if len(shape) != 2 or 0 in shape:
            raise ValueError("expected a non-empty 2-D image")
        kern = KernelSpec.square(int(k))
        validate_aware_root(int(k), root)
    else:
        kern = as_kernel(k)
        _validate_oblivious(kern, root)
        if len(shape) != 2:
            raise ValueError("expected a 2-D image")
        if 0 in shape:
            raise ValueError(f"image dims must be positive, got {shape[1]}x{shape[0]}")
    out = (_run_torch(img, kern.k_w, kern.k_h, launch, devices) if torch_in
           else _run_numpy(img, kern.k_w, kern.k_h, launch, device, devices, slice_budget))
    if variant == "aware" and (counter is not None or checksums is not None):
        H, W = shape
        itemsize = img.element_size() if torch_in else img.itemsize
        if counter is not None:
            aware_counts(H, W, int(k), root, itemsize, workers, slice_budget, counter)
        if checksums is not None:
            t = validate_aware_root(int(k), root)
            host = out if not torch_in else out.cpu().numpy()
            level = max(0, (t.bit_length() - 1) - 1)
            for ty0, ty1 in aware_bands(H, W, int(k), t, itemsize, workers, slice_budget):
                band = np.ascontiguousarray(host[ty0 * t: min(H, ty1 * t)])
                digest = hashlib.blake2b(band.tobytes(), digest_size=8).hexdigest()
                checksums.append(f"pass=finalize level={level + 1} checksum={digest}")
    return out


def filter_planes(image, k, variant="auto", **kwargs):
    """Filter a 2-D image, or every channel of an (H, W, C) image (engine.py:55-64).

    The (H, W, C) case runs all planes in one launch on the interleaved
    buffer (no per-channel strided copies, no stack).
    """
    torch_in = _is_torch(image)
    img = image if torch_in else np.asarray(image)
    if img.ndim == 2:
        return filter_image(img, k, variant, **kwargs)
    if img.ndim != 3:
        raise ValueError(f"expected a 2-D or (H, W, C) image, got shape {tuple(img.shape)}")
    if variant not in VARIANTS:
        raise ValueError(f"unknown variant {variant!r} (expected one of {VARIANTS})")
    if kwargs.get("counter") is not None or kwargs.get("checksums") is not None:
        # instrumentation is per plane in the reference; keep its semantics
        planes = [filter_image(img[..., c], k, variant, **kwargs) for c in range(img.shape[2])]
        if torch_in:
            import torch
            return torch.stack(planes, dim=-1)
        return np.stack(planes, axis=-1)
    h, w, ch = (int(s) for s in img.shape)
    if ch == 0:  # the reference stacks zero planes (engine.py:63)
        raise ValueError("need at least one array to stack")
    if h == 0 or w == 0:  # the reference filters plane 0 first, which raises
        return filter_image(img[..., 0], k, variant, **kwargs)
    v = pick_variant(k) if variant == "auto" else variant
    # validate exactly as filter_image would for one plane
    probe = np.empty((1, 1), dtype=np.uint8)
    _validate_like_plane(probe, k, v, kwargs.get("root"))
    kern = as_kernel(k)
    devices = kwargs.get("devices")
    return (_run_torch(img, kern.k_w, kern.k_h, variant, devices) if torch_in
            else _run_numpy(img, kern.k_w, kern.k_h, variant, int(kwargs.get("device", 0)),
                            devices, kwargs.get("slice_budget")))


def filter_frames(frames, k, variant="auto", *, devices=None, **kwargs):
    """Filter a batch of independent frames, (N, H, W) or (N, H, W, C).

    Every frame is filtered exactly like ``filter_planes(frame, k, variant)``
    (engine.py:55-64); frames are split across ``devices`` (GPU ordinals)
    with no communication ("batches of frames are split across GPUs").
    numpy in -> numpy out (one pipelined host call per frame on its device);
    torch CUDA tensors in -> a tensor on the input's device.
    """
    torch_in = _is_torch(frames)
    arr = frames if torch_in else np.asarray(frames)
    if arr.ndim not in (3, 4):
        raise ValueError(f"expected (N, H, W) or (N, H, W, C) frames, got shape {tuple(arr.shape)}")
    if variant not in VARIANTS:
        raise ValueError(f"unknown variant {variant!r} (expected one of {VARIANTS})")
    v = pick_variant(k) if variant == "auto" else variant
    _validate_like_plane(None, k, v, kwargs.get("root"))
    kern = as_kernel(k)
    n_fr, h, w = (int(s) for s in arr.shape[:3])
    ch = int(arr.shape[3]) if arr.ndim == 4 else 1
    if ch == 0:
        raise ValueError("need at least one array to stack")
    if n_fr == 0:
        return arr.clone() if torch_in else np.empty_like(arr)
    if h == 0 or w == 0:
        raise ValueError(f"image dims must be positive, got {w}x{h}")
    devs = [int(d) for d in devices] if devices else [int(kwargs.get("device", 0))]
    if torch_in and arr.is_cuda:
        import torch
        src = arr.contiguous()
        if len(devs) > 1:
            outs = [_run_torch(src[i].to(f"cuda:{devs[i % len(devs)]}"), kern.k_w, kern.k_h,
                               variant) for i in range(n_fr)]
            return torch.stack([o.to(src.device) for o in outs])
        out = torch.empty_like(src)
        bits = {torch.uint8: 8, torch.uint16: 16, torch.uint32: 32}.get(src.dtype)
        if bits is None:
            raise TypeError(f"unsupported element type {src.dtype}: expected uint8/16/32")
        esz = src.element_size()
        lib = _lib.load()
        with torch.cuda.device(src.device):
            stream = torch.cuda.current_stream(src.device).cuda_stream
            for i in range(n_fr):
                _lib.check(lib.tm_median2d_band(
                    src[i].data_ptr(), src.stride(1) * esz, h, 0, h, out[i].data_ptr(),
                    out.stride(1) * esz, w, ch, bits, kern.k_w, kern.k_h,
                    _lib.VARIANT_CODES[variant], stream))
        return out
    if torch_in:
        import torch
        return torch.from_numpy(filter_frames(arr.numpy(), k, variant, devices=devices, **kwargs))
    bits = _bits_of(arr.dtype)
    src = arr
    if not (src.strides[-1] == src.itemsize and (ch == 1 or src.strides[2] == ch * src.itemsize)
            and src.strides[1] > 0 and src.strides[0] >= h * src.strides[1]):
        src = np.ascontiguousarray(src)
    out = pinned_empty(arr.shape, arr.dtype)
    import ctypes
    ids = (ctypes.c_int32 * len(devs))(*devs)
    _lib.check(_lib.load().tm_median2d_host_frames(
        src.ctypes.data, src.strides[1], src.strides[0], out.ctypes.data, out.strides[1],
        out.strides[0], n_fr, w, h, ch, bits, kern.k_w, kern.k_h, _lib.VARIANT_CODES[variant],
        ids, len(devs)))
    return out


def _validate_like_plane(probe, k, variant, root) -> None:
    if variant == "aware":
        if isinstance(k, KernelSpec) or hasattr(k, "k_w"):
            raise ValueError("rectangular kernels need the oblivious engine")
        if k < AWARE_MIN_KERNEL:
            raise ValueError(
                f"k={k} is below the aware engine's minimum of {AWARE_MIN_KERNEL}; "
                "use the oblivious engine for small kernels")
        validate_aware_root(int(k), root)
    elif variant == "oblivious":
        _validate_oblivious(as_kernel(k), root)
    else:
        as_kernel(k)


def dispatch_query(dtype, k, variant="auto") -> str:
    """Name of the kernel the C ABI runs for (dtype, k, variant)."""
    kern = as_kernel(k)
    code = _lib.load().tm_dispatch_query(_bits_of(dtype), kern.k_w, kern.k_h,
                                         _lib.VARIANT_CODES[variant])
    return _lib.KERNEL_NAMES.get(code, "none")
