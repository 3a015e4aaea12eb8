"""Row-band sharding of one image across ranks, with a k/2-row halo exchange.

Multi-GPU form of the reference's banding (oblivious.py:351-394 processes
bands of tile rows; aware.py:455-491 runs bands that re-read +-k/2 halo rows
of the original image and stitches them, exact by construction).  Here every
rank owns rows [y0, y1) of the image on its own GPU; before filtering it
receives h = k_h/2 rows from each neighbour over the process group (NCCL over
NVLink/NVSwitch on GPUs, gloo on CPU for tests) into the halo rows of one
contiguous buffer, then filters its band with the C ABI's band entry point.
Replicate clamping therefore happens only at the true image edges (ranks 0
and N-1), so the stitched result is byte-identical to the 1-GPU result.
"""
from __future__ import annotations


def band_rows(height: int, world: int, rank: int) -> tuple[int, int]:
    """Rows [y0, y1) owned by ``rank`` (balanced split, earlier ranks get +1)."""
    base, extra = divmod(height, world)
    y0 = rank * base + min(rank, extra)
    return y0, y0 + base + (1 if rank < extra else 0)


def halo_buffer(band, halo: int, top: bool, bottom: bool):
    """Allocate [halo_top + band + halo_bottom] rows and copy the band in.

    Returns (buffer, out_row0): out_row0 is the first band row inside it.
    """
    import torch
    h_top = halo if top else 0
    h_bot = halo if bottom else 0
    shape = (band.shape[0] + h_top + h_bot,) + tuple(band.shape[1:])
    buf = torch.empty(shape, dtype=band.dtype, device=band.device)
    buf[h_top:h_top + band.shape[0]].copy_(band)
    return buf, h_top


def exchange_halo(buf, out_row0: int, n_rows: int, halo: int, group=None):
    """Fill the halo rows of ``buf`` from the neighbouring ranks (in place).

    ``buf`` rows [out_row0, out_row0 + n_rows) hold this rank's band.  Each
    rank sends its first/last ``halo`` rows up/down and receives the
    neighbours' into rows [0, out_row0) and [out_row0 + n_rows, ...).
    All ranks need n_rows >= halo (checked).  Uses batched P2P ops, so the
    two directions overlap.
    """
    import torch.distributed as dist
    if halo == 0 or not dist.is_initialized():
        return
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if halo == 0 or world == 1:
        return
    if n_rows < halo:
        raise ValueError(f"band of {n_rows} rows is thinner than the {halo}-row halo")
    ops = []
    if rank > 0:
        ops.append(dist.P2POp(dist.isend, buf[out_row0:out_row0 + halo].contiguous(), rank - 1, group))
        ops.append(dist.P2POp(dist.irecv, buf[0:out_row0], rank - 1, group))
    if rank < world - 1:
        end = out_row0 + n_rows
        ops.append(dist.P2POp(dist.isend, buf[end - halo:end].contiguous(), rank + 1, group))
        ops.append(dist.P2POp(dist.irecv, buf[end:end + halo], rank + 1, group))
    for req in dist.batch_isend_irecv(ops):
        req.wait()


def filter_band(buf, out_row0: int, n_rows: int, k: int, variant: str = "auto"):
    """Filter the band held in ``buf`` (a CUDA tensor with halo rows) on its device."""
    import torch
    from . import _lib
    bits = {torch.uint8: 8, torch.uint16: 16, torch.uint32: 32}[buf.dtype]
    v = variant  # "auto": the C ABI's measured per-(dtype, k) table
    W = buf.shape[1]
    ch = 1 if buf.ndim == 2 else buf.shape[2]
    out = torch.empty((n_rows,) + tuple(buf.shape[1:]), dtype=buf.dtype, device=buf.device)
    esz = buf.element_size()
    with torch.cuda.device(buf.device):
        stream = torch.cuda.current_stream(buf.device).cuda_stream
        rc = _lib.load().tm_median2d_band(buf.data_ptr(), buf.stride(0) * esz, buf.shape[0],
                                          out_row0, n_rows, out.data_ptr(), out.stride(0) * esz,
                                          W, ch, bits, k, k, _lib.VARIANT_CODES[v], stream)
    _lib.check(rc)
    return out


def filter_sharded(image, kw: int, kh: int, variant: str, devices):
    """Filter a CUDA tensor as one row band per GPU in ``devices`` (one process).

    Every band is copied to its GPU into a buffer with k_h/2 halo rows of
    slack on both sides; the C ABI's ``tm_median2d_bands`` fills the halos
    from the neighbouring bands (peer copies over NVLink) and filters each
    band on its own device and current stream.  The bands are gathered back on
    the input's device, bit-identical to one GPU.
    """
    import ctypes

    import torch
    from . import _lib
    bits = {torch.uint8: 8, torch.uint16: 16, torch.uint32: 32}[image.dtype]
    H = int(image.shape[0])
    halo = kh // 2
    n = max(1, min(len(devices), H // max(halo, 1) if halo else H))
    rest = tuple(image.shape[1:])
    W = int(rest[0])
    ch = 1 if image.ndim == 2 else int(rest[1])
    esz = image.element_size()
    bufs, outs, rows, ids, streams = [], [], [], [], []
    for i in range(n):
        y0, y1 = band_rows(H, n, i)
        dev = torch.device("cuda", int(devices[i]))
        buf = torch.empty((halo + (y1 - y0) + halo,) + rest, dtype=image.dtype, device=dev)
        buf[halo:halo + y1 - y0].copy_(image[y0:y1])
        bufs.append(buf)
        outs.append(torch.empty((y1 - y0,) + rest, dtype=image.dtype, device=dev))
        rows.append(y1 - y0)
        ids.append(int(devices[i]))
        streams.append(torch.cuda.current_stream(dev).cuda_stream)
    arr = lambda ty, xs: (ty * n)(*xs)  # noqa: E731
    rc = _lib.load().tm_median2d_bands(
        arr(ctypes.c_void_p, [b.data_ptr() for b in bufs]),
        arr(ctypes.c_int64, [b.stride(0) * esz for b in bufs]),
        arr(ctypes.c_void_p, [o.data_ptr() for o in outs]),
        arr(ctypes.c_int64, [o.stride(0) * esz for o in outs]),
        arr(ctypes.c_int32, rows), arr(ctypes.c_int32, ids), n, W, ch, bits, kw, kh,
        _lib.VARIANT_CODES[variant], arr(ctypes.c_void_p, streams))
    _lib.check(rc)
    return torch.cat([o.to(image.device) for o in outs], dim=0)
