"""Row-band sharding with halo exchange, world_size 2 and 3 on CPU (gloo).

The multi-GPU path (bench.py --mode bands, paper_2507_19926_b200/bands.py)
exchanges k/2 halo rows with the neighbours, then filters each band with the
C ABI's band entry point.  Here the same exchange runs over gloo on CPU
tensors and each band is filtered by the CPU oracle on its halo buffer with
the same (out_row0, n_rows) contract; the stitched image must equal the
whole-image oracle byte for byte (the invariant of test_aware.py:236-247).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2507_19926_b200 import bands


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, k, H, W, dtype, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle_median_filter_c
        rng = np.random.default_rng(7)
        img = rng.integers(0, np.iinfo(dtype).max, size=(H, W), dtype=dtype, endpoint=True)
        y0, y1 = bands.band_rows(H, world, rank)
        band = torch.from_numpy(img[y0:y1].astype(np.int64))
        halo = k // 2
        buf, r0 = bands.halo_buffer(band, halo, rank > 0, rank < world - 1)
        bands.exchange_halo(buf, r0, y1 - y0, halo)
        src = buf.numpy().astype(dtype)
        # the band contract: output rows [r0, r0 + n) of a source that carries its halo
        full_band = oracle_median_filter_c(src, k)[r0:r0 + (y1 - y0)]
        q.put((rank, y0, y1, full_band))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,k,H,W,dtype", [
    (2, 9, 61, 45, np.uint8),
    (3, 5, 40, 33, np.uint16),
    (2, 17, 70, 23, np.uint32),
])
def test_band_halo_exchange_is_exact(world, k, H, W, dtype):
    from oracle import oracle_median_filter_c
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, k, H, W, dtype, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(7)
    img = rng.integers(0, np.iinfo(dtype).max, size=(H, W), dtype=dtype, endpoint=True)
    out = np.empty_like(img)
    for _, y0, y1, band in parts:
        out[y0:y1] = band
    assert np.array_equal(out, oracle_median_filter_c(img, k))


def test_band_rows_partition():
    for H in (1, 7, 100, 4097):
        for world in (1, 2, 3, 8):
            if world > H:
                continue
            spans = [bands.band_rows(H, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == H
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def test_halo_buffer_layout():
    band = torch.arange(12).reshape(4, 3)
    buf, r0 = bands.halo_buffer(band, 2, True, False)
    assert r0 == 2 and buf.shape == (6, 3)
    assert torch.equal(buf[2:], band)
    buf, r0 = bands.halo_buffer(band, 2, False, True)
    assert r0 == 0 and buf.shape == (6, 3) and torch.equal(buf[:4], band)
