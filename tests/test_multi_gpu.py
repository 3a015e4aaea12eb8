"""Multi-GPU entry points, exercised on the GPUs this box has (GPU required).

* ``filter_image(numpy, k, devices=[...])`` -> ``tm_median2d_host_multi``:
  one row band per device, each re-reading its k/2 halo rows from the host;
* ``filter_image(tensor, k, devices=[...])`` -> ``tm_median2d_bands``:
  device-resident bands whose halo rows are exchanged between the GPUs;
* ranks over a process group (bench.py --mode bands): gloo exchanges the
  halos of host copies between 2-3 processes that all filter their band with
  the CUDA band entry point on this GPU.
With one GPU the device lists repeat ordinal 0 -- the same code paths (peer
copies become device-local copies), so stitching exactness is covered; the
cross-device copies themselves run only where several GPUs exist.
All results must be byte-identical to the whole-image oracle (the invariant
of the reference's band tests, test_aware.py:236-247).
"""
import os
import socket

import numpy as np
import pytest

from oracle import TestImageSpec, generate, oracle_median_filter_c

pytestmark = pytest.mark.gpu

from paper_2507_19926_b200 import bands, filter_image, filter_planes  # noqa: E402


def _devices(n):
    import torch
    cnt = torch.cuda.device_count()
    return [i % cnt for i in range(n)]


@pytest.mark.parametrize("bits,k,shape,n", [(8, 17, (301, 203), 3), (16, 49, (260, 130), 2),
                                            (32, 9, (97, 61), 4), (8, 75, (150, 90), 2)])
def test_host_multi_device_bands(bits, k, shape, n):
    img = generate(TestImageSpec("random", shape[1], shape[0], bits, seed=k))
    out = filter_image(img, k, devices=_devices(n))
    assert np.array_equal(out, oracle_median_filter_c(img, k))


def test_host_multi_planes():
    rng = np.random.default_rng(3)
    img = rng.integers(0, 256, (140, 90, 3), dtype=np.uint8)
    out = filter_planes(img, 17, devices=_devices(3))
    for c in range(3):
        assert np.array_equal(out[..., c], oracle_median_filter_c(np.ascontiguousarray(img[..., c]), 17))


@pytest.mark.parametrize("bits,k,n", [(8, 9, 3), (16, 27, 2), (32, 49, 3), (8, 33, 8)])
def test_device_bands_halo_exchange(bits, k, n):
    import torch
    tdt = {8: torch.uint8, 16: torch.uint16, 32: torch.uint32}[bits]
    img = generate(TestImageSpec("random", 173, 240, bits, seed=100 + k))
    t = torch.from_numpy(img.astype(np.int64)).to(tdt).cuda()
    out = filter_image(t, k, devices=_devices(n))
    assert out.device == t.device and out.shape == t.shape
    assert np.array_equal(out.cpu().numpy().astype(img.dtype), oracle_median_filter_c(img, k))


def test_device_bands_rejects_thin_bands():
    import ctypes

    import torch
    from paper_2507_19926_b200 import _lib
    lib = _lib.load()
    W, rows, h = 16, [3, 3], 4  # k = 9: halo 4 > 3-row bands
    bufs = [torch.zeros((2 * h + r, W), dtype=torch.uint8, device="cuda") for r in rows]
    outs = [torch.zeros((r, W), dtype=torch.uint8, device="cuda") for r in rows]
    arr = lambda ty, xs: (ty * 2)(*xs)  # noqa: E731
    rc = lib.tm_median2d_bands(arr(ctypes.c_void_p, [b.data_ptr() for b in bufs]),
                               arr(ctypes.c_int64, [W, W]),
                               arr(ctypes.c_void_p, [o.data_ptr() for o in outs]),
                               arr(ctypes.c_int64, [W, W]), arr(ctypes.c_int32, rows),
                               arr(ctypes.c_int32, [0, 0]), 2, W, 1, 8, 9, 9, 0, None)
    with pytest.raises(ValueError, match="halo"):
        _lib.check(rc)


def test_second_device_after_first():
    """Launch facts are cached per device: the >48 KB shared-memory opt-in of the
    u32 rank kernel (k = 49) must hold on every device of the process."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    img = generate(TestImageSpec("random", 200, 150, 32, seed=9))
    ref = oracle_median_filter_c(img, 49)
    for d in (0, 1):
        t = torch.from_numpy(img.astype(np.int64)).to(torch.uint32).to(f"cuda:{d}")
        assert np.array_equal(filter_image(t, 49).cpu().numpy().astype(np.uint32), ref)
        assert np.array_equal(filter_image(img, 49, device=d), ref)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_worker(rank, world, port, k, H, W, bits, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        img = generate(TestImageSpec("random", W, H, bits, seed=k))
        y0, y1 = bands.band_rows(H, world, rank)
        halo = k // 2
        band = torch.from_numpy(img[y0:y1].astype(np.int64))
        buf, r0 = bands.halo_buffer(band, halo, rank > 0, rank < world - 1)
        bands.exchange_halo(buf, r0, y1 - y0, halo)  # gloo on host tensors
        tdt = {8: torch.uint8, 16: torch.uint16, 32: torch.uint32}[bits]
        dev = buf.to(tdt).cuda()
        out = bands.filter_band(dev, r0, y1 - y0, k)  # the CUDA band entry point
        q.put((rank, y0, y1, out.cpu().to(torch.int64).numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,k,bits", [(2, 17, 8), (3, 25, 16), (2, 49, 32)])
def test_ranks_gloo_exchange_cuda_filter(world, k, bits):
    import torch.multiprocessing as mp
    H, W = 150, 111
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_worker, args=(r, world, port, k, H, W, bits, q))
             for r in range(world)]
    for p in procs:
        p.start()
    parts = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    img = generate(TestImageSpec("random", W, H, bits, seed=k))
    out = np.empty(img.shape, np.int64)
    for _, y0, y1, band in parts:
        out[y0:y1] = band
    assert np.array_equal(out, oracle_median_filter_c(img, k).astype(np.int64))


@pytest.mark.parametrize("bits,k,shape,n_dev", [(8, 17, (5, 90, 70, 3), 2), (16, 27, (3, 64, 80), 1),
                                                (32, 9, (4, 33, 47), 3)])
def test_filter_frames_numpy(bits, k, shape, n_dev):
    from paper_2507_19926_b200 import filter_frames
    dt = {8: np.uint8, 16: np.uint16, 32: np.uint32}[bits]
    rng = np.random.default_rng(k)
    frames = rng.integers(0, np.iinfo(dt).max, size=shape, dtype=dt, endpoint=True)
    out = filter_frames(frames, k, devices=_devices(n_dev))
    assert out.shape == frames.shape and out.dtype == frames.dtype
    for f in range(shape[0]):
        assert np.array_equal(out[f], filter_planes(frames[f], k)), f
        plane = frames[f] if frames.ndim == 3 else np.ascontiguousarray(frames[f][..., 0])
        got = out[f] if frames.ndim == 3 else out[f][..., 0]
        assert np.array_equal(got, oracle_median_filter_c(plane, k)), f


def test_filter_frames_torch():
    import torch
    from paper_2507_19926_b200 import filter_frames
    rng = np.random.default_rng(1)
    frames = rng.integers(0, 256, size=(4, 70, 61, 3), dtype=np.uint8)
    t = torch.from_numpy(frames).cuda()
    for devs in (None, _devices(2)):
        out = filter_frames(t, 11, devices=devs)
        assert out.is_cuda and out.shape == t.shape
        got = out.cpu().numpy()
        for f in range(4):
            for c in range(3):
                assert np.array_equal(got[f, ..., c],
                                      oracle_median_filter_c(np.ascontiguousarray(frames[f, ..., c]), 11))


def test_filter_frames_validation():
    from paper_2507_19926_b200 import filter_frames
    with pytest.raises(ValueError):
        filter_frames(np.zeros((4, 4), np.uint8), 3)
    with pytest.raises(ValueError):
        filter_frames(np.zeros((2, 4, 4), np.uint8), 4)
    with pytest.raises(ValueError, match="minimum"):
        filter_frames(np.zeros((2, 4, 4), np.uint8), 7, "aware")
    assert filter_frames(np.zeros((0, 4, 4), np.uint8), 3).shape == (0, 4, 4)


@pytest.mark.parametrize("budget", [1, 4096, 200_000])
def test_slice_budget_banding(budget):
    """slice_budget bounds the device bytes per band of the host path; the
    result never depends on it (test_acceptance.py:126-143)."""
    img = generate(TestImageSpec("random", 211, 157, 16, seed=4))
    ref = oracle_median_filter_c(img, 25)
    assert np.array_equal(filter_image(img, 25, slice_budget=budget), ref)
    assert np.array_equal(filter_image(img, 25, "aware", slice_budget=budget), ref)
