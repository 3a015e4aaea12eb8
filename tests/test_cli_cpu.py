"""PNM / MF32 files and the command line's argument handling (CPU).

Mirrors the reference's test_pnm.py round trips and malformed-header cases
and test_cli.py's usage errors (exit status 2); the filtering itself runs on
the GPU (tests/test_cli_gpu.py).
"""
import numpy as np
import pytest

from paper_2507_19926_b200 import cli, pnm
from paper_2507_19926_b200.synth import generate_host


@pytest.mark.parametrize("dtype,shape", [(np.uint8, (7, 11)), (np.uint16, (5, 9)),
                                         (np.uint32, (6, 4)), (np.uint8, (3, 5, 3))])
def test_round_trip(tmp_path, dtype, shape):
    rng = np.random.default_rng(0)
    img = rng.integers(0, np.iinfo(dtype).max, size=shape, dtype=dtype, endpoint=True)
    p = tmp_path / "x.img"
    pnm.write_image(p, img)
    back = pnm.read_image(p)
    assert back.dtype == img.dtype and np.array_equal(back, img)


def test_formats_on_disk(tmp_path):
    p = tmp_path / "a.pgm"
    pnm.write_image(p, np.array([[1, 2], [3, 4]], np.uint16))
    assert p.read_bytes() == b"P5\n2 2\n65535\n\x00\x01\x00\x02\x00\x03\x00\x04"
    p = tmp_path / "b.mf32"
    pnm.write_image(p, np.array([[7]], np.uint32))
    assert p.read_bytes() == b"MF32" + b"\x01\x00\x00\x00" * 2 + b"\x07\x00\x00\x00"


def test_header_comments_and_errors(tmp_path):
    p = tmp_path / "c.pgm"
    p.write_bytes(b"P5\n# a comment\n2 1\n# another\n255\n\x05\x06")
    assert pnm.read_image(p).tolist() == [[5, 6]]
    p.write_bytes(b"P5\n2 1\n255\n\x05")
    with pytest.raises(ValueError, match="raster holds 1 samples, expected 2"):
        pnm.read_image(p)
    p.write_bytes(b"P5\n2 x\n255\n")
    with pytest.raises(ValueError, match="bad header token"):
        pnm.read_image(p)
    p.write_bytes(b"P5\n2 1\n70000\n\x00\x00")
    with pytest.raises(ValueError, match="unsupported maxval"):
        pnm.read_image(p)
    p.write_bytes(b"XX")
    with pytest.raises(ValueError, match="unrecognised image magic"):
        pnm.read_image(p)
    with pytest.raises(ValueError, match="multi-channel output"):
        pnm.write_image(tmp_path / "d", np.zeros((2, 2, 4), np.uint8))
    with pytest.raises(ValueError, match="no container"):
        pnm.write_image(tmp_path / "d", np.zeros((2, 2), np.int16))


def test_synth_matches_the_reference_generator():
    from oracle import TestImageSpec, generate
    for pat in ("constant", "gradient", "random", "impulse"):
        for depth in (8, 16, 32):
            a = generate_host(pat, 37, 21, depth, seed=5, density=0.2)
            b = generate(TestImageSpec(pat, 37, 21, depth, seed=5, density=0.2))
            assert a.dtype == b.dtype and np.array_equal(a, b), (pat, depth)


@pytest.mark.parametrize("argv", [["filter", "--in", "synth:random:8x8:8", "--out", "o", "--k", "4"],
                                  ["filter", "--in", "synth:random:8x8:8", "--out", "o", "--k", "7",
                                   "--variant", "aware"],
                                  ["filter", "--in", "/nonexistent.pgm", "--out", "o", "--k", "3"],
                                  ["filter", "--in", "synth:random:8x8", "--out", "o", "--k", "3"]])
def test_usage_errors_exit_2(argv, capsys):
    with pytest.raises(SystemExit) as e:
        cli.main(argv)
    assert e.value.code == 2
