"""``python -m paper_2507_19926_b200.cli filter`` end to end (GPU): the
reference's test_cli.py flow -- synth: and file inputs, P5 / P6 / MF32
outputs -- checked against the oracle."""
import numpy as np
import pytest

from oracle import TestImageSpec, generate, oracle_median_filter_c

pytestmark = pytest.mark.gpu

from paper_2507_19926_b200 import cli, pnm  # noqa: E402


@pytest.mark.parametrize("depth,k,variant", [(8, 3, "auto"), (16, 9, "aware"), (32, 5, "oblivious"),
                                             (16, 25, "auto")])
def test_filter_synth(tmp_path, capsys, depth, k, variant):
    out = tmp_path / "out.img"
    rc = cli.main(["filter", "--in", f"synth:random:61x47:{depth}", "--out", str(out), "--k", str(k),
                   "--variant", variant, "--seed", "3"])
    assert rc == 0
    assert f"wrote {out}: 61x47" in capsys.readouterr().out
    img = generate(TestImageSpec("random", 61, 47, depth, seed=3))
    assert np.array_equal(pnm.read_image(out), oracle_median_filter_c(img, k))


def test_filter_rgb_file(tmp_path):
    rng = np.random.default_rng(2)
    rgb = rng.integers(0, 256, (40, 52, 3), dtype=np.uint8)
    src, out = tmp_path / "in.ppm", tmp_path / "out.ppm"
    pnm.write_image(src, rgb)
    assert cli.main(["filter", "--in", str(src), "--out", str(out), "--k", "17"]) == 0
    got = pnm.read_image(out)
    for c in range(3):
        assert np.array_equal(got[..., c], oracle_median_filter_c(np.ascontiguousarray(rgb[..., c]), 17))


def test_dump_checksums(tmp_path, capsys):
    out = tmp_path / "o.pgm"
    assert cli.main(["filter", "--in", "synth:impulse:40x40:8", "--out", str(out), "--k", "9",
                     "--variant", "aware", "--dump-checksums"]) == 0
    assert "pass=finalize" in capsys.readouterr().out
