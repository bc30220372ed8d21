"""Command line and codecs (cli.py:56-98,190-235, imaging.py:68-139 of the
reference).  The cases follow the reference's own test_cli.py / test_imaging.py: usage errors
exit 2, runtime errors exit 1 with 'error:', `foveate` writes exactly what `foveate()` returns,
zero strength is byte-identical, identical invocations are byte-identical."""

import csv
import warnings

import numpy as np
import pytest

import paper_2012_08655_b200 as fk
from paper_2012_08655_b200.cli import main
from paper_2012_08655_b200.imaging import load_image, save_image
from paper_2012_08655_b200.retinal import load_params, parse_params_text


def scene(seed=7, shape=(160, 160, 3)):
    rng = np.random.default_rng(seed)
    h, w, c = shape
    yy, xx = np.mgrid[0:h, 0:w]
    base = 128 + 90 * np.sin(xx / 5.0) * np.cos(yy / 8.0)
    return fk.RasterImage.from_array(
        np.clip(base[..., None] + rng.integers(-20, 21, shape), 0, 255).astype(np.uint8))


# ------------------------------------------------------------------------------ CPU side
def test_usage_error_exits_2():
    with pytest.raises(SystemExit) as exc:
        main(["foveate", "--bogus-flag"])
    assert exc.value.code == 2
    with pytest.raises(SystemExit):
        main([])


def test_missing_input_exits_1(tmp_path, capsys):
    rc = main(["foveate", "--input", str(tmp_path / "no.png"), "--output", str(tmp_path / "o.png")])
    assert rc == 1
    assert "error:" in capsys.readouterr().err


@pytest.mark.parametrize("ext,channels", [(".ppm", 3), (".pgm", 1), (".png", 3), (".png", 1), (".pnm", 3)])
def test_codec_round_trip(tmp_path, ext, channels):
    img = scene(3, (37, 53, channels))
    path = tmp_path / f"img{ext}"
    save_image(img, path)
    assert load_image(path) == img


def test_codec_errors(tmp_path):
    img = scene(3, (8, 8, 3))
    with pytest.raises(ValueError, match="unsupported output format"):
        save_image(img, tmp_path / "x.jpg")
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"GIF89a....")
    with pytest.raises(ValueError, match="unsupported format"):
        load_image(bad)
    trunc = tmp_path / "t.ppm"
    trunc.write_bytes(b"P6\n4 4\n255\n" + bytes(10))
    with pytest.raises(ValueError, match="truncated PNM payload"):
        load_image(trunc)
    deep = tmp_path / "d.pgm"
    deep.write_bytes(b"P5\n2 2\n65535\n" + bytes(8))
    with pytest.raises(ValueError, match="only maxval 255"):
        load_image(deep)
    comment = tmp_path / "c.pgm"
    comment.write_bytes(b"P5\n# made by hand\n2 2\n255\n" + bytes([1, 2, 3, 4]))
    assert load_image(comment).data[:, :, 0].tolist() == [[1, 2], [3, 4]]


def test_png_alpha_is_dropped_with_a_warning(tmp_path):
    from PIL import Image

    rgba = np.zeros((5, 6, 4), np.uint8)
    rgba[..., 0], rgba[..., 3] = 200, 128
    path = tmp_path / "a.png"
    Image.fromarray(rgba, mode="RGBA").save(path)
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        img = load_image(path)
    assert img.channels == 3 and img.data[0, 0].tolist() == [200, 0, 0]
    assert any("alpha channel dropped" in str(x.message) for x in w)


def test_params_file(tmp_path):
    p = parse_params_text("# comment\nfragment_size = 16\nfixation=10, 20.5\ne2=1.5 # alt fit\n")
    assert p.fragment_size == 16 and p.fixation == (10.0, 20.5) and p.e2 == 1.5
    with pytest.raises(ValueError, match="unknown key 'bogus'"):
        parse_params_text("bogus=1")
    with pytest.raises(ValueError, match="line 2: expected key=value"):
        parse_params_text("e2=2\nnonsense")
    f = tmp_path / "p.cfg"
    f.write_text("strength=0.5\n")
    assert load_params(f, fk.FoveationParams(fragment_size=8)).strength == 0.5


# ------------------------------------------------------------------------------ GPU side
@pytest.fixture()
def scene_png(tmp_path):
    path = tmp_path / "scene.png"
    save_image(scene(), path)
    return path


@pytest.mark.gpu
def test_foveate_writes_output_and_stats(tmp_path, scene_png, capsys):
    out_path = tmp_path / "out.png"
    rc = main(["foveate", "--input", str(scene_png), "--output", str(out_path), "--fragment", "16",
               "--fixation", "80,80", "--e-corner", "20"])
    assert rc == 0
    captured = capsys.readouterr().out
    assert "regions" in captured and "render_ms" in captured
    expect, *_ = fk.foveate(scene(), fk.FoveationParams(fragment_size=16, fixation=(80, 80), e_corner=20.0))
    assert load_image(out_path) == expect


@pytest.mark.gpu
def test_foveate_zero_strength_and_repeatability(tmp_path, scene_png):
    out_path = tmp_path / "out.png"
    assert main(["foveate", "--input", str(scene_png), "--output", str(out_path), "--strength", "0"]) == 0
    assert out_path.read_bytes() == scene_png.read_bytes()
    a, b = tmp_path / "a.png", tmp_path / "b.png"
    argv = ["foveate", "--input", str(scene_png), "--fragment", "16"]
    assert main(argv + ["--output", str(a)]) == 0
    assert main(argv + ["--output", str(b)]) == 0
    assert a.read_bytes() == b.read_bytes()


@pytest.mark.gpu
def test_foveate_with_config_file_and_density_map(tmp_path, scene_png):
    cfg = tmp_path / "p.cfg"
    cfg.write_text("fragment_size=16\nfixation=40,100\n")
    dm = tmp_path / "map.pgm"
    ramp = np.tile(np.linspace(0, 255, 40, dtype=np.uint8), (40, 1))
    save_image(fk.RasterImage.from_array(ramp), dm)
    out_path = tmp_path / "o.ppm"
    rc = main(["foveate", "--input", str(scene_png), "--output", str(out_path), "--config", str(cfg),
               "--map", str(dm), "--sigma-max", "3.0", "--no-shift"])
    assert rc == 0
    expect, *_ = fk.foveate(scene(), fk.FoveationParams(fragment_size=16, fixation=(40, 100)),
                            density=fk.RasterImage.from_array(ramp), sigma_max=3.0, use_shift=False)
    assert load_image(out_path) == expect


@pytest.mark.gpu
def test_grid_dump(tmp_path, scene_png, capsys):
    out_path = tmp_path / "grid.txt"
    assert main(["grid", "--input", str(scene_png), "--output", str(out_path), "--fragment", "16"]) == 0
    text = out_path.read_text()
    assert text.startswith("fragment 16") and "index_matrix" in text
    assert main(["grid", "--input", str(scene_png), "--fragment", "16"]) == 0
    assert capsys.readouterr().out.strip() == text.strip()


@pytest.mark.gpu
def test_ssim_command(tmp_path, scene_png, capsys):
    blurred, *_ = fk.foveate(scene(), fk.FoveationParams(fragment_size=16))
    test_path = tmp_path / "blurred.png"
    save_image(blurred, test_path)
    map_path = tmp_path / "map.png"
    rc = main(["ssim", "--ref", str(scene_png), "--test", str(test_path), "--map-out", str(map_path)])
    assert rc == 0
    out = capsys.readouterr().out
    assert out.startswith("mean ") and "argmin" in out
    m = load_image(map_path)
    assert m.channels == 1 and m.size == (150, 150)


@pytest.mark.gpu
def test_bench_command(tmp_path, capsys):
    img_path = tmp_path / "img.ppm"
    save_image(scene(0, (48, 48, 3)), img_path)
    out_path = tmp_path / "bench.csv"
    rc = main(["bench", "--images", str(img_path), "--output", str(out_path), "--fragments", "16",
               "--e-corners", "10", "--methods", "blockwise"])
    assert rc == 0
    with open(out_path) as fh:
        rows = list(csv.DictReader(fh))
    assert len(rows) == 1 and rows[0]["method"] == "blockwise" and rows[0]["image_w"] == "48"
    assert "wrote 1 rows" in capsys.readouterr().out
    assert main(["bench", "--images", str(img_path), "--output", str(out_path), "--methods", "pyramid"]) == 1
