"""CPU-side checks of the boundary: libfovea.so loads, exports everything include/fovea.h
declares, struct layouts agree with the ctypes mirror, and the host-side mirror of the
reference API behaves like the reference (no compute calls here -- no GPU needed)."""

import ctypes
import re
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

ROOT = Path(__file__).resolve().parent.parent

import paper_2012_08655_b200 as fk  # noqa: E402
from paper_2012_08655_b200 import _native  # noqa: E402
from oracle import fovea_oracle as fo  # noqa: E402


def test_library_loads_and_exports_every_declared_symbol():
    lib = _native.lib()
    header = (ROOT / "include" / "fovea.h").read_text()
    declared = sorted(set(re.findall(r"\b(fk_[a-z0-9_]+)\s*\(", header)))
    assert declared, "no declarations parsed"
    assert sorted(_native.EXPORTS) == declared
    for name in declared:
        assert hasattr(lib, name), f"libfovea.so does not export {name}"
    assert lib.fk_abi_version() == 1


def test_struct_layouts_match_the_header(tmp_path):
    src = tmp_path / "sz.c"
    src.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "fovea.h"\n'
        "int main(void){printf(\"%zu %zu %zu %zu %zu %zu\\n\", sizeof(fk_params),"
        " offsetof(fk_params, fragment_size), sizeof(fk_plan_view), offsetof(fk_plan_view, sigma),"
        " sizeof(fk_device_info), offsetof(fk_device_info, name));return 0;}\n")
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True,
                                          check=True).stdout.split()]
    want = [ctypes.sizeof(_native.FkParams), _native.FkParams.fragment_size.offset,
            ctypes.sizeof(_native.FkPlanView), _native.FkPlanView.sigma.offset,
            ctypes.sizeof(_native.FkDeviceInfo), _native.FkDeviceInfo.name.offset]
    assert got == want


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_no_cpu_fallback_without_a_gpu():
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        fk.Engine(0)
    img = fk.RasterImage.from_array(np.zeros((32, 32, 3), np.uint8))
    with pytest.raises(RuntimeError):
        fk.foveate(img, fk.FoveationParams())
    # argument errors still surface as the reference's ValueError before any device work
    lib = _native.lib()
    assert lib.fk_create(0, None) == _native.FK_EINVAL
    assert "NULL" in _native.last_error()


def test_hypot_replica_matches_libm():
    exe = Path("/tmp/fk_test_hypot")
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-I",
                    str(ROOT / "paper_2012_08655_b200" / "csrc"),
                    str(ROOT / "tests" / "c" / "test_hypot.c"), "-o", str(exe), "-lm"], check=True)
    res = subprocess.run([str(exe)], capture_output=True, text=True)
    assert res.returncode == 0, res.stdout
    assert res.stdout.startswith("0 mismatches")


# ---------------------------------------------------------------- host mirror parity
def test_shift_matches_reference_kats():
    # test_blockwise.py:45-69
    assert fk.compute_fragment_shift((16, 16), 32) == (0, 0)
    assert fk.compute_fragment_shift((0, 0), 32) == (16, 16)
    assert fk.compute_fragment_shift((960.0, 540.0), 32) == (16, 12)
    with pytest.raises(ValueError, match="fragment_size must be >= 4"):
        fk.compute_fragment_shift((0, 0), 2)
    rng = np.random.default_rng(1)
    for _ in range(200):
        F = int(rng.integers(4, 70))
        fx, fy = rng.uniform(0, 4000, 2)
        assert fk.compute_fragment_shift((fx, fy), F) == fo.np_fragment_shift((fx, fy), F)


def test_spans_match_oracle_and_cover_image():
    rng = np.random.default_rng(2)
    for _ in range(300):
        F = int(rng.integers(4, 70))
        extent = int(rng.integers(1, 500))
        off = int(rng.integers(0, F))
        a = fk.fragment_spans(extent, F, off)
        assert np.array_equal(a, fo.np_fragment_spans(extent, F, off))
        assert a[0, 0] == 0 and a[-1, 1] == extent and np.all(a[1:, 0] == a[:-1, 1])
        from paper_2012_08655_b200.tiling import span_count
        assert span_count(extent, F, off) == len(a)
    with pytest.raises(ValueError):
        fk.fragment_spans(0, 8, 0)
    with pytest.raises(ValueError):
        fk.fragment_spans(10, 8, 8)


def test_filter_length_and_taps_kats():
    # test_filters.py:41-47,105-112
    assert fk.filter_length(1.0) == 7 and fk.filter_length(0.0) == 1
    assert list(fk.filter_length(np.array([0.1, 0.2, 1.0, 5.0]))) == [1, 3, 7, 31]
    g = fk.gaussian_filter_1d(1.0)
    assert len(g) == 7 and abs(g[3] - 0.3990502797) < 1e-9 and abs(g[2] - 0.2420362294) < 1e-9
    with pytest.raises(ValueError):
        fk.filter_length(-1.0)
    with pytest.raises(ValueError):
        fk.filter_length(np.nan)


def test_params_validation_messages():
    # retinal.py:46-61,67-75
    for kw, pat in [(dict(alpha=0), "alpha"), (dict(e2=-1), "e2"), (dict(ct0=1.0), "ct0"),
                    (dict(e_corner=-1), "e_corner"), (dict(f_max=0), "f_max"),
                    (dict(strength=-0.1), "strength"), (dict(fragment_size=3), "fragment_size")]:
        with pytest.raises(ValueError, match=pat):
            fk.FoveationParams(**kw)
    p = fk.FoveationParams(fixation=(100, 5))
    assert p.fixation_for((200, 10)) == (100.0, 5.0)
    with pytest.raises(ValueError, match="outside"):
        p.fixation_for((100, 10))
    assert fk.FoveationParams().fixation_for((1920, 1080)) == (960.0, 540.0)
    # test_retinal.py:72-95
    assert abs(fk.cutoff_cpd(0.0, fk.FoveationParams()) - 39.2347) < 1e-3
    assert abs(fk.sigma_at(0.0, fk.FoveationParams()) - 1 / np.pi) < 1e-12
    assert abs(fk.sigma_at(2.3, fk.FoveationParams()) - 2 / np.pi) < 1e-12


def test_raster_image_contract():
    # imaging.py:26-65
    with pytest.raises(ValueError, match="uint8"):
        fk.RasterImage(2, 2, 1, np.zeros((2, 2, 1), np.float32))
    with pytest.raises(ValueError, match="channels"):
        fk.RasterImage.from_array(np.zeros((2, 2, 2), np.uint8))
    a = fk.RasterImage.from_array(np.arange(12, dtype=np.uint8).reshape(3, 4))
    assert a.size == (4, 3) and a.channels == 1
    assert a == fk.RasterImage.from_array(a.data.copy())


def test_shard_range_partitions():
    for n in (0, 1, 7, 256, 65536):
        for world in (1, 2, 3, 4, 8):
            parts = [fk.shard_range(n, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        fk.shard_range(10, 2, 2)


def test_handover_protocol_model_holds_for_one_and_two_raw_buffers():
    """tools/handover_model.py: the item slots, the request cursor and the rotating hand-over of
    fk_blur_tma under random interleavings of its four warps -- no slot read before it holds the
    wanted item, no cursor more than two items ahead, no wait without end -- for the buffer
    counts the kernel uses; with a third buffer the model finds the read that precedes its
    publication (why the kernel stops at two)."""
    import importlib.util
    import pathlib

    path = pathlib.Path(__file__).resolve().parents[1] / "tools" / "handover_model.py"
    spec = importlib.util.spec_from_file_location("handover_model", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    assert mod.check(1, 2, 400) == []
    assert mod.check(2, 2, 400) == []
    assert mod.check(3, 4, 400) != []
