"""Latest-wins streaming layer (reference service.py:58-63,121-146,192-238)."""

import queue
import time

import numpy as np
import pytest

import paper_2012_08655_b200 as fk
from paper_2012_08655_b200.streaming import FoveationStream, clamp_fixation


def test_clamp_fixation_matches_reference_rule():
    # service.py:58-63: clamp into [0, w-1] x [0, h-1] and report whether the point moved
    assert clamp_fixation(10.0, 20.0, (640, 480)) == (10.0, 20.0, False)
    assert clamp_fixation(-3.0, 20.0, (640, 480)) == (0.0, 20.0, True)
    assert clamp_fixation(700.0, 500.0, (640, 480)) == (639.0, 479.0, True)
    assert clamp_fixation(639.0, 479.0, (640, 480)) == (639.0, 479.0, False)


@pytest.mark.gpu
def test_stream_frames_equal_foveate_and_latest_wins():
    rng = np.random.default_rng(3)
    img = rng.integers(0, 256, (360, 640, 3), dtype=np.uint8)
    base = fk.FoveationParams(fragment_size=32)
    with FoveationStream(img, base) as s:
        # one request at a time: every frame is rendered and equals foveate()
        for (x, y) in [(320.0, 180.0), (0.0, 0.0), (639.0, 359.0), (100.5, 200.25)]:
            s.submit(x, y)
            out, stats = s.get(timeout=30)
            ref, grid, bank, rs = fk.foveate(fk.RasterImage.from_array(img),
                                             fk.FoveationParams(fragment_size=32, fixation=(x, y)))
            assert np.array_equal(out, ref.data)
            assert stats["regions"] == rs.regions and stats["shift"] == list(rs.shift)
            assert stats["method"] == "blockwise" and stats["fragment"] == 32
            assert "warning" not in stats
        # overrides persist (service.py:121-146) and out-of-image fixations are clamped
        s.submit(900.0, -5.0, strength=2.0, fragment=16)
        out, stats = s.get(timeout=30)
        assert stats["warning"] == "fixation clamped to image bounds"
        assert (stats["x"], stats["y"]) == (639.0, 0.0) and stats["fragment"] == 16
        ref, *_ = fk.foveate(fk.RasterImage.from_array(img),
                             fk.FoveationParams(fragment_size=16, strength=2.0, fixation=(639.0, 0.0)))
        assert np.array_equal(out, ref.data)
        s.submit(10.0, 10.0)
        out, stats = s.get(timeout=30)
        assert stats["fragment"] == 16      # the override persisted
        # a burst: requests overwrite each other, the newest one is always rendered last
        n0 = s.rendered
        for i in range(200):
            s.submit(float(i), 50.0)
        last = None
        deadline = time.time() + 30
        while time.time() < deadline:
            try:
                last = s.get(timeout=0.5)
            except queue.Empty:
                break
        assert last is not None and last[1]["x"] == 199.0
        assert 1 <= s.rendered - n0 <= 200
        # a request the reference would reject comes back as a ValueError
        s.submit(5.0, 5.0, fragment=2)
        with pytest.raises(ValueError):
            s.get(timeout=30)
        with pytest.raises(ValueError):
            s.submit(1.0, 1.0, gamma=2)


def test_harness_config_validation_matches_reference():
    # bench.py:48-56: warm-up >= 3, iterations >= 10, no empty axes
    from paper_2012_08655_b200 import harness
    img = fk.RasterImage.from_array(np.zeros((64, 64, 3), np.uint8))
    with pytest.raises(ValueError, match="warmup"):
        harness.BenchConfig(images=(img,), warmup=2)
    with pytest.raises(ValueError, match="iterations"):
        harness.BenchConfig(images=(img,), iterations=5)
    with pytest.raises(ValueError, match="empty"):
        harness.BenchConfig(images=())
    assert harness.CSV_COLUMNS[:4] == ["method", "image_w", "image_h", "fragment"]
    with pytest.raises(ValueError, match="unknown method"):
        harness.run_benchmark(harness.BenchConfig(images=(img,), methods=("pyramid",)))


@pytest.mark.gpu
def test_harness_rows_and_csv(tmp_path):
    from paper_2012_08655_b200 import harness
    rng = np.random.default_rng(11)
    img = fk.RasterImage.from_array(rng.integers(0, 256, (270, 480, 3), dtype=np.uint8))
    cfg = harness.BenchConfig(images=(img,), fragments=(16, 32), e_corners=(20.0, 60.0),
                              fixations=("center", "corner", (100, 50)))
    rows = harness.run_benchmark(cfg)
    assert len(rows) == 2 * 2 * 3 and all(set(r) == set(harness.CSV_COLUMNS) for r in rows)
    assert [r["fragment"] for r in rows[:6]] == [16] * 6          # the reference's sweep order
    assert rows[1]["fixation_x"] == 0.0 and rows[2]["fixation_x"] == 100.0
    # stronger foveation -> at least as many regions and taps (test_acceptance.py:208-248 trends)
    assert rows[3]["max_filter"] >= rows[0]["max_filter"]
    harness.write_csv(rows, tmp_path / "b.csv")
    head = (tmp_path / "b.csv").read_text().splitlines()[0]
    assert head == ",".join(harness.CSV_COLUMNS)
