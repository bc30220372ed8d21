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


@pytest.mark.gpu
def test_two_streams_on_one_image_size_run_side_by_side():
    """Two service-style callers on the same geometry (service.py:231: one connection per
    worker thread): each stream owns its plan, CUDA stream and request graphs, so their
    frames interleave freely and every one of them still equals foveate()."""
    import threading

    rng = np.random.default_rng(8)
    imgs = [rng.integers(0, 256, (270, 480, 3), dtype=np.uint8) for _ in range(2)]
    pts = [(float(x), float(y)) for x, y in rng.integers(0, 270, (12, 2))]
    results = [[], []]

    def client(k):
        with FoveationStream(imgs[k], fk.FoveationParams(fragment_size=32)) as s:
            for (x, y) in pts:
                s.submit(x, y)
                out, stats = s.get(timeout=60)
                results[k].append((x, y, out.copy()))

    threads = [threading.Thread(target=client, args=(k,)) for k in range(2)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(120)
    for k in range(2):
        assert len(results[k]) == len(pts)
        for (x, y, out) in results[k]:
            ref, *_ = fk.foveate(fk.RasterImage.from_array(imgs[k]),
                                 fk.FoveationParams(fragment_size=32, fixation=(x, y)))
            assert np.array_equal(out, ref.data)


@pytest.mark.gpu
def test_frame_request_graph_equals_foveate_float32_and_reports_plan():
    """fk_request_*: the captured plan -> render -> copy graph on a float32 frame, replayed
    for several fixations, equals foveate_batch bit for bit and reports the plan header."""
    import torch
    from paper_2012_08655_b200.engine import DevicePlan, FrameRequest, get_engine, pinned_empty

    rng = np.random.default_rng(4)
    frame = torch.from_numpy(rng.random((200, 320, 3), dtype=np.float32)).cuda()
    out = torch.empty_like(frame)
    host = pinned_empty((200, 320, 3), np.float32)
    eng = get_engine(0)
    params = fk.FoveationParams(fragment_size=16, strength=1.7)
    plan = DevicePlan(eng, (320, 200), 16, 1)
    stream = torch.cuda.Stream()
    req = FrameRequest(eng, plan, params, frame, out, host, stream)
    try:
        for (x, y) in [(160.0, 100.0), (0.0, 0.0), (319.0, 199.0), (33.5, 150.25)]:
            req.launch(x, y)
            stream.synchronize()
            ref = fk.foveate_batch(frame[None], np.asarray([[x, y]]), params)[0]
            assert torch.equal(out, ref)
            assert np.array_equal(host, ref.cpu().numpy())
            info = req.info()
            exp = fk.compute_fragment_shift((x, y), 16)
            assert info["shift"] == tuple(exp)
            assert info["length"].shape == (info["grid"][1], info["grid"][0])
        with pytest.raises(ValueError):
            req.launch(320.0, 10.0)
    finally:
        req.close()
        plan.close()


@pytest.mark.gpu
@pytest.mark.parametrize("split", ["0", "30", "55"])
def test_frame_request_in_two_bands_equals_foveate(split, monkeypatch):
    """A request renders frames of a megabyte and more in two bands from two plans so that the
    copy of the upper band runs under the render of the lower one (fk_request_create,
    FK_REQUEST_SPLIT): whatever the split row, the frame on the device and in pinned host memory
    equals foveate_batch -- fixations above, below and on the split row, RGB and gray."""
    import torch
    from paper_2012_08655_b200.engine import DevicePlan, FrameRequest, get_engine, pinned_empty

    monkeypatch.setenv("FK_REQUEST_SPLIT", split)
    rng = np.random.default_rng(21)
    eng = get_engine(0)
    for shape, F in (((1080, 1920, 3), 32), ((720, 1600, 1), 32), ((600, 800, 3), 16)):
        h, w, _ = shape
        frame = torch.from_numpy(rng.integers(0, 256, shape, dtype=np.uint8)).cuda()
        out = torch.empty_like(frame)
        host = pinned_empty(shape, np.uint8)
        params = fk.FoveationParams(fragment_size=F)
        plan = DevicePlan(eng, (w, h), F, 1)
        stream = torch.cuda.Stream()
        req = FrameRequest(eng, plan, params, frame, out, host, stream)
        try:
            ys = h * int(split) // 100
            for (x, y) in [(w / 2.0, h / 2.0), (3.0, 2.0), (w - 1.0, h - 1.0), (w / 3.0, float(ys)),
                           (w / 3.0, max(ys - 1.0, 0.0))]:
                out.zero_()
                host[...] = 0
                req.launch(x, y)
                stream.synchronize()
                ref = fk.foveate_batch(frame[None], np.asarray([[x, y]]), params)[0]
                assert torch.equal(out, ref), (shape, split, x, y)
                assert np.array_equal(host, ref.cpu().numpy()), (shape, split, x, y)
                assert req.info()["shift"] == tuple(fk.compute_fragment_shift((x, y), F))
        finally:
            req.close()
            plan.close()


@pytest.mark.gpu
def test_stream_single_channel_image():
    """Gray sources go through the row-partitioned kernel inside the request graph."""
    rng = np.random.default_rng(12)
    img = rng.integers(0, 256, (200, 300), dtype=np.uint8)
    with FoveationStream(img, fk.FoveationParams(fragment_size=32)) as s:
        for (x, y) in [(150.0, 100.0), (299.0, 0.0)]:
            s.submit(x, y)
            out, stats = s.get(timeout=30)
            ref, *_ = fk.foveate(fk.RasterImage.from_array(img),
                                 fk.FoveationParams(fragment_size=32, fixation=(x, y)))
            assert out.shape == (200, 300, 1) and np.array_equal(out, ref.data)
