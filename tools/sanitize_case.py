import sys
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2012_08655_b200 as fk
rng = np.random.default_rng(0)
for (h, w, F, fix) in [(270, 480, 32, (301.0, 77.0)), (200, 320, 32, (0.0, 0.0)), (128, 256, 16, (255.0, 127.0))]:
    img = rng.integers(0, 256, (2, h, w, 3), dtype=np.uint8)
    frames = torch.from_numpy(img).cuda()
    fx = np.asarray([fix, (w / 2.0, h / 2.0)])
    out = fk.foveate_batch(frames, fx, fk.FoveationParams(fragment_size=F, strength=1.5))
    torch.cuda.synchronize()
    f32 = torch.from_numpy(rng.random((1, h, w, 3), dtype=np.float32)).cuda()
    out2 = fk.foveate_batch(f32, fx[:1], fk.FoveationParams(fragment_size=F))
    torch.cuda.synchronize()
print("done")
