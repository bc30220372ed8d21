import numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_2012_08655_b200 as fk
rng = np.random.default_rng(13)
img = rng.integers(0, 256, (1, 96, 128, 1), dtype=np.uint8)
frames = torch.from_numpy(img).cuda()
out = fk.foveate_batch(frames, np.asarray([[100.0, 40.0]]), fk.FoveationParams(fragment_size=32))
torch.cuda.synchronize()
print("ok", int(out.sum()))
