import sys
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2012_08655_b200 as fk
eng = fk.get_engine(0)
rng = np.random.default_rng(0)
h, w = 270, 480
img = rng.integers(0, 256, (1, h, w, 3), dtype=np.uint8)
frames = torch.from_numpy(img).cuda()
fx = np.asarray([[240.0, 135.0]])
p = fk.FoveationParams(fragment_size=32)
eng.set_kernel_variant(1); ref = fk.foveate_batch(frames, fx, p).clone(); torch.cuda.synchronize()
eng.set_kernel_variant(5); out = fk.foveate_batch(frames, fx, p); torch.cuda.synchronize()
d = (out.int() - ref.int()).abs()
print("max diff", int(d.max()), "mismatch px", int((d.amax(dim=3) > 0).sum()))
