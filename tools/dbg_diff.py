"""Debug: where does the default kernel differ from the generic one?  (GPU box)"""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2012_08655_b200 as fk

W, H = 1920, 1080
fix = (float(sys.argv[1]), float(sys.argv[2])) if len(sys.argv) > 2 else (960.0, 540.0)
img = np.random.default_rng(0).integers(0, 256, (H, W, 3), dtype=np.uint8)
eng = fk.get_engine(0)
p = fk.FoveationParams(fragment_size=32, fixation=fix)
outs = {}
import os
VAR = int(os.environ.get('FK_VARIANT', '0'))
for v in (1, VAR):
    eng.set_kernel_variant(v)
    out, grid, bank, stats = fk.foveate(fk.RasterImage.from_array(img), p)
    outs[v] = out.data.astype(np.int16)
eng.set_kernel_variant(0)
d = np.abs(outs[VAR] - outs[1]).max(axis=2)
ys, xs = np.nonzero(d)
print("mismatching pixels:", len(ys), "max", d.max())
if len(ys):
    print("rows", ys.min(), ys.max(), "cols", xs.min(), xs.max())
    sx, sy = grid.shift
    cells = {}
    for y, x in zip(ys[:200000], xs[:200000]):
        gy = 0 if y < sy else (y - sy) // 32 + (1 if sy > 0 else 0)
        gx = 0 if x < sx else (x - sx) // 32 + (1 if sx > 0 else 0)
        cells.setdefault((gy, gx), []).append((y, x))
    lengths = np.asarray(bank.lengths)[np.asarray(grid.index)]
    for (gy, gx), pts in sorted(cells.items())[:40]:
        pts = np.asarray(pts)
        print(f"cell ({gy},{gx}) L={lengths[gy, gx]} n={len(pts)} rows {pts[:,0].min()}-{pts[:,0].max()} cols {pts[:,1].min()}-{pts[:,1].max()}")
    print("cells with mismatches:", len(cells))
