"""Density-map sigma fields (mirror of foveakit.retinal.ingest_density_map,
retinal.py:180-231).  The bilinear resampling of the map at the fragment midpoints and the
value -> sigma mapping run in the plan kernel (csrc/fk_plan.cu), bit-identically to the
reference."""

from __future__ import annotations

from .retinal import SigmaField
from .tiling import span_count


def ingest_density_map(density, sigma_max, image_size, fragment_size, shift, *, device=0):
    """Sigma field from an arbitrary 1-channel retinal-density map: sample value v in
    [0, 255] maps to sigma = sigma_max * (1 - v / 255)."""
    from .engine import get_engine

    if density.channels != 1:
        raise ValueError(f"density map must be 1-channel, got {density.channels}")
    if sigma_max < 0:
        raise ValueError(f"sigma_max must be >= 0, got {sigma_max}")
    w, h = image_size
    if w < 1 or h < 1:
        raise ValueError(f"extent must be positive, got {w}x{h}")
    for off in shift:
        if not 0 <= off < fragment_size:
            raise ValueError(f"offset {off} outside [0, {fragment_size})")
    eng = get_engine(device)
    with eng._lock:
        plan = eng.plan_for(image_size, fragment_size, 1)
        plan.density(density.data[:, :, 0], sigma_max, fragment_size, [(0.0, 0.0)], shift=shift)
        got = plan.read(0)
    assert got["grid"] == (span_count(w, fragment_size, shift[0]),
                           span_count(h, fragment_size, shift[1]))
    return SigmaField(grid_width=got["grid"][0], grid_height=got["grid"][1], sigma=got["sigma"])
