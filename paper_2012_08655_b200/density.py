"""Density-map sigma fields (foveakit.retinal.ingest_density_map, retinal.py:180-231).

SURVEY.md 8(f) rank 1 -- a "next" row, not yet built on the device.  The argument checks
and error messages of the reference are in place so callers fail the same way."""

from __future__ import annotations


def ingest_density_map(density, sigma_max, image_size, fragment_size, shift, *, device=0):
    if density.channels != 1:
        raise ValueError(f"density map must be 1-channel, got {density.channels}")
    if sigma_max < 0:
        raise ValueError(f"sigma_max must be >= 0, got {sigma_max}")
    raise NotImplementedError(
        "density-map sigma fields are not built yet in the B200 path (SURVEY.md 8f rank 1)")
