"""B200-native blockwise foveated rendering -- drop-in for the ``plan`` / ``render`` /
``foveate`` path of foveakit (arXiv 2012.08655), backed by hand-written sm_100a CUDA
kernels behind a C ABI (include/fovea.h, csrc/).

Only the hot path and its "next" rows are here: plan / render /
foveate, density-map sigma fields, the latest-wins streaming layer, the SSIM checker
(``quality``) and ``adapter``, which routes the reference's own command line, timing harness
and service onto this path when foveakit is importable.  The reference's file codecs, web
service, pyramid baseline and per-pixel oracle are out of scope.  There is no CPU fallback: importing works anywhere, but every compute entry point
needs a CUDA device.
"""

from .imaging import RasterImage
from .retinal import (
    FoveationParams,
    SigmaField,
    build_sigma_field,
    contrast_threshold,
    cutoff_cpd,
    cutoff_cpp,
    eccentricity_of,
    sigma_at,
)
from .filters import (
    FilterBank,
    build_bank,
    filter_length,
    gaussian_filter_1d,
    total_coefficients,
)
from .tiling import cell_of, fragment_spans, span_midpoints
from .blockwise import (
    BlurGrid,
    RenderStats,
    Tile,
    build_blur_grid,
    compute_fragment_shift,
    foveate,
    foveate_batch,
    plan,
    render,
)
from .density import ingest_density_map
from .engine import Engine, get_engine, pinned_empty, shard_range
from .streaming import FoveationStream
from .quality import SSIMMap, mean_ssim_map, ssim_map

__version__ = "0.1.0"

__all__ = [
    "RasterImage", "SSIMMap", "ssim_map", "mean_ssim_map",
    "FoveationParams", "SigmaField", "build_sigma_field", "contrast_threshold",
    "cutoff_cpd", "cutoff_cpp", "eccentricity_of", "ingest_density_map", "sigma_at",
    "FilterBank", "build_bank", "filter_length", "gaussian_filter_1d", "total_coefficients",
    "cell_of", "fragment_spans", "span_midpoints",
    "BlurGrid", "RenderStats", "Tile", "build_blur_grid", "compute_fragment_shift", "foveate",
    "foveate_batch", "plan", "render",
    "Engine", "get_engine", "pinned_empty", "shard_range", "FoveationStream",
]
