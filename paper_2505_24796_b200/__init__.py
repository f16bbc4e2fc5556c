"""B200-native TC-GS forward renderer (arxiv 2505.24796) -- a drop-in for the
reference package ``tilesplat``'s render entry point.

    import paper_2505_24796_b200 as tcgs
    img, stats = tcgs.render(scene, cam)          # tilesplat.render(scene, cam, backend)

Preprocess, binning/sort and tensor-core alpha + blending run as hand-written
sm_100a CUDA kernels in libtcgs.so (include/tcgs.h), loaded through ctypes;
there is no CPU fallback.  Names mirror /root/reference/pkg/src/tilesplat/
__init__.py:16-40 for the render path.
"""

from .raster import (  # noqa: F401
    ALPHA_CULL_THRESHOLD,
    TERMINATION_THRESHOLD,
    TILE_SIZE,
    Backend,
    Frame,
    FragmentStats,
    GaussianCloud,
    ImageBuffer,
    Renderer,
    ViewRenderer,
    computation_model,
    make_backend,
    rasterize,
    render,
)

from .pipeline import FramePipeline  # noqa: F401,E402
from .ply import SceneFormatError, SceneValidationError, load_ply, read_ply, write_ply  # noqa: F401,E402

__all__ = [
    "FramePipeline",
    "SceneFormatError",
    "SceneValidationError",
    "load_ply",
    "read_ply",
    "write_ply",
    "ALPHA_CULL_THRESHOLD",
    "TERMINATION_THRESHOLD",
    "TILE_SIZE",
    "Backend",
    "Frame",
    "FragmentStats",
    "GaussianCloud",
    "ImageBuffer",
    "Renderer",
    "ViewRenderer",
    "computation_model",
    "make_backend",
    "rasterize",
    "render",
]
