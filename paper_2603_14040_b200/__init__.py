"""B200-native matrix-free geometric-multigrid Stokes solver (arXiv 2603.14040 hot path).

The numerical path lives in libstokes_b200.so (hand-written sm_100a CUDA kernels behind
the C ABI of include/stokes.h); this package is its thin Python binding.
"""
from .stokes import (FREE_SLIP, NO_SLIP, Opts, Stokes, StokesDist, StokesError, default_opts, lib,  # noqa: F401
                     nccl_unique_id, shapes, tile_windows)

__all__ = ["Stokes", "StokesDist", "tile_windows", "nccl_unique_id", "StokesError", "Opts", "default_opts", "lib", "shapes", "FREE_SLIP", "NO_SLIP"]
