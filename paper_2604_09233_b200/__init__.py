"""B200-native non-Fourier SENSE reconstruction hot path (arXiv 2604.09233).

Drop-in for the reference package's engine API (nfs/__init__.py:18-27): the same names
and signatures, backed by hand-written sm_100a CUDA kernels behind a C ABI
(include/nfs_b200.h).  See DESIGN.md.
"""

from .core import Grid, ReconImage, grid_coordinates
from .engine import (
    CGLog,
    DatasetSamples,
    DeviceRMSE,
    DeviceSens,
    DeviceSSIM,
    DeviceSpatial,
    EncodingInputs,
    EngineError,
    MemoryBudgetError,
    apply_E,
    apply_EH,
    build_bases,
    choose_block_starts,
    intensity_correction,
    phase_block,
    recon_full,
    recon_slices,
    recon_split,
)

__all__ = [
    "CGLog", "DatasetSamples", "DeviceRMSE", "DeviceSens", "DeviceSSIM", "DeviceSpatial", "EncodingInputs", "EngineError", "Grid", "MemoryBudgetError", "ReconImage",
    "apply_E", "apply_EH", "build_bases", "choose_block_starts", "grid_coordinates", "intensity_correction",
    "phase_block", "recon_full", "recon_slices", "recon_split",
]

__version__ = "0.1.0"
