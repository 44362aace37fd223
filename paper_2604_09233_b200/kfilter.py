"""k-space filter application on the device.

`apply_filter` = IFFT(fftshift-centred FFT(image) * filter) exactly as nfs/kfilter.py:83-97,
run with cuFFT through torch on the GPU that holds the reconstruction.  The filter itself
(convex hull of the trajectory, nfs/kfilter.py:37-64) is calibration and stays on the host.
"""

from __future__ import annotations

import numpy as np

from .core import Grid
from .errors import EngineError, NativeUnavailable


def apply_filter(image: np.ndarray, filt: np.ndarray, grid: Grid, device: int | None = None) -> np.ndarray:
    import torch

    if not torch.cuda.is_available():
        raise NativeUnavailable("apply_filter runs on the GPU (cuFFT); no CUDA device visible")
    image = np.asarray(image).reshape(-1)
    filt = np.asarray(filt, dtype=float).reshape(-1)
    if image.size != grid.nvox or filt.size != grid.nvox:
        raise EngineError("image/filter length does not match the grid")
    nx, ny, nz = grid.dims
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    # x-fastest flat vector == C-order (nz, ny, nx); an all-axes FFT is axis-order agnostic
    vol = torch.from_numpy(np.ascontiguousarray(image, dtype=np.complex128)).to(dev).reshape(nz, ny, nx)
    f = torch.from_numpy(np.ascontiguousarray(filt)).to(dev).reshape(nz, ny, nx)
    spec = torch.fft.fftshift(torch.fft.fftn(vol)) * f
    out = torch.fft.ifftn(torch.fft.ifftshift(spec))
    return out.reshape(-1).cpu().numpy()
