"""Exception classes of the engine boundary (nfs/engine.py:22-27)."""


class EngineError(Exception):
    """Shape mismatch, non-finite data, CG breakdown or non-finite iterate."""


class MemoryBudgetError(EngineError):
    """Full phase matrix (or device memory) would not fit; use the split variant."""


class DeviceError(EngineError):
    """CUDA / NCCL failure inside the native extension."""


class NativeUnavailable(EngineError):
    """The CUDA extension is not built or cannot be loaded: there is no CPU fallback."""
