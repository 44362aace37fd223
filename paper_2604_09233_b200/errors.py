"""Exception classes of the engine boundary (nfs/engine.py:22-27).

When the reference package `nfsense` is importable, `EngineError` and `MemoryBudgetError`
DERIVE from its classes, so callers that catch the reference's exceptions -- the CLI's exit-code
mapping (`nfs/cli.py:351-356`: MemoryBudgetError -> 4, EngineError -> 5) and the reference
tests' `pytest.raises(engine.EngineError)` -- catch the GPU path's errors unchanged.  Set
NFS_B200_STANDALONE=1 to skip the lookup.
"""

from __future__ import annotations

import os
import sys


def _reference_bases():
    """(EngineError, MemoryBudgetError) of the reference package, or (Exception, None)."""
    if os.environ.get("NFS_B200_STANDALONE") == "1":
        return Exception, None
    mod = sys.modules.get("nfsense.engine")   # already (possibly partially) imported
    if mod is None:
        try:
            import nfsense.engine as mod  # noqa: F811
        except Exception:
            return Exception, None
    eng, bud = getattr(mod, "EngineError", None), getattr(mod, "MemoryBudgetError", None)
    if not (isinstance(eng, type) and issubclass(eng, Exception)):
        return Exception, None
    return eng, bud if isinstance(bud, type) and issubclass(bud, eng) else None


_REF_ENGINE_ERROR, _REF_BUDGET_ERROR = _reference_bases()


class EngineError(_REF_ENGINE_ERROR):
    """Shape mismatch, non-finite data, CG breakdown or non-finite iterate."""


if _REF_BUDGET_ERROR is not None:
    class MemoryBudgetError(EngineError, _REF_BUDGET_ERROR):
        """Full phase matrix (or device memory) would not fit; use the split variant."""
else:
    class MemoryBudgetError(EngineError):
        """Full phase matrix (or device memory) would not fit; use the split variant."""


class DeviceError(EngineError):
    """CUDA / NCCL failure inside the native extension."""


class NativeUnavailable(EngineError):
    """The CUDA extension is not built or cannot be loaded: there is no CPU fallback."""


def bound_to_reference() -> bool:
    """True when the classes above derive from the reference package's exceptions."""
    return _REF_ENGINE_ERROR is not Exception
