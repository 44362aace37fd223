"""Reference-side dispatch: route the reference package's engine entry points to the GPU path.

The binding a maintainer adds at the END of the reference's `nfs/engine.py`:

    if os.environ.get("NFSENSE_BACKEND") == "b200":
        from paper_2604_09233_b200.dispatch import install
        install()

`install()` rebinds `phase_block`, `apply_E`, `apply_EH`, `recon_full` and `recon_split` in
`nfsense.engine` and in the `nfsense` package namespace (nfs/__init__.py:18-27) to the GPU
implementations; `EncodingInputs`, `CGLog`, `choose_block_starts` and `build_bases` stay the
reference's own (host-side).  Results come back as the reference's `ReconImage` / `CGLog`, and
the GPU path's `EngineError` / `MemoryBudgetError` derive from the reference's classes
(errors.py), so `pipeline.run_recon`, the CLI's exit codes (nfs/cli.py:351-356) and the
reference tests see no difference.  `CALLS` counts the routed calls (evidence that the GPU path
ran).
"""

from __future__ import annotations

import functools
import sys

ROUTED = ("phase_block", "apply_E", "apply_EH", "recon_full", "recon_split")
CALLS = {name: 0 for name in ROUTED}
_installed = False


def _counted(name, fn):
    @functools.wraps(fn)
    def wrapper(*args, **kwargs):
        CALLS[name] += 1
        return fn(*args, **kwargs)
    return wrapper


def install() -> None:
    """Rebind the reference's engine entry points to the GPU path (idempotent)."""
    global _installed
    if _installed:
        return
    ref = sys.modules.get("nfsense.engine")
    if ref is None:
        import nfsense.engine as ref  # noqa: F811
    from . import engine as gpu
    from .errors import bound_to_reference

    if not bound_to_reference():
        raise ImportError("paper_2604_09233_b200 was imported with NFS_B200_STANDALONE=1 or before "
                          "nfsense was importable; its exceptions cannot derive from the reference's")
    core = sys.modules.get("nfsense.core")
    if core is None:
        import nfsense.core as core  # noqa: F811
    gpu.RESULT_TYPES["ReconImage"] = core.ReconImage
    gpu.RESULT_TYPES["CGLog"] = ref.CGLog
    pkg = sys.modules.get("nfsense")
    for name in ROUTED:
        fn = _counted(name, getattr(gpu, name))
        setattr(ref, name, fn)
        if pkg is not None and hasattr(pkg, name):
            setattr(pkg, name, fn)
    _installed = True
