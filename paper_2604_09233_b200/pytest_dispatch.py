"""pytest plugin: run the reference's own test files through the GPU dispatch.

    NFSENSE_BACKEND=b200 PYTHONPATH=baseline/_ref:. python -m pytest \
        -p paper_2604_09233_b200.pytest_dispatch baseline/_ref_tests/test_engine.py

`pytest_configure` runs before the test modules are imported, so their
`from nfsense import recon_full` bindings already see the GPU functions.  The session summary
line `b200 dispatch calls: {...}` shows how many calls took the GPU path.
"""

import os


def pytest_configure(config):
    if os.environ.get("NFSENSE_BACKEND") == "b200":
        from .dispatch import install
        install()


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    if os.environ.get("NFSENSE_BACKEND") == "b200":
        from .dispatch import CALLS
        terminalreporter.write_line(f"b200 dispatch calls: {CALLS}")
