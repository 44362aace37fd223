"""The drop-in contract seen from the reference's side.

The UNMODIFIED reference package is staged by `tools/stage_reference.sh` into the git-ignored
`baseline/_ref` (pip install) and `baseline/_ref_tests` (its own test files); both travel to the
GPU box with the snapshot.  The reference's tests then run unchanged with the GPU dispatch
installed (`-p paper_2604_09233_b200.pytest_dispatch`, NFSENSE_BACKEND=b200):

* CPU (here): the error contract -- EncodingInputs validation, the budget rule
  (`pytest.raises(MemoryBudgetError, match="split")`, tests/test_engine.py:111-115), split
  without block starts, and the CLI's exit code 4 for `recon --memory-budget 64`
  (tests/test_cli.py:203-205, nfs/cli.py:351-353) -- none of which reach the device;
* GPU: the reference's whole tests/test_engine.py and tests/test_acceptance.py plus the CLI
  chain through `recon` on the B200 path in FP64 parity mode, with the routed-call counter
  proving the GPU functions ran.
"""

import os
import subprocess
import sys
import textwrap

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
REF_TESTS = os.path.join(ROOT, "baseline", "_ref_tests")


def _staged():
    if os.path.isdir(os.path.join(REF, "nfsense")) and os.path.isdir(REF_TESTS):
        return True
    if os.path.isdir("/root/reference/pkg"):   # build container: stage it now
        subprocess.run(["bash", os.path.join(ROOT, "tools", "stage_reference.sh")], check=True,
                       capture_output=True)
        return True
    return False


needs_ref = pytest.mark.skipif(not _staged(), reason="reference package not staged (tools/stage_reference.sh)")


def _env(**extra):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, ROOT] + ([env["PYTHONPATH"]] if env.get("PYTHONPATH") else []))
    env["NFSENSE_BACKEND"] = "b200"
    env.pop("NFS_B200_STANDALONE", None)
    env.update(extra)
    return env


def run_reference_tests(tmp_path, selectors, k=None, timeout=1200, **env):
    ini = tmp_path / "pytest.ini"
    ini.write_text("[pytest]\n")
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "paper_2604_09233_b200.pytest_dispatch",
           "-p", "no:cacheprovider", "--rootdir", REF_TESTS, "-c", str(ini), *selectors]
    if k:
        cmd += ["-k", k]
    r = subprocess.run(cmd, cwd=REF_TESTS, env=_env(**env), capture_output=True, text=True, timeout=timeout)
    return r.returncode, r.stdout + r.stderr


def dispatch_calls(out):
    line = [ln for ln in out.splitlines() if ln.startswith("b200 dispatch calls:")]
    assert line, out[-3000:]
    return eval(line[-1].split(":", 1)[1])   # a dict literal printed by the plugin


CLI_SCRIPT = textwrap.dedent("""
    import os, sys, pathlib
    from paper_2604_09233_b200.dispatch import install, CALLS
    install()
    from nfsense.cli import main
    from nfsense.pipeline import read_cg_log_csv
    d = pathlib.Path(sys.argv[1])
    (d / "config.toml").write_text('''{config}''')
    ds = str(d / "ds")
    assert main(["simulate", "--config", str(d / "config.toml"), "--out", ds, "--seed", "11"]) == 0
    for argv in (["masks", ds], ["sensmaps", ds], ["b0map", ds], ["kfilter", ds]):
        assert main(argv) == 0, argv
    rc = main(["recon", ds, "--iters", "2", "--memory-budget", "64"])
    print("budget_rc", rc)
    if sys.argv[2] == "gpu":
        rc = main(["recon", ds, "--iters", "8", "--log", str(d / "cg_log.csv")])
        print("recon_rc", rc, "log_rows", len(read_cg_log_csv(str(d / "cg_log.csv"))))
    print("calls", CALLS["recon_full"] + CALLS["recon_split"])
""")

# tests/test_cli.py:8-36 (the reference CLI test configuration)
CLI_CONFIG = """[grid]
dims = [20, 20, 1]
fov_m = [0.2, 0.2, 0.002]
[phantom]
kind = "discs"
smooth_phase = true
[coils]
count = 5
[prescan]
echoes = 6
noise_sd = 0.02
[trajectory]
kind = "spiral"
samples = 700
turns = 10
[b0]
pattern = "linear"
amplitude = 50.0
[noise]
sigma_sd = 0.002
"""


def run_cli(tmp_path, mode):
    script = CLI_SCRIPT.replace("{config}", CLI_CONFIG)
    r = subprocess.run([sys.executable, "-c", script, str(tmp_path), mode], env=_env(), capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    out = {}
    for ln in r.stdout.splitlines():   # the CLI prints its own progress lines too
        w = ln.split()
        if w and w[0] in ("budget_rc", "recon_rc", "calls"):
            out.update(zip(w[::2], w[1::2]))
    return out


@needs_ref
def test_errors_derive_from_reference_classes():
    code = ("import nfsense.engine as ref; from paper_2604_09233_b200 import errors as e;"
            "assert issubclass(e.MemoryBudgetError, ref.MemoryBudgetError);"
            "assert issubclass(e.EngineError, ref.EngineError);"
            "assert issubclass(e.DeviceError, ref.EngineError);"
            "assert issubclass(e.MemoryBudgetError, e.EngineError); print('ok')")
    r = subprocess.run([sys.executable, "-c", code], env=_env(), capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr


@needs_ref
def test_reference_error_contract_through_dispatch(tmp_path):
    """The reference's own validation / budget / split tests, which never reach the device."""
    rc, out = run_reference_tests(
        tmp_path, ["test_engine.py"],
        k="test_memory_budget or Validation or ChooseBlockStarts or BuildBases or needs_block_starts")
    assert rc == 0, out[-4000:]
    assert "11 passed" in out, out[-2000:]
    calls = dispatch_calls(out)
    assert calls["recon_full"] >= 1 and calls["recon_split"] >= 1   # the routed functions raised


@needs_ref
def test_reference_cli_budget_exit_code(tmp_path):
    """`nfsense recon --memory-budget 64` exits 4 with the GPU dispatch (nfs/cli.py:351-353)."""
    out = run_cli(tmp_path, "cpu")
    assert out["budget_rc"] == "4"
    assert int(out["calls"]) >= 1


@pytest.mark.gpu
@needs_ref
def test_reference_engine_tests_on_gpu(tmp_path):
    """The reference's tests/test_engine.py, unchanged, on the B200 path (FP64 parity mode)."""
    rc, out = run_reference_tests(tmp_path, ["test_engine.py"], NFS_B200_PRECISION="fp64")
    assert rc == 0, out[-6000:]
    calls = dispatch_calls(out)
    assert calls["recon_full"] >= 5 and calls["apply_E"] >= 2 and calls["phase_block"] >= 4, calls


@pytest.mark.gpu
@needs_ref
def test_reference_acceptance_engine_cases_on_gpu(tmp_path):
    """The engine-facing cases of the reference's tests/test_acceptance.py (oracle equivalence,
    exact recovery, parallel imaging, B0 benefit, split/full equivalence, CG over-iteration,
    pipeline determinism) on the B200 path, unchanged."""
    rc, out = run_reference_tests(
        tmp_path, ["test_acceptance.py"],
        k="oracle_equivalence or exact_recovery or parallel_imaging or b0_correction or "
          "split_full or cg_over_iteration or pipeline_determinism",
        NFS_B200_PRECISION="fp64")
    assert rc == 0, out[-6000:]
    assert "7 passed" in out, out[-3000:]
    calls = dispatch_calls(out)
    assert calls["recon_full"] >= 6 and calls["recon_split"] >= 4, calls


@pytest.mark.gpu
@needs_ref
def test_reference_cli_recon_on_gpu(tmp_path):
    out = run_cli(tmp_path, "gpu")
    assert out["budget_rc"] == "4"
    assert out["recon_rc"] == "0" and int(out["log_rows"]) >= 1
    assert int(out["calls"]) >= 2
