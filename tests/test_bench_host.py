"""Host logic of bench.py that the JSON contract depends on (no GPU): the clock sampler keeps
only the nvidia-smi samples taken inside the timed region and reports every throttle reason
seen there."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402


def _row(mhz, power_cap=False, thermal=False):
    return [str(mhz), "1965", "0x0", "Not Active", "Not Active",
            "Active" if thermal else "Not Active", "Active" if power_cap else "Not Active"]


def test_clock_sampler_window_and_reasons():
    s = bench.ClockSampler(0)
    s.rows = [(0.5, _row(1965)), (1.1, _row(1800, power_cap=True)), (1.2, _row(1700)),
              (1.3, _row(1750)), (2.5, _row(1000, thermal=True))]
    out = s.summary(1.0, 2.0)
    assert out["samples"] == 3
    assert out["sm_mhz"] == 1750.0 and out["sm_max_mhz"] == 1965.0
    assert out["reasons"] == ["sw_power_cap"]          # the thermal sample lies outside


def test_clock_sampler_short_region_and_unsampled():
    s = bench.ClockSampler(0)
    s.rows = [(0.0, _row(1965)), (5.0, _row(1500))]
    # shorter than the sampling period: the nearest samples
    assert s.summary(0.1, 0.2)["sm_mhz"] in (1965.0, 1732.5, 1500.0)
    empty = bench.ClockSampler(0)
    assert empty.summary()["reasons"] == ["unsampled"]


def test_both_arms_print_the_same_config():
    """The driver compares the two arms' `config` dicts: they are built by one function."""
    for cfg in ("B", "D"):
        assert bench.bench_config(cfg) == bench.bench_config(cfg)
        assert set(bench.bench_config(cfg)) == {"workload", "cg_iterations_e2e", "l2"}


def test_reference_cpu_sample_runs_the_staged_reference():
    """The CPU legs time the unmodified reference (baseline/_ref) through its own recon_split;
    a tiny row sample of config B is enough to exercise the path."""
    if bench.load_reference() is None:
        import pytest
        pytest.skip("reference not staged (tools/stage_reference.sh)")
    prob = bench._problem("B")
    v, dt, kind = bench.cpu_apply_sample(prob, rows=8)
    assert kind == "reference" and v > 0 and dt > 0


def test_host_info_records_cpu_and_blas():
    info = bench.host_info()
    assert info["cores"] >= 1 and "threadpools" in info
