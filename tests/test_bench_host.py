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
    s.window(1.0, 2.0)
    out = s.summary()
    assert out["samples"] == 3
    assert out["sm_mhz"] == 1750.0 and out["sm_max_mhz"] == 1965.0
    assert out["reasons"] == ["sw_power_cap"]          # the thermal sample lies outside


def test_clock_sampler_short_region_and_unsampled():
    s = bench.ClockSampler(0)
    s.rows = [(0.0, _row(1965)), (5.0, _row(1500))]
    s.window(0.1, 0.2)                                    # shorter than the sampling period
    assert s.summary()["sm_mhz"] in (1965.0, 1732.5, 1500.0)
    empty = bench.ClockSampler(0)
    assert empty.summary()["reasons"] == ["unsampled"]
