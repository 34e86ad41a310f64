"""Host logic of bench.py (no GPU): the clock sampler keeps only the samples
inside the timed window (or the nearest two when the window is shorter than
the sampling period) and reports the throttle reasons seen there."""
import importlib.util
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


class _Done:
    def terminate(self):
        pass

    def wait(self, timeout=None):
        return 0

    def poll(self):
        return 0

    def kill(self):
        pass


def sampler_with(bench, tmp_path, lines):
    s = bench.ClockSampler(0)
    s.path = str(tmp_path / "smi.csv")
    with open(s.path, "w") as f:
        f.write("\n".join(lines) + "\n")
    s.proc = _Done()
    return s


def line(ts, sm, power_cap="Not Active", hw="Not Active"):
    return f"{ts}, {sm}, 1965, 700.0, 0x0, {hw}, Not Active, Not Active, {power_cap}"


def test_window_filter_and_reasons(bench, tmp_path):
    import datetime
    t = datetime.datetime(2026, 10, 20, 1, 2, 3)
    lines = [line((t + datetime.timedelta(seconds=0.1 * k)).strftime("%Y/%m/%d %H:%M:%S.%f")[:-3],
                  1000 + 100 * k, "Active" if k == 7 else "Not Active") for k in range(10)]
    s = sampler_with(bench, tmp_path, lines)
    t0 = (t + datetime.timedelta(seconds=0.35)).timestamp()
    t1 = (t + datetime.timedelta(seconds=0.75)).timestamp()
    r = s.stop(t0, t1)
    assert r["samples"] == 4                           # samples 4, 5, 6, 7
    assert r["sm_mhz"] == 1550.0 and r["sm_max_mhz"] == 1965.0
    assert r["reasons"] == ["sw_power_cap"]


def test_short_window_takes_nearest(bench, tmp_path):
    import datetime
    t = datetime.datetime(2026, 10, 20, 1, 2, 3)
    lines = [line((t + datetime.timedelta(seconds=0.1 * k)).strftime("%Y/%m/%d %H:%M:%S.%f")[:-3], 1900 + k)
             for k in range(5)]
    s = sampler_with(bench, tmp_path, lines)
    t0 = (t + datetime.timedelta(seconds=0.21)).timestamp()
    r = s.stop(t0, t0 + 0.01)
    assert r["samples"] == 2 and r["reasons"] == []


def test_window_starts(bench):
    """Five timed windows of K iterations spread over stage B (250-999) after the
    warm-up; as many as fit, at least one."""
    s = bench.window_starts(250, 5, 20)
    assert len(s) == 5 and s[0] == 255 and s[-1] + 20 <= 1000 and all(b - a >= 20 for a, b in zip(s, s[1:]))
    s = bench.window_starts(250, 20, 200)
    assert len(s) == 3 and s[0] == 270 and s[-1] + 200 <= 1000
    assert bench.window_starts(250, 20, 1000) == [270]
