"""Host-side pieces of bench.py (no GPU): the nvidia-smi clock summary and the e2e window's block-phase
alignment."""
import importlib.util
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def test_clock_summary_median_and_reasons():
    b = _bench()
    c = b.Clocks(0)
    c.out = "".join(f"0, {mhz}, 1965, 900, Not Active, Not Active, Not Active, {cap}\n"
                    for mhz, cap in [(1800, "Active"), (1900, "Not Active"), (1850, "Not Active")])
    s = c.summary()
    assert s["sm_mhz"] == 1850.0 and s["sm_max_mhz"] == 1965.0 and s["samples"] == 3
    assert s["reasons"] == ["sw_power_cap"]
    c.out = ""
    assert c.summary()["reasons"] == ["unsampled"]


def test_e2e_window_starts_at_the_timed_windows_block_phase():
    # bench.py runs (warmup - (warmup + steps)) % (B + 1) untimed steps between the timed and the e2e
    # windows, so the e2e window starts at the timed window's phase of the (B decode + 1 flush) cycle
    for B in (4, 16, 32):
        cyc = B + 1
        for warmup in (3, 5):
            for steps in (1, 10, 17, 30, 100):
                align = (warmup - (warmup + steps)) % cyc
                assert (warmup + steps + align) % cyc == warmup % cyc
                assert 0 <= align < cyc
