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


def test_window_starts_three_disjoint_windows_same_block_phase():
    b = _bench()
    for B, gen in ((4, 256), (16, 512), (32, 1024)):
        cyc = B + 1
        T = gen // B * cyc
        for warmup in (3, 5, 8):
            for steps in (1, 10, 17, 20, 30):
                st = b.window_starts(T, warmup, steps, cyc)
                assert st[0] == warmup and len(st) == 3
                assert all(s % cyc == warmup % cyc for s in st)            # same decode/flush mix
                assert all(b2 >= a + steps + 2 for a, b2 in zip(st, st[1:]))  # disjoint (+ profile pass)
                assert st[-1] + steps <= T
    assert b.window_starts(40, 5, 30, 17) == [5]                          # too short for three


def test_plan_requests_weak_and_lpt_strong():
    b = _bench()
    from synth import get_config
    c3 = get_config("C3")
    g0, l0, sc = b.plan_requests(c3, 2, 0)
    g1, _, _ = b.plan_requests(c3, 2, 1)
    assert sc == "weak" and g0 == list(range(64)) and g1 == list(range(64, 128)) and set(l0.values()) == {1024}
    c4 = get_config("C4")
    shards = [b.plan_requests(c4, 4, r) for r in range(4)]
    assert all(s[2] == "strong" for s in shards)
    assert sorted(sum((s[0] for s in shards), [])) == list(range(256))
    assert {len(s[0]) for s in shards} == {64}
    loads = [sum(s[1].values()) for s in shards]
    assert max(loads) / min(loads) < 1.01
    assert all(256 <= L <= 4096 for s in shards for L in s[1].values())


def test_gpus_n_relaunches_under_torchrun_and_rank0_prints_one_line():
    """bench.py --gpus 2 outside torchrun re-launches itself with 2 ranks (127.0.0.1 rendezvous); the
    reference arm runs on rank 0 only, the other rank exits 0 without work."""
    import json
    import subprocess
    import sys
    b = _bench()
    cmd = b.relaunch_cmd(["--gpus", "2"], 2, 12345)
    assert cmd[1:3] == ["-m", "torch.distributed.run"] and "--nproc-per-node=2" in cmd and "127.0.0.1" in cmd
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--impl", "reference",
                          "--workload", "C1", "--steps", "2", "--warmup", "3"], capture_output=True, text=True,
                         timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
