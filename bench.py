"""Decoded tokens/sec of the FOCUS block-diffusion decode step on B200 (BASELINE.json metric).

  python bench.py [--gpus N --steps K --warmup W]            # our CUDA path (libfocus.so)
  python bench.py --impl reference [--steps K --warmup W]    # the CPU oracle on a bounded sample

Workload (per GPU): C3 = SDAR-8B-shaped random-init model (36 layers, d 4096, GQA 32/8, d_ff 12288,
vocab 151936), block 16, 64 requests, prompt 1024, gen 512 (BASELINE.json configs[2]).  Under
torchrun each rank owns 64 requests of its own (request-level data parallel, weak scaling).
A step = focus_step_block + focus_commit over all requests of the rank (the whole hot path).
Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decoded tokens/sec (SDAR-8B-shaped, block 16) at 1/2/4/8 B200; % roofline"
UNIT = "tokens/s"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return dict(hbm=float(d["hbm_gbs"]), tc=float(d["bf16_tflops"]), tc_sus=float(d["bf16_tflops_sustained"]),
                    src="measured (MEASURED_PEAKS.json)")
    return dict(hbm=6650.0, tc=1590.0, tc_sus=1400.0, src="fallback (B200_PROFILING.md)")


class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu, self.p, self.lines, self.th = gpu, None, [], None
        self.t0 = self.t1 = 0.0

    def _reader(self):
        for line in self.p.stdout:
            self.lines.append((time.time(), line))

    def __enter__(self):
        # the sampler is started and its first sample awaited BEFORE the timed region begins (nvidia-smi
        # takes a few hundred ms to start, longer than a short timed region); samples are time-stamped
        # on arrival and the summary keeps those that fall inside the region
        import threading
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + self.Q, "--format=csv,noheader,nounits",
                                       "-lms", "25"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._reader, daemon=True)
            self.th.start()
            deadline = time.time() + 10.0
            while not self.lines and time.time() < deadline and self.p.poll() is None:
                time.sleep(0.01)
        except Exception:
            self.p = None
        self.t0 = time.time()
        return self

    def __exit__(self, *a):
        self.t1 = time.time()
        time.sleep(0.06)                                 # let the in-flight sample arrive
        if self.p is not None:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except Exception:
                pass
            if self.th is not None:
                self.th.join(timeout=2)
        inside = [ln for (t, ln) in self.lines if self.t0 - 0.03 <= t <= self.t1 + 0.03]
        self.out = "".join(inside)

    def summary(self):
        rows = [r.split(",") for r in (self.out or "").strip().splitlines() if r.count(",") >= 7]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(r[1]) for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if "Active" in r[4 + k] and "Not" not in r[4 + k]})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": float(rows[0][2]), "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------------------------------ algorithmic work
def step_work(model, B, counters, states, rids):
    """SURVEY 8(d) per-step algorithmic FLOPs / bytes by kernel family, from the step's live sizes."""
    d, ff, V, L = model.d_model, model.d_ff, model.vocab, model.n_layers
    qkv = model.qkv_dim
    qd = model.n_q_heads * model.head_dim
    MP, MS, ML = counters
    Wqkv, Wo, Wgu, Wd = d * qkv, qd * d, 2 * d * ff, d * ff
    fl = {
        "gemm_qkv": 2 * Wqkv * (2 * MP + (L - 2) * MS),
        "gemm_o": 2 * Wo * (MP + (L - 1) * MS),
        "gemm_gu": 2 * Wgu * (MP + (L - 1) * MS),
        "gemm_down": 2 * Wd * (MP + (L - 1) * MS),
        "gemm_lm": 2 * d * V * ML,
    }
    # weight bytes each GEMM family must stream once per step (bf16)
    wb = {"gemm_qkv": 2 * Wqkv * L, "gemm_o": 2 * Wo * L, "gemm_gu": 2 * Wgu * L, "gemm_down": 2 * Wd * L,
          "gemm_lm": 2 * d * V}
    kvb = 4 * model.n_kv_heads * model.head_dim          # K+V bf16 bytes per token per layer
    attn_bytes = 0
    for r in rids:
        s = states[r]
        if not s.active:
            continue
        attn_bytes += kvb * (2 * (s.s + B) + (L - 2) * (s.s + s.R_new + 1))
    return fl, wb, attn_bytes


def build_ctx(run, n_req):
    from paper_2601_23278_b200 import FocusContext, make_config
    return FocusContext(make_config(run, max_requests=n_req))


def run_focus(args):
    import torch
    from paper_2601_23278_b200 import dist as D
    from paper_2601_23278_b200.focus import focus_commit_result
    from synth import get_config
    from synth.gen import prompt_tokens

    rank, world, local = D.init("nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    run = get_config(args.workload)
    n_req = run.n_requests
    gids = list(range(rank * n_req, (rank + 1) * n_req))          # weak scaling: 64 requests per rank
    ctx = build_ctx(run, n_req)
    rids = list(range(n_req))
    t0 = time.time()
    for i, r in enumerate(rids):
        ctx.focus_kv_append(r, prompt_tokens(gids[i], run.prompt_len, run.model.vocab), run.gen_len)
    torch.cuda.synchronize()
    prefill_s = time.time() - t0
    st = ctx.stream

    def tok_sum():
        s = ctx.states()
        return sum(int(s[r].token_sum) for r in rids)

    for _ in range(args.warmup):
        ctx.focus_step_block(rids)
        ctx.focus_commit(rids)
    ctx.focus_sync()

    # ---- timed: K steps, inputs resident in HBM, device-timed with events on the library stream
    dec0 = tok_sum()
    l0 = ctx.launches()
    D.barrier(dev)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ncu_step = bool(os.environ.get("FOCUS_NCU_STEP"))  # ncu --profile-from-start off: capture timed step 1 only
    with Clocks(local) as clk:
        ev0.record(st)
        for i in range(args.steps):
            if ncu_step and i == 0:
                torch.cuda.profiler.start()
            ctx.focus_step_block(rids)
            ctx.focus_commit(rids)
            if ncu_step and i == 0:
                torch.cuda.profiler.stop()
        ev1.record(st)
        torch.cuda.synchronize()
    D.barrier(dev)
    ms = ev0.elapsed_time(ev1)
    launches = ctx.launches() - l0
    dec = tok_sum() - dec0
    ms_max = D.reduce_max(ms, dev)
    dec_all = D.reduce_sum(dec, dev)
    value = dec_all / (ms_max / 1e3)

    # ---- e2e: through the C ABI with host buffers; every step uploads the request list from host
    # memory and copies its commit results (newly decoded tokens per request) back into pinned host
    # memory.  The readback is double-buffered like a serving loop: step t's results are read on the
    # host (event wait + parse) while step t+1 runs, since all decode state stays on the device.
    rsz = __import__("ctypes").sizeof(focus_commit_result)
    res = [torch.empty(n_req * rsz, dtype=torch.uint8).pin_memory() for _ in range(2)]
    done = [None, None]
    e2e_steps = max(1, min(args.steps, 20))
    # start the e2e window at the same phase of the block cycle (B decode steps + 1 flush step per
    # block under the synthetic dynamics) as the timed window, so both windows hold the same mix of
    # decode and flush steps; the phase-alignment steps are untimed
    cyc = run.method.block_size + 1
    for _ in range((args.warmup - (args.warmup + args.steps)) % cyc):
        ctx.focus_step_block(rids)
        ctx.focus_commit(rids)
    ctx.focus_sync()
    dec0 = tok_sum()
    host_decoded = 0

    def consume(k):
        nonlocal host_decoded
        done[k].synchronize()
        arr = (focus_commit_result * n_req).from_address(res[k].data_ptr())
        host_decoded += sum(int(r.n_new) for r in arr)

    D.barrier(dev)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(e2e_steps):
        k = i & 1
        if done[k] is not None:
            consume(k)
            done[k] = None
        ctx.focus_step_block(rids)
        ctx.focus_commit(rids, res[k].data_ptr())
        done[k] = torch.cuda.Event()
        done[k].record(st)
    for i in (e2e_steps - 2, e2e_steps - 1):       # drain the last two steps' readbacks, in order
        if i >= 0 and done[i & 1] is not None:
            consume(i & 1)
            done[i & 1] = None
    ctx.focus_sync()
    e2e_s = time.perf_counter() - t0
    e2e_dec = tok_sum() - dec0
    assert host_decoded == e2e_dec, (host_decoded, e2e_dec)
    e2e_val = D.reduce_sum(e2e_dec, dev) / D.reduce_max(e2e_s, dev)

    # ---- kernel breakdown: per-launch CUDA events (separate pass, 2 steps)
    ctx.focus_set_profile(True)
    fl_tot, wb_tot, ab_tot = {}, {}, 0
    prof_steps = 2
    for _ in range(prof_steps):
        ctx.focus_step_block(rids)
        ctx.focus_sync()
        c = ctx.counters()
        fl, wb, ab = step_work(run.model, run.method.block_size, (int(c[0]), int(c[1]), int(c[2])), ctx.states(), rids)
        for k in fl:
            fl_tot[k] = fl_tot.get(k, 0) + fl[k]
            wb_tot[k] = wb_tot.get(k, 0) + wb[k]
        ab_tot += ab
        ctx.focus_commit(rids)
    ctx.focus_sync()
    prof = ctx.profile()
    ctx.focus_set_profile(False)
    pk = peaks()
    total_ms = sum(v["total_ms"] for v in prof.values()) or 1.0
    kernels = {}
    for k, v in prof.items():
        if not v["launches"]:
            continue
        e = {"launches": v["launches"] // prof_steps, "ms_per_step": round(v["total_ms"] / prof_steps, 4),
             "share": round(v["total_ms"] / total_ms, 4)}
        if k in fl_tot:
            tf = fl_tot[k] / (v["total_ms"] / 1e3) / 1e12
            e.update(tflops=round(tf, 2), tc_frac=round(tf / pk["tc_sus"], 4),
                     weight_gbs=round(wb_tot[k] / (v["total_ms"] / 1e3) / 1e9, 1))
        if k == "attention":
            gbs = ab_tot / (v["total_ms"] / 1e3) / 1e9
            e.update(kv_gbs=round(gbs, 1), hbm_frac=round(gbs / pk["hbm"], 4))
        kernels[k] = e
    # roofline of the dominant kernel (largest share of the step), with per-launch DRAM traffic from the
    # committed ncu capture (profiles/traffic.json) when present
    traffic_map = {}
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        traffic_map = json.load(open(tp)).get("dram_bytes_per_launch", {})
    cands = [k for k in ("attention", "gemm_gu", "gemm_down", "gemm_qkv", "gemm_o", "gemm_lm") if prof[k]["launches"]]
    dom = max(cands, key=lambda k: prof[k]["total_ms"])
    n_l = prof[dom]["launches"]
    ms_l = prof[dom]["total_ms"] / n_l
    if dom == "attention":
        per_launch = ab_tot / n_l
        ach = per_launch / (ms_l / 1e3) / 1e9
        roofline = {"bound": "hbm", "kernel": "k_attn_tc (block-diffusion paged attention, tcgen05) per layer",
                    "achieved": round(ach, 1), "peak": pk["hbm"], "unit": "GB/s", "frac": round(ach / pk["hbm"], 4),
                    "traffic": traffic_map.get(dom), "algorithmic_bytes_per_launch": round(per_launch),
                    "peak_src": pk["src"] + " HBM copy"}
    else:
        per_launch = fl_tot[dom] / n_l
        ach = per_launch / (ms_l / 1e3) / 1e12
        roofline = {"bound": "tensor", "kernel": f"k_gemm_tc ({dom}) per layer", "achieved": round(ach, 2),
                    "peak": pk["tc_sus"], "unit": "TFLOP/s", "frac": round(ach / pk["tc_sus"], 4),
                    "traffic": traffic_map.get(dom), "flops_per_launch": round(per_launch),
                    "peak_src": pk["src"] + " sustained bf16"}
    roofline.update(launch_ms=round(ms_l, 4), launches_per_step=n_l // prof_steps,
                    share_of_step=round(prof[dom]["total_ms"] / total_ms, 4),
                    timing="CUDA events around every launch on the library stream, 2 profiled steps after the timed region")
    proj = ["gemm_qkv", "gemm_o", "gemm_gu", "gemm_down"]
    g_ms = sum(prof[k]["total_ms"] for k in proj)
    g_fl = sum(fl_tot[k] for k in proj)
    ach_all = g_fl / (g_ms / 1e3) / 1e12
    roofline_gemms = {"bound": "tensor", "kernel": "all projection GEMMs", "achieved": round(ach_all, 2),
                      "peak": pk["tc_sus"], "unit": "TFLOP/s", "frac": round(ach_all / pk["tc_sus"], 4),
                      "share_of_step": round(g_ms / total_ms, 4)}
    stats = D.all_gather_stats([int(dec), int(launches), int(prefill_s * 1e3)], dev)

    out = None
    if rank == 0:
        cpu = None if (args.no_cpu_baseline or world > 1) else cpu_baseline(args, run)
        out = {"metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 3), "higher_is_better": True,
               "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded prompts, random-init weights)",
               "config": {"workload": f"{run.name}: {run.description}", "model": "SDAR-8B-shaped (random init)",
                          "requests_per_gpu": n_req, "global_batch": n_req * world, "block": run.method.block_size,
                          "prompt_len": run.prompt_len, "gen_len": run.gen_len, "seq_len": run.prompt_len + run.gen_len,
                          "alpha": "3/2", "tau": run.method.conf_threshold, "cache": "DC+",
                          "parallelism": f"request-sharded dp{world}",
                          "l2": "inputs larger than L2 every step (16.4 GB bf16 weights + KV stream)",
                          "timed_steps_from": f"step {args.warmup + 1} of the decode (context {run.prompt_len}+)",
                          "prefill_s": round(prefill_s, 2)},
               "e2e": {"value": round(e2e_val, 2), "unit": UNIT, "h2d_bytes_per_step": 4 * n_req,
                       "d2h_bytes_per_step": n_req * rsz + 32, "steps": e2e_steps,
                       "readback": "every step's commit results to pinned host memory, double-buffered"},
               "gpu_launches": int(launches), "roofline": roofline, "roofline_gemms": roofline_gemms,
               "kernels": kernels,
               "clocks": clk.summary(), "decoded_in_window": int(dec_all), "per_rank": stats}
        if cpu is not None:
            out["cpu_baseline"] = cpu
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return out


# ------------------------------------------------------------------------------------ CPU oracle legs
def _oracle_sample(run, seed=123):
    """One request of the workload, started from a synthetic (seeded) context KV of the workload's
    prompt length (prefill is excluded from the metric); the oracle exactly as it stands."""
    import numpy as np
    from oracle.engine import OracleEngine
    from oracle.model import OracleWeights
    m = run.model
    w = OracleWeights(m, run.weight_seed, cache=True)
    eng = OracleEngine(run.with_(n_requests=1), "ref", weights=w)
    rng = np.random.default_rng(seed)
    K = [rng.standard_normal((run.prompt_len, m.n_kv_heads, m.head_dim)).astype(np.float32) for _ in range(m.n_layers)]
    V = [rng.standard_normal((run.prompt_len, m.n_kv_heads, m.head_dim)).astype(np.float32) for _ in range(m.n_layers)]
    eng.set_context_kv(0, run.prompt_len, run.gen_len, K, V)
    for l in range(m.n_layers):                      # materialise weights outside the timed region
        w.layer(l)
    w.lm_head()
    return eng


def _threads():
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        return max((i.get("num_threads", 1) for i in info), default=1), [i.get("internal_api") for i in info]
    except Exception:
        return len(os.sched_getaffinity(0)), []


def cpu_baseline(args, run, budget_s: float = 25.0):
    eng = _oracle_sample(run)
    t0 = time.perf_counter()
    steps = dec = 0
    while time.perf_counter() - t0 < budget_s and steps < 6:
        eng.step_one(0)
        dec += len(eng.commit_one(0).decoded)
        steps += 1
    dt = time.perf_counter() - t0
    th, apis = _threads()
    return {"value": round(dec / dt, 4), "unit": UNIT, "cores": th, "kind": "oracle",
            "sample": f"{run.name}, 1 request x {steps} decode steps ({dec} tokens) from a synthetic {run.prompt_len}-token "
                      f"context, binary64 NumPy ({'/'.join(a for a in apis if a)}), {dt:.1f} s",
            "host_cpus": len(os.sched_getaffinity(0))}


def run_reference(args):
    from paper_2601_23278_b200 import dist as D
    from synth import get_config
    rank, world, _ = D.env_world()
    if rank != 0:
        return None
    run = get_config(args.workload)
    eng = _oracle_sample(run)
    for _ in range(args.warmup):
        eng.step_one(0)
        eng.commit_one(0)
    t0 = time.perf_counter()
    dec = 0
    for _ in range(args.steps):
        eng.step_one(0)
        dec += len(eng.commit_one(0).decoded)
    dt = time.perf_counter() - t0
    th, apis = _threads()
    value = dec / dt
    sample = (f"{run.name}, 1 request x {args.steps} decode steps ({dec} tokens) per run from a synthetic "
              f"{run.prompt_len}-token context; the CPU oracle (binary64 NumPy) as it stands")
    out = {"impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt / args.steps * 1e3, 1),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "config": {"workload": f"{run.name}: {run.description}", "requests": 1},
           "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": th, "kind": "oracle", "sample": sample},
           "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="focus", choices=["focus", "reference"])
    ap.add_argument("--workload", default="C3")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_focus(args)


if __name__ == "__main__":
    main()
