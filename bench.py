"""Decoded tokens/sec of the FOCUS block-diffusion decode step on B200 (BASELINE.json metric).

  python bench.py [--gpus N --steps K --warmup W]            # our CUDA path (libfocus.so)
  python bench.py --impl reference [--steps K --warmup W]    # the CPU oracle on a bounded sample

Default workload (per GPU): C3 = SDAR-8B-shaped random-init model (36 layers, d 4096, GQA 32/8, d_ff
12288, vocab 151936), block 16, 64 requests, prompt 1024, gen 512 (BASELINE.json configs[2]).  With
N GPUs each rank owns 64 requests of its own (request-level data parallel, weak scaling, no collective
on the data path).  `--workload C4` is BASELINE configs[3]: 256 requests with prompt lengths uniform
in [256, 4096], LPT-sharded over the N ranks (strong scaling: the global batch is fixed).
`--gpus N` without a torchrun environment re-launches itself under torch.distributed.run.

A step = focus_step_block + focus_commit over all requests of the rank (the whole hot path).  Each
run decodes the WHOLE generation (every request to its gen_len) after an untimed prefill:
  - W warm-up steps, then three device-timed windows of exactly K steps at the start, middle and end
    of the generation (same phase of the B-decode + 1-flush block cycle, so context spans 1024-1536
    at C3); `value` = the median window (barrier + synchronize around each window, CUDA events on the
    library stream, max over ranks); `generation` = every post-warm-up step, device-timed;
  - e2e: the whole generation again through the C ABI from host buffers (request list uploaded and
    commit results read back to pinned memory every step), wall clock after the W warm-up steps;
  - box-local baselines on the same inputs: strategy NONE (no eviction, the LMDeploy-like regime the
    paper compares with, fig:ablation_throughput P:538-545) and the calibrated logit_scale run
    (about 0.1 B tokens decoded per request-step);
  - redundancy N_processed / N_decoded at layers 2+ (tab:reduce_ratio P:480-504) from device counters;
  - per-kernel CUDA-event breakdown (2 profiled steps after the middle window) and the roofline of the
    dominant kernel: max(FLOPs / tensor peak, bytes / HBM peak) per launch.
Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import socket
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decoded tokens/sec (SDAR-8B-shaped, block 16) at 1/2/4/8 B200; % roofline"
UNIT = "tokens/s"
# calibrated LM-head scale per workload: mean decoded tokens per request-step ~ 0.1 B (the
# fig:decoding_stats regime); C3 measured 1.59 at 16 (scripts/calibrate_logit_scale.py)
CALIBRATED_SCALE = {"C2": 16.0, "C3": 16.0, "C4": 16.0, "C5": 16.0}
MODEL_NAME = {"C2": "SDAR-1.7B-shaped (random init)", "C3": "SDAR-8B-shaped (random init)",
              "C4": "SDAR-8B-shaped (random init)", "C5": "SDAR-8B-shaped (random init)",
              "C3B64": "SDAR-8B-shaped (random init)", "C6": "LLaDA2.0-mini-shaped MoE (random init)",
              "C1": "tiny block-diffusion model (random init)"}


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
        self.spans = []
        self.out = ""

    def _reader(self):
        for line in self.p.stdout:
            self.lines.append((time.time(), line))

    def start(self):
        # the sampler is started and its first sample awaited BEFORE the first timed window (nvidia-smi
        # takes a few hundred ms to start); samples are time-stamped on arrival and the summary keeps
        # those that fall inside a timed window
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
        return self

    def span(self, t0, t1):
        self.spans.append((t0, t1))

    def stop(self):
        time.sleep(0.06)                                 # let the in-flight sample arrive
        if self.p is not None:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except Exception:
                pass
            if self.th is not None:
                self.th.join(timeout=2)
        inside = [ln for (t, ln) in self.lines if any(a - 0.03 <= t <= b + 0.03 for a, b in self.spans)]
        self.out = "".join(inside)

    def summary(self):
        rows = [r.split(",") for r in (self.out or "").strip().splitlines() if r.count(",") >= 7]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(r[1]) for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if "Active" in r[4 + k] and "Not" not in r[4 + k]})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": float(rows[0][2]), "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------------------------------ host planning
def gen_steps(run) -> int:
    """Steps of a whole generation under the synthetic dynamics: each block takes B
    decode steps (one fallback decode per request-step) + 1 flush step."""
    B = run.method.block_size
    return run.gen_len // B * (B + 1)


def window_starts(total: int, warmup: int, steps: int, cyc: int) -> list:
    """Starts of the three timed K-step windows: right after the warm-up, in the middle and at the end
    of the generation, all at the warm-up's phase of the block cycle (same decode/flush mix); fewer
    windows when the generation is too short to hold three disjoint ones."""
    ph = warmup % cyc
    last = total - steps
    starts = [warmup]
    if last >= warmup:
        late = last - ((last - ph) % cyc)
        mid = (warmup + late) // 2
        mid -= (mid - ph) % cyc
        for s in (mid, late):
            if s >= starts[-1] + steps + 2 and s + steps <= total:    # disjoint, room for the profile pass
                starts.append(s)
    return starts


def plan_requests(run, world: int, rank: int):
    """(global request ids of this rank, {gid: prompt length}, scaling).  C4: fixed global batch with
    mixed prompt lengths, LPT-sharded by cost L_prompt + gen/2 -> strong scaling.
    Otherwise run.n_requests requests per rank (weak scaling)."""
    from paper_2601_23278_b200 import dist as D
    from synth.gen import prompt_lengths
    if run.prompt_len_hi is not None:
        lens = prompt_lengths(run.n_requests, run.prompt_len, run.prompt_len_hi).tolist()
        costs = [L + run.gen_len / 2 for L in lens]
        mine = D.shard_requests(run.n_requests, world, rank, costs)
        return mine, {g: lens[g] for g in mine}, "strong"
    n = run.n_requests
    gids = list(range(rank * n, (rank + 1) * n))
    return gids, {g: run.prompt_len for g in gids}, "weak"


# ------------------------------------------------------------------------------------ algorithmic work
def step_work(model, B, counters, states, rids):
    """SURVEY 8(d) per-step algorithmic FLOPs and bytes by kernel family, from the step's live sizes.
    GEMM bytes: weights once + activation rows in/out; attention bytes: the K/V each request streams
    (ctx + B at layers 0-1, ctx + R' + 1 at layers >= 2), FLOPs 4 H_q d_h per (query row, key)."""
    d, ff, V, L = model.d_model, model.d_ff, model.vocab, model.n_layers
    qkv = model.qkv_dim
    qd = model.n_q_heads * model.head_dim
    MP, MS, ML = counters
    # dense FFN layers (rows: layer 0 on P, layers >= 1 on S); MoE models replace layers >= n_dense_layers
    moe_layers = [l for l in range(L) if model.is_moe_layer(l)]
    dense_parts = [(MP if l == 0 else MS, 1) for l in range(L) if not model.is_moe_layer(l)]
    shapes = {  # family: (N, K, rows per step [(rows, launches)], out bytes per element read+written)
        "gemm_qkv": (qkv, d, [(MP, 2), (MS, L - 2)], 2),
        "gemm_o": (d, qd, [(MP, 1), (MS, L - 1)], 8),
        "gemm_gu": (2 * ff, d, dense_parts, 1),
        "gemm_down": (d, ff, dense_parts, 8),
        "gemm_lm": (V, d, [(ML, 1)], 4),
    }
    fl, by = {}, {}
    for k, (N, K, parts, ob) in shapes.items():
        fl[k] = sum(2 * r * N * K * n for r, n in parts)
        by[k] = sum((2 * N * K + 2 * r * K + ob * r * N) * n for r, n in parts)
    if moe_layers:
        # MoE (A-M5): router GEMM; routed + shared experts (each row runs top_k + n_shared SwiGLU experts);
        # weight bytes: every routed expert (all are touched at these row counts) and the shared ones
        E, de, act = model.n_experts, model.d_expert, model.top_k + model.n_shared_experts
        rows = [MP if l == 0 else MS for l in moe_layers]
        fl["moe_route"] = sum(2 * r * d * E for r in rows)
        by["moe_route"] = sum(2 * E * d + 2 * r * d + 4 * r * E for r in rows)
        fl["moe_experts"] = sum(2 * r * act * 3 * d * de for r in rows)
        by["moe_experts"] = sum(2 * (E + model.n_shared_experts) * 3 * d * de + r * act * (2 * d + 4 * d) for r in rows)
    kvb = 4 * model.n_kv_heads * model.head_dim          # K+V bf16 bytes per token per layer
    attn_bytes = attn_flops = 0
    for r in rids:
        s = states[r]
        if not s.active or s.finished:
            continue
        nP = bin(int(s.P)).count("1")
        nS = bin(int(s.S)).count("1")
        attn_bytes += kvb * ((s.s + B) + (L - 2) * (s.s + s.R_new + 1) + (s.s + B))
        attn_flops += 4 * qd * (nP * (s.s + B) + nS * (s.s + B) + (L - 2) * nS * (s.s + s.R_new + 1))
    fl["attention"], by["attention"] = attn_flops, attn_bytes
    return fl, by


# ------------------------------------------------------------------------------------ the CUDA path
class Rank:
    """One rank's decode loop over the C ABI (libfocus through the ctypes binding)."""

    def __init__(self, run, gids, lens, dev, **cfg_kw):
        from paper_2601_23278_b200 import FocusContext, make_config
        self.run, self.gids, self.lens, self.dev = run, gids, lens, dev
        hi = max(lens.values()) if lens else run.prompt_len
        # the KV page pool holds exactly this rank's requests (prompt + generation), not max_requests x
        # max_seq_len: the mixed-length C4 batch (256 requests, prompts 256-4096) would otherwise reserve
        # 183 GiB of pages for ~90 GiB of tokens
        ps = run.page_size
        pages = sum((lens[g] + run.gen_len + ps - 1) // ps for g in gids) if gids else 0
        cfg_kw.setdefault("kv_pages", pages)
        self.ctx = FocusContext(make_config(run, max_requests=max(1, len(gids)), max_seq_len=hi + run.gen_len,
                                            **cfg_kw))
        self.rids = list(range(len(gids)))

    def prefill(self):
        import torch
        from synth.gen import prompt_tokens
        t0 = time.time()
        for r, g in zip(self.rids, self.gids):
            self.ctx.focus_kv_append(r, prompt_tokens(g, self.lens[g], self.run.model.vocab), self.run.gen_len)
        torch.cuda.synchronize()
        return time.time() - t0

    def release(self):
        for r in self.rids:
            self.ctx.focus_release(r)

    def step(self):
        self.ctx.focus_step_block(self.rids)
        self.ctx.focus_commit(self.rids)

    def tok_sum(self):
        s = self.ctx.states()
        return sum(int(s[r].token_sum) for r in self.rids)

    def all_finished(self):
        s = self.ctx.states()
        return all(s[r].finished for r in self.rids)

    def close(self):
        import torch
        self.ctx.focus_destroy()
        del self.ctx
        torch.cuda.empty_cache()


def _all_finished(rk, D):
    return D.reduce_min(1.0 if rk.all_finished() else 0.0, rk.dev) > 0.5


def decode_generation(rk, D, warmup, steps, starts, clk=None, prof_after=None, max_steps=100000):
    """Decode the whole generation of the rank's requests.  Returns per-window and whole-generation
    device timings (max over ranks) and the profiled step data when `prof_after` names a window."""
    import torch
    st, dev = rk.ctx.stream, rk.dev
    cyc = rk.run.method.block_size + 1
    for _ in range(warmup):
        rk.step()
    torch.cuda.synchronize()
    windows, segs, prof = [], [], None
    t = warmup
    seg_dec0, seg_ev0 = rk.tok_sum(), None
    D.barrier(dev)

    def seg_begin():
        e = torch.cuda.Event(enable_timing=True)
        e.record(st)
        return e

    def seg_end(e0, dec0, kind):
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record(st)
        torch.cuda.synchronize()
        segs.append((kind, e0.elapsed_time(e1), rk.tok_sum() - dec0))

    seg_ev0 = seg_begin()
    n_since_check = 0
    while t < max_steps:
        if t in starts:
            seg_end(seg_ev0, seg_dec0, "gap")
            D.barrier(dev)
            torch.cuda.synchronize()
            dec0, l0 = rk.tok_sum(), rk.ctx.launches()
            if clk is not None and not windows:
                clk.start()
            w0 = time.time()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(steps):
                rk.step()
            e1.record(st)
            torch.cuda.synchronize()
            if clk is not None:
                clk.span(w0, time.time())
            D.barrier(dev)
            ms = e0.elapsed_time(e1)
            dec = rk.tok_sum() - dec0
            windows.append(dict(start=t, ms=ms, decoded=dec, launches=rk.ctx.launches() - l0))
            segs.append(("window", ms, dec))
            t += steps
            if prof_after is not None and len(windows) == prof_after:
                prof = profile_steps(rk, 2)
                t += 2
            seg_dec0, seg_ev0 = rk.tok_sum(), seg_begin()
            n_since_check = 0
            continue
        rk.step()
        t += 1
        n_since_check += 1
        if n_since_check >= cyc and t not in starts:
            seg_end(seg_ev0, seg_dec0, "gap")
            n_since_check = 0
            if _all_finished(rk, D):
                seg_ev0 = None
                break
            seg_dec0, seg_ev0 = rk.tok_sum(), seg_begin()
    if seg_ev0 is not None:
        seg_end(seg_ev0, seg_dec0, "gap")
    while not _all_finished(rk, D) and t < max_steps:
        e0, d0 = seg_begin(), rk.tok_sum()
        rk.step()
        t += 1
        seg_end(e0, d0, "gap")
    gen_ms = sum(ms for _, ms, _ in segs)
    gen_dec = sum(dec for _, _, dec in segs)
    return dict(windows=windows, gen_ms=gen_ms, gen_dec=gen_dec, steps_total=t, prof=prof)


def profile_steps(rk, n):
    """n steps with CUDA events around every launch (FOCUS_PROF kinds) plus the live sizes."""
    c = rk.ctx
    c.focus_set_profile(True)
    fl_tot, by_tot = {}, {}
    for _ in range(n):
        c.focus_step_block(rk.rids)
        c.focus_sync()
        cnt = c.counters()
        fl, by = step_work(rk.run.model, rk.run.method.block_size, (int(cnt[0]), int(cnt[1]), int(cnt[2])),
                           c.states(), rk.rids)
        for k in fl:
            fl_tot[k] = fl_tot.get(k, 0) + fl[k]
            by_tot[k] = by_tot.get(k, 0) + by[k]
        c.focus_commit(rk.rids)
    c.focus_sync()
    prof = c.profile()
    c.focus_set_profile(False)
    return dict(prof=prof, flops=fl_tot, bytes=by_tot, steps=n, M_S=max(1, int(cnt[1])))


def e2e_generation(rk, D, warmup):
    """The whole generation through the C ABI from host buffers, wall clock after `warmup` untimed
    steps: every step uploads the request list (focus_step_block reads it from host memory) and reads
    the commit results back into pinned host memory, double-buffered like a serving loop (step t's
    results are parsed while step t+1 runs); it ends when the host has seen every request finish."""
    import ctypes
    import torch
    from paper_2601_23278_b200.focus import focus_commit_result
    c, st, dev, n = rk.ctx, rk.ctx.stream, rk.dev, len(rk.rids)
    for _ in range(warmup):
        rk.step()
    c.focus_sync()
    rsz = ctypes.sizeof(focus_commit_result)
    res = [torch.empty(max(n, 1) * rsz, dtype=torch.uint8).pin_memory() for _ in range(2)]
    done = [None, None]
    dec0 = rk.tok_sum()
    host_decoded, steps = 0, 0
    finished = set()

    def consume(k):
        nonlocal host_decoded
        done[k].synchronize()
        arr = (focus_commit_result * n).from_address(res[k].data_ptr())
        for x in arr:
            host_decoded += int(x.n_new)
            if x.finished:
                finished.add(int(x.req_id))
        done[k] = None

    D.barrier(dev)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    i = 0
    while len(finished) < n:
        k = i & 1
        if done[k] is not None:
            consume(k)
            if len(finished) >= n:
                break
        c.focus_step_block(rk.rids)
        c.focus_commit(rk.rids, res[k].data_ptr())
        done[k] = torch.cuda.Event()
        done[k].record(st)
        i += 1
        steps += 1
        if steps > 1000000:
            raise RuntimeError("e2e generation did not finish")
    for k in (0, 1):
        if done[k] is not None:
            consume(k)
    c.focus_sync()
    wall = time.perf_counter() - t0
    dec = rk.tok_sum() - dec0
    assert host_decoded == dec, (host_decoded, dec)
    return dict(wall_s=wall, decoded=dec, steps=steps, rsz=rsz)


def _agg_windows(win_lists, D, dev):
    """Per window: decoded summed over ranks / device ms max over ranks."""
    out = []
    for w in win_lists:
        ms = D.reduce_max(w["ms"], dev)
        dec = D.reduce_sum(w["decoded"], dev)
        out.append(dict(start=w["start"], ms=round(ms, 3), decoded=int(dec), launches=int(w["launches"]),
                        value=round(dec / (ms / 1e3), 2)))
    return out


def roofline_report(pd, pk, workload):
    """Per kernel family: T_roof = max(FLOPs / tensor peak, bytes / HBM peak) against the CUDA-event
    time of its launches (SURVEY 8(d) reporting); the dominant kernel's object for the JSON line."""
    prof, fl, by, n = pd["prof"], pd["flops"], pd["bytes"], pd["steps"]
    total_ms = sum(v["total_ms"] for v in prof.values()) or 1.0
    traffic = {}
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get("workloads", {}).get(workload, {})   # ncu capture of THIS workload only
    kernels, troof_sum = {}, 0.0
    for k, v in prof.items():
        if not v["launches"]:
            continue
        e = {"launches": v["launches"] // n, "ms_per_step": round(v["total_ms"] / n, 4),
             "share": round(v["total_ms"] / total_ms, 4)}
        if k in fl:
            t_tc = fl[k] / (pk["tc_sus"] * 1e12) * 1e3
            t_hbm = by[k] / (pk["hbm"] * 1e9) * 1e3
            t_roof = max(t_tc, t_hbm)
            troof_sum += t_roof
            e.update(bound="tensor" if t_tc >= t_hbm else "hbm", roofline_ms=round(t_roof / n, 4),
                     frac=round(t_roof / v["total_ms"], 4),
                     tflops=round(fl[k] / (v["total_ms"] / 1e3) / 1e12, 2),
                     gbs=round(by[k] / (v["total_ms"] / 1e3) / 1e9, 1))
        kernels[k] = e
    cands = [k for k in kernels if k in fl and prof[k]["launches"]]
    dom = max(cands, key=lambda k: prof[k]["total_ms"])
    n_l = prof[dom]["launches"]
    ms_l = prof[dom]["total_ms"] / n_l
    e = kernels[dom]
    if e["bound"] == "hbm":
        ach = by[dom] / n_l / (ms_l / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": round(ach, 1), "peak": pk["hbm"], "unit": "GB/s",
                "frac": round(ach / pk["hbm"], 4), "algorithmic_bytes_per_launch": round(by[dom] / n_l),
                "peak_src": pk["src"] + " HBM copy"}
    else:
        ach = fl[dom] / n_l / (ms_l / 1e3) / 1e12
        roof = {"bound": "tensor", "achieved": round(ach, 2), "peak": pk["tc_sus"], "unit": "TFLOP/s",
                "frac": round(ach / pk["tc_sus"], 4), "flops_per_launch": round(fl[dom] / n_l),
                "peak_src": pk["src"] + " sustained bf16"}
    names = {"attention": "k_attn_tc (block-diffusion paged attention, tcgen05) per layer"}
    roof.update(kernel=names.get(dom, f"k_gemm_pair ({dom}) per layer"), traffic=traffic.get(dom),
                launch_ms=round(ms_l, 4), launches_per_step=n_l // n, share_of_step=e["share"],
                timing="CUDA events around every launch on the library stream, 2 profiled (eager) steps after the middle "
                       "window, each held on the device until the host has enqueued it (k_hold), so the intervals "
                       "are device time, not host launch latency")
    proj = [k for k in ("gemm_qkv", "gemm_o", "gemm_gu", "gemm_down", "moe_experts") if prof.get(k, {}).get("launches")]
    g_ms = sum(prof[k]["total_ms"] for k in proj)
    g_fl = sum(fl[k] for k in proj)
    ach_all = g_fl / (g_ms / 1e3) / 1e12
    gemms = {"bound": "tensor", "kernel": "all projection GEMMs", "achieved": round(ach_all, 2),
             "peak": pk["tc_sus"], "unit": "TFLOP/s", "frac": round(ach_all / pk["tc_sus"], 4),
             "share_of_step": round(g_ms / total_ms, 4)}
    step = {"roofline_ms_per_step": round(troof_sum / n, 4), "measured_ms_per_step": round(total_ms / n, 4),
            "frac": round(troof_sum / total_ms, 4),
            "note": "sum over kernel families of max(F/TC, B/HBM) vs the profiled step (events serialise launches)"}
    return roof, gemms, kernels, step


def cublas_reference(model, M, dev):
    """cuBLAS (torch.matmul, bf16) at the projection shapes of the profiled step's S rows, weights
    cold (a 256 MB buffer is rewritten between reps, as the step streams its weights from HBM): the
    library baseline the hand-written tcgen05 GEMMs are compared with."""
    import torch
    d, ff = model.d_model, model.d_ff
    qd = model.n_q_heads * model.head_dim
    shapes = {"gemm_qkv": (model.qkv_dim, d), "gemm_o": (d, qd), "gemm_gu": (2 * ff, d), "gemm_down": (d, ff)}
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    out = {}
    for k, (N, K) in shapes.items():
        A = torch.randn(M, K, device=dev, dtype=torch.bfloat16)
        W = torch.randn(N, K, device=dev, dtype=torch.bfloat16)
        best = 1e9
        for r in range(6):
            flush.zero_()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            torch.matmul(A, W.t())
            e1.record()
            torch.cuda.synchronize()
            if r:
                best = min(best, e0.elapsed_time(e1))
        out[k] = {"M": M, "N": N, "K": K, "us": round(best * 1e3, 1), "tflops": round(2 * M * N * K / (best * 1e-3) / 1e12, 1)}
    del flush
    torch.cuda.empty_cache()
    return out


def run_focus(args):
    import torch
    from paper_2601_23278_b200 import dist as D
    from synth import get_config

    rank, world, local = D.init("nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    run = get_config(args.workload)
    if args.logit_scale != 1.0:
        run = run.with_(model=dataclasses.replace(run.model, logit_scale=args.logit_scale))
    gids, lens, scaling = plan_requests(run, world, rank)
    B = run.method.block_size
    cyc = B + 1
    T = gen_steps(run)
    starts = window_starts(T, args.warmup, args.steps, cyc)
    kw = dict(batch_invariant=args.batch_invariant)

    # ---- FOCUS: whole generation, three timed windows, profile pass after the middle window
    rk = Rank(run, gids, lens, dev, **kw)
    prefill_s = rk.prefill()
    rows0 = rk.ctx.cumulative_rows()
    clk = Clocks(local)
    g = decode_generation(rk, D, args.warmup, args.steps, starts, clk, prof_after=min(2, len(starts)))
    clk.stop()
    rows1 = rk.ctx.cumulative_rows()
    wins = _agg_windows(g["windows"], D, dev)
    med = sorted(wins, key=lambda w: w["value"])[len(wins) // 2]
    value = med["value"]
    gen_ms = D.reduce_max(g["gen_ms"], dev)
    gen_dec = D.reduce_sum(g["gen_dec"], dev)
    dec_total = D.reduce_sum(sum(int(rk.ctx.states()[r].token_sum) for r in rk.rids), dev)
    red_S = D.reduce_sum(rows1["sum_S"] - rows0["sum_S"], dev) / max(dec_total, 1)
    red_P = D.reduce_sum(rows1["sum_P"] - rows0["sum_P"], dev) / max(dec_total, 1)

    # ---- e2e: the whole generation again from host buffers (same context, graphs already captured)
    rk.release()
    rk.prefill()
    e = e2e_generation(rk, D, args.warmup)
    e2e_val = D.reduce_sum(e["decoded"], dev) / D.reduce_max(e["wall_s"], dev)
    rk.close()

    # ---- box-local baselines on the same inputs
    extras = {}
    if not args.no_extras:
        from synth.configs import STRATEGY_NONE
        for name, r2 in (("no_eviction", run.with_(method=dataclasses.replace(run.method, strategy=STRATEGY_NONE))),
                         ("calibrated", run.with_(model=dataclasses.replace(
                             run.model, logit_scale=CALIBRATED_SCALE.get(args.workload, 16.0))))):
            rb = Rank(r2, gids, lens, dev, **kw)
            rb.prefill()
            c0 = rb.ctx.cumulative_rows()
            gb = decode_generation(rb, D, args.warmup, args.steps, starts if name == "no_eviction" else [])
            c1 = rb.ctx.cumulative_rows()
            dec_b = D.reduce_sum(sum(int(rb.ctx.states()[r].token_sum) for r in rb.rids), dev)
            st_b = D.reduce_sum(sum(int(rb.ctx.states()[r].total_steps) for r in rb.rids), dev)
            gms = D.reduce_max(gb["gen_ms"], dev)
            gdec = D.reduce_sum(gb["gen_dec"], dev)
            x = {"generation": {"value": round(gdec / (gms / 1e3), 2), "decoded": int(gdec), "ms": round(gms, 1),
                                "steps": gb["steps_total"]},
                 "redundancy_layer2plus": round(D.reduce_sum(c1["sum_S"] - c0["sum_S"], dev) / max(dec_b, 1), 3),
                 "redundancy_layers01": round(D.reduce_sum(c1["sum_P"] - c0["sum_P"], dev) / max(dec_b, 1), 3),
                 "decoded_per_request_step": round(dec_b / max(st_b, 1), 3)}
            if gb["windows"]:
                wb = _agg_windows(gb["windows"], D, dev)
                x["windows"] = wb
                x["value"] = sorted(wb, key=lambda w: w["value"])[len(wb) // 2]["value"]
            if name == "calibrated":
                x["logit_scale"] = r2.model.logit_scale
            rb.close()
            extras[name] = x
        fg = gen_dec / (gen_ms / 1e3)
        extras["no_eviction"]["focus_speedup_generation"] = round(fg / extras["no_eviction"]["generation"]["value"], 3)
        if "value" in extras["no_eviction"]:
            extras["no_eviction"]["focus_speedup_windows"] = round(value / extras["no_eviction"]["value"], 3)

    pk = peaks()
    roof = gemms = kernels = stepr = cub = None
    if g["prof"] is not None:
        roof, gemms, kernels, stepr = roofline_report(g["prof"], pk, run.name)
        if rank == 0 and not args.no_extras:
            cub = cublas_reference(run.model, g["prof"]["M_S"], dev)
            for k, v in cub.items():
                if k in kernels:
                    ours = kernels[k]["ms_per_step"] * 1e3 / max(1, kernels[k]["launches"])
                    v["ours_us_per_launch"] = round(ours, 1)
                    v["ours_over_cublas"] = round(ours / v["us"], 3)
    stats = D.all_gather_stats([int(g["gen_dec"]), len(gids), int(prefill_s * 1e3)], dev)
    global_batch = int(D.reduce_sum(len(gids), dev))

    out = None
    if rank == 0:
        cpu = None if (args.no_cpu_baseline or world > 1) else cpu_baseline(args, run)
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": round(med["ms"] / args.steps, 3), "higher_is_better": True,
               "scaling": scaling, "vs_baseline": None, "dtype": "bf16",
               "data": "synthetic (seeded prompts, random-init weights)",
               "config": {"workload": f"{run.name}: {run.description}", "model": MODEL_NAME.get(run.name, run.name),
                          "requests_per_gpu": len(gids), "global_batch": global_batch,
                          "block": B, "prompt_len": run.prompt_len if run.prompt_len_hi is None else
                          f"{run.prompt_len}-{run.prompt_len_hi} (uniform, LPT-sharded)",
                          "gen_len": run.gen_len, "alpha": f"{run.method.alpha_num}/{run.method.alpha_den}",
                          "tau": run.method.conf_threshold, "cache": "DC+", "logit_scale": run.model.logit_scale,
                          "batch_invariant": bool(args.batch_invariant),
                          "parallelism": f"request-sharded dp{world}",
                          "l2": "inputs larger than L2 every step (16.4 GB bf16 weights + KV stream)",
                          "timed": f"median of {len(wins)} windows of {args.steps} steps at decode steps {[w['start'] + 1 for w in wins]} of {g['steps_total']}",
                          "prefill_s": round(prefill_s, 2)},
               "windows": wins,
               "generation": {"value": round(gen_dec / (gen_ms / 1e3), 2), "decoded": int(gen_dec),
                              "ms": round(gen_ms, 1), "steps": g["steps_total"],
                              "note": "every post-warm-up step of the whole generation, device time (profiled steps excluded)"},
               "e2e": {"value": round(e2e_val, 2), "unit": UNIT, "h2d_bytes_per_step": 4 * len(gids),
                       "d2h_bytes_per_step": len(gids) * e["rsz"], "steps": e["steps"],
                       "readback": "every step's commit results to pinned host memory, double-buffered; whole generation after the warm-up"},
               "gpu_launches": int(med["launches"]),
               "redundancy": {"layer2plus": round(red_S, 3), "layers01": round(red_P, 3),
                              "definition": "N_processed / N_decoded over the whole generation (tab:reduce_ratio P:480-504)"},
               "clocks": clk.summary(), "per_rank": stats}
        if roof is not None:
            out.update(roofline=roof, roofline_gemms=gemms, kernels=kernels, step_roofline=stepr)
        if cub is not None:
            out["cublas_reference"] = {"note": "torch.matmul bf16 at the profiled step's S-row shapes, cold weights; "
                                               "ours = CUDA-event time per launch averaged over the step's launches "
                                               "(layers 0-1 run the P rows)", **cub}
        out.update(extras)
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


# ------------------------------------------------------------------------------------ launcher
def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def relaunch_cmd(argv, n: int, port: int) -> list:
    """`bench.py --gpus N` outside torchrun: the same command under torch.distributed.run, one rank
    per GPU, rendezvous on 127.0.0.1."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
            "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + list(argv)


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="focus", choices=["focus", "reference"])
    ap.add_argument("--workload", default="C3")
    ap.add_argument("--logit-scale", type=float, default=1.0)
    ap.add_argument("--batch-invariant", type=int, default=0)
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    return args


def main():
    args = parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(subprocess.call(relaunch_cmd(sys.argv[1:], args.gpus, _free_port())))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_focus(args)


if __name__ == "__main__":
    main()
