"""Stage-wise parity of every kernel of the step at SDAR-8B / 1.7B layer shapes (fewer layers),
through the tap buffers of the C ABI: the oracle is fed each stage's GPU input and compared with the
stage's GPU output.  Shapes span several GEMM tiles with ragged M,
several KV pages, GQA packing and block sizes 4/16."""
import json
import os

import numpy as np
import pytest

from oracle import focus as F
from oracle.model import OracleWeights
from oracle.numerics import attend, bf16_round, f32, rms_norm, rope, silu
from oracle.engine import request_prompts
from synth import get_config
from synth.configs import MethodConfig, ModelConfig
from synth.gen import TID_LMHEAD, weight_matrix

from gpu_helpers import bits, gpu_importance_sums, rel_l2

pytestmark = pytest.mark.gpu

M8B4 = ModelConfig(n_layers=4, d_model=4096, n_q_heads=32, n_kv_heads=8, head_dim=128, d_ff=12288, vocab=151936,
                   rope_theta=1e6)
M1P7B3 = ModelConfig(n_layers=3, d_model=2048, n_q_heads=16, n_kv_heads=8, head_dim=128, d_ff=6144, vocab=151936,
                     rope_theta=1e6)
# small-width models with long contexts: several key splits per (request, kv head) in the tensor-core
# attention (split merge), page sizes below / above the 128-key tile, GQA groups 4 and 2, several
# query chunks per request (B=64)
MINI128 = ModelConfig(n_layers=3, d_model=512, n_q_heads=8, n_kv_heads=2, head_dim=128, d_ff=512, vocab=4096,
                      rope_theta=1e6)
MINI_G2 = ModelConfig(n_layers=3, d_model=512, n_q_heads=8, n_kv_heads=4, head_dim=128, d_ff=512, vocab=4096,
                      rope_theta=1e6)


# GEMM stage tolerance (DESIGN.md §7 "numerics"): the tensor core accumulates the K bf16 products in
# fp32 in its own order; the rounding errors of the partial sums add up like a random walk, ~sqrt(K) * u
# relative (u = 2^-24).  Bound: 3 sqrt(K) u (K = 12288: 2.0e-5; K = 4096: 1.1e-5).  Measured on B200
# (profiles/r2_gemm_errors.jsonl, every stage of this test): max 7.1e-6 at K = 6144 / 12288, 3.5e-6 at
# K = 4096, i.e. at most half the bound.
def gemm_tol(K):
    return 3.0 * np.sqrt(K) * 2.0 ** -24



def _log_err(stage, K, err):
    """Append a measured GEMM stage error to $FOCUS_TEST_LOG (JSON lines) when set: the distribution
    behind gemm_tol (profiles/r2_gemm_errors.jsonl)."""
    path = os.environ.get("FOCUS_TEST_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps({"stage": stage, "K": int(K), "rel_l2": float(err)}) + "\n")


def _bf16_close(got, want, tag, frac=0.95, tol=4e-3):
    assert rel_l2(got, want) < tol, (tag, rel_l2(got, want))
    assert np.mean(got == want) > frac, (tag, np.mean(got == want))


@pytest.mark.parametrize("model,B,nreq,prompt,taps,page", [
    (M8B4, 16, 3, 100, (0, 1, 3), 64),
    (M8B4, 16, 26, 40, (0, 1), 64),          # ~400 P rows: 4 m-tiles
    (M1P7B3, 4, 5, 70, (0, 1, 2), 64),
    (MINI128, 16, 3, 1100, (0, 1, 2), 16),
    (MINI128, 64, 2, 700, (0, 1, 2), 32),
    (MINI_G2, 32, 2, 1500, (0, 1, 2), 128),
    (MINI_G2, 8, 3, 2900, (0, 1, 2), 256),
])
def test_layer_stages(model, B, nreq, prompt, taps, page):
    from paper_2601_23278_b200 import FocusContext, make_config
    run = get_config("C3").with_(model=model, method=MethodConfig(block_size=B), n_requests=nreq, prompt_len=prompt,
                                 gen_len=4 * B, page_size=page)
    ctx = FocusContext(make_config(run, debug_taps=True))
    prompts = request_prompts(run)
    for r in range(nreq):
        ctx.focus_kv_append(r, prompts[r], run.gen_len)
    W = OracleWeights(model, run.weight_seed)
    d, qd, hq, hkv, dh, G = model.d_model, model.n_q_heads * model.head_dim, model.n_q_heads, model.n_kv_heads, \
        model.head_dim, model.group
    live = list(range(nreq))
    ctx.focus_step_block(live)                     # one untapped step so U / committed sets are non-trivial
    ctx.commit_results(live)
    for l in taps:
        ctx.focus_set_tap(l)
        pre = ctx.states()
        ctx.focus_step_block(live)
        ctx.focus_sync()
        st = ctx.states()
        cnt = ctx.counters()
        MP, MS, ML = int(cnt[0]), int(cnt[1]), int(cnt[2])
        rowsP, rowsS, rowsL = ctx.rows("P"), ctx.rows("S"), ctx.rows("L")
        Mq = MP if l <= 1 else MS
        rows_q = rowsP if l <= 1 else rowsS
        Ma = MP if l == 0 else MS
        rows_a = rowsP if l == 0 else rowsS
        w = W.layer(l)
        x_in = ctx.export_f32("TAP_X_IN", (Mq, d)).astype(np.float64)
        h = ctx.export_bf16("TAP_H", (Mq, d))
        _bf16_close(h, bf16_round(rms_norm(x_in, 1.0, model.rms_eps)), ("rmsnorm", l), frac=0.99)
        qkv = ctx.export_bf16("TAP_QKV", (Mq, (hq + 2 * hkv) * dh))
        pos = rows_q[:, 2]
        y = f32(h @ np.concatenate([w["q"], w["k"], w["v"]]).T)
        q_o = bf16_round(rope(f32(y[:, :qd].reshape(Mq, hq, dh)), pos, model.rope_theta)).reshape(Mq, -1)
        k_o = bf16_round(rope(f32(y[:, qd:qd + hkv * dh].reshape(Mq, hkv, dh)), pos, model.rope_theta)).reshape(Mq, -1)
        v_o = bf16_round(y[:, qd + hkv * dh:])
        _bf16_close(qkv, np.concatenate([q_o, k_o, v_o], 1), ("qkv+rope", l))
        # the QKV GEMM before its bf16 rounding is not exported; its fp32 accumulation shows in the
        # fraction of bf16 outputs identical to the fp64 reference's rounding
        _log_err("qkv bf16-mismatch-fraction", d, 1.0 - float(np.mean(qkv == np.concatenate([q_o, k_o, v_o], 1))))
        # importance (layers 0, 1) from the GPU's q, k over P
        if l <= 1:
            Iraw = np.frombuffer(ctx.focus_debug_export("I0" if l == 0 else "I1"), np.float32)
            Ig = gpu_importance_sums(Iraw, cnt, [st[r].P for r in live], hkv, B)
            for i, r in enumerate(live):
                s = st[r]
                if s.flush:
                    continue
                P = bits(s.P, B)
                qb = np.zeros((B, hq, dh)); kb = np.zeros((B, hkv, dh))
                for n in range(Mq):
                    if rows_q[n][0] == r:
                        qb[rows_q[n][1]] = qkv[n, :qd].reshape(hq, dh)
                        kb[rows_q[n][1]] = qkv[n, qd:qd + hkv * dh].reshape(hkv, dh)
                Io = F.importance(qb, kb, P, G, 3)
                floor = 1e-6 * len(P) * hq
                err = np.abs(Ig[i][P] - Io[P]) / np.maximum(np.abs(Io[P]), floor)
                assert err.max() <= 1e-3, (l, r, err.max())
        # attention (queries: layer-1 uses the compacted q rows)
        q_att = ctx.export_bf16("TAP_QS", (MS, qd)) if l == 1 else qkv[:, :qd]
        att = ctx.export_bf16("TAP_ATTN", (Ma, qd))
        ref = np.zeros_like(att)
        for n in range(Ma):
            r, j = int(rows_a[n][0]), int(rows_a[n][1])
            s = st[r]
            ext = B if l <= 1 else s.R_new + 1
            nk = s.s + ext
            K = ctx.export_bf16("KV_K", (s.s + B, hkv, dh), req_id=r, layer=l)[:nk]
            V = ctx.export_bf16("KV_V", (s.s + B, hkv, dh), req_id=r, layer=l)[:nk]
            qr = q_att[n].reshape(hq, dh)
            ref[n] = np.concatenate([attend(qr[hh:hh + 1], K[:, hh // G], V[:, hh // G])[0] for hh in range(hq)])
        assert rel_l2(att, ref) <= 1e-2, ("attention", l, rel_l2(att, ref))
        # O projection + residual (layer 1: residual rows are the gathered P rows)
        if l == 1:
            idx = {(int(a), int(b)): n for n, (a, b, _, _) in enumerate(rowsP[:MP])}
            x_res = np.stack([x_in[idx[(int(a), int(b))]] for a, b, _, _ in rowsS[:MS]])
        else:
            x_res = x_in
        x_mid = ctx.export_f32("TAP_X_MID", (Ma, d)).astype(np.float64)
        inc = att @ w["o"].T
        _log_err("o-proj", qd, rel_l2(x_mid - x_res, inc))
        assert rel_l2(x_mid - x_res, inc) < gemm_tol(qd), ("o-proj", l, rel_l2(x_mid - x_res, inc))
        h2 = ctx.export_bf16("TAP_H2", (Ma, d))
        _bf16_close(h2, bf16_round(rms_norm(x_mid, 1.0, model.rms_eps)), ("rmsnorm2", l), frac=0.99)
        act = ctx.export_bf16("TAP_ACT", (Ma, model.d_ff))
        _bf16_close(act, bf16_round(silu(f32(h2 @ w["gate"].T)) * f32(h2 @ w["up"].T)), ("swiglu", l))
        x_out = ctx.export_f32("TAP_X_OUT", (Ma, d)).astype(np.float64)
        inc = act @ w["down"].T
        _log_err("down", model.d_ff, rel_l2(x_out - x_mid, inc))
        assert rel_l2(x_out - x_mid, inc) < gemm_tol(model.d_ff), ("down", l, rel_l2(x_out - x_mid, inc))
        # LM head on S cap M rows (sampled vocab columns) after the last layer
        if l == model.n_layers - 1 and ML:
            hl = ctx.export_bf16("HL", (ML, d))
            srcL = [int(np.flatnonzero((rowsS[:MS, 0] == a) & (rowsS[:MS, 1] == b))[0]) for a, b, _, _ in rowsL[:ML]]
            _bf16_close(hl, bf16_round(rms_norm(x_out[srcL], 1.0, model.rms_eps)), "final-norm", frac=0.99)
            logits = ctx.export_f32("LOGITS", (ML, model.vocab))
            for lo in (0, model.vocab - 2048):
                wl = weight_matrix(TID_LMHEAD, model.vocab, d, d, run.weight_seed, lo, lo + 2048).astype(np.float64)
                _log_err("lm-head", d, rel_l2(logits[:, lo:lo + 2048], hl @ wl.T))
                assert rel_l2(logits[:, lo:lo + 2048], hl @ wl.T) < gemm_tol(d), ("lm-head", lo)
        ctx.commit_results(live)
    ctx.focus_set_tap(-1)
    ctx.focus_sync()


def test_layer_stages_multicast_gemm(monkeypatch):
    """Same stage-wise parity with the opt-in 4-CTA TMA-multicast GEMM clusters (4 m-tiles of rows) of
    the one-CTA-per-tile GEMM."""
    monkeypatch.setenv("FOCUS_GEMM_PAIR", "0")
    monkeypatch.setenv("FOCUS_GEMM_MC", "1")
    test_layer_stages(M8B4, 16, 26, 40, (0, 1), 64)


def test_layer_stages_single_cta_gemm(monkeypatch):
    """Stage-wise parity with the one-CTA-per-tile tcgen05 GEMM (cta_group::1) instead of CTA pairs."""
    monkeypatch.setenv("FOCUS_GEMM_PAIR", "0")
    test_layer_stages(M8B4, 16, 26, 40, (0, 1), 64)


def test_layer_stages_pair_stream_k_gemm(monkeypatch):
    """Stage-wise parity with the opt-in stream-K schedule of the CTA-pair GEMM (units cut at pair
    boundaries, later pieces' fp32 partials added by the first piece in pair order), including grids
    where some pairs own no stage (tiny GEMMs)."""
    monkeypatch.setenv("FOCUS_GEMM_PSK", "1")
    test_layer_stages(M8B4, 16, 26, 40, (0, 1), 64)
    test_layer_stages(MINI128, 16, 3, 1100, (0, 1, 2), 16)


def test_layer_stages_stream_k_attention(monkeypatch):
    """Stage-wise parity with the opt-in stream-K attention schedule (pairs cut at CTA boundaries,
    merged in-kernel by the last-arriving piece) on a long-context, multi-request case."""
    monkeypatch.setenv("FOCUS_ATTN_SK", "1")
    test_layer_stages(MINI128, 16, 3, 1100, (0, 1, 2), 16)


def test_layer_stages_tail_split(monkeypatch):
    """Stage-wise parity with the opt-in tail split (the units of the last partial round of the attention
    grid are cut into key ranges, one per idle CTA, merged in-kernel by the last-arriving piece)."""
    monkeypatch.setenv("FOCUS_ATTN_TAIL", "1")
    test_layer_stages(MINI128, 16, 3, 1100, (0, 1, 2), 16)


def test_layer_stages_unplanned_attention(monkeypatch):
    """Stage-wise parity with the attention unit table built in the kernel prologue (no plan kernel)."""
    monkeypatch.setenv("FOCUS_ATTN_NOPLAN", "1")
    test_layer_stages(MINI_G2, 8, 3, 2900, (0, 1, 2), 256)


def test_layer_stages_swap_ab_gemm(monkeypatch):
    """Stage-wise parity with the swap-AB decode GEMM (default for M_max <= 256 live rows: weights on
    the MMA M side, K ranges of a tile in one thread-block cluster, reduced in order through distributed
    shared memory) for every projection, at the 8B and 1.7B layer shapes, including a ragged live row
    count that is not a multiple of the 32-row activation box."""
    monkeypatch.setenv("FOCUS_GEMM_SWAP", "1")
    test_layer_stages(M8B4, 16, 3, 100, (0, 1, 3), 64)
    test_layer_stages(M1P7B3, 4, 5, 70, (0, 1, 2), 64)
    test_layer_stages(M1P7B3, 4, 13, 70, (0, 2), 64)
    # 128- and 256-token capacities (M_max 80, 192; gate-up stays on the CTA-pair kernel above 64 rows)
    test_layer_stages(M8B4, 16, 5, 100, (0, 2), 64)
    test_layer_stages(M8B4, 16, 12, 60, (0, 2), 64)


def test_layer_stages_pair_gemm_small_m(monkeypatch):
    """The same small-M stages on the CTA-pair GEMM (FOCUS_GEMM_SWAP=0), which the swap-AB kernel
    replaces by default at these row counts."""
    monkeypatch.setenv("FOCUS_GEMM_SWAP", "0")
    test_layer_stages(M8B4, 16, 3, 100, (0, 1, 3), 64)
    test_layer_stages(M1P7B3, 4, 5, 70, (0, 1, 2), 64)


def test_layer_stages_frequent_rescale(monkeypatch):
    """Stage-wise parity with the lazy-softmax threshold cut from 2^8 to 2^0.25 (FOCUS_ATTN_RESCALE_LOG2),
    so the running max, which starts from each unit's first key, moves on most tiles: the exact per-row
    max and the O^T / row-sum rescale of the tensor-core attention run constantly (at the default
    threshold they never fire on these random-weight logits)."""
    monkeypatch.setenv("FOCUS_ATTN_RESCALE_LOG2", "0.25")
    test_layer_stages(MINI128, 16, 3, 1100, (0, 1, 2), 16)
    test_layer_stages(M8B4, 16, 5, 100, (0, 2), 64)
