"""Algorithm 1 composed per request (App. C P:628-665 + App. E state).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Each request is processed on its own (requests do not interact; batch
invariance S:444), in plain loops.  One FOCUS step for request r at step t
(SURVEY c.3 / DESIGN.md "the step"):

 1. P = uncommitted block positions, M = masked, U = P \\ M; flush <=> M empty.
 2. x_j = E[tok_j] for j in P.
 3. Layer 0 fully on P; K0/V0 stored for P; keys = context [0,s) + block [s, s+B).
    I0 = Importance(layer-0 q, k over P)                        (Alg.1)
 4. Layer 1 projections on P; K1/V1 stored for ALL of P before eviction.
    I1 = Importance(layer-1 q, k over P).
 5. S = Select(dI, ...)  (flush: S = P)                          (Alg.1)
 6. R' = max(R, max S)                                           (reading A-E5)
 7. Layer 1 suffix on S (keys context + whole block, A-K2); layers 2.. on S with keys
    context + block [s, s+R'] (evicted positions keep their last KV, A-K1).
 8. Logits for S cap M; Decode_and_Verify; statistics; DC+ commit; R <- R'; block advance.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from synth.configs import RunConfig
from synth.gen import prompt_lengths, prompt_tokens

from . import focus as F
from .model import Backbone, OracleWeights


@dataclass
class RequestState:
    rid: int
    prompt: np.ndarray
    gen_len: int
    B: int
    s: int = 0                     # block start (absolute position) = committed context length
    b: int = 0                     # block index
    tok: list = field(default_factory=list)
    dstep: list = field(default_factory=list)     # step index at which decoded; None = masked
    committed: set = field(default_factory=set)
    R: int = -1                    # rightmost processed position in the block (App.E)
    token_sum: int = 0             # App.E
    total_steps: int = 0           # App.E
    t: int = 0                     # steps executed so far for this request
    finished: bool = False
    output: list = field(default_factory=list)
    written: dict = field(default_factory=dict)   # layer -> set of block positions holding KV

    def open_block(self, mask_id: int):
        self.tok = [mask_id] * self.B
        self.dstep = [None] * self.B
        self.committed = set()
        self.R = -1
        self.written = {}


@dataclass
class StepRecord:
    """What one step computed for one request (for tests / taps)."""
    P: list
    M: list
    U: list
    flush: bool
    I0: Optional[np.ndarray] = None
    I1: Optional[np.ndarray] = None
    sel: Optional[F.Selection] = None
    S: list = field(default_factory=list)
    R_new: int = -1
    logit_rows: list = field(default_factory=list)     # positions j in S cap M (ascending)
    logits: Optional[np.ndarray] = None
    q0: Optional[np.ndarray] = None
    k0: Optional[np.ndarray] = None
    q1: Optional[np.ndarray] = None
    k1: Optional[np.ndarray] = None


@dataclass
class CommitRecord:
    decoded: list                  # positions decoded this step
    tokens: list                   # their token ids
    conf: dict                     # position -> confidence
    new_committed: set
    block_done: bool
    finished: bool


class OracleEngine:
    def __init__(self, run: RunConfig, mode: str = "ref", weights: OracleWeights | None = None):
        self.run, self.cfg, self.meth = run, run.model, run.method
        self.w = weights or OracleWeights(self.cfg, run.weight_seed)
        self.bb = Backbone(self.cfg, self.w, mode)
        self.req: dict[int, RequestState] = {}
        self.K: dict[int, list] = {}   # rid -> per layer K [cap, Hkv, dh]
        self.V: dict[int, list] = {}
        self.pending: dict[int, StepRecord] = {}
        # OracleTrace-style scripted mode: {(rid, t): {"dI": {j: v}, "conf": {j: c},
        # "tok": {j: id}}} replaces the model forward so the rules can be driven directly.
        self.script: dict | None = None

    # ------------------------------------------------------------------ prefill
    def kv_append(self, rid: int, prompt, gen_len: int):
        """Prefill (focus_kv_append): causal attention over the prompt at every layer fills the
        exact KV cache K/V[0..Lp-1] (reading A-K5), then block 0 opens at s = Lp."""
        c, B = self.cfg, self.meth.block_size
        prompt = np.asarray(prompt, dtype=np.int32)
        Lp = len(prompt)
        cap = Lp + gen_len
        self.K[rid] = [np.zeros((cap, c.n_kv_heads, c.head_dim)) for _ in range(c.n_layers)]
        self.V[rid] = [np.zeros((cap, c.n_kv_heads, c.head_dim)) for _ in range(c.n_layers)]
        x = self.bb.embed(prompt)
        pos = np.arange(Lp)
        for l in range(c.n_layers):
            q, k, v = self.bb.qkv(l, x, pos)
            self.K[rid][l][:Lp], self.V[rid][l][:Lp] = k, v
            o = self.bb.attention_causal(q, self.K[rid][l], self.V[rid][l], 0)
            x = self.bb.o_proj(l, x, o)
            x = self.bb.mlp(l, x)
        st = RequestState(rid=rid, prompt=prompt, gen_len=gen_len, B=B, s=Lp)
        st.open_block(c.mask_token_id)
        self.req[rid] = st

    def set_context_kv(self, rid: int, prompt_len: int, gen_len: int, K: list, V: list):
        """Start a request from a given prompt KV cache (timing baselines: prefill excluded)."""
        c, B = self.cfg, self.meth.block_size
        cap = prompt_len + gen_len
        self.K[rid] = [np.zeros((cap, c.n_kv_heads, c.head_dim)) for _ in range(c.n_layers)]
        self.V[rid] = [np.zeros((cap, c.n_kv_heads, c.head_dim)) for _ in range(c.n_layers)]
        for l in range(c.n_layers):
            self.K[rid][l][:prompt_len] = K[l]
            self.V[rid][l][:prompt_len] = V[l]
        st = RequestState(rid=rid, prompt=np.zeros(prompt_len, np.int32), gen_len=gen_len, B=B, s=prompt_len)
        st.open_block(c.mask_token_id)
        self.req[rid] = st

    # ------------------------------------------------------------------ step
    def _store(self, rid, l, j_list, k, v):
        st = self.req[rid]
        for n, j in enumerate(j_list):
            assert j not in st.committed, "write to a committed KV slot (S:319-320)"
            self.K[rid][l][st.s + j] = k[n]
            self.V[rid][l][st.s + j] = v[n]
            st.written.setdefault(l, set()).add(j)

    def _keys(self, rid, l, extent):
        """Key set of a block query: context [0, s) and block slots [s, s+extent)."""
        st = self.req[rid]
        for j in range(extent):
            assert j in st.written.get(l, set()) or j in st.committed, \
                f"layer {l} slot {j} read before written (Placeholder Integrity)"
        n = st.s + extent
        return self.K[rid][l][:n], self.V[rid][l][:n]

    def step_one(self, rid: int) -> StepRecord:
        c, m, bb = self.cfg, self.meth, self.bb
        st = self.req[rid]
        assert not st.finished
        B, s = st.B, st.s
        st.t += 1
        P = [j for j in range(B) if j not in st.committed]
        M = [j for j in P if st.dstep[j] is None]
        U = [j for j in P if st.dstep[j] is not None]
        rec = StepRecord(P=P, M=M, U=U, flush=not M)
        if self.script is not None:
            return self._scripted_step(rid, st, rec)
        x = bb.embed([st.tok[j] for j in P])
        pos = np.array([s + j for j in P])
        # layer 0 fully (Alg.1)
        q, k, v = bb.qkv(0, x, pos)
        self._store(rid, 0, P, k, v)
        Kc, Vc = self._keys(rid, 0, B)
        x = bb.mlp(0, bb.o_proj(0, x, bb.attention(q, Kc, Vc)))
        qb = np.zeros((B, c.n_q_heads, c.head_dim)); kb = np.zeros((B, c.n_kv_heads, c.head_dim))
        qb[P], kb[P] = q, k
        rec.q0, rec.k0 = qb, kb
        if not rec.flush:
            rec.I0 = F.importance(qb, kb, P, c.group, m.maxpool_kernel)
        # layer 1 projections on P, KV filled before eviction
        q1, k1, v1 = bb.qkv(1, x, pos)
        self._store(rid, 1, P, k1, v1)
        qb1 = np.zeros_like(qb); kb1 = np.zeros_like(kb)
        qb1[P], kb1[P] = q1, k1
        rec.q1, rec.k1 = qb1, kb1
        if rec.flush:
            S = list(P)
        else:
            rec.I1 = F.importance(qb1, kb1, P, c.group, m.maxpool_kernel)
            d = F.delta(rec.I0, rec.I1)
            dfull = [0.0] * B
            for j in P:
                dfull[j] = d[j]
            rec.sel = F.select(dfull, M, U, st.committed, st.R, st.token_sum, st.total_steps, B,
                               m.alpha_num, m.alpha_den, m.placeholder_mode, m.strategy, m.fixed_k,
                               request_id=rid, step=st.t, seed=self.run.weight_seed)
            S = sorted(rec.sel.S)
        rec.S = S
        rec.R_new = max(st.R, max(S))
        idx = [P.index(j) for j in S]
        x = x[idx]
        # layer 1 suffix on S: keys = context + whole block (A-K2)
        Kc, Vc = self._keys(rid, 1, B)
        x = bb.mlp(1, bb.o_proj(1, x, bb.attention(q1[idx], Kc, Vc)))
        spos = np.array([s + j for j in S])
        for l in range(2, c.n_layers):
            q, k, v = bb.qkv(l, x, spos)
            self._store(rid, l, S, k, v)
            Kc, Vc = self._keys(rid, l, rec.R_new + 1)
            x = bb.mlp(l, bb.o_proj(l, x, bb.attention(q, Kc, Vc)))
        Mset = set(M)
        rows = [n for n, j in enumerate(S) if j in Mset]
        rec.logit_rows = [S[n] for n in rows]
        rec.logits = bb.logits(x[rows]) if rows else np.zeros((0, c.vocab))
        self.pending[rid] = rec
        return rec

    def _scripted_step(self, rid, st, rec):
        m, B = self.meth, st.B
        sc = self.script.get((rid, st.t), {})
        if rec.flush:
            rec.S = list(rec.P)
        else:
            if "I0" in sc:                       # importance fed from elsewhere (parity protocol)
                rec.I0, rec.I1 = np.asarray(sc["I0"]), np.asarray(sc["I1"])
            else:
                dI = sc["dI"]
                rec.I0 = np.zeros(B)
                rec.I1 = np.array([dI.get(j, 0.0) for j in range(B)])
            d = F.delta(rec.I0, rec.I1)
            rec.sel = F.select(d, rec.M, rec.U, st.committed, st.R, st.token_sum, st.total_steps, B,
                               m.alpha_num, m.alpha_den, m.placeholder_mode, m.strategy, m.fixed_k,
                               request_id=rid, step=st.t, seed=self.run.weight_seed)
            rec.S = sorted(rec.sel.S)
        rec.R_new = max(st.R, max(rec.S))
        Mset = set(rec.M)
        rec.logit_rows = [j for j in rec.S if j in Mset]
        self.pending[rid] = rec
        rec.script = sc
        return rec

    def commit_one(self, rid: int, conf_override: dict | None = None) -> CommitRecord:
        """Decode_and_Verify, statistics update (App.E; flush steps leave them untouched,
        A-B4), KV commit with Neighbor-Aware Stability, R <- R', block reset / finish."""
        c, m = self.cfg, self.meth
        st, rec = self.req[rid], self.pending.pop(rid)
        toks, conf = {}, {}
        if self.script is not None:
            sc = getattr(rec, "script", {})
            for j in rec.logit_rows:
                conf[j] = sc.get("conf", {}).get(j, 0.0)
                toks[j] = sc.get("tok", {}).get(j, 0)
        else:
            for n, j in enumerate(rec.logit_rows):
                toks[j], conf[j] = F.confidence(rec.logits[n])
        if conf_override is not None:
            conf = dict(conf_override)
        D = [] if rec.flush else F.decide(conf, float(np.float32(m.conf_threshold)))
        for j in D:
            assert toks[j] != c.mask_token_id
            st.tok[j] = toks[j]
            st.dstep[j] = st.t
        if not rec.flush:
            st.token_sum += len(D)
            st.total_steps += 1
        new = F.kv_commit(st.dstep, st.committed, rec.P, st.t, st.B, m.cache_mode)
        st.committed |= new
        st.R = rec.R_new
        block_done = len(st.committed) == st.B
        if block_done:
            st.output.extend(st.tok)
            st.b += 1
            st.s += st.B
            if st.b * st.B >= st.gen_len:
                st.finished = True
            else:
                st.open_block(c.mask_token_id)
        return CommitRecord(decoded=D, tokens=[toks[j] for j in D], conf=conf, new_committed=new,
                            block_done=block_done, finished=st.finished)

    def step(self, rids):
        return {r: self.step_one(r) for r in rids}

    def commit(self, rids):
        return {r: self.commit_one(r) for r in rids}


def request_prompts(run: RunConfig) -> list:
    """Synthetic prompts of the run (synth recipe)."""
    if run.prompt_len_hi is not None:
        lens = prompt_lengths(run.n_requests, run.prompt_len, run.prompt_len_hi).tolist()
    else:
        lens = [run.prompt_len] * run.n_requests
    return [prompt_tokens(r, lens[r], run.model.vocab) for r in range(run.n_requests)]


def run_to_completion(run: RunConfig, mode: str = "ref", rids=None, max_steps: int = 100000):
    """Prefill every request, then step + commit until all finish.  Returns (engine, per-step log)."""
    eng = OracleEngine(run, mode)
    prompts = request_prompts(run)
    rids = list(range(run.n_requests)) if rids is None else list(rids)
    for r in rids:
        eng.kv_append(r, prompts[r], run.gen_len)
    log = []
    for _ in range(max_steps):
        live = [r for r in rids if not eng.req[r].finished]
        if not live:
            break
        recs = eng.step(live)
        coms = eng.commit(live)
        log.append((recs, coms))
    return eng, log
