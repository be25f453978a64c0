"""Thin ctypes binding of libfocus (include/focus.h): argument marshalling only.

Every step of the decode path runs in the CUDA kernels of libfocus.so; this module only converts
Python values to the C structs, owns the device arena (a torch uint8 CUDA tensor) and passes the
current torch CUDA stream.  There is no CPU fallback: if the shared library is missing or no CUDA
device is present, the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libfocus.so")

FOCUS_OK, FOCUS_ERR_CONFIG, FOCUS_ERR_INVARIANT, FOCUS_ERR_IO = 0, 2, 3, 4
FOCUS_ERR_NOMEM, FOCUS_ERR_STATE, FOCUS_ERR_CUDA = 5, 6, 7

DBG = dict(STATE=1, COUNTERS=2, ROWS_P=3, ROWS_S=4, ROWS_L=5, I0=6, I1=7, LOGITS=8, TOKCONF=9, KV_K=10, KV_V=11,
           TAP_X_IN=20, TAP_H=21, TAP_QKV=22, TAP_ATTN=23, TAP_X_MID=24, TAP_H2=25, TAP_ACT=26, TAP_X_OUT=27,
           TAP_QS=28, HL=29, LAUNCHES=30, PROFILE=31, ATTN_TRACE=32, MOE_SEL=33, MOE_WT=34,
           MOE_ROWS=35, MOE_Y=36, MOE_AG=37)
PROF_KINDS = ["setup", "embed", "rmsnorm", "gemm_qkv", "rope_store", "attention", "importance", "gemm_o",
              "gemm_gu", "silu_mul", "gemm_down", "select", "gather", "gemm_lm", "vocab_reduce", "commit",
              "moe_route", "moe_experts", "moe_combine"]

EXPORTED = ["focus_required_bytes", "focus_init", "focus_destroy", "focus_kv_append", "focus_step_block",
            "focus_commit", "focus_sync", "focus_get_tokens", "focus_release", "focus_set_tap",
            "focus_debug_export", "focus_status_str", "focus_set_profile"]


class focus_config(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("d_model", C.c_int32), ("n_q_heads", C.c_int32),
                ("n_kv_heads", C.c_int32), ("head_dim", C.c_int32), ("d_ff", C.c_int32), ("vocab", C.c_int32),
                ("rope_theta", C.c_float), ("rms_eps", C.c_float),
                ("block_size", C.c_int32), ("alpha_num", C.c_int32), ("alpha_den", C.c_int32),
                ("conf_threshold", C.c_float), ("maxpool_kernel", C.c_int32), ("cache_mode", C.c_int32),
                ("placeholder_mode", C.c_int32), ("strategy", C.c_int32), ("fixed_k", C.c_int32),
                ("max_requests", C.c_int32), ("max_seq_len", C.c_int32), ("page_size", C.c_int32),
                ("max_prefill_chunk", C.c_int32), ("kv_pages", C.c_int64), ("weight_seed", C.c_uint64),
                ("debug_taps", C.c_int32), ("logit_scale", C.c_float), ("batch_invariant", C.c_int32),
                ("n_experts", C.c_int32), ("top_k", C.c_int32), ("d_expert", C.c_int32),
                ("n_shared_experts", C.c_int32), ("n_dense_layers", C.c_int32)]


class focus_commit_result(C.Structure):
    _fields_ = [("req_id", C.c_int32), ("n_new", C.c_int32), ("block_done", C.c_int32), ("finished", C.c_int32),
                ("n_committed", C.c_int32), ("pos", C.c_int32 * 64), ("tok", C.c_int32 * 64)]


class focus_req_state(C.Structure):
    _fields_ = [("active", C.c_int32), ("finished", C.c_int32), ("s", C.c_int32), ("b", C.c_int32),
                ("gen_len", C.c_int32), ("prompt_len", C.c_int32), ("R", C.c_int32), ("t", C.c_int32),
                ("token_sum", C.c_int64), ("total_steps", C.c_int64), ("committed", C.c_uint64),
                ("masked", C.c_uint64), ("P", C.c_uint64), ("M", C.c_uint64), ("S", C.c_uint64),
                ("R_new", C.c_int32), ("K", C.c_int32), ("n_sigma", C.c_int32), ("k_hist", C.c_int32),
                ("flush", C.c_int32), ("n_new", C.c_int32), ("n_committed", C.c_int32), ("pad_", C.c_int32),
                ("tok", C.c_int32 * 64), ("dstep", C.c_int32 * 64)]


class FocusError(RuntimeError):
    def __init__(self, code: int, where: str):
        self.code = code
        msg = _lib().focus_status_str(code).decode() if _LIB is not None else str(code)
        super().__init__(f"{where}: {msg} ({code})")


_LIB: Optional[C.CDLL] = None


def _lib() -> C.CDLL:
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libfocus.so not built ({LIB_PATH}); run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        L.focus_required_bytes.restype = C.c_size_t
        L.focus_required_bytes.argtypes = [C.POINTER(focus_config)]
        L.focus_init.argtypes = [C.POINTER(focus_config), C.c_void_p, C.c_size_t, C.c_void_p, C.POINTER(C.c_void_p)]
        L.focus_destroy.argtypes = [C.c_void_p]
        L.focus_kv_append.argtypes = [C.c_void_p, C.c_int32, C.POINTER(C.c_int32), C.c_int32, C.c_int32]
        L.focus_step_block.argtypes = [C.c_void_p, C.POINTER(C.c_int32), C.c_int32]
        L.focus_commit.argtypes = [C.c_void_p, C.POINTER(C.c_int32), C.c_int32, C.c_void_p]
        L.focus_sync.argtypes = [C.c_void_p]
        L.focus_get_tokens.argtypes = [C.c_void_p, C.c_int32, C.POINTER(C.c_int32), C.c_int32, C.POINTER(C.c_int32)]
        L.focus_release.argtypes = [C.c_void_p, C.c_int32]
        L.focus_set_tap.argtypes = [C.c_void_p, C.c_int32]
        L.focus_set_profile.argtypes = [C.c_void_p, C.c_int32]
        L.focus_debug_export.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_size_t,
                                         C.POINTER(C.c_size_t)]
        L.focus_status_str.restype = C.c_char_p
        L.focus_status_str.argtypes = [C.c_int]
        for name in EXPORTED:
            if name not in ("focus_required_bytes", "focus_status_str"):
                getattr(L, name).restype = C.c_int
        _LIB = L
    return _LIB


def _check(rc: int, where: str):
    if rc != FOCUS_OK:
        raise FocusError(rc, where)


def make_config(run, max_requests: Optional[int] = None, max_seq_len: Optional[int] = None,
                max_prefill_chunk: int = 1024, debug_taps: bool = False, kv_pages: int = 0,
                batch_invariant: bool = False) -> focus_config:
    """focus_config from a synth.RunConfig (plain data)."""
    m, me = run.model, run.method
    if max_seq_len is None:
        hi = run.prompt_len_hi if run.prompt_len_hi is not None else run.prompt_len
        max_seq_len = hi + run.gen_len
    return focus_config(
        n_layers=m.n_layers, d_model=m.d_model, n_q_heads=m.n_q_heads, n_kv_heads=m.n_kv_heads,
        head_dim=m.head_dim, d_ff=m.d_ff, vocab=m.vocab, rope_theta=m.rope_theta, rms_eps=m.rms_eps,
        block_size=me.block_size, alpha_num=me.alpha_num, alpha_den=me.alpha_den,
        conf_threshold=me.conf_threshold, maxpool_kernel=me.maxpool_kernel, cache_mode=me.cache_mode,
        placeholder_mode=me.placeholder_mode, strategy=me.strategy, fixed_k=me.fixed_k,
        max_requests=max_requests or run.n_requests, max_seq_len=max_seq_len, page_size=run.page_size,
        max_prefill_chunk=max_prefill_chunk, kv_pages=kv_pages, weight_seed=run.weight_seed,
        debug_taps=1 if debug_taps else 0, logit_scale=m.logit_scale, batch_invariant=1 if batch_invariant else 0,
        n_experts=m.n_experts, top_k=m.top_k, d_expert=m.d_expert, n_shared_experts=m.n_shared_experts,
        n_dense_layers=m.n_dense_layers)


def focus_required_bytes(cfg: focus_config) -> int:
    return int(_lib().focus_required_bytes(C.byref(cfg)))


class FocusContext:
    """One libfocus context on the current CUDA device: owns the torch arena tensor."""

    def __init__(self, cfg: focus_config, device: str = "cuda", stream=None):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("libfocus needs a CUDA device (no CPU fallback)")
        L = _lib()
        self.cfg = cfg
        nbytes = focus_required_bytes(cfg)
        if nbytes == 0:
            raise FocusError(FOCUS_ERR_CONFIG, "focus_required_bytes")
        self.arena = torch.empty(nbytes, dtype=torch.uint8, device=device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.arena.device)
        h = C.c_void_p()
        _check(L.focus_init(C.byref(cfg), C.c_void_p(self.arena.data_ptr()), nbytes,
                            C.c_void_p(self.stream.cuda_stream), C.byref(h)), "focus_init")
        self.h = h
        self.B = cfg.block_size
        self._res = None
        self._res_n = 0

    # -- C ABI calls (same names) --------------------------------------------------------------
    def focus_kv_append(self, req_id: int, prompt: Sequence[int], gen_len: int):
        arr = np.ascontiguousarray(np.asarray(prompt, dtype=np.int32))
        _check(_lib().focus_kv_append(self.h, req_id, arr.ctypes.data_as(C.POINTER(C.c_int32)), len(arr), gen_len),
               "focus_kv_append")

    def focus_step_block(self, req_ids: Sequence[int]):
        ids = np.ascontiguousarray(np.asarray(req_ids, dtype=np.int32))
        _check(_lib().focus_step_block(self.h, ids.ctypes.data_as(C.POINTER(C.c_int32)), len(ids)),
               "focus_step_block")

    def focus_commit(self, req_ids: Sequence[int], pinned_out=None):
        ids = np.ascontiguousarray(np.asarray(req_ids, dtype=np.int32))
        ptr = C.c_void_p(pinned_out) if pinned_out is not None else None
        _check(_lib().focus_commit(self.h, ids.ctypes.data_as(C.POINTER(C.c_int32)), len(ids), ptr), "focus_commit")

    def focus_sync(self):
        _check(_lib().focus_sync(self.h), "focus_sync")

    def focus_get_tokens(self, req_id: int, cap: int = 1 << 20) -> list:
        buf = (C.c_int32 * cap)()
        n = C.c_int32()
        _check(_lib().focus_get_tokens(self.h, req_id, buf, cap, C.byref(n)), "focus_get_tokens")
        return list(buf[: n.value])

    def focus_release(self, req_id: int):
        _check(_lib().focus_release(self.h, req_id), "focus_release")

    def focus_set_tap(self, layer: int):
        _check(_lib().focus_set_tap(self.h, layer), "focus_set_tap")

    def focus_set_profile(self, on: bool):
        _check(_lib().focus_set_profile(self.h, 1 if on else 0), "focus_set_profile")

    def launches(self) -> int:
        return int(np.frombuffer(self.focus_debug_export("LAUNCHES", cap=8), dtype=np.uint64)[0])

    def profile(self) -> dict:
        raw = self.focus_debug_export("PROFILE", cap=16 * len(PROF_KINDS))
        a = np.frombuffer(raw, dtype=np.dtype([("kind", "<i4"), ("n", "<i4"), ("ms", "<f4"), ("max", "<f4")]))
        return {PROF_KINDS[int(e["kind"])]: dict(launches=int(e["n"]), total_ms=float(e["ms"]), max_ms=float(e["max"]))
                for e in a}

    def focus_debug_export(self, what, req_id: int = 0, layer: int = 0, cap: int = 1 << 31) -> bytes:
        code = DBG[what] if isinstance(what, str) else int(what)
        buf = (C.c_char * cap)() if cap <= (1 << 26) else None
        if buf is None:
            arr = np.empty(cap, dtype=np.uint8)
            ptr = arr.ctypes.data
        else:
            ptr = C.addressof(buf)
        n = C.c_size_t()
        _check(_lib().focus_debug_export(self.h, code, req_id, layer, C.c_void_p(ptr), cap, C.byref(n)),
               "focus_debug_export")
        return bytes(buf[: n.value]) if buf is not None else arr[: n.value].tobytes()

    def focus_destroy(self):
        if getattr(self, "h", None) is not None:
            _check(_lib().focus_destroy(self.h), "focus_destroy")
            self.h = None

    def __del__(self):
        try:
            self.focus_destroy()
        except Exception:
            pass

    # -- convenience ---------------------------------------------------------------------------
    def commit_results(self, req_ids: Sequence[int]) -> list:
        """focus_commit into a pinned host buffer + sync; returns a list of dicts."""
        import torch
        n = len(req_ids)
        if self._res is None or self._res_n < n:
            self._res = torch.empty(max(n, 1) * C.sizeof(focus_commit_result), dtype=torch.uint8).pin_memory()
            self._res_n = max(n, 1)
        self.focus_commit(req_ids, self._res.data_ptr())
        self.focus_sync()
        arr = (focus_commit_result * n).from_address(self._res.data_ptr())
        return [dict(req_id=r.req_id, n_new=r.n_new, block_done=r.block_done, finished=r.finished,
                     n_committed=r.n_committed, pos=list(r.pos[: r.n_new]), tok=list(r.tok[: r.n_new]))
                for r in arr]

    def states(self) -> list:
        raw = self.focus_debug_export("STATE", cap=self.cfg.max_requests * C.sizeof(focus_req_state))
        arr = (focus_req_state * self.cfg.max_requests).from_buffer_copy(raw)
        return list(arr)

    def counters(self) -> np.ndarray:
        """int32[8]: M_P, M_S, M_logit, invariant, rows per attention chunk, chunks, pad, pad."""
        return np.frombuffer(self.focus_debug_export("COUNTERS", cap=64)[:32], dtype=np.int32).copy()

    def cumulative_rows(self) -> dict:
        """Rows processed since focus_init: sum M_P, sum M_S, sum M_logit and the step count."""
        a = np.frombuffer(self.focus_debug_export("COUNTERS", cap=64)[32:64], dtype=np.int64)
        return dict(sum_P=int(a[0]), sum_S=int(a[1]), sum_L=int(a[2]), steps=int(a[3]))

    def rows(self, which: str) -> np.ndarray:
        return np.frombuffer(self.focus_debug_export("ROWS_" + which), dtype=np.int32).reshape(-1, 4).copy()

    def export_f32(self, what: str, shape) -> np.ndarray:
        n = int(np.prod(shape))
        raw = self.focus_debug_export(what, cap=n * 4)
        return np.frombuffer(raw, dtype=np.float32)[:n].reshape(shape).copy()

    def export_bf16(self, what: str, shape, req_id: int = 0, layer: int = 0) -> np.ndarray:
        n = int(np.prod(shape))
        raw = self.focus_debug_export(what, req_id=req_id, layer=layer, cap=n * 2)
        u = np.frombuffer(raw, dtype=np.uint16)[:n].astype(np.uint32) << np.uint32(16)
        return u.view(np.float32).astype(np.float64).reshape(shape)
