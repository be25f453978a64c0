/* focus.h — C ABI of the B200-native FOCUS block-diffusion decode step.
 *
 * FOCUS (arxiv 2601.23278): one step of block-diffusion decoding (Alg.1).
 * A block of B masked tokens per request attends bidirectionally within the block and causally to
 * an exact paged KV cache; attention-derived importance deltas of layers 0 and 1
 * (Eq.2, Eq.3) select the tokens likely to be decodable (Eq.4-5, §4.2
 * P:292-303); the survivors are compacted and run through the remaining layers; confidence-based
 * unmasking commits tokens, and the Neighbor-Aware delayed KV cache (§4.3)
 * decides which block positions are re-processed.
 *
 * One context = one GPU + one CUDA stream.  A context is not thread-safe; distinct contexts are
 * independent.  All work is stream-ordered on the stream given to focus_init; no call performs a
 * device-wide synchronisation except focus_sync / focus_get_tokens / focus_debug_export.
 *
 * Memory ownership: the caller allocates ONE device arena (focus_required_bytes) and keeps it alive
 * until focus_destroy; the context carves weights, the paged KV pool, per-request state and all
 * workspaces out of it and never allocates device memory after focus_init.  Host input arrays are
 * read before a call returns.  Host output buffers of focus_commit are written asynchronously and are
 * valid after the next focus_sync.
 *
 * Errors: every call returns a focus_status and never aborts the process.  Device-detected invariant
 * violations (write to a committed KV slot, empty retained set, a decoded token equal to the mask id)
 * set a device flag reported as FOCUS_ERR_INVARIANT by the next focus_sync.
 */
#ifndef FOCUS_H_
#define FOCUS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  FOCUS_OK = 0,
  FOCUS_ERR_CONFIG = 2,     /* invalid configuration (SPEC S:663 class 2)                     */
  FOCUS_ERR_INVARIANT = 3,  /* device invariant flag set (SPEC S:663 class 3)                 */
  FOCUS_ERR_IO = 4,         /* host buffer too small / bad pointer                            */
  FOCUS_ERR_NOMEM = 5,      /* arena too small or KV page pool exhausted                      */
  FOCUS_ERR_STATE = 6,      /* unknown / duplicate request id, step without commit, ...      */
  FOCUS_ERR_CUDA = 7        /* a CUDA runtime error                                           */
} focus_status;

/* cache_mode (§4.3; ablation tab:ablation_cache P:519-536) */
enum { FOCUS_CACHE_NONE = 0, FOCUS_CACHE_DC = 1, FOCUS_CACHE_DC_PLUS = 2 };
/* placeholder_mode (§4.2; Alg.1 P:652 literal = ALL_MASKED; App.E P:775 = UNPROCESSED_ONLY) */
enum { FOCUS_PLACEHOLDER_UNPROCESSED_ONLY = 0, FOCUS_PLACEHOLDER_ALL_MASKED = 1 };
/* strategy (FOCUS = Eq.4 budget + top-K by importance delta; NONE = K=B, no eviction;
   FIXED_* = tab:selection_strategy P:308-353 with K = fixed_k) */
enum { FOCUS_STRATEGY_FOCUS = 0, FOCUS_STRATEGY_NONE = 1, FOCUS_STRATEGY_FIXED_TOP = 2,
       FOCUS_STRATEGY_FIXED_RANDOM = 3, FOCUS_STRATEGY_FIXED_BOTTOM = 4 };

typedef struct {
  /* backbone (SURVEY A-M1: Qwen3-like GQA + RoPE + SwiGLU + RMSNorm; weights random-init) */
  int32_t n_layers;        /* >= 2 (layer 0 and layer 1 are structurally distinct, Alg.1)      */
  int32_t d_model;         /* multiple of 64, at most 8192                                      */
  int32_t n_q_heads, n_kv_heads;  /* n_q_heads % n_kv_heads == 0 (GQA)                         */
  int32_t head_dim;        /* even, multiple of 16, <= 128                                     */
  int32_t d_ff;            /* multiple of 128                                                  */
  int32_t vocab;           /* mask token id = vocab - 1 (reading A-M2)                         */
  float rope_theta, rms_eps;
  /* method (Alg.1 hyper-parameters) */
  int32_t block_size;      /* B in [1, 64]: per-request masks are uint64                       */
  int32_t alpha_num, alpha_den;   /* alpha = num/den > 1 exact rational (Eq.4, reading A-B3)   */
  float conf_threshold;    /* tau in (0, 1]                                     */
  int32_t maxpool_kernel;  /* odd >= 1, default 3                                      */
  int32_t cache_mode, placeholder_mode, strategy, fixed_k;
  /* capacity */
  int32_t max_requests;    /* request ids are slots 0 .. max_requests-1                       */
  int32_t max_seq_len;     /* prompt + generation per request                                 */
  int32_t page_size;       /* KV page size (positions per page)                               */
  int32_t max_prefill_chunk; /* rows per prefill pass                                         */
  int64_t kv_pages;        /* pages in the pool; 0 = max_requests * ceil(max_seq_len/page_size) */
  uint64_t weight_seed;    /* synthetic weights: counter hash of (seed, tensor, index)         */
  int32_t debug_taps;      /* 1 = reserve per-layer tap buffers for focus_debug_export         */
  float logit_scale;       /* synthetic LM-head scale: W_lm = logit_scale * (recipe weights), so
                              z = logit_scale * z_1 exactly.  A power of two in [2^-16, 2^16]
                              (keeps W_lm exact in bf16); 0 means 1.  Sets the confidence regime
                              of random weights: at 1 the max softmax probability over V = 151936
                              stays far below tau (one fallback decode per step);
                              larger scales make conf >= tau fire for several
                              positions per step ("calibrated" run).  FOCUS_ERR_CONFIG otherwise. */
  int32_t batch_invariant; /* 1 = a request's results never depend on which other requests share
                              its steps (S:444 batch invariance, bit for bit): turns off the
                              attention's load-balancing tail split, whose cut units merge two
                              partial softmaxes (equal up to fp32 rounding).  Set it when requests
                              are sharded across GPUs and per-request outputs must be identical at
                              every world size.  0 = fastest (default).        */
  /* Mixture-of-Experts FFN (LLaDA2.0-mini-shaped workload; readings A-M5, A-M6): with
     n_experts > 0 the layers l >= n_dense_layers replace the dense SwiGLU by a router (top_k of
     n_experts by logit, softmax over the selected logits), n_experts routed SwiGLU experts of width
     d_expert and n_shared_experts shared ones; run on the compacted rows like every layer.
     n_experts <= 1024, 1 <= top_k <= min(16, n_experts), d_expert % 128 == 0; 0 = dense model. */
  int32_t n_experts, top_k, d_expert, n_shared_experts, n_dense_layers;
} focus_config;

typedef struct focus_ctx focus_ctx;

/* Per-request result of one focus_commit (host, pinned recommended). */
typedef struct {
  int32_t req_id;
  int32_t n_new;           /* tokens unmasked this step (0 on a flush step)                    */
  int32_t block_done;      /* the block committed completely this step                         */
  int32_t finished;        /* all gen_len tokens committed                                     */
  int32_t n_committed;     /* KV positions committed this step (DC+ rule)                      */
  int32_t pos[64];         /* block positions decoded this step, ascending                    */
  int32_t tok[64];         /* their token ids                                                  */
} focus_commit_result;

/* Bytes of device memory the arena must provide for `cfg` (0 if cfg is invalid). */
size_t focus_required_bytes(const focus_config* cfg);

/* Validate cfg, carve the arena (caller-owned device pointer, >= focus_required_bytes), generate
 * the synthetic bf16 weights on `cuda_stream` (a cudaStream_t; NULL = legacy default stream).
 * Returns FOCUS_ERR_CONFIG / FOCUS_ERR_NOMEM / FOCUS_ERR_CUDA on failure; *out is untouched then. */
focus_status focus_init(const focus_config* cfg, void* dev_arena, size_t arena_bytes,
                        void* cuda_stream, focus_ctx** out);
focus_status focus_destroy(focus_ctx* ctx);

/* New request in slot req_id: allocate its KV pages, run the causal prefill over the prompt at
 * every layer (exact AR-style KV; reading A-K5) and open block 0 (all masked, R = -1).
 * prompt_tokens_host: n_tokens ids in [0, vocab-1).  gen_len: multiple of block_size.
 * FOCUS_ERR_STATE if the slot is in use; FOCUS_ERR_NOMEM if the page pool is exhausted. */
focus_status focus_kv_append(focus_ctx* ctx, int32_t req_id, const int32_t* prompt_tokens_host,
                             int32_t n_tokens, int32_t gen_len);

/* One FOCUS step (Alg.1 lines 3-19: layer 0, layer-1 projections, importance delta, budget,
 * selection, compaction, remaining layers on the survivors, logits + confidences) for each listed
 * request.  Finished requests in the list are skipped (no rows).  Must be followed by focus_commit
 * with the identical list before the next step (FOCUS_ERR_STATE otherwise): the budget's N_bar and
 * the DC+ state are strictly per step. */
focus_status focus_step_block(focus_ctx* ctx, const int32_t* req_ids_host, int32_t n_req);

/* Decode_and_Verify + statistics + Neighbor-Aware KV commit + block advance (Alg.1 lines 18-22,
 * App.E) for the requests of the preceding focus_step_block.  If pinned_out is non-NULL
 * it receives n_req results (async; valid after focus_sync). */
focus_status focus_commit(focus_ctx* ctx, const int32_t* req_ids_host, int32_t n_req,
                          focus_commit_result* pinned_out);

/* Stream synchronisation; surfaces the device invariant flag and CUDA errors. */
focus_status focus_sync(focus_ctx* ctx);

/* Committed generated tokens of a request (synchronous).  *n_out = number written (<= cap). */
focus_status focus_get_tokens(focus_ctx* ctx, int32_t req_id, int32_t* out_host, int32_t cap,
                              int32_t* n_out);

/* Release a request slot and its KV pages (synchronous w.r.t. the stream). */
focus_status focus_release(focus_ctx* ctx, int32_t req_id);

/* ---- parity taps (test infrastructure; synchronous) ------------------------------------- */
/* Select the layer whose intermediates the next focus_step_block copies into tap buffers
 * (needs cfg.debug_taps = 1); -1 disables. */
focus_status focus_set_tap(focus_ctx* ctx, int32_t layer);

enum {
  FOCUS_DBG_STATE = 1,      /* focus_req_state[max_requests]                                 */
  FOCUS_DBG_COUNTERS = 2,   /* int32[8] M_P, M_S, M_logit, invariant flag, rows per attention
                               chunk, chunks per request, 2 pad; then int64[4] cumulative since
                               focus_init: sum M_P, sum M_S, sum M_logit, steps               */
  FOCUS_DBG_ROWS_P = 3,     /* int32[M_P][4] (slot, j, abs pos, list index) of processed rows */
  FOCUS_DBG_ROWS_S = 4,     /* int32[M_S][4] retained rows                                   */
  FOCUS_DBG_ROWS_L = 5,     /* int32[M_logit][4] logit rows (S cap M)                        */
  FOCUS_DBG_I0 = 6,         /* float[n_req][n_kv_heads][B] per-kv-head partial importance    */
  FOCUS_DBG_I1 = 7,
  FOCUS_DBG_LOGITS = 8,     /* float[M_logit][vocab] (stored only when cfg.debug_taps = 1: the LM
                               head's epilogue otherwise emits just the per-row confidence
                               statistics, and the logits never reach HBM)                   */
  FOCUS_DBG_TOKCONF = 9,    /* struct {int32 tok; float conf;}[M_logit]                      */
  FOCUS_DBG_KV_K = 10,      /* bf16[s+B][n_kv_heads][head_dim] of (req_id, layer)            */
  FOCUS_DBG_KV_V = 11,
  FOCUS_DBG_TAP_X_IN = 20,  /* float[rows][d]   residual entering the tapped layer           */
  FOCUS_DBG_TAP_H = 21,     /* bf16[rows][d]    RMSNorm output fed to the QKV GEMM           */
  FOCUS_DBG_TAP_QKV = 22,   /* bf16[rows][(Hq+2Hkv)dh] q|k|v after RoPE                      */
  FOCUS_DBG_TAP_ATTN = 23,  /* bf16[rows][Hq dh] attention output                            */
  FOCUS_DBG_TAP_X_MID = 24, /* float[rows][d]   after O-projection + residual                */
  FOCUS_DBG_TAP_H2 = 25,    /* bf16[rows][d]    RMSNorm output fed to the gate/up GEMM       */
  FOCUS_DBG_TAP_ACT = 26,   /* bf16[rows][d_ff] silu(gate)*up                                */
  FOCUS_DBG_TAP_X_OUT = 27, /* float[rows][d]   layer output                                 */
  FOCUS_DBG_TAP_QS = 28,    /* bf16[M_S][Hq dh] compacted layer-1 queries (tap layer 1)      */
  FOCUS_DBG_HL = 29,        /* bf16[M_logit][d] final-norm rows fed to the LM head           */
  FOCUS_DBG_LAUNCHES = 30,  /* uint64: kernels launched by this context so far                */
  FOCUS_DBG_PROFILE = 31,   /* focus_prof_entry[FOCUS_PROF_KINDS] accumulated since the last
                               focus_set_profile(ctx, 1)                                       */
  FOCUS_DBG_ATTN_TRACE = 32, /* uint64[grid][8 roles][512]: clock64 event trace of the last
                               tensor-core attention launch of layer FOCUS_ATTN_TRACE_LAYER
                               (env var read at focus_init; empty otherwise)                   */
  FOCUS_DBG_MOE_SEL = 33,   /* int32[M_S][top_k]: experts selected for the rows of the last MoE
                               layer of the last step (selection order)                        */
  FOCUS_DBG_MOE_WT = 34,    /* float[M_S][top_k]: their routing weights                        */
  FOCUS_DBG_MOE_ROWS = 35,  /* int32[M_S * top_k] token row of each gathered (expert-contiguous)
                               row, then int32[n_experts + 1] expert offsets                   */
  FOCUS_DBG_MOE_Y = 36,     /* float[M_S * top_k][d] expert outputs of the gathered rows        */
  FOCUS_DBG_MOE_AG = 37     /* bf16[M_S * top_k][d] gathered expert inputs                      */
};

/* Per-kernel-kind device time measured with CUDA events on the context stream around every launch
 * while profiling is on (for the roofline report; adds event records between launches). */
enum {
  FOCUS_PROF_SETUP = 0, FOCUS_PROF_EMBED, FOCUS_PROF_RMSNORM, FOCUS_PROF_GEMM_QKV, FOCUS_PROF_ROPE_STORE /* RoPE: unfused store, or the per-row factor tables */,
  FOCUS_PROF_ATTN, FOCUS_PROF_IMPORTANCE, FOCUS_PROF_GEMM_O, FOCUS_PROF_GEMM_GU, FOCUS_PROF_SILU,
  FOCUS_PROF_GEMM_DOWN, FOCUS_PROF_SELECT, FOCUS_PROF_GATHER, FOCUS_PROF_GEMM_LM, FOCUS_PROF_VOCAB,
  FOCUS_PROF_COMMIT, FOCUS_PROF_MOE_ROUTE /* router GEMM, top-k, placement, gather */,
  FOCUS_PROF_MOE_EXPERTS /* grouped expert GEMMs + shared expert */, FOCUS_PROF_MOE_COMBINE, FOCUS_PROF_KINDS
};
typedef struct {
  int32_t kind, launches;
  float total_ms, max_ms;
} focus_prof_entry;

/* Enable (1) / disable (0) per-launch event timing; enabling resets the accumulators. */
focus_status focus_set_profile(focus_ctx* ctx, int32_t on);

/* Copy a debug view to host memory (synchronous).  *n_written = bytes copied. */
focus_status focus_debug_export(focus_ctx* ctx, int32_t what, int32_t req_id, int32_t layer,
                                void* dst_host, size_t cap, size_t* n_written);

/* Mirror of the device per-request state (FOCUS_DBG_STATE). */
typedef struct {
  int32_t active, finished;
  int32_t s;               /* block start = committed context length                          */
  int32_t b;               /* block index                                                     */
  int32_t gen_len, prompt_len;
  int32_t R;               /* rightmost processed position (App.E), -1 at block open    */
  int32_t t;               /* steps executed                                                  */
  int64_t token_sum, total_steps;   /* App.E                                        */
  uint64_t committed;      /* bit j: KV of block position j committed                         */
  uint64_t masked;         /* bit j: position j still masked                                  */
  uint64_t P, M, S;        /* last step: processed / masked / retained sets                   */
  int32_t R_new, K, n_sigma, k_hist;
  int32_t flush, n_new, n_committed, pad_;
  int32_t tok[64];         /* block tokens (mask id where masked)                             */
  int32_t dstep[64];       /* step at which decoded, INT32_MAX while masked                   */
} focus_req_state;

const char* focus_status_str(focus_status s);

#ifdef __cplusplus
}
#endif
#endif /* FOCUS_H_ */
