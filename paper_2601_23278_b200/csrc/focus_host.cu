// libfocus host orchestration: config validation, arena carving, synthetic weights, page
// allocator, the per-step kernel sequence and the C ABI of include/focus.h.
//
// The step (focus_step_block) is a fixed sequence of stream-ordered launches with no host sync and
// no device->host copy; ragged sizes (M_P, M_S, M_logit) live in device counters and every kernel
// reads them, so grids are sized by host-known upper bounds (n_req * B).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <new>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "common.cuh"

using namespace focus;

namespace {
// NVTX phase ranges: host-side markers around the step's phases, visible in Nsight
// Systems / ncu --nvtx (header-only NVTX v3; no-ops without an attached tool)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

namespace focus {
void launch_gemm_simt(const bf16* A, int lda, const bf16* W, int N, int K, float* C, int ldc, const int* M_dev,
                      int M_max, GemmMode mode, cudaStream_t s);
bool launch_gemm_tc(const bf16* A, int lda, int a_rows, const bf16* W, int N, int K, float* C, int ldc,
                    const int* M_dev, int M_max, GemmMode mode, const GemmWs& ws, cudaStream_t s,
                    const GemmEpi* epi = nullptr, int m_est = 0);

void launch_gemm(const bf16* A, int lda, int a_rows, const bf16* W, int N, int K, float* C, int ldc, const int* M_dev,
                 int M_max, GemmMode mode, const GemmWs& ws, cudaStream_t s, int m_est) {
  if (gemm_backend() == 1 && launch_gemm_tc(A, lda, a_rows, W, N, K, C, ldc, M_dev, M_max, mode, ws, s, nullptr, m_est))
    return;
  launch_gemm_simt(A, lda, W, N, K, C, ldc, M_dev, M_max, mode, s);
}
}  // namespace focus

namespace {

constexpr int kTapCount = 10;
constexpr size_t kMaxGraphs = 32;    // whole-step graphs kept (least recently used evicted)
enum { TAP_X_IN = 0, TAP_H, TAP_QKV, TAP_ATTN, TAP_X_MID, TAP_H2, TAP_ACT, TAP_X_OUT, TAP_QS, TAP_ROWS };

struct Upload {                 // pinned staging ring for small host->device copies
  char* host = nullptr;
  size_t cap = 0, head = 0;
  static constexpr int kSlots = 16;
  cudaEvent_t ev[kSlots];
  size_t slot_end[kSlots];
  int next = 0;
};

int weight_exp(int fan_in) {
  return -(int)std::ceil(std::log2(255.0 * std::sqrt((double)fan_in / 3.0)));
}

bool is_moe(const focus_config& c, int layer) { return c.n_experts > 0 && layer >= c.n_dense_layers; }

// synth/gen.py expert_tid: routed expert e of layer l, kind 0 gate / 1 up / 2 down
uint64_t expert_tid(int layer, int kind, int e) { return (1ull << 20) + ((uint64_t)(3 * layer + kind) << 12) + e; }

}  // namespace

struct focus_ctx {
  focus_config cfg;
  cudaStream_t stream;
  char* arena = nullptr;
  size_t arena_bytes = 0;
  // geometry
  int B, G, qkv_dim, q_dim, max_rows, max_pages_per_req, n_chunks, nch_vocab, mask_id, max_gen;
  size_t kv_layer_elems;
  int64_t kv_pages;
  // attention path: tcgen05 kernel (head_dim 64/128) or the SIMT kernel (other head dims)
  bool attn_tc = false;
  int attn_rpc = 0, split_tiles = 8, max_nsplit = 1;
  CUtensorMap mapK, mapV, mapQ_qkv, mapQ_qs;
  float* attn_part = nullptr;
  float* attn_scratch = nullptr;
  unsigned long long* attn_trace = nullptr;
  void* plan_units[4] = {};       // per-step attention unit tables: layer 0, layer-1 importance,
  int* plan_n[4] = {};            // layer-1 suffix, layers >= 2
  int trace_layer = -1;
  int pf_tiles = 0, pf_grid = 0;  // QKV-GEMM L2 prefetch of the attention's first K/V tiles (per CTA)
  int* attn_sem = nullptr;
  // weights
  bf16* E = nullptr;
  bf16* Wlm = nullptr;
  std::vector<bf16*> Wqkv, Wo, Wgu, Wd;
  // MoE layers (A-M5): router [E][d], routed experts gate/up [E][2 de][d] (interleaved by 128 rows per
  // expert) and down [E][d][de], shared experts gate/up [2 ns de][d] and down [d][ns de]
  std::vector<bf16*> Wr, Wxgu, Wxd, Wsgu, Wsd;
  int* moe_sel = nullptr;          // [rows][top_k] selected experts (selection order)
  float* moe_wt = nullptr;         // [rows][top_k] routing weights
  int* moe_cnt = nullptr;          // [E] tokens per expert
  int* moe_off = nullptr;          // [E + 1] expert offsets into the gathered rows
  int* moe_tok = nullptr;          // [rows * top_k] gathered row -> token row
  int* moe_slot = nullptr;         // [rows][top_k] token row, k -> gathered row
  bf16* moe_Ag = nullptr;          // [rows * top_k + 64][d] gathered expert inputs
  bf16* moe_act = nullptr;         // [rows * top_k + 64][de] expert SwiGLU activations
  float* moe_y = nullptr;          // [rows * top_k][d] expert outputs
  // KV pool
  bf16* Kpool = nullptr;
  bf16* Vpool = nullptr;
  float* rope_cos = nullptr;
  float* rope_sin = nullptr;
  float* ropeT_P = nullptr;     // per-row RoPE factors of the P rows / S rows ([128][max_rows])
  float* ropeT_S = nullptr;
  int* page_table = nullptr;
  focus_req_state* st = nullptr;
  int* out_tokens = nullptr;
  // workspace
  float *x = nullptr, *x2 = nullptr, *f32tmp = nullptr, *logits = nullptr;
  bf16 *h = nullptr, *qkv = nullptr, *qS = nullptr, *attn = nullptr, *act = nullptr;
  RowInfo *rowP = nullptr, *rowS = nullptr, *rowL = nullptr;
  int *offP = nullptr, *offS = nullptr, *offL = nullptr, *srcP = nullptr, *srcL = nullptr, *tokP = nullptr;
  int* req_dev = nullptr;
  Counters* cnt = nullptr;
  float *I0p = nullptr, *I1p = nullptr;
  VocabPartial* vpart = nullptr;
  focus_status sticky = FOCUS_OK;  // launch-time failure reported by the next focus_sync
  VocabPartial* vtiles = nullptr;  // LM-head epilogue partials [logit row][64-column group]
  bool vocab_fused = false;        // LM head emits vtiles (tensor-core GEMM); logits stored only with taps
  TokConf* tokconf = nullptr;
  focus_commit_result* res_dev = nullptr;
  GemmWs gws{};
  // pinned 2-slot ring of the device counters: step n copies its counters into slot n % 2 (after the
  // step, outside any graph) and records cnt_ev[n % 2]; step n + 2 waits for that event and uses them
  // as its tile-shape estimates.  The estimate of every step is thus a deterministic function of the
  // computation (never of how far the host runs ahead), and the host stays at most ~2 steps ahead.
  Counters* cnt_host = nullptr;
  cudaEvent_t cnt_ev[2] = {};
  bool cnt_valid[2] = {false, false};
  uint64_t step_no = 0;
  Counters est{};                 // this step's estimate (set by focus_step_block)
  void* taps[kTapCount] = {};
  size_t tap_bytes[kTapCount] = {};
  // host state
  std::vector<int> slot_used;                 // 0 free, 1 allocated
  std::vector<std::vector<int>> slot_pages;
  std::vector<int> free_pages;
  std::vector<int> last_list, pending_list;
  bool step_pending = false;
  int last_n_req = 0;
  int tap_layer = -1;
  Upload up;
  // launch accounting / profiling
  uint64_t launches = 0;
  bool prof_on = false;
  std::vector<cudaEvent_t> prof_events;
  size_t prof_used = 0;
  std::vector<int> prof_kind;                    // per record
  focus_prof_entry prof_acc[FOCUS_PROF_KINDS];
  // whole-step CUDA graphs: the launch sequence of focus_step_block for one request
  // list and one set of GEMM tile configurations, captured once and replayed
  struct StepGraph {
    std::vector<int32_t> list;
    std::vector<int> key;           // tile configurations of the step's GEMMs (shape_key)
    cudaGraphExec_t exec = nullptr;
    int32_t* list_host = nullptr;   // pinned copy of the list: the captured H2D copy reads it
    uint64_t launches = 0;
    uint64_t last_use = 0;
  };
  std::vector<StepGraph> graphs;
  uint64_t graph_clock = 0;
  const int32_t* upload_src = nullptr;   // graph capture: the request list's pinned source
  cudaStream_t cap_stream = nullptr;      // capture stream (the context stream may be the legacy one)
};

namespace {

focus_status cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return FOCUS_OK;
  std::fprintf(stderr, "[focus] CUDA error: %s\n", cudaGetErrorString(e));
  return FOCUS_ERR_CUDA;
}

bool valid_config(const focus_config& c) {
  if (c.n_layers < 2 || c.d_model <= 0 || c.d_model % 64 || c.d_model > 8192) return false;   // rmsnorm: row in registers
  if (c.n_q_heads <= 0 || c.n_kv_heads <= 0 || c.n_q_heads % c.n_kv_heads) return false;
  if (!(c.head_dim == 16 || c.head_dim == 32 || c.head_dim == 64 || c.head_dim == 128)) return false;
  if (c.d_ff <= 0 || c.d_ff % kGuGroup) return false;
  if (c.vocab < 2) return false;
  if (c.block_size < 1 || c.block_size > kMaxB) return false;
  if (c.alpha_den <= 0 || c.alpha_num <= c.alpha_den) return false;       // alpha > 1
  if (!(c.conf_threshold > 0.f && c.conf_threshold <= 1.f)) return false;
  if (c.maxpool_kernel < 1 || c.maxpool_kernel % 2 == 0) return false;
  if (c.cache_mode < 0 || c.cache_mode > 2 || c.placeholder_mode < 0 || c.placeholder_mode > 1) return false;
  if (c.strategy < 0 || c.strategy > 4) return false;
  if (c.strategy >= FOCUS_STRATEGY_FIXED_TOP && c.fixed_k < 1) return false;
  if (c.max_requests < 1 || c.max_requests > 1024 || c.max_seq_len < 1 || c.page_size < 1) return false;
  if (c.max_prefill_chunk < 1) return false;
  const int G = c.n_q_heads / c.n_kv_heads;
  if (G > kAttnQRows) return false;
  if ((c.n_q_heads * c.head_dim) % 64) return false;
  if (c.batch_invariant < 0 || c.batch_invariant > 1) return false;
  if (c.n_experts < 0 || c.n_experts > 1024) return false;
  if (c.n_experts > 0) {
    if (c.top_k < 1 || c.top_k > 16 || c.top_k > c.n_experts) return false;
    if (c.d_expert <= 0 || c.d_expert % 128 || c.n_shared_experts < 0 || c.n_shared_experts > 8) return false;
    if (c.n_dense_layers < 0 || c.n_dense_layers > c.n_layers) return false;
  }
  if (c.logit_scale != 0.f) {                     // a power of two in [2^-16, 2^16] (W_lm stays exact)
    int e = 0;
    const float m = std::frexp(c.logit_scale, &e);
    if (!(m == 0.5f) || e < -15 || e > 17) return false;
  }
  return true;
}

// log2 of the LM-head scale (focus_config::logit_scale; 0 = 1)
int logit_scale_log2(const focus_config& c) {
  if (c.logit_scale == 0.f) return 0;
  int e = 0;
  std::frexp(c.logit_scale, &e);
  return e - 1;
}

// Carve (or, with base == nullptr, size) the arena.  Returns bytes used.
size_t carve(focus_ctx* x, char* base) {
  const focus_config& c = x->cfg;
  size_t off = 0;
  auto take = [&](size_t bytes) -> char* {
    off = (off + 255) & ~size_t(255);
    char* p = base ? base + off : nullptr;
    off += bytes;
    return p;
  };
  const size_t d = c.d_model, ff = c.d_ff, V = c.vocab;
  const size_t qkv = x->qkv_dim, qd = x->q_dim, L = c.n_layers;
  x->E = (bf16*)take(V * d * 2);
  x->Wlm = (bf16*)take(V * d * 2);
  x->Wqkv.assign(L, nullptr); x->Wo.assign(L, nullptr); x->Wgu.assign(L, nullptr); x->Wd.assign(L, nullptr);
  x->Wr.assign(L, nullptr); x->Wxgu.assign(L, nullptr); x->Wxd.assign(L, nullptr);
  x->Wsgu.assign(L, nullptr); x->Wsd.assign(L, nullptr);
  const size_t E = c.n_experts, de = c.d_expert, ns = c.n_shared_experts;
  for (size_t l = 0; l < L; ++l) {
    x->Wqkv[l] = (bf16*)take(qkv * d * 2);
    x->Wo[l] = (bf16*)take(d * qd * 2);
    if (is_moe(c, (int)l)) {
      x->Wr[l] = (bf16*)take(E * d * 2);
      x->Wxgu[l] = (bf16*)take(E * 2 * de * d * 2);
      x->Wxd[l] = (bf16*)take(E * d * de * 2);
      if (ns) {
        x->Wsgu[l] = (bf16*)take(2 * ns * de * d * 2);
        x->Wsd[l] = (bf16*)take(d * ns * de * 2);
      }
    } else {
      x->Wgu[l] = (bf16*)take(2 * ff * d * 2);
      x->Wd[l] = (bf16*)take(d * ff * 2);
    }
  }
  x->Kpool = (bf16*)take(L * x->kv_layer_elems * 2);
  x->Vpool = (bf16*)take(L * x->kv_layer_elems * 2);
  const size_t half = c.head_dim / 2;
  x->rope_cos = (float*)take((size_t)c.max_seq_len * half * 4);
  x->rope_sin = (float*)take((size_t)c.max_seq_len * half * 4);
  x->page_table = (int*)take((size_t)c.max_requests * x->max_pages_per_req * 4);
  x->st = (focus_req_state*)take((size_t)c.max_requests * sizeof(focus_req_state));
  x->out_tokens = (int*)take((size_t)c.max_requests * x->max_gen * 4);
  const size_t R = x->max_rows;
  x->x = (float*)take(R * d * 4);
  x->x2 = (float*)take(R * d * 4);
  x->f32tmp = (float*)take(R * std::max(qkv, 2 * ff) * 4);
  x->h = (bf16*)take(R * std::max(d, ff) * 2);
  x->qkv = (bf16*)take(R * qkv * 2);
  x->qS = (bf16*)take(R * qd * 2);
  x->attn = (bf16*)take(R * qd * 2);
  x->act = (bf16*)take(R * ff * 2);
  const size_t RL = (size_t)c.max_requests * x->B;   // logit rows <= retained masked rows
  x->logits = (float*)take(RL * V * 4);
  x->ropeT_P = (float*)take(R * 128 * 4);
  x->ropeT_S = (float*)take(R * 128 * 4);
  x->rowP = (RowInfo*)take(R * sizeof(RowInfo));
  x->rowS = (RowInfo*)take(R * sizeof(RowInfo));
  x->rowL = (RowInfo*)take(RL * sizeof(RowInfo));
  x->offP = (int*)take((c.max_requests + 1) * 4);
  x->offS = (int*)take((c.max_requests + 1) * 4);
  x->offL = (int*)take((c.max_requests + 1) * 4);
  x->srcP = (int*)take(R * 4);
  x->srcL = (int*)take(RL * 4);
  x->tokP = (int*)take(R * 4);
  x->req_dev = (int*)take(c.max_requests * 4);
  x->cnt = (Counters*)take(sizeof(Counters));
  const size_t nparts = (size_t)x->n_chunks * c.n_kv_heads;
  x->I0p = (float*)take(c.max_requests * nparts * x->B * 4);
  x->I1p = (float*)take(c.max_requests * nparts * x->B * 4);
  x->vpart = (VocabPartial*)take(RL * x->nch_vocab * sizeof(VocabPartial));
  x->vtiles = (VocabPartial*)take(RL * ((V + 63) / 64) * sizeof(VocabPartial));
  x->tokconf = (TokConf*)take(RL * sizeof(TokConf));
  x->res_dev = (focus_commit_result*)take(c.max_requests * sizeof(focus_commit_result));
  if (E) {
    const size_t RK = R * c.top_k;
    x->moe_sel = (int*)take(RK * 4);
    x->moe_wt = (float*)take(RK * 4);
    x->moe_cnt = (int*)take(E * 4);
    x->moe_off = (int*)take((E + 1) * 4);
    x->moe_tok = (int*)take(RK * 4);
    x->moe_slot = (int*)take(RK * 4);
    x->moe_Ag = (bf16*)take((RK + 64) * d * 2);
    x->moe_act = (bf16*)take((RK + 64) * de * 2);
    x->moe_y = (float*)take(RK * d * 4);
  }
  if (x->attn_tc) {
    const size_t pairs = (size_t)c.max_requests * x->n_chunks * c.n_kv_heads;
    x->attn_part = (float*)take(pairs * x->max_nsplit * ((size_t)128 * c.head_dim + 256) * 4);
    x->attn_sem = (int*)take(pairs * 4);
    x->attn_scratch = (float*)take((size_t)1024 * 128 * kMaxB * 4);   // >= grid (one CTA per SM)
    for (int k = 0; k < 4; ++k) {
      x->plan_units[k] = take((size_t)1024 * attn_tc_plan_capacity() * 80);
      x->plan_n[k] = (int*)take(1024 * 4);
    }
    const char* tl = getenv("FOCUS_ATTN_TRACE_LAYER");
    x->trace_layer = tl ? atoi(tl) : -1;
    if (x->trace_layer >= 0) x->attn_trace = (unsigned long long*)take((size_t)1024 * 8 * kTraceEv * 8);
  }
  x->gws.bytes = (size_t)64 << 20;
  x->gws.ptr = (float*)take(x->gws.bytes);
  x->gws.sem_count = kSwapSemBase + 4096;
  x->gws.no_swap = c.batch_invariant ? 1 : 0;
  x->gws.sem = (int*)take(x->gws.sem_count * 4);
  if (c.debug_taps) {
    const size_t sz[kTapCount] = {R * d * 4, R * d * 2, R * qkv * 2, R * qd * 2, R * d * 4,
                                  R * d * 2, R * ff * 2, R * d * 4, R * qd * 2, R * sizeof(RowInfo)};
    for (int t = 0; t < kTapCount; ++t) {
      x->taps[t] = take(sz[t]);
      x->tap_bytes[t] = sz[t];
    }
  }
  return off + 256;
}

void derive(focus_ctx* x) {
  const focus_config& c = x->cfg;
  x->B = c.block_size;
  x->G = c.n_q_heads / c.n_kv_heads;
  x->q_dim = c.n_q_heads * c.head_dim;
  x->qkv_dim = (c.n_q_heads + 2 * c.n_kv_heads) * c.head_dim;
  x->max_rows = std::max(c.max_requests * c.block_size, c.max_prefill_chunk);
  x->max_pages_per_req = (c.max_seq_len + c.page_size - 1) / c.page_size;
  const int64_t pages = c.kv_pages > 0 ? c.kv_pages : (int64_t)c.max_requests * x->max_pages_per_req;
  x->kv_pages = pages;
  x->kv_layer_elems = (size_t)pages * c.n_kv_heads * c.page_size * c.head_dim;
  // (the tensor-core kernel's importance epilogue unrolls MaxPool windows up to k = 5; wider windows take
  // the SIMT kernel)
  x->attn_tc = attn_tc_supported(c.head_dim, c.page_size, x->G) && c.maxpool_kernel <= 5 &&
               getenv("FOCUS_ATTN_SIMT") == nullptr;
  x->attn_rpc = x->attn_tc ? attn_tc_rows_per_chunk(x->G) : kAttnQRows / x->G;
  x->n_chunks = (x->B + x->attn_rpc - 1) / x->attn_rpc;
  x->split_tiles = 16;                         // 128-key tiles per split (the kernel may enlarge it)
  if (const char* e = getenv("FOCUS_ATTN_SPLIT_TILES")) x->split_tiles = std::max(2, atoi(e));
  x->max_nsplit = std::max(16, ((c.max_seq_len + 127) / 128 + x->split_tiles - 1) / x->split_tiles + 1);
  // LM head with the vocab-statistics epilogue (default on the tensor-core GEMM path; FOCUS_VOCAB_FUSED=0:
  // store the fp32 logits and reduce them in k_vocab_reduce)
  x->vocab_fused = gemm_backend() == 1 && !(getenv("FOCUS_VOCAB_FUSED") && getenv("FOCUS_VOCAB_FUSED")[0] == '0');
  x->nch_vocab = x->vocab_fused ? 1 : std::max(1, std::min(16, c.vocab / 8192));
  x->mask_id = c.vocab - 1;
  x->max_gen = c.max_seq_len;
}

KVView kv_view(focus_ctx* x, int layer) {
  KVView v;
  v.K = x->Kpool + (size_t)layer * x->kv_layer_elems;
  v.V = x->Vpool + (size_t)layer * x->kv_layer_elems;
  v.page_table = x->page_table;
  v.max_pages = x->max_pages_per_req;
  v.page_size = x->cfg.page_size;
  v.n_kv_heads = x->cfg.n_kv_heads;
  v.head_dim = x->cfg.head_dim;
  return v;
}

int prof_begin(focus_ctx* x) {
  if (!x->prof_on) return -1;
  if (x->prof_used + 2 > x->prof_events.size()) {
    for (int i = 0; i < 512; ++i) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      x->prof_events.push_back(e);
    }
  }
  const int e0 = (int)x->prof_used;
  x->prof_used += 2;
  cudaEventRecord(x->prof_events[e0], x->stream);
  return e0;
}

void prof_end(focus_ctx* x, int kind, int e0) {
  ++x->launches;
  if (e0 < 0) return;
  cudaEventRecord(x->prof_events[e0 + 1], x->stream);
  x->prof_kind.push_back(kind);
}

// Fold recorded event pairs into the per-kind accumulators (caller synchronised the stream).
void prof_collect(focus_ctx* x) {
  for (size_t r = 0; r < x->prof_kind.size(); ++r) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, x->prof_events[2 * r], x->prof_events[2 * r + 1]);
    focus_prof_entry& e = x->prof_acc[x->prof_kind[r]];
    e.launches += 1;
    e.total_ms += ms;
    e.max_ms = std::max(e.max_ms, ms);
  }
  x->prof_kind.clear();
  x->prof_used = 0;
}

#define LAUNCH(kind, call)                  \
  do {                                      \
    const int e0_ = prof_begin(x);          \
    call;                                   \
    prof_end(x, FOCUS_PROF_##kind, e0_);    \
  } while (0)

// Stage `bytes` of host data in the pinned ring and copy them to `dst` on the stream.
focus_status upload(focus_ctx* x, void* dst, const void* src, size_t bytes) {
  if (x->upload_src)   // graph capture: a memcpy node reading the graph's own pinned buffer
    return cuda_status(cudaMemcpyAsync(dst, x->upload_src, bytes, cudaMemcpyHostToDevice, x->stream));
  Upload& u = x->up;
  if (bytes > u.cap / Upload::kSlots) {           // large: synchronous copy
    return cuda_status(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, x->stream)) == FOCUS_OK
               ? cuda_status(cudaStreamSynchronize(x->stream)) : FOCUS_ERR_CUDA;
  }
  const int s = u.next;
  u.next = (u.next + 1) % Upload::kSlots;
  cudaEventSynchronize(u.ev[s]);                   // previous use of this slot finished
  char* h = u.host + (size_t)s * (u.cap / Upload::kSlots);
  std::memcpy(h, src, bytes);
  cudaError_t e = cudaMemcpyAsync(dst, h, bytes, cudaMemcpyHostToDevice, x->stream);
  cudaEventRecord(u.ev[s], x->stream);
  return cuda_status(e);
}

void tap(focus_ctx* x, int layer, int which, const void* src, size_t bytes) {
  if (!x->cfg.debug_taps || layer != x->tap_layer || !x->taps[which]) return;
  cudaMemcpyAsync(x->taps[which], src, std::min(bytes, x->tap_bytes[which]), cudaMemcpyDeviceToDevice, x->stream);
}

// ---------------------------------------------------------------- one transformer layer, pieces
struct RowSpace {             // the rows a layer piece runs on
  const int* M_dev;           // device row count (nullptr: M_host exact)
  int M_max;
  const RowInfo* rows;
  int M_est;                  // host estimate of the live count (last step's counter; tile-shape choice only)
  const float* ropeT;         // launch_rope_rows table of these rows (fused QKV epilogue)
  bool pf_attn = false;       // the following attention launch uses plan slot 3 (layers >= 2)
};

// fused QKV epilogue (tensor-core GEMM, head_dim 128) in use: it reads the per-row RoPE tables
bool fused_qkv(const focus_ctx* x) { return gemm_backend() == 1 && x->cfg.head_dim == 128; }

void qkv_piece(focus_ctx* x, int l, int tl, float* xr, const RowSpace& rs) {
  const focus_config& c = x->cfg;
  cudaStream_t s = x->stream;
  tap(x, tl, TAP_X_IN, xr, (size_t)rs.M_max * c.d_model * 4);
  LAUNCH(RMSNORM, launch_rmsnorm(xr, nullptr, rs.M_dev, rs.M_max, c.d_model, c.rms_eps, x->h, s));
  tap(x, tl, TAP_H, x->h, (size_t)rs.M_max * c.d_model * 2);
  // tensor-core GEMM with the RoPE + paged-KV-store epilogue (head_dim 128); otherwise GEMM -> fp32 ->
  // k_rope_store
  GemmEpi e{};
  e.out = x->qkv; e.ldo = x->qkv_dim; e.rows = rs.rows; e.ropeT = rs.ropeT; e.rope_ld = x->max_rows;
  e.st = x->st; e.kv = kv_view(x, l); e.n_q_heads = c.n_q_heads; e.cnt = x->cnt;
  if (rs.pf_attn && x->pf_tiles > 0) {         // layers >= 2: warm L2 with the attention's first K/V tiles
    e.pf_units = static_cast<const AttnUnit*>(x->plan_units[3]);
    e.pf_n = x->plan_n[3];
    e.pf_grid = x->pf_grid;
    e.pf_ucap = attn_tc_plan_capacity();
    e.pf_tiles = x->pf_tiles;
  }
  bool fused = false;
  LAUNCH(GEMM_QKV, fused = fused_qkv(x) &&
                           launch_gemm_tc(x->h, c.d_model, x->max_rows, x->Wqkv[l], x->qkv_dim, c.d_model, nullptr, 0,
                                          rs.M_dev, rs.M_max, GEMM_QKV_ROPE, x->gws, s, &e, rs.M_est));
  if (!fused) {
    --x->launches;                            // the fused attempt launched nothing
    LAUNCH(GEMM_QKV, launch_gemm(x->h, c.d_model, x->max_rows, x->Wqkv[l], x->qkv_dim, c.d_model, x->f32tmp,
                                 x->qkv_dim, rs.M_dev, rs.M_max, GEMM_STORE, x->gws, s, rs.M_est));
    LAUNCH(ROPE_STORE, launch_rope_store(x->f32tmp, rs.rows, rs.M_dev, rs.M_max, c.n_q_heads, x->rope_cos,
                                         x->rope_sin, x->st, kv_view(x, l), x->qkv, x->cnt, s));
  }
  tap(x, tl, TAP_QKV, x->qkv, (size_t)rs.M_max * x->qkv_dim * 2);
  tap(x, tl, TAP_ROWS, rs.rows, (size_t)rs.M_max * sizeof(RowInfo));
}

// MoE FFN of layer l on the rows `rs` (A-M5, A-M6): h = RMSNorm(x) is in x->h.  Router GEMM -> top-k
// routing -> expert-contiguous placement -> gathered rows -> grouped expert GEMMs (gate/up + SwiGLU,
// down) -> shared expert (x += shared(h)) -> x += sum_k w_k y_k (selection order).
void moe_piece(focus_ctx* x, int l, int tl, float* xr, const RowSpace& rs) {
  const focus_config& c = x->cfg;
  cudaStream_t s = x->stream;
  const int E = c.n_experts, K = c.top_k, d = c.d_model, de = c.d_expert;
  const int RK = x->max_rows * K;
  LAUNCH(MOE_ROUTE, {
    launch_gemm(x->h, d, x->max_rows, x->Wr[l], E, d, x->f32tmp, E, rs.M_dev, rs.M_max, GEMM_STORE, x->gws, s, rs.M_est);
    launch_moe_route(x->f32tmp, E, rs.M_dev, rs.M_max, E, K, x->moe_sel, x->moe_wt, x->moe_cnt, s);
    launch_moe_place(x->moe_sel, x->moe_cnt, rs.M_dev, rs.M_max, E, K, x->moe_off, x->moe_tok, x->moe_slot, s);
    launch_moe_gather(x->h, x->moe_tok, rs.M_dev, rs.M_max, K, d, x->moe_Ag, s);
  });
  x->launches += 3;                               // the group above launched 4 kernels
  bool ok = true;
  LAUNCH(MOE_EXPERTS, {
    GemmEpi e{};
    e.out = x->moe_act;
    e.ldo = de;
    ok = launch_gemm_grouped(x->moe_Ag, RK + 64, x->Wxgu[l], E, 2 * de, d, nullptr, 0, x->moe_off,
                             rs.M_max, GEMM_SWIGLU, &e, s) &&
         launch_gemm_grouped(x->moe_act, RK + 64, x->Wxd[l], E, d, de, x->moe_y, d, x->moe_off, rs.M_max,
                             GEMM_STORE, nullptr, s);
    if (c.n_shared_experts) {                     // shared experts: dense SwiGLU on every row, residual add
      GemmEpi es{};
      es.out = x->act;
      es.ldo = c.n_shared_experts * de;
      const int nsd = c.n_shared_experts * de;
      ok = ok && launch_gemm_tc(x->h, d, x->max_rows, x->Wsgu[l], 2 * nsd, d, nullptr, 0, rs.M_dev, rs.M_max,
                                GEMM_SWIGLU, x->gws, s, &es, rs.M_est);
      launch_gemm(x->act, nsd, x->max_rows, x->Wsd[l], d, nsd, xr, d, rs.M_dev, rs.M_max, GEMM_ADD, x->gws, s,
                  rs.M_est);
    }
  });
  x->launches += c.n_shared_experts ? 3 : 1;
  if (!ok) x->sticky = FOCUS_ERR_CUDA;
  tap(x, tl, TAP_ACT, x->moe_act, (size_t)rs.M_max * de * 2);
  LAUNCH(MOE_COMBINE, launch_moe_combine(x->moe_y, x->moe_slot, x->moe_wt, rs.M_dev, rs.M_max, K, d, xr, x->moe_cnt, E, s));
  tap(x, tl, TAP_X_OUT, xr, (size_t)rs.M_max * d * 4);
}

void out_mlp_piece(focus_ctx* x, int l, int tl, float* xr, const RowSpace& rs) {
  const focus_config& c = x->cfg;
  cudaStream_t s = x->stream;
  tap(x, tl, TAP_ATTN, x->attn, (size_t)rs.M_max * x->q_dim * 2);
  LAUNCH(GEMM_O, launch_gemm(x->attn, x->q_dim, x->max_rows, x->Wo[l], c.d_model, x->q_dim, xr, c.d_model,
                             rs.M_dev, rs.M_max, GEMM_ADD, x->gws, s, rs.M_est));
  tap(x, tl, TAP_X_MID, xr, (size_t)rs.M_max * c.d_model * 4);
  LAUNCH(RMSNORM, launch_rmsnorm(xr, nullptr, rs.M_dev, rs.M_max, c.d_model, c.rms_eps, x->h, s));
  tap(x, tl, TAP_H2, x->h, (size_t)rs.M_max * c.d_model * 2);
  if (is_moe(c, l)) {
    moe_piece(x, l, tl, xr, rs);
    return;
  }
  // tensor-core GEMM with the SwiGLU epilogue; otherwise GEMM -> fp32 -> k_silu_mul
  GemmEpi e{};
  e.out = x->act; e.ldo = c.d_ff;
  bool fused = false;
  LAUNCH(GEMM_GU, fused = gemm_backend() == 1 &&
                          launch_gemm_tc(x->h, c.d_model, x->max_rows, x->Wgu[l], 2 * c.d_ff, c.d_model, nullptr, 0,
                                         rs.M_dev, rs.M_max, GEMM_SWIGLU, x->gws, s, &e, rs.M_est));
  if (!fused) {
    --x->launches;
    LAUNCH(GEMM_GU, launch_gemm(x->h, c.d_model, x->max_rows, x->Wgu[l], 2 * c.d_ff, c.d_model, x->f32tmp,
                                2 * c.d_ff, rs.M_dev, rs.M_max, GEMM_STORE, x->gws, s, rs.M_est));
    LAUNCH(SILU, launch_silu_mul(x->f32tmp, rs.M_dev, rs.M_max, c.d_ff, x->act, s));
  }
  tap(x, tl, TAP_ACT, x->act, (size_t)rs.M_max * c.d_ff * 2);
  LAUNCH(GEMM_DOWN, launch_gemm(x->act, c.d_ff, x->max_rows, x->Wd[l], c.d_model, c.d_ff, xr, c.d_model, rs.M_dev,
                                rs.M_max, GEMM_ADD, x->gws, s, rs.M_est));
  tap(x, tl, TAP_X_OUT, xr, (size_t)rs.M_max * c.d_model * 4);
}

AttnArgs attn_args(focus_ctx* x, int l, const bf16* q, int ldq, int n_req, const int* row_off, int ext_mode) {
  AttnArgs a{};
  a.q = q;
  a.ldq = ldq;
  a.out = x->attn;
  a.ldo = x->q_dim;
  a.kv = kv_view(x, l);
  a.req_list = x->req_dev;
  a.row_off = row_off;
  a.st = x->st;
  a.n_req = n_req;
  a.B = x->B;
  a.n_q_heads = x->cfg.n_q_heads;
  a.ext_mode = ext_mode;
  a.n_chunks = x->n_chunks;
  a.mp_kernel = x->cfg.maxpool_kernel;
  a.scale = 1.0f / std::sqrt((float)x->cfg.head_dim);
  a.layer = l;
  a.kv_pages = x->kv_pages;
  a.split_tiles = x->split_tiles;
  a.max_nsplit = x->max_nsplit;
  a.part = x->attn_part;
  a.sem = x->attn_sem;
  a.stream_k = getenv("FOCUS_ATTN_SK") ? 1 : 0;   // opt-in stream-K (measured slower than the tail split)
  // tail split on by default (FOCUS_ATTN_TAIL=0: off): with the bulk-store epilogue and evict-first KV
  // loads it shortens the layer launch by ~10% (clock64 trace) and the C3 step by ~1.5%
  a.tail_split = (x->cfg.batch_invariant || (getenv("FOCUS_ATTN_TAIL") && getenv("FOCUS_ATTN_TAIL")[0] == '0')) ? 0 : 1;
  a.l2_prefetch = getenv("FOCUS_ATTN_PF") ? std::max(0, atoi(getenv("FOCUS_ATTN_PF"))) : 0;   // opt-in
  a.nch_fixed = getenv("FOCUS_ATTN_NCH4") ? 1 : 0;
  a.debug_check = getenv("FOCUS_ATTN_CHECK") ? 1 : 0;
  {
    const char* e = getenv("FOCUS_ATTN_RESCALE_LOG2");
    a.rescale_log2 = e ? std::max(0.0f, std::min(64.0f, (float)atof(e))) : 8.0f;
  }
  a.page_skip = (getenv("FOCUS_ATTN_PAGESKIP") && getenv("FOCUS_ATTN_PAGESKIP")[0] == '0') ? 0 : 1;
  a.kv_hint = (getenv("FOCUS_ATTN_L2HINT") && getenv("FOCUS_ATTN_L2HINT")[0] == '0') ? 0 : 1;
  a.imp_scratch = x->attn_scratch;
  static int pre_pf = -1;
  if (pre_pf < 0) {                              // FOCUS_ATTN_PRE_PF=n: first-unit tiles prefetched pre-wait
    const char* e = getenv("FOCUS_ATTN_PRE_PF");
    pre_pf = e ? std::max(0, atoi(e)) : 0;   // measured: 2 or 4 tiles slow the C3 attention by ~3-4 %
  }
  a.pre_pf_tiles = pre_pf;
  a.max_slots = x->cfg.max_requests;
  a.trace = (l == x->trace_layer && x->cfg.debug_taps >= 0) ? x->attn_trace : nullptr;
  return a;
}

// Precompute the unit table of an attention launch shape into plan slot k; on success the args point
// the kernel at it (otherwise the kernel builds its own table).
bool plan_attention(focus_ctx* x, AttnArgs& a, int k) {
  a.plan_units = x->plan_units[k];
  a.plan_n = x->plan_n[k];
  if (getenv("FOCUS_ATTN_NOPLAN") || !launch_attention_plan(a, x->stream)) {
    a.plan_units = nullptr;
    a.plan_n = nullptr;
    return false;
  }
  return true;
}

void run_attention(focus_ctx* x, const AttnArgs& a0) {
  AttnArgs a = a0;
  // debug: FOCUS_ATTN_TRACE_IMP=1 traces the layer's importance-only launch instead of its attention
  static const int trace_imp = getenv("FOCUS_ATTN_TRACE_IMP") ? 1 : 0;
  if (a.trace && trace_imp != a.imp_only) a.trace = nullptr;
  if (a.trace) cudaMemsetAsync(a.trace, 0, (size_t)num_sms() * 8 * kTraceEv * 8, x->stream);
  if (x->attn_tc) launch_attention_tc(x->mapK, x->mapV, a.q == x->qS ? x->mapQ_qs : x->mapQ_qkv, a, x->stream);
  else launch_attention(a, x->stream);
}

}  // namespace

// ======================================================================= C ABI
extern "C" {

const char* focus_status_str(focus_status s) {
  switch (s) {
    case FOCUS_OK: return "ok";
    case FOCUS_ERR_CONFIG: return "invalid configuration";
    case FOCUS_ERR_INVARIANT: return "device invariant violated";
    case FOCUS_ERR_IO: return "host buffer error";
    case FOCUS_ERR_NOMEM: return "out of memory (arena or KV pages)";
    case FOCUS_ERR_STATE: return "invalid request state";
    case FOCUS_ERR_CUDA: return "CUDA error";
  }
  return "unknown";
}

size_t focus_required_bytes(const focus_config* cfg) {
  if (!cfg || !valid_config(*cfg)) return 0;
  focus_ctx tmp;
  tmp.cfg = *cfg;
  derive(&tmp);
  return carve(&tmp, nullptr);
}

focus_status focus_init(const focus_config* cfg, void* dev_arena, size_t arena_bytes, void* cuda_stream,
                        focus_ctx** out) {
  if (!cfg || !out || !valid_config(*cfg)) return FOCUS_ERR_CONFIG;
  focus_ctx* x = new (std::nothrow) focus_ctx();
  if (!x) return FOCUS_ERR_NOMEM;
  x->cfg = *cfg;
  derive(x);
  const size_t need = carve(x, nullptr);
  if (!dev_arena || arena_bytes < need) { delete x; return FOCUS_ERR_NOMEM; }
  x->arena = (char*)dev_arena;
  x->arena_bytes = arena_bytes;
  carve(x, (char*)(((uintptr_t)dev_arena + 255) & ~uintptr_t(255)) - 0);
  x->stream = (cudaStream_t)cuda_stream;
  const focus_config& c = x->cfg;
  cudaStream_t s = x->stream;
  // pinned staging ring
  x->up.cap = Upload::kSlots * 65536;
  if (cudaMallocHost(&x->up.host, x->up.cap) != cudaSuccess) { delete x; return FOCUS_ERR_CUDA; }
  if (cudaMallocHost(&x->cnt_host, 2 * sizeof(Counters)) != cudaSuccess) { cudaFreeHost(x->up.host); delete x; return FOCUS_ERR_CUDA; }
  std::memset(x->cnt_host, 0, 2 * sizeof(Counters));
  for (int i = 0; i < 2; ++i) cudaEventCreateWithFlags(&x->cnt_ev[i], cudaEventDisableTiming);
  for (int i = 0; i < Upload::kSlots; ++i) {
    cudaEventCreateWithFlags(&x->up.ev[i], cudaEventDisableTiming);
    cudaEventRecord(x->up.ev[i], s);
  }
  // synthetic weights (synth/gen.py recipe; tensor ids: E=1, W_lm=2, layer l: 16(l+1)+kind)
  const uint64_t seed = c.weight_seed;
  const int d = c.d_model, ff = c.d_ff, qd = x->q_dim, kd = c.n_kv_heads * c.head_dim;
  launch_init_weights(x->E, c.vocab, d, 1, seed, weight_exp(d), 0, 0, s);
  launch_init_weights(x->Wlm, c.vocab, d, 2, seed, weight_exp(d) + logit_scale_log2(c), 0, 0, s);
  for (int l = 0; l < c.n_layers; ++l) {
    const uint64_t t0 = 16ull * (l + 1);
    launch_init_weights(x->Wqkv[l], qd, d, t0 + 0, seed, weight_exp(d), 0, 0, s);
    launch_init_weights(x->Wqkv[l] + (size_t)qd * d, kd, d, t0 + 1, seed, weight_exp(d), 0, 0, s);
    launch_init_weights(x->Wqkv[l] + (size_t)(qd + kd) * d, kd, d, t0 + 2, seed, weight_exp(d), 0, 0, s);
    launch_init_weights(x->Wo[l], d, qd, t0 + 3, seed, weight_exp(qd), 0, 0, s);
    if (is_moe(c, l)) {
      const int E = c.n_experts, de = c.d_expert, nsd = c.n_shared_experts * c.d_expert;
      launch_init_weights(x->Wr[l], E, d, t0 + 7, seed, weight_exp(d), 0, 0, s);
      for (int e = 0; e < E; ++e) {
        bf16* gu = x->Wxgu[l] + (size_t)e * 2 * de * d;
        launch_init_weights(gu, de, d, expert_tid(l, 0, e), seed, weight_exp(d), kGuGroup, 0, s);
        launch_init_weights(gu, de, d, expert_tid(l, 1, e), seed, weight_exp(d), kGuGroup, 1, s);
        launch_init_weights(x->Wxd[l] + (size_t)e * d * de, d, de, expert_tid(l, 2, e), seed, weight_exp(de), 0, 0, s);
      }
      if (nsd) {
        launch_init_weights(x->Wsgu[l], nsd, d, t0 + 8, seed, weight_exp(d), kGuGroup, 0, s);
        launch_init_weights(x->Wsgu[l], nsd, d, t0 + 9, seed, weight_exp(d), kGuGroup, 1, s);
        launch_init_weights(x->Wsd[l], d, nsd, t0 + 10, seed, weight_exp(nsd), 0, 0, s);
      }
    } else {
      launch_init_weights(x->Wgu[l], ff, d, t0 + 4, seed, weight_exp(d), kGuGroup, 0, s);
      launch_init_weights(x->Wgu[l], ff, d, t0 + 5, seed, weight_exp(d), kGuGroup, 1, s);
      launch_init_weights(x->Wd[l], d, ff, t0 + 6, seed, weight_exp(ff), 0, 0, s);
    }
  }
  // RoPE table in binary64 on the host (angle pos * theta^(-2k/dh), rotate-half pairs)
  {
    const int half = c.head_dim / 2;
    std::vector<float> cs((size_t)c.max_seq_len * half), sn(cs.size());
    for (int p = 0; p < c.max_seq_len; ++p)
      for (int k = 0; k < half; ++k) {
        const double ang = (double)p * std::pow((double)c.rope_theta, -2.0 * k / c.head_dim);
        cs[(size_t)p * half + k] = (float)std::cos(ang);
        sn[(size_t)p * half + k] = (float)std::sin(ang);
      }
    cudaMemcpyAsync(x->rope_cos, cs.data(), cs.size() * 4, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(x->rope_sin, sn.data(), sn.size() * 4, cudaMemcpyHostToDevice, s);
    cudaStreamSynchronize(s);
  }
  cudaMemsetAsync(x->st, 0, (size_t)c.max_requests * sizeof(focus_req_state), s);
  {
    Counters c0{};
    c0.attn_rpc = x->attn_rpc;
    c0.n_chunks = x->n_chunks;
    cudaMemcpyAsync(x->cnt, &c0, sizeof(c0), cudaMemcpyHostToDevice, s);
  }
  // KV pool zeroed once: key tiles past a request's written slots read finite zeros (P * V = 0)
  cudaMemsetAsync(x->Kpool, 0, (size_t)c.n_layers * x->kv_layer_elems * 2, s);
  cudaMemsetAsync(x->Vpool, 0, (size_t)c.n_layers * x->kv_layer_elems * 2, s);
  if (x->attn_tc) {
    cudaMemsetAsync(x->attn_sem, 0, (size_t)c.max_requests * x->n_chunks * c.n_kv_heads * 4, s);
    const size_t rows = (size_t)c.n_layers * x->kv_pages * c.n_kv_heads * c.page_size;
    if (!attn_tc_make_maps(x->Kpool, x->Vpool, rows, c.head_dim, c.page_size, &x->mapK, &x->mapV) ||
        !attn_tc_make_qmap(x->qkv, x->max_rows, x->qkv_dim, c.n_q_heads, x->G, &x->mapQ_qkv) ||
        !attn_tc_make_qmap(x->qS, x->max_rows, x->q_dim, c.n_q_heads, x->G, &x->mapQ_qs)) {
      cudaStreamSynchronize(s);
      cudaFreeHost(x->up.host);
      delete x;
      return FOCUS_ERR_CUDA;
    }
  }
  cudaMemsetAsync(x->gws.sem, 0, x->gws.sem_count * 4, s);
  if (x->moe_cnt) cudaMemsetAsync(x->moe_cnt, 0, (size_t)c.n_experts * 4, s);
  cudaMemsetAsync(x->page_table, 0, (size_t)c.max_requests * x->max_pages_per_req * 4, s);
  cudaMemsetAsync(x->out_tokens, 0, (size_t)c.max_requests * x->max_gen * 4, s);
  for (int k = 0; k < FOCUS_PROF_KINDS; ++k) x->prof_acc[k] = focus_prof_entry{k, 0, 0.f, 0.f};
  x->slot_used.assign(c.max_requests, 0);
  x->slot_pages.assign(c.max_requests, {});
  const int64_t pages = x->kv_layer_elems / ((size_t)c.n_kv_heads * c.page_size * c.head_dim);
  x->free_pages.reserve(pages);
  for (int64_t p = pages - 1; p >= 0; --p) x->free_pages.push_back((int)p);
  focus_status st = cuda_status(cudaStreamSynchronize(s));
  if (st != FOCUS_OK) {
    cudaFreeHost(x->up.host);
    delete x;
    return st;
  }
  *out = x;
  return FOCUS_OK;
}

focus_status focus_destroy(focus_ctx* x) {
  if (!x) return FOCUS_ERR_STATE;
  cudaStreamSynchronize(x->stream);
  for (int i = 0; i < Upload::kSlots; ++i) cudaEventDestroy(x->up.ev[i]);
  for (cudaEvent_t e : x->prof_events) cudaEventDestroy(e);
  for (int i = 0; i < 2; ++i) cudaEventDestroy(x->cnt_ev[i]);
  for (auto& g : x->graphs) {
    cudaGraphExecDestroy(g.exec);
    cudaFreeHost(g.list_host);
  }
  if (x->cap_stream) cudaStreamDestroy(x->cap_stream);
  cudaFreeHost(x->up.host);
  cudaFreeHost(x->cnt_host);
  delete x;
  return FOCUS_OK;
}

focus_status focus_kv_append(focus_ctx* x, int32_t req_id, const int32_t* prompt, int32_t n_tokens, int32_t gen_len) {
  if (!x) return FOCUS_ERR_STATE;
  NvtxRange nv("focus_kv_append (prefill)");
  const focus_config& c = x->cfg;
  if (x->step_pending) return FOCUS_ERR_STATE;
  if (req_id < 0 || req_id >= c.max_requests || x->slot_used[req_id]) return FOCUS_ERR_STATE;
  if (!prompt || n_tokens < 1 || gen_len < x->B || gen_len % x->B) return FOCUS_ERR_CONFIG;
  if (n_tokens + gen_len > c.max_seq_len) return FOCUS_ERR_NOMEM;
  for (int i = 0; i < n_tokens; ++i)
    if (prompt[i] < 0 || prompt[i] >= c.vocab - 1) return FOCUS_ERR_CONFIG;
  const int np = (n_tokens + gen_len + c.page_size - 1) / c.page_size;
  if ((int)x->free_pages.size() < np) return FOCUS_ERR_NOMEM;
  std::vector<int> pt(x->max_pages_per_req, 0);
  for (int i = 0; i < np; ++i) {
    pt[i] = x->free_pages.back();
    x->free_pages.pop_back();
    x->slot_pages[req_id].push_back(pt[i]);
  }
  x->slot_used[req_id] = 1;
  cudaStream_t s = x->stream;
  focus_status rc = upload(x, x->page_table + (size_t)req_id * x->max_pages_per_req, pt.data(), pt.size() * 4);
  if (rc != FOCUS_OK) return rc;
  // state: prefill is in progress (not active for steps yet)
  focus_req_state st{};
  st.active = 0;
  st.s = n_tokens;
  st.gen_len = gen_len;
  st.prompt_len = n_tokens;
  st.R = -1;
  st.masked = full_mask(x->B);
  for (int j = 0; j < kMaxB; ++j) { st.tok[j] = x->mask_id; st.dstep[j] = 0x7fffffff; }
  rc = upload(x, x->st + req_id, &st, sizeof(st));
  if (rc != FOCUS_OK) return rc;
  // causal prefill in chunks
  std::vector<RowInfo> rows;
  for (int c0 = 0; c0 < n_tokens; c0 += c.max_prefill_chunk) {
    const int n = std::min(c.max_prefill_chunk, n_tokens - c0);
    rows.resize(n);
    for (int i = 0; i < n; ++i) rows[i] = RowInfo{req_id, -1, c0 + i, 0};
    if ((rc = upload(x, x->tokP, prompt + c0, (size_t)n * 4)) != FOCUS_OK) return rc;
    if ((rc = upload(x, x->rowP, rows.data(), (size_t)n * sizeof(RowInfo))) != FOCUS_OK) return rc;
    LAUNCH(EMBED, launch_embed(x->tokP, nullptr, n, x->E, c.d_model, x->x, s));
    RowSpace rs{nullptr, n, x->rowP, n, x->ropeT_P};
    if (fused_qkv(x))
      LAUNCH(ROPE_STORE, launch_rope_rows(x->rowP, nullptr, n, x->rope_cos, x->rope_sin, x->ropeT_P, x->max_rows, s));
    for (int l = 0; l < c.n_layers; ++l) {
      qkv_piece(x, l, -1000, x->x, rs);
      AttnArgs a = attn_args(x, l, x->qkv, x->qkv_dim, 0, nullptr, 2);
      a.prefill_slot = req_id;
      a.prefill_pos0 = c0;
      a.prefill_rows = n;
      LAUNCH(ATTN, run_attention(x, a));
      out_mlp_piece(x, l, -1000, x->x, rs);
    }
  }
  // activate: the request takes part in steps from now on
  st.active = 1;
  rc = upload(x, x->st + req_id, &st, sizeof(st));
  if (rc != FOCUS_OK) return rc;
  return cuda_status(cudaStreamSynchronize(s));
}

focus_status focus_release(focus_ctx* x, int32_t req_id) {
  if (!x) return FOCUS_ERR_STATE;
  if (x->step_pending) return FOCUS_ERR_STATE;
  if (req_id < 0 || req_id >= x->cfg.max_requests || !x->slot_used[req_id]) return FOCUS_ERR_STATE;
  focus_status rc = cuda_status(cudaStreamSynchronize(x->stream));
  if (rc != FOCUS_OK) return rc;
  for (int p : x->slot_pages[req_id]) x->free_pages.push_back(p);
  x->slot_pages[req_id].clear();
  x->slot_used[req_id] = 0;
  focus_req_state st{};
  rc = upload(x, x->st + req_id, &st, sizeof(st));
  if (rc != FOCUS_OK) return rc;
  x->last_list.clear();
  return cuda_status(cudaStreamSynchronize(x->stream));
}

static focus_status check_list(focus_ctx* x, const int32_t* ids, int32_t n) {
  if (n < 0 || n > x->cfg.max_requests || (n > 0 && !ids)) return FOCUS_ERR_STATE;
  std::vector<char> seen(x->cfg.max_requests, 0);
  for (int i = 0; i < n; ++i) {
    const int r = ids[i];
    if (r < 0 || r >= x->cfg.max_requests || !x->slot_used[r] || seen[r]) return FOCUS_ERR_STATE;
    seen[r] = 1;
  }
  return FOCUS_OK;
}

static focus_status enqueue_step(focus_ctx* x, const int32_t* ids, int32_t n_req);
static focus_status step_graph(focus_ctx* x, const int32_t* ids, int32_t n_req, bool same_list);

static bool graphs_enabled(const focus_ctx* x) {
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("FOCUS_GRAPH");
    env = (e && e[0] == '0') ? 0 : 1;
  }
  return env == 1 && !x->prof_on && x->cfg.debug_taps == 0 && x->trace_layer < 0;
}

focus_status focus_step_block(focus_ctx* x, const int32_t* ids, int32_t n_req) {
  if (!x) return FOCUS_ERR_STATE;
  NvtxRange nv("focus_step_block");
  if (x->step_pending) return FOCUS_ERR_STATE;
  focus_status rc = check_list(x, ids, n_req);
  if (rc != FOCUS_OK) return rc;
  const bool same_list = x->last_list.size() == (size_t)n_req && std::equal(ids, ids + n_req, x->last_list.begin());
  x->pending_list.assign(ids, ids + n_req);
  x->step_pending = true;
  if (n_req == 0) return FOCUS_OK;
  // tile-shape estimate: the live row counts of the step before the previous one (see cnt_ev), in
  // units of 256-row CTA-pair tiles -- the only granularity the GEMM launch shapes depend on
  const int maxP = n_req * x->B;
  {
    const int slot = (int)(x->step_no & 1);
    Counters e{};
    if (x->cnt_valid[slot]) {
      cudaEventSynchronize(x->cnt_ev[slot]);
      e = x->cnt_host[slot];
    }
    if (e.M_P <= 0 || e.M_P > maxP) { e.M_P = maxP; e.M_S = maxP; e.M_L = maxP; }
    e.M_S = std::min(std::max(e.M_S, 1), maxP);
    e.M_L = std::min(std::max(e.M_L, 1), maxP);
    x->est = e;
  }
  focus_status st = FOCUS_OK;
  if (x->prof_on) {   // profiled (eager) step: the device starts it only once the host has enqueued it
    static long long hold_us = -1;
    if (hold_us < 0) hold_us = getenv("FOCUS_PROF_HOLD_US") ? std::max(0, atoi(getenv("FOCUS_PROF_HOLD_US"))) : 30000;
    if (hold_us > 0) launch_hold(hold_us * 1000, x->stream);
  }
  if (!graphs_enabled(x)) st = enqueue_step(x, ids, n_req);
  else st = step_graph(x, ids, n_req, same_list);
  if (st != FOCUS_OK) return st;
  const int slot = (int)(x->step_no & 1);
  cudaMemcpyAsync(x->cnt_host + slot, x->cnt, sizeof(Counters), cudaMemcpyDeviceToHost, x->stream);
  cudaEventRecord(x->cnt_ev[slot], x->stream);
  x->cnt_valid[slot] = true;
  ++x->step_no;
  return cuda_status(cudaGetLastError());
}

// The launch choices a step bakes in: the tile configuration of every GEMM shape of the step at this
// step's row-count estimates (P rows: layers 0-1; S rows: layer-1 suffix and layers >= 2; logit rows).
static std::vector<int> shape_key(const focus_ctx* x, int maxP, const Counters& e) {
  const focus_config& c = x->cfg;
  std::vector<int> k;
  if (gemm_backend() != 1) return k;
  const GemmMode qm = fused_qkv(x) ? GEMM_QKV_ROPE : GEMM_STORE;
  for (int m : {e.M_P, e.M_S}) {
    k.push_back(gemm_tc_choice(x->qkv_dim, c.d_model, qm, maxP, m, !x->gws.no_swap));
    k.push_back(gemm_tc_choice(c.d_model, x->q_dim, GEMM_ADD, maxP, m, !x->gws.no_swap));
    k.push_back(gemm_tc_choice(2 * c.d_ff, c.d_model, GEMM_SWIGLU, maxP, m, !x->gws.no_swap));
    k.push_back(gemm_tc_choice(c.d_model, c.d_ff, GEMM_ADD, maxP, m, !x->gws.no_swap));
  }
  k.push_back(gemm_tc_choice(c.vocab, c.d_model, GEMM_STORE, maxP, e.M_L, !x->gws.no_swap));
  if (c.n_experts > 0) {                          // MoE: router and shared-expert GEMMs (S rows)
    const int nsd = c.n_shared_experts * c.d_expert;
    k.push_back(gemm_tc_choice(c.n_experts, c.d_model, GEMM_STORE, maxP, e.M_S, !x->gws.no_swap));
    if (nsd) {
      k.push_back(gemm_tc_choice(2 * nsd, c.d_model, GEMM_SWIGLU, maxP, e.M_S, !x->gws.no_swap));
      k.push_back(gemm_tc_choice(c.d_model, nsd, GEMM_ADD, maxP, e.M_S, !x->gws.no_swap));
    }
  }
  return k;
}

// Capture the step's launch sequence for the row-count estimate e into a new graph of the cache.
static focus_status capture_graph(focus_ctx* x, const int32_t* ids, int32_t n_req, const Counters& e,
                                  const std::vector<int>& key) {
  focus_status rc;
  focus_ctx::StepGraph g;
  g.list.assign(ids, ids + n_req);
  g.key = key;
  if (cudaMallocHost(&g.list_host, (size_t)n_req * 4) != cudaSuccess) return FOCUS_ERR_CUDA;
  std::memcpy(g.list_host, ids, (size_t)n_req * 4);
  cudaGraph_t graph = nullptr;
  const uint64_t l0 = x->launches;
  if (!x->cap_stream && cudaStreamCreateWithFlags(&x->cap_stream, cudaStreamNonBlocking) != cudaSuccess) {
    cudaFreeHost(g.list_host);
    return FOCUS_ERR_CUDA;
  }
  // capture on the private stream (capturing the legacy default stream is not allowed); the graph is
  // then launched on the context stream, so stream order is unchanged
  cudaStream_t user = x->stream;
  const Counters est_saved = x->est;
  const std::vector<int32_t> last_saved = x->last_list;
  x->est = e;
  x->stream = x->cap_stream;
  if ((rc = cuda_status(cudaStreamBeginCapture(x->stream, cudaStreamCaptureModeThreadLocal))) != FOCUS_OK) {
    x->stream = user;
    x->est = est_saved;
    cudaFreeHost(g.list_host);
    return rc;
  }
  x->upload_src = g.list_host;
  rc = enqueue_step(x, ids, n_req);
  x->upload_src = nullptr;
  const cudaError_t ec = cudaStreamEndCapture(x->stream, &graph);
  x->stream = user;
  x->est = est_saved;
  x->last_list = last_saved;
  if (rc == FOCUS_OK && ec == cudaSuccess) rc = cuda_status(cudaGraphInstantiate(&g.exec, graph, 0));
  else if (rc == FOCUS_OK) rc = cuda_status(ec);
  if (graph) cudaGraphDestroy(graph);
  g.launches = x->launches - l0;
  x->launches = l0;                               // capturing launches nothing
  if (rc != FOCUS_OK) {
    cudaFreeHost(g.list_host);
    return rc;
  }
  g.last_use = x->graph_clock;
  if (x->graphs.size() >= kMaxGraphs) {            // keep the most recently used
    auto lru = std::min_element(x->graphs.begin(), x->graphs.end(),
                                [](const focus_ctx::StepGraph& a, const focus_ctx::StepGraph& b) { return a.last_use < b.last_use; });
    cudaGraphExecDestroy(lru->exec);
    cudaFreeHost(lru->list_host);
    x->graphs.erase(lru);
  }
  x->graphs.push_back(g);
  return FOCUS_OK;
}

static focus_ctx::StepGraph* find_graph(focus_ctx* x, const int32_t* ids, int32_t n_req, const std::vector<int>* key) {
  for (auto& g : x->graphs) {
    if (g.list.size() != (size_t)n_req || !std::equal(ids, ids + n_req, g.list.begin())) continue;
    if (key == nullptr || g.key == *key) return &g;
  }
  return nullptr;
}

static focus_status step_graph(focus_ctx* x, const int32_t* ids, int32_t n_req, bool same_list) {
  // graph key: the request list and the GEMM tile configurations the launch sequence bakes in;
  // device-side row counts keep any replay exact
  const int maxP = n_req * x->B;
  const std::vector<int> key = shape_key(x, maxP, x->est);
  ++x->graph_clock;
  focus_ctx::StepGraph* g = find_graph(x, ids, n_req, &key);
  if (g == nullptr) {
    // capture only in a steady state (the same list as the previous step); otherwise launch eagerly
    if (!same_list) return enqueue_step(x, ids, n_req);
    focus_status rc;
    if (find_graph(x, ids, n_req, nullptr) == nullptr) {
      // first steady-state step of this list: capture every tile configuration its row counts can
      // select (estimates of 1 .. maxP/256 pair tiles per row space), so no capture lands in a
      // later step
      std::vector<std::vector<int>> seen;
      const int mp = (maxP + 255) / 256;
      for (int a = 1; a <= mp; ++a)
        for (int b = 1; b <= mp; ++b)
          for (int l = 1; l <= mp; ++l) {
            Counters e = x->est;
            e.M_P = std::min(a * 256, maxP);
            e.M_S = std::min(b * 256, maxP);
            e.M_L = std::min(l * 256, maxP);
            const std::vector<int> k = shape_key(x, maxP, e);
            if (std::find(seen.begin(), seen.end(), k) != seen.end() || seen.size() >= kMaxGraphs / 2) continue;
            seen.push_back(k);
            if ((rc = capture_graph(x, ids, n_req, e, k)) != FOCUS_OK) return rc;
          }
    }
    g = find_graph(x, ids, n_req, &key);
    if (g == nullptr) {
      if ((rc = capture_graph(x, ids, n_req, x->est, key)) != FOCUS_OK) return rc;
      g = &x->graphs.back();
    }
  }
  g->last_use = x->graph_clock;
  x->launches += g->launches;
  x->last_list = x->pending_list;
  return cuda_status(cudaGraphLaunch(g->exec, x->stream));
}

static focus_status enqueue_step(focus_ctx* x, const int32_t* ids, int32_t n_req) {
  focus_status rc;
  const focus_config& c = x->cfg;
  cudaStream_t s = x->stream;
  // the request list is uploaded every step (pinned staging, async): the step's host input
  if ((rc = upload(x, x->req_dev, ids, (size_t)n_req * 4)) != FOCUS_OK) return rc;
  x->last_list = x->pending_list;
  const int maxP = n_req * x->B;
  // A0 setup, A1 embedding
  nvtxRangePushA("A0-A1 setup, embedding");
  LAUNCH(SETUP, launch_step_setup(x->req_dev, n_req, x->st, x->B, x->rowP, x->offP, x->tokP, x->cnt, s));
  const int* MP = &x->cnt->M_P;
  const int* MS = &x->cnt->M_S;
  const int* ML = &x->cnt->M_L;
  LAUNCH(EMBED, launch_embed(x->tokP, MP, maxP, x->E, c.d_model, x->x, s));
  const Counters& est = x->est;   // tile-shape estimates (focus_step_block)
  RowSpace rsP{MP, maxP, x->rowP, est.M_P, x->ropeT_P};
  RowSpace rsS{MS, maxP, x->rowS, est.M_S, x->ropeT_S};
  if (fused_qkv(x))
    LAUNCH(ROPE_STORE, launch_rope_rows(x->rowP, MP, maxP, x->rope_cos, x->rope_sin, x->ropeT_P, x->max_rows, s));
  nvtxRangePop();
  nvtxRangePushA("A2-A3 layer 0, layer-1 prefix, importance");
  // A2 layer 0 fully on P (+ fused importance I0)
  // attention unit tables of the P-row launches (layer 0, layer-1 importance), once per step
  AttnArgs a0 = attn_args(x, 0, x->qkv, x->qkv_dim, n_req, x->offP, 0);
  a0.imp = x->I0p;
  AttnArgs a1 = attn_args(x, 1, x->qkv, x->qkv_dim, n_req, x->offP, 0);
  a1.imp = x->I1p;
  a1.imp_only = 1;
  a1.out = nullptr;
  if (x->attn_tc && plan_attention(x, a0, 0)) ++x->launches;
  // layer-1 importance (block keys only, O(B^2 H d_h) work): the persistent tensor-core kernel's
  // importance-only mode (default; 0.063 ms per C3 step) or, with FOCUS_IMP_TC=0, the CUDA-core kernel
  // (one CTA per (request, chunk, kv head); measured 0.124 ms)
  static int imp_tc = -1;
  if (imp_tc < 0) imp_tc = (getenv("FOCUS_IMP_TC") && getenv("FOCUS_IMP_TC")[0] == '0') ? 0 : 1;
  if (x->attn_tc && imp_tc && plan_attention(x, a1, 1)) ++x->launches;
  qkv_piece(x, 0, 0, x->x, rsP);
  LAUNCH(ATTN, run_attention(x, a0));
  out_mlp_piece(x, 0, 0, x->x, rsP);
  // A3 layer-1 projections on P, K1/V1 stored before eviction, importance-only I1
  qkv_piece(x, 1, 1, x->x, rsP);
  if (x->attn_tc && !imp_tc) LAUNCH(IMPORTANCE, launch_attention(a1, s));
  else LAUNCH(IMPORTANCE, run_attention(x, a1));
  nvtxRangePop();
  nvtxRangePushA("A4-A5 selection, compaction");
  // A4 selection + compaction plan, A5 gather
  {
    SelectArgs sa{};
    sa.req_list = x->req_dev;
    sa.n_req = n_req;
    sa.st = x->st;
    sa.I0p = x->I0p;
    sa.I1p = x->I1p;
    sa.n_chunks = x->n_chunks;
    sa.n_kv_heads = c.n_kv_heads;
    sa.attn_rpc = x->attn_rpc;
    sa.B = x->B;
    sa.alpha_num = c.alpha_num;
    sa.alpha_den = c.alpha_den;
    sa.placeholder_mode = c.placeholder_mode;
    sa.strategy = c.strategy;
    sa.fixed_k = c.fixed_k;
    sa.seed = c.weight_seed;
    sa.offP = x->offP;
    sa.rowS = x->rowS; sa.srcP = x->srcP; sa.offS = x->offS;
    sa.rowL = x->rowL; sa.srcL = x->srcL; sa.offL = x->offL;
    sa.cnt = x->cnt;
    LAUNCH(SELECT, launch_select_plan(sa, s));
  }
  if (fused_qkv(x) && c.n_layers > 1)
    LAUNCH(ROPE_STORE, launch_rope_rows(x->rowS, MS, maxP, x->rope_cos, x->rope_sin, x->ropeT_S, x->max_rows, s));
  LAUNCH(GATHER, launch_gather_rows(x->x, x->qkv, x->qkv_dim, x->q_dim, x->srcP, MS, maxP, c.d_model, x->x2, x->qS, s));
  tap(x, 1, TAP_QS, x->qS, (size_t)maxP * x->q_dim * 2);
  // attention unit tables of the S-row launches (layer-1 suffix, layers >= 2), once per step
  AttnArgs a2 = attn_args(x, 1, x->qS, x->q_dim, n_req, x->offS, 0);
  AttnArgs a3 = attn_args(x, 2, x->qkv, x->qkv_dim, n_req, x->offS, 1);
  if (x->attn_tc && plan_attention(x, a2, 2)) ++x->launches;
  x->pf_tiles = 0;
  if (x->attn_tc && c.n_layers > 2 && plan_attention(x, a3, 3)) {
    ++x->launches;
    static int pf_env = -1;
    if (pf_env < 0) {
      const char* e = getenv("FOCUS_ATTN_L2PF_TILES");
      pf_env = e ? std::max(0, atoi(e)) : 0;
    }
    x->pf_tiles = pf_env;
    x->pf_grid = attn_tc_grid(a3);
  }
  nvtxRangePop();
  nvtxRangePushA("A6-A7 layers 1-suffix .. L-1 on S");
  // A6 layer-1 suffix on S: keys = context + whole block
  LAUNCH(ATTN, run_attention(x, a2));
  out_mlp_piece(x, 1, 1, x->x2, rsS);
  // A7 layers 2.. on S: keys = context + block [0, R'] (same unit table for every layer)
  RowSpace rsS2 = rsS;
  rsS2.pf_attn = true;
  for (int l = 2; l < c.n_layers; ++l) {
    qkv_piece(x, l, l, x->x2, rsS2);
    AttnArgs a = a3;
    const AttnArgs al = attn_args(x, l, x->qkv, x->qkv_dim, n_req, x->offS, 1);
    a.kv = al.kv;
    a.layer = l;
    a.trace = al.trace;
    LAUNCH(ATTN, run_attention(x, a));
    out_mlp_piece(x, l, l, x->x2, rsS);
  }
  nvtxRangePop();
  nvtxRangePushA("A8 final norm, LM head, vocab statistics");
  // A8 final norm + LM head on S cap M, vocab reduction
  LAUNCH(RMSNORM, launch_rmsnorm(x->x2, x->srcL, ML, maxP, c.d_model, c.rms_eps, x->h, s));
  if (x->vocab_fused) {
    // the LM head's epilogue emits per-row vocab statistics per 64 columns; the fp32 logits reach HBM
    // only when debug taps are on (parity tests read them)
    GemmEpi e{};
    e.vpart = x->vtiles;
    e.vp_ld = (c.vocab + 63) / 64;
    e.mask_id = x->mask_id;
    bool ok = false;
    LAUNCH(GEMM_LM, ok = launch_gemm_tc(x->h, c.d_model, x->max_rows, x->Wlm, c.vocab, c.d_model,
                                        c.debug_taps ? x->logits : nullptr, c.vocab, ML, maxP, GEMM_STORE, x->gws,
                                        s, &e, est.M_L));
    if (!ok) { nvtxRangePop(); return FOCUS_ERR_CUDA; }
    LAUNCH(VOCAB, launch_vocab_combine(x->vtiles, e.vp_ld, ML, maxP, x->vpart, s));
  } else {
    LAUNCH(GEMM_LM, launch_gemm(x->h, c.d_model, x->max_rows, x->Wlm, c.vocab, c.d_model, x->logits, c.vocab, ML,
                                maxP, GEMM_STORE, x->gws, s, est.M_L));
    LAUNCH(VOCAB, launch_vocab_reduce(x->logits, ML, maxP, c.vocab, x->mask_id, x->nch_vocab, x->vpart, s));
  }
  nvtxRangePop();
  return cuda_status(cudaGetLastError());
}

focus_status focus_commit(focus_ctx* x, const int32_t* ids, int32_t n_req, focus_commit_result* out) {
  if (!x) return FOCUS_ERR_STATE;
  NvtxRange nv("focus_commit (A9-A10)");
  if (!x->step_pending || n_req != (int)x->pending_list.size()) return FOCUS_ERR_STATE;
  for (int i = 0; i < n_req; ++i)
    if (!ids || ids[i] != x->pending_list[i]) return FOCUS_ERR_STATE;
  x->step_pending = false;
  if (n_req == 0) return FOCUS_OK;
  CommitArgs a{};
  a.req_list = x->req_dev;
  a.n_req = n_req;
  a.st = x->st;
  a.rowL = x->rowL;
  a.offL = x->offL;
  a.part = x->vpart;
  a.nch = x->nch_vocab;
  a.tau = x->cfg.conf_threshold;
  a.B = x->B;
  a.cache_mode = x->cfg.cache_mode;
  a.mask_id = x->mask_id;
  a.max_gen = x->max_gen;
  a.out_tokens = x->out_tokens;
  a.tokconf = x->tokconf;
  a.res = x->res_dev;
  a.cnt = x->cnt;
  LAUNCH(COMMIT, launch_commit(a, x->stream));
  if (out)
    cudaMemcpyAsync(out, x->res_dev, (size_t)n_req * sizeof(focus_commit_result), cudaMemcpyDeviceToHost, x->stream);
  return cuda_status(cudaGetLastError());
}

focus_status focus_sync(focus_ctx* x) {
  if (!x) return FOCUS_ERR_STATE;
  if (x->sticky != FOCUS_OK) return x->sticky;
  focus_status rc = cuda_status(cudaStreamSynchronize(x->stream));
  if (rc != FOCUS_OK) return rc;
  int inv = 0;
  rc = cuda_status(cudaMemcpy(&inv, &x->cnt->invariant, 4, cudaMemcpyDeviceToHost));
  if (rc != FOCUS_OK) return rc;
  return inv ? FOCUS_ERR_INVARIANT : FOCUS_OK;
}

focus_status focus_get_tokens(focus_ctx* x, int32_t req_id, int32_t* out_host, int32_t cap, int32_t* n_out) {
  if (!x || req_id < 0 || req_id >= x->cfg.max_requests || !x->slot_used[req_id]) return FOCUS_ERR_STATE;
  if (!out_host || !n_out) return FOCUS_ERR_IO;
  focus_status rc = cuda_status(cudaStreamSynchronize(x->stream));
  if (rc != FOCUS_OK) return rc;
  focus_req_state st;
  rc = cuda_status(cudaMemcpy(&st, x->st + req_id, sizeof(st), cudaMemcpyDeviceToHost));
  if (rc != FOCUS_OK) return rc;
  const int n = std::min(cap, st.b * x->B);
  rc = cuda_status(cudaMemcpy(out_host, x->out_tokens + (size_t)req_id * x->max_gen, (size_t)n * 4,
                              cudaMemcpyDeviceToHost));
  *n_out = n;
  return rc;
}

focus_status focus_set_profile(focus_ctx* x, int32_t on) {
  if (!x) return FOCUS_ERR_STATE;
  focus_status rc = cuda_status(cudaStreamSynchronize(x->stream));
  if (rc != FOCUS_OK) return rc;
  prof_collect(x);
  if (on) {
    for (int k = 0; k < FOCUS_PROF_KINDS; ++k) x->prof_acc[k] = focus_prof_entry{k, 0, 0.f, 0.f};
  }
  x->prof_on = on != 0;
  return FOCUS_OK;
}

focus_status focus_set_tap(focus_ctx* x, int32_t layer) {
  if (!x) return FOCUS_ERR_STATE;
  if (!x->cfg.debug_taps && layer >= 0) return FOCUS_ERR_CONFIG;
  x->tap_layer = layer;
  return FOCUS_OK;
}

focus_status focus_debug_export(focus_ctx* x, int32_t what, int32_t req_id, int32_t layer, void* dst, size_t cap,
                                size_t* n_written) {
  if (!x || !dst || !n_written) return FOCUS_ERR_IO;
  focus_status rc = cuda_status(cudaStreamSynchronize(x->stream));
  if (rc != FOCUS_OK) return rc;
  const focus_config& c = x->cfg;
  Counters cnt;
  cudaMemcpy(&cnt, x->cnt, sizeof(cnt), cudaMemcpyDeviceToHost);
  const int n_req = x->last_list.size();
  const void* src = nullptr;
  size_t bytes = 0;
  switch (what) {
    case FOCUS_DBG_STATE: src = x->st; bytes = (size_t)c.max_requests * sizeof(focus_req_state); break;
    case FOCUS_DBG_COUNTERS: src = x->cnt; bytes = sizeof(Counters); break;
    case FOCUS_DBG_ROWS_P: src = x->rowP; bytes = (size_t)cnt.M_P * sizeof(RowInfo); break;
    case FOCUS_DBG_ROWS_S: src = x->rowS; bytes = (size_t)cnt.M_S * sizeof(RowInfo); break;
    case FOCUS_DBG_ROWS_L: src = x->rowL; bytes = (size_t)cnt.M_L * sizeof(RowInfo); break;
    case FOCUS_DBG_I0: src = x->I0p; bytes = (size_t)n_req * x->n_chunks * c.n_kv_heads * x->B * 4; break;
    case FOCUS_DBG_I1: src = x->I1p; bytes = (size_t)n_req * x->n_chunks * c.n_kv_heads * x->B * 4; break;
    case FOCUS_DBG_LOGITS: src = x->logits; bytes = (size_t)cnt.M_L * c.vocab * 4; break;
    case FOCUS_DBG_TOKCONF: src = x->tokconf; bytes = (size_t)cnt.M_L * sizeof(TokConf); break;
    case FOCUS_DBG_HL: src = x->h; bytes = (size_t)cnt.M_L * c.d_model * 2; break;
    case FOCUS_DBG_MOE_SEL: src = x->moe_sel; bytes = x->moe_sel ? (size_t)cnt.M_S * c.top_k * 4 : 0; break;
    case FOCUS_DBG_MOE_WT: src = x->moe_wt; bytes = x->moe_wt ? (size_t)cnt.M_S * c.top_k * 4 : 0; break;
    case FOCUS_DBG_MOE_AG: src = x->moe_Ag; bytes = x->moe_Ag ? (size_t)cnt.M_S * c.top_k * c.d_model * 2 : 0; break;
    case FOCUS_DBG_MOE_Y: src = x->moe_y; bytes = x->moe_y ? (size_t)cnt.M_S * c.top_k * c.d_model * 4 : 0; break;
    case FOCUS_DBG_MOE_ROWS: {
      if (!x->moe_tok) { *n_written = 0; return FOCUS_OK; }
      const size_t a = (size_t)cnt.M_S * c.top_k * 4, b = (size_t)(c.n_experts + 1) * 4;
      if (cap < a + b) return FOCUS_ERR_IO;
      cudaMemcpy(dst, x->moe_tok, a, cudaMemcpyDeviceToHost);
      cudaMemcpy((char*)dst + a, x->moe_off, b, cudaMemcpyDeviceToHost);
      *n_written = a + b;
      return cuda_status(cudaGetLastError());
    }
    case FOCUS_DBG_ATTN_TRACE: src = x->attn_trace; bytes = x->attn_trace ? (size_t)num_sms() * 8 * kTraceEv * 8 : 0; break;
    case FOCUS_DBG_LAUNCHES:
      if (cap < 8) return FOCUS_ERR_IO;
      std::memcpy(dst, &x->launches, 8);
      *n_written = 8;
      return FOCUS_OK;
    case FOCUS_DBG_PROFILE: {
      prof_collect(x);
      const size_t nb = sizeof(x->prof_acc);
      if (cap < nb) return FOCUS_ERR_IO;
      std::memcpy(dst, x->prof_acc, nb);
      *n_written = nb;
      return FOCUS_OK;
    }
    case FOCUS_DBG_KV_K:
    case FOCUS_DBG_KV_V: {
      if (req_id < 0 || req_id >= c.max_requests || !x->slot_used[req_id] || layer < 0 || layer >= c.n_layers)
        return FOCUS_ERR_STATE;
      focus_req_state st;
      cudaMemcpy(&st, x->st + req_id, sizeof(st), cudaMemcpyDeviceToHost);
      const int n = std::min(st.s + x->B, c.max_seq_len);
      const size_t row = (size_t)c.n_kv_heads * c.head_dim;
      if (cap < (size_t)n * row * 2) return FOCUS_ERR_IO;
      const bf16* pool = (what == FOCUS_DBG_KV_K ? x->Kpool : x->Vpool) + (size_t)layer * x->kv_layer_elems;
      char* out = (char*)dst;
      const auto& pages = x->slot_pages[req_id];
      for (int p = 0; p < n; ++p) {
        const int page = pages[p / c.page_size], off = p % c.page_size;
        for (int h = 0; h < c.n_kv_heads; ++h) {
          const size_t e = (((size_t)page * c.n_kv_heads + h) * c.page_size + off) * c.head_dim;
          cudaMemcpy(out + ((size_t)p * row + (size_t)h * c.head_dim) * 2, pool + e, (size_t)c.head_dim * 2,
                     cudaMemcpyDeviceToHost);
        }
      }
      *n_written = (size_t)n * row * 2;
      return cuda_status(cudaGetLastError());
    }
    default: {
      const int t = what - FOCUS_DBG_TAP_X_IN;
      if (t < 0 || t >= kTapCount - 1 || !x->taps[t]) return FOCUS_ERR_IO;
      src = x->taps[t];
      bytes = x->tap_bytes[t];
      if (t == TAP_QS) bytes = std::min(bytes, (size_t)cnt.M_S * x->q_dim * 2);
    }
  }
  bytes = std::min(bytes, cap);
  rc = cuda_status(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost));
  *n_written = bytes;
  return rc;
}

}  // extern "C"
