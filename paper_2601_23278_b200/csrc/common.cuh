// Internal declarations shared by the libfocus CUDA translation units (sm_100a only).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "focus.h"

typedef __nv_bfloat16 bf16;

namespace focus {

// ---------------------------------------------------------------- programmatic dependent launch
// Every kernel of the step triggers its dependents at entry and waits for its predecessor (full
// completion + memory flush) before touching data produced earlier in the stream; setup that only
// reads launch parameters / weights (barrier init, TMEM alloc, tensor-map prefetch) runs before the
// wait and overlaps the previous kernel's tail.  Without the launch attribute both are no-ops.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

constexpr int kMaxB = 64;          // per-request masks are uint64 (focus.h)
constexpr int kGuGroup = 128;      // gate/up rows interleaved in groups of 128 (Wgu layout)
constexpr int kAttnQRows = 64;     // query rows (G x block rows) per attention CTA
constexpr int kAttnKT = 32;        // keys per attention tile (SIMT path)
constexpr int kTraceEv = 512;      // attention trace events per (CTA, role)

// One processed / retained / logit row of the ragged batch.
struct RowInfo {
  int slot;   // request slot
  int j;      // block position (-1 for prefill rows)
  int pos;    // absolute position (RoPE angle, KV slot)
  int ri;     // index of the request in the call's req list
};

struct Counters {
  int M_P, M_S, M_L, invariant;
  int attn_rpc;     // query block rows per attention chunk (importance partials are per chunk)
  int n_chunks;     // chunks per request (ceil(B / attn_rpc))
  int pad[2];
  // cumulative since focus_init (redundancy statistics, tab:reduce_ratio P:480-504): rows processed
  // at layers 0-1 (sum M_P), rows kept for the later layers (sum M_S), logit rows (sum M_L), steps
  long long sum_P, sum_S, sum_L, steps;
};

struct VocabPartial {   // running (max, sum exp(x - max), argmax) of a vocab chunk
  float m, s;
  int idx, pad;
};

struct TokConf {
  int tok;
  float conf;
};

// Device pointers + geometry of the paged KV pool of one layer.
struct KVView {
  bf16* K;
  bf16* V;
  const int* page_table;   // [max_requests][max_pages]
  int max_pages, page_size, n_kv_heads, head_dim;
};

__device__ __forceinline__ size_t kv_offset(const KVView& kv, int slot, int pos, int kvh) {
  int page = kv.page_table[(size_t)slot * kv.max_pages + pos / kv.page_size];
  int off = pos % kv.page_size;
  return (((size_t)page * kv.n_kv_heads + kvh) * kv.page_size + off) * kv.head_dim;
}

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;

__host__ __device__ __forceinline__ uint64_t full_mask(int B) {
  return B >= 64 ? ~0ull : ((1ull << B) - 1ull);
}

// ---------------------------------------------------------------- launchers (kernels_*.cu)
void launch_init_weights(bf16* dst, int rows, int cols, uint64_t tid, uint64_t seed, int exp2,
                         int gu_group, int gu_off, cudaStream_t st);

void launch_step_setup(const int* req_list, int n_req, focus_req_state* st, int B, RowInfo* rowP,
                       int* offP, int* tokP, Counters* cnt, cudaStream_t s);
void launch_hold(long long ns, cudaStream_t s);
void launch_embed(const int* tok, const int* M_dev, int M_max, const bf16* E, int d, float* x,
                  cudaStream_t s);
void launch_rmsnorm(const float* x, const int* src_map, const int* M_dev, int M_max, int d, float eps,
                    bf16* out, cudaStream_t s);
void launch_rope_store(const float* qkv_f32, const RowInfo* rows, const int* M_dev, int M_max,
                       int n_q_heads, const float* rope_cos, const float* rope_sin,
                       const focus_req_state* st, KVView kv, bf16* qkv_out, Counters* cnt,
                       cudaStream_t s);
// Per-row RoPE factors, transposed: out[f][r] = cos(pos_r * w_f), out[64 + f][r] = sin(pos_r * w_f)
// (ld = row stride), copied from the fp64-built tables, for the fused QKV epilogue (head_dim 128).
void launch_rope_rows(const RowInfo* rows, const int* M_dev, int M_max, const float* rcos, const float* rsin,
                      float* out, int ld, cudaStream_t s);
void launch_silu_mul(const float* gu, const int* M_dev, int M_max, int d_ff, bf16* act, cudaStream_t s);
void launch_gather_rows(const float* x, const bf16* qkv, int qkv_dim, int q_dim, const int* src,
                        const int* M_dev, int M_max, int d, float* x_out, bf16* q_out, cudaStream_t s);

// GEMM: C[M x N] (fp32) = A[M x K] (bf16, row stride lda) . W[N x K]^T (bf16), store or accumulate.
enum GemmMode { GEMM_STORE = 0, GEMM_ADD = 1, GEMM_SWIGLU = 2, GEMM_QKV_ROPE = 3 };
struct GemmWs {                 // split-K partials + per-tile semaphores (carved from the arena)
  float* ptr;
  size_t bytes;
  int* sem;
  size_t sem_count;
  int no_swap;                  // 1: never the swap-AB decode GEMM (batch_invariant: the path would
                                // otherwise depend on the batch's row-count bound)
};
constexpr int kSwapSemBase = 4096;   // swap-AB split-K tile counters: sem[kSwapSemBase + tile]
// One work unit of the tensor-core attention kernel (request i of the call, query-row chunk, kv head,
// key split; key tiles [t_lo, t_hi) of 128 keys), as planned once per step by k_attn_plan.
struct AttnUnit {
  int i, chunk, kvh, sp, nsplit, slot, r0, nr, nq, kbeg, kend, t_lo, t_hi, s0, pos_base, pair;
  uint64_t P;
  int want_imp, pad;
};

// Fused-epilogue parameters (tensor-core GEMM only).
struct GemmEpi {
  bf16* out; int ldo;                  // SWIGLU: act [M][d_ff]; QKV_ROPE: qkv [M][(Hq+2Hkv) dh]
  const RowInfo* rows;                 // QKV_ROPE: per-row (slot, j, pos) for RoPE angle and KV slot
  const float* ropeT; int rope_ld;     // QKV_ROPE: launch_rope_rows table of these rows ([128][rope_ld])
  const focus_req_state* st;
  KVView kv;
  int n_q_heads;
  Counters* cnt;
  // QKV_ROPE, layers >= 2: L2 prefetch of the next attention launch's context K/V.  While the GEMM
  // runs, its idle warp prefetches the first pf_tiles key tiles (context keys only: the block's own
  // slots are being written by this GEMM) of the units the attention CTAs run first
  const AttnUnit* pf_units;            // plan [pf_grid][pf_ucap] (nullptr: off)
  const int* pf_n;                     // [pf_grid] units per attention CTA
  int pf_grid, pf_ucap, pf_tiles;
  // STORE (LM head): per row and 64-column group, (max, sum exp(z - max), lowest argmax) of the logits
  // (mask id excluded) -> vpart[row][group] (ld vp_ld); C may then be nullptr (logits never stored)
  VocabPartial* vpart; int vp_ld; int mask_id;
};
// a_rows: allocated rows of A (TMA bounds); M_dev/M_max: live / maximum rows of this call.
void launch_gemm(const bf16* A, int lda, int a_rows, const bf16* W, int N, int K, float* C, int ldc,
                 const int* M_dev, int M_max, GemmMode mode, const GemmWs& ws, cudaStream_t s, int m_est = 0);
int gemm_backend();
// tile configuration a tensor-core GEMM of this shape takes at m_est expected live rows (the graph
// cache keys on it; kernels_gemm_tc.cu)
int gemm_tc_choice(int N, int K, GemmMode mode, int M_max, int m_est, bool allow_swap = true);
int num_sms();
void gemm_set_backend(int b);

struct AttnArgs {
  const bf16* q;  int ldq;      // query rows; head h at column h*head_dim
  bf16* out;      int ldo;      // [rows][n_q_heads*head_dim] (nullptr in importance-only mode)
  KVView kv;
  const int* req_list;          // decode: request slots of the call
  const int* row_off;           // decode: rows of list index i are [row_off[i], row_off[i+1])
  const focus_req_state* st;
  int n_req, B, n_q_heads;
  int ext_mode;                 // 0: keys [0, s+B)  1: keys [0, s+R_new+1)  2: causal prefill
  int imp_only;                 // 1: keys = block [s, s+B) only, no output (layer-1 importance)
  int prefill_slot, prefill_pos0, prefill_rows;
  float* imp;                   // [n_req][n_chunks][n_kv_heads][B] partial importance or nullptr
  int n_chunks;                 // query-row chunks per request (decode)
  int mp_kernel;                // MaxPool1D kernel (odd)
  float scale;                  // 1/sqrt(head_dim)
  // tensor-core path (kernels_attn_tc.cu)
  int layer;                    // pool layer (TMA row base = layer * kv_pages * n_kv_heads * page_size)
  long long kv_pages;           // pages per layer
  int split_tiles;              // 64-key tiles per key split (>= 2)
  int max_nsplit;               // split slots per (request, chunk, kv head) in `part`
  float* part;                  // split partials [pair][max_nsplit][128 * head_dim + 2 * 128]
  float* imp_scratch;           // per-CTA block-score scratch [grid][128][64] (importance epilogue)
  unsigned long long* trace;    // debug: clock64 events [grid][8][kTraceEv] or nullptr
  int* sem;                     // per (request, chunk, kv head): arrival count of split pieces (zeroed)
  int stream_k;                 // 1: stream-K over key tiles (balanced CTAs; attention without importance)
  int tail_split;               // 1: units of the last partial round are key-split across the idle CTAs
  int l2_prefetch;              // K/V tiles past the smem rings to prefetch into L2
  int kv_hint;                  // 1: K/V tiles loaded with the L2 evict-first policy
  int page_skip;                // 1: K/V boxes holding no key of the unit are not loaded
  int nch_fixed;                // 1: every non-causal unit runs the 64-row softmax variant (one hot copy)
  void* plan_units;             // unit table [grid][UCAP] precomputed by k_attn_plan, or nullptr
  int* plan_n;                  // [grid] units per CTA (nullptr: the kernel builds its table itself)
  int pre_pf_tiles;             // key tiles of the first unit prefetched into L2 before the PDL wait
  int max_slots;                // request slots (rows of the page table)
  int debug_check;              // 1: unit-table sanity checks (trap with a message; FOCUS_ATTN_CHECK=1)
  float rescale_log2;           // lazy softmax: the running max moves when a score exceeds it by this
                                // (log2 units; 8 by default, FOCUS_ATTN_RESCALE_LOG2 for tests)
};
void launch_attention(const AttnArgs& a, cudaStream_t s);
bool attn_tc_supported(int head_dim, int page_size, int group);
bool attn_tc_make_qmap(const bf16* q, size_t rows, int ld, int n_heads, int group, CUtensorMap* mq);
int attn_tc_rows_per_chunk(int group);
bool attn_tc_make_maps(const bf16* Kpool, const bf16* Vpool, size_t rows, int head_dim, int page_size,
                       CUtensorMap* mk, CUtensorMap* mv);
void launch_attention_tc(const CUtensorMap& mk, const CUtensorMap& mv, const CUtensorMap& mq, const AttnArgs& a,
                         cudaStream_t s);
bool launch_attention_plan(const AttnArgs& a, cudaStream_t s);
int attn_tc_plan_capacity();
int attn_tc_grid(const AttnArgs& a);   // CTAs of a tensor-core attention launch (0: nothing to do)

struct SelectArgs {
  const int* req_list; int n_req;
  focus_req_state* st;
  const float* I0p; const float* I1p;                 // partial importance [n_req][n_chunks][n_kv_heads][B]
  int n_chunks, n_kv_heads, attn_rpc;                 // chunk c of a request exists iff c * attn_rpc < |P|
  int B, alpha_num, alpha_den, placeholder_mode, strategy, fixed_k;
  uint64_t seed;
  const int* offP;
  RowInfo* rowS; int* srcP; int* offS;
  RowInfo* rowL; int* srcL; int* offL;
  Counters* cnt;
};
void launch_select_plan(const SelectArgs& a, cudaStream_t s);

void launch_vocab_reduce(const float* logits, const int* M_dev, int M_max, int V, int mask_id, int nch,
                         VocabPartial* part, cudaStream_t s);
// MoE FFN (kernels_moe.cu, grouped expert GEMM in kernels_gemm_tc.cu)
void launch_moe_route(const float* z, int ldz, const int* M_dev, int M_max, int E, int K, int* sel, float* wt, int* cnt,
                      cudaStream_t s);
void launch_moe_place(const int* sel, const int* cnt, const int* M_dev, int M_max, int E, int K, int* off, int* tok_of,
                      int* slot_of, cudaStream_t s);
void launch_moe_gather(const bf16* h, const int* tok_of, const int* M_dev, int M_max, int K, int d, bf16* Ag,
                       cudaStream_t s);
void launch_moe_combine(const float* y, const int* slot_of, const float* wt, const int* M_dev, int M_max, int K, int d,
                        float* x, int* cnt, int E, cudaStream_t s);
bool launch_gemm_grouped(const bf16* A, int a_rows, const bf16* W, int n_experts, int wrows, int K, float* C, int ldc,
                         const int* off, int M_max_rows, GemmMode mode, const GemmEpi* epi, cudaStream_t s);
// combine the LM-head epilogue's per-64-column partials of each logit row (fixed order) -> out[row]
void launch_vocab_combine(const VocabPartial* tiles, int ngroups, const int* M_dev, int M_max, VocabPartial* out,
                          cudaStream_t s);

struct CommitArgs {
  const int* req_list; int n_req;
  focus_req_state* st;
  const RowInfo* rowL; const int* offL;
  const VocabPartial* part; int nch;
  float tau;
  int B, cache_mode, mask_id, max_gen;
  int* out_tokens;              // [max_requests][max_gen]
  TokConf* tokconf;             // [M_logit]
  focus_commit_result* res;     // [n_req]
  Counters* cnt;
};
void launch_commit(const CommitArgs& a, cudaStream_t s);

}  // namespace focus
