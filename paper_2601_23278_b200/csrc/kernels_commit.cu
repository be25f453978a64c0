// Confidence-based unmasking and the Neighbor-Aware delayed KV commit.
//
// k_vocab_reduce: per logit row (S cap M) and vocab chunk, one streaming pass with 16-byte loads
//   keeps (max, sum exp(z - max), lowest argmax) — the max softmax probability is
//   conf = 1 / sum_v exp(z_v - max) (reading A-CF1; mask id excluded; ties -> lowest id, A-CF4).
// k_commit: per request (one warp): combine the chunk partials in a fixed order, Decode_and_Verify
//   (conf >= tau, else the single best position, ties to the lowest position; A-CF2),
//   statistics (App.E; untouched on flush steps, A-B4), KV commit (§4.3; DC+ =
//   decoded at an earlier step and right neighbour decoded by now / whole block decoded for the last
//   position, A-DC1..A-DC3), R <- R', block reset / advance / finish (App.E).
#include <math_constants.h>

#include "common.cuh"

namespace focus {

__device__ __forceinline__ VocabPartial vp_combine(VocabPartial a, VocabPartial b);
__device__ __forceinline__ VocabPartial vp_combine(VocabPartial a, float4 b4, int) {   // b as raw 16 bytes
  VocabPartial b;
  b.m = b4.x;
  b.s = b4.y;
  b.idx = __float_as_int(b4.z);
  b.pad = 0;
  return vp_combine(a, b);
}
__device__ __forceinline__ VocabPartial vp_combine(VocabPartial a, VocabPartial b) {
  if (b.m == -CUDART_INF_F) return a;
  if (a.m == -CUDART_INF_F) return b;
  VocabPartial r;
  r.m = fmaxf(a.m, b.m);
  r.s = a.s * expf(a.m - r.m) + b.s * expf(b.m - r.m);
  r.idx = a.m > b.m ? a.idx : (b.m > a.m ? b.idx : min(a.idx, b.idx));
  r.pad = 0;
  return r;
}

__global__ void __launch_bounds__(256) k_vocab_reduce(const float* __restrict__ logits, const int* __restrict__ M_dev,
                                                      int M_max, int V, int mask_id, int nch,
                                                      VocabPartial* __restrict__ part) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x, c = blockIdx.y;
  if (r >= min(*M_dev, M_max)) return;
  const int per = ((V + nch - 1) / nch + 3) & ~3;
  const int lo = c * per, hi = min(V, lo + per);
  const float* row = logits + (size_t)r * V;
  VocabPartial acc{-CUDART_INF_F, 0.f, 0x7fffffff, 0};
  // V is a multiple of 4 for 16-byte loads when the row stride allows it; otherwise scalar.
  const bool vec = (V % 4) == 0;
  if (vec) {
    for (int k = lo + threadIdx.x * 4; k < hi; k += blockDim.x * 4) {
      const float4 v4 = *reinterpret_cast<const float4*>(row + k);
      const float vv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int id = k + e;
        if (id >= hi || id == mask_id) continue;
        const float v = vv[e];
        if (v > acc.m) { acc.s = acc.s * expf(acc.m - v) + 1.f; acc.m = v; acc.idx = id; }
        else acc.s += expf(v - acc.m);
      }
    }
  } else {
    for (int k = lo + threadIdx.x; k < hi; k += blockDim.x) {
      if (k == mask_id) continue;
      const float v = row[k];
      if (v > acc.m) { acc.s = acc.s * expf(acc.m - v) + 1.f; acc.m = v; acc.idx = k; }
      else acc.s += expf(v - acc.m);
    }
  }
  for (int off = 16; off; off >>= 1) {
    VocabPartial o;
    o.m = __shfl_xor_sync(0xffffffffu, acc.m, off);
    o.s = __shfl_xor_sync(0xffffffffu, acc.s, off);
    o.idx = __shfl_xor_sync(0xffffffffu, acc.idx, off);
    acc = vp_combine(acc, o);
  }
  __shared__ VocabPartial red[8];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    VocabPartial t = red[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) t = vp_combine(t, red[w]);
    part[(size_t)r * nch + c] = t;
  }
}

void launch_vocab_reduce(const float* logits, const int* M_dev, int M_max, int V, int mask_id, int nch,
                         VocabPartial* part, cudaStream_t s) {
  if (M_max <= 0) return;
  dim3 grid(M_max, nch);
  launch_pdl(k_vocab_reduce, grid, dim3(256), 0, s, logits, M_dev, M_max, V, mask_id, nch, part);
}

// One CTA per logit row: thread t combines groups t, t + 256, ... in order, then a fixed butterfly per
// warp and the 8 warps in order (vp_combine is commutative, so the result does not depend on timing);
// (max, sum exp(z - max), lowest argmax) of the whole row goes to out[row].  The LM-head epilogue wrote
// the per-64-column partials, so the fp32 logits never reach HBM.
__global__ void __launch_bounds__(256) k_vocab_combine(const VocabPartial* __restrict__ tiles, int ngroups,
                                                       const int* __restrict__ M_dev, int M_max,
                                                       VocabPartial* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const int row = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (row >= min(*M_dev, M_max)) return;
  const VocabPartial* t = tiles + (size_t)row * ngroups;
  VocabPartial acc{-CUDART_INF_F, 0.f, 0x7fffffff, 0};
  for (int g = threadIdx.x; g < ngroups; g += 256) acc = vp_combine(acc, __ldcg(reinterpret_cast<const float4*>(t + g)) , 0);
  for (int off = 1; off < 32; off <<= 1) {
    VocabPartial o;
    o.m = __shfl_xor_sync(0xffffffffu, acc.m, off);
    o.s = __shfl_xor_sync(0xffffffffu, acc.s, off);
    o.idx = __shfl_xor_sync(0xffffffffu, acc.idx, off);
    o.pad = 0;
    acc = vp_combine(acc, o);
  }
  __shared__ VocabPartial red[8];
  if (lane == 0) red[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    VocabPartial r = red[0];
    for (int w = 1; w < 8; ++w) r = vp_combine(r, red[w]);
    out[row] = r;
  }
}

void launch_vocab_combine(const VocabPartial* tiles, int ngroups, const int* M_dev, int M_max, VocabPartial* out,
                          cudaStream_t s) {
  if (M_max <= 0) return;
  launch_pdl(k_vocab_combine, dim3(M_max), dim3(256), 0, s, tiles, ngroups, M_dev, M_max, out);
}

__global__ void __launch_bounds__(1024) k_commit(CommitArgs a) {
  pdl_trigger();
  pdl_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int B = a.B;
  const uint64_t full = full_mask(B);
  for (int i = warp; i < a.n_req; i += 32) {
    const int slot = a.req_list[i];
    focus_req_state& st = a.st[slot];
    focus_commit_result* res = a.res ? a.res + i : nullptr;
    const bool live = st.active && !st.finished;
    if (!live) {
      if (res && lane == 0) { res->req_id = slot; res->n_new = 0; res->block_done = 0; res->finished = st.finished; res->n_committed = 0; }
      continue;
    }
    const int lo = __ldcg(a.offL + i), nL = __ldcg(a.offL + i + 1) - lo;   // written by the selection, kernels back
    // per logit row: combine chunk partials (fixed order)
    float cf[2] = {-1.f, -1.f};
    int tk[2] = {0, 0}, jp[2] = {-1, -1};
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const int k = lane + 32 * t;
      if (k < nL) {
        VocabPartial p = a.part[(size_t)(lo + k) * a.nch];
        for (int c = 1; c < a.nch; ++c) p = vp_combine(p, a.part[(size_t)(lo + k) * a.nch + c]);
        cf[t] = 1.0f / p.s;
        tk[t] = p.idx;
        jp[t] = __ldcg(&a.rowL[lo + k].j);
        if (tk[t] < 0 || tk[t] >= a.mask_id || !(cf[t] >= 0.f)) {
          // no valid argmax (non-finite logits): flag the step instead of committing an out-of-range id
          // (which the next step's embedding gather would read past the table with)
          atomicExch(&a.cnt->invariant, 1);
          tk[t] = 0;
          cf[t] = -CUDART_INF_F;
        }
        a.tokconf[lo + k] = TokConf{p.idx, cf[t]};
      }
    }
    // Decode_and_Verify: D = {conf >= tau} as a position mask
    uint64_t Dl = 0ull;
#pragma unroll
    for (int t = 0; t < 2; ++t)
      if (jp[t] >= 0 && cf[t] >= a.tau) Dl |= 1ull << jp[t];
    for (int off = 16; off; off >>= 1) Dl |= __shfl_xor_sync(0xffffffffu, Dl, off);
    uint64_t D = Dl;
    if (D == 0ull && nL > 0) {
      // fallback: highest confidence, ties to the lowest position
      float bc = -1.f;
      int bj = 0x7fffffff;
#pragma unroll
      for (int t = 0; t < 2; ++t)
        if (jp[t] >= 0 && (cf[t] > bc || (cf[t] == bc && jp[t] < bj))) { bc = cf[t]; bj = jp[t]; }
      for (int off = 16; off; off >>= 1) {
        const float oc = __shfl_xor_sync(0xffffffffu, bc, off);
        const int oj = __shfl_xor_sync(0xffffffffu, bj, off);
        if (oc > bc || (oc == bc && oj < bj)) { bc = oc; bj = oj; }
      }
      if (bj < 64) D = 1ull << bj;
      else atomicExch(&a.cnt->invariant, 1);      // every confidence invalid (flagged above): decode nothing
    }
    // apply decisions (each lane its own rows)
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      if (jp[t] >= 0 && ((D >> jp[t]) & 1ull)) {
        st.tok[jp[t]] = tk[t];
        st.dstep[jp[t]] = st.t;
        if (tk[t] == a.mask_id) atomicExch(&a.cnt->invariant, 1);
        if (res) { const int k = __popcll(D & ((1ull << jp[t]) - 1ull)); res->pos[k] = jp[t]; res->tok[k] = tk[t]; }
      }
    }
    __syncwarp();
    if (lane == 0) {
      const uint64_t dec_before = full & ~st.masked;           // decoded at an earlier step
      const uint64_t dec_now = dec_before | D;
      const bool flush = st.flush;
      if (!flush) {
        st.token_sum += __popcll(D);
        st.total_steps += 1;
      }
      st.masked &= ~D;
      const uint64_t cand = st.P & dec_before & ~st.committed;
      uint64_t nw;
      if (a.cache_mode == FOCUS_CACHE_NONE) {
        nw = dec_before == full ? st.P : 0ull;
      } else if (a.cache_mode == FOCUS_CACHE_DC) {
        nw = cand;
      } else {
        uint64_t nb = dec_now >> 1;
        if (dec_now == full) nb |= 1ull << (B - 1);
        nw = cand & nb;
      }
      st.committed |= nw;
      st.R = st.R_new;
      st.n_new = __popcll(D);
      st.n_committed = __popcll(nw);
      int block_done = 0;
      if (st.committed == full) {
        block_done = 1;
        for (int j = 0; j < B; ++j) a.out_tokens[(size_t)slot * a.max_gen + (size_t)st.b * B + j] = st.tok[j];
        st.b += 1;
        st.s += B;
        if (st.b * B >= st.gen_len) {
          st.finished = 1;
        } else {
          st.committed = 0ull;
          st.masked = full;
          st.R = -1;
          for (int j = 0; j < B; ++j) { st.tok[j] = a.mask_id; st.dstep[j] = 0x7fffffff; }
        }
      }
      if (res) {
        res->req_id = slot;
        res->n_new = __popcll(D);
        res->block_done = block_done;
        res->finished = st.finished;
        res->n_committed = __popcll(nw);
      }
    }
  }
}

void launch_commit(const CommitArgs& a, cudaStream_t s) {
  launch_pdl(k_commit, dim3(1), dim3(1024), 0, s, a);
}

}  // namespace focus
