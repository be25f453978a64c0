// Mixture-of-Experts FFN of the LLaDA2.0-mini-shaped workload (readings A-M5,
// A-M6).  The FOCUS step is unchanged: an MoE layer runs on the compacted S rows like every layer >= 1
// ("routing after compaction"), so evicted tokens never reach the router or the experts.  Per layer:
//   router GEMM (tcgen05, fp32 logits [M][E])  ->  k_moe_route (top-k per row + weights, expert counts)
//   -> k_moe_place (expert-contiguous, row-ordered positions: deterministic)  ->  k_moe_gather (bf16 rows)
//   -> grouped expert GEMMs (kernels_gemm_tc.cu: gate/up + SwiGLU, down)  ->  shared expert (dense GEMMs,
//   residual add)  ->  k_moe_combine (x += sum_k w_k y_k in selection order).
#include <math_constants.h>

#include "common.cuh"

namespace focus {

__device__ __forceinline__ int live(const int* M_dev, int M_max) { return M_dev ? min(*M_dev, M_max) : M_max; }

// One warp per row: the top-k experts by router logit (ties to the lower expert id; softmax is monotonic,
// so this is the top-k by probability), weights = softmax over the selected logits (A-M6), and the
// per-expert token counts.  E <= 1024, k <= 16.
__global__ void __launch_bounds__(256) k_moe_route(const float* __restrict__ z, int ldz, const int* __restrict__ M_dev,
                                                   int M_max, int E, int K, int* __restrict__ sel,
                                                   float* __restrict__ wt, int* __restrict__ cnt) {
  pdl_trigger();
  pdl_wait();
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (row >= live(M_dev, M_max)) return;
  const float* zr = z + (size_t)row * ldz;
  // the row's logits in registers once (lane holds experts lane + 32 i): one batch of L2 loads instead
  // of K passes of dependent loads
  float v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = lane + 32 * i < E ? __ldcg(zr + lane + 32 * i) : -CUDART_INF_F;
  unsigned taken = 0u;                                   // bit i: expert lane + 32 i already chosen
  float zk[16];
  int ek[16];
  for (int k = 0; k < K; ++k) {
    float best = -CUDART_INF_F;
    int bi = 0x7fffffff, fe = 0x7fffffff;                // fe: lowest expert not yet chosen (fallback)
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const int e = lane + 32 * i;
      if (e < E && !((taken >> i) & 1u)) {
        if (v[i] > best || (v[i] == best && e < bi)) { best = v[i]; bi = e; }
        fe = min(fe, e);
      }
    }
    for (int o = 16; o; o >>= 1) {
      const float ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      fe = min(fe, __shfl_xor_sync(0xffffffffu, fe, o));
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    if (bi >= E) bi = fe;                                // no comparable logit (NaN row): lowest free expert
    zk[k] = best;
    ek[k] = bi;
    if ((bi & 31) == lane) taken |= 1u << (bi >> 5);
  }
  if (lane == 0) {
    float s = 0.f;
    float ex[16];
    for (int k = 0; k < K; ++k) { ex[k] = expf(zk[k] - zk[0]); s += ex[k]; }
    for (int k = 0; k < K; ++k) {
      sel[(size_t)row * K + k] = ek[k];
      wt[(size_t)row * K + k] = ex[k] / s;
      atomicAdd(&cnt[ek[k]], 1);                          // a count: order-independent
    }
  }
}

// One CTA per expert: the expert's offset (prefix of the counts), then its (row, k) entries in row order
// by a block scan, so position p = off[e] + rank is the same on every run: tok_of[p] = row,
// slot_of[row][k] = p.  off[E] = total.
__global__ void __launch_bounds__(256) k_moe_place(const int* __restrict__ sel, const int* __restrict__ cnt,
                                                   const int* __restrict__ M_dev, int M_max, int E, int K,
                                                   int* __restrict__ off, int* __restrict__ tok_of,
                                                   int* __restrict__ slot_of) {
  pdl_trigger();
  pdl_wait();
  const int e = blockIdx.x;
  const int M = live(M_dev, M_max);
  __shared__ int base_sh, wsum[8];
  if (threadIdx.x < 32) {
    int s = 0;
    for (int i = threadIdx.x; i < e; i += 32) s += __ldcg(cnt + i);
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) {
      base_sh = s;
      off[e] = s;
      if (e == E - 1) off[E] = s + __ldcg(cnt + e);
    }
  }
  __syncthreads();
  int run = base_sh;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int r0 = 0; r0 < M; r0 += 256) {
    const int r = r0 + threadIdx.x;
    int kk = -1;
    if (r < M) {
      int sk[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) sk[k] = k < K ? __ldcg(sel + (size_t)r * K + k) : -1;   // one batch of loads
#pragma unroll
      for (int k = 0; k < 16; ++k)
        if (sk[k] == e) kk = k;                        // an expert is selected at most once per row
    }
    const int flag = kk >= 0;
    const unsigned b = __ballot_sync(0xffffffffu, flag);
    if (lane == 0) wsum[warp] = __popc(b);
    __syncthreads();
    int before = 0, total = 0;
    for (int w = 0; w < 8; ++w) { if (w < warp) before += wsum[w]; total += wsum[w]; }
    if (flag) {
      const int p = run + before + __popc(b & ((1u << lane) - 1u));
      tok_of[p] = r;
      slot_of[(size_t)r * K + kk] = p;
    }
    run += total;
    __syncthreads();
  }
}

// Gathered expert inputs: A_g[p] = h[tok_of[p]] (bf16 rows of d), p < M K.  One warp per row, 16-B copies.
__global__ void __launch_bounds__(256) k_moe_gather(const bf16* __restrict__ h, const int* __restrict__ tok_of,
                                                    const int* __restrict__ M_dev, int M_max, int K, int d,
                                                    bf16* __restrict__ Ag) {
  pdl_trigger();
  pdl_wait();
  const int p = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (p >= live(M_dev, M_max) * K) return;
  const uint4* src = reinterpret_cast<const uint4*>(h + (size_t)__ldcg(tok_of + p) * d);
  uint4* dst = reinterpret_cast<uint4*>(Ag + (size_t)p * d);
  for (int c = lane; c < d / 8; c += 32) dst[c] = src[c];
  // the rows are read next by TMA (async proxy) in a programmatically dependent grid
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// x[r] += sum_k w_k y[slot_of[r][k]] (fp32, selection order: fixed).  One CTA per row.  CTA 0 also
// re-zeroes the expert counts for the next MoE layer (every reader of them has completed: the expert
// GEMMs ran after k_moe_place), so no memset node sits between the layer's kernels.
__global__ void __launch_bounds__(256) k_moe_combine(const float* __restrict__ y, const int* __restrict__ slot_of,
                                                     const float* __restrict__ wt, const int* __restrict__ M_dev,
                                                     int M_max, int K, int d, float* __restrict__ x,
                                                     int* __restrict__ cnt, int E) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x;
  if (r == 0)
    for (int e = threadIdx.x; e < E; e += blockDim.x) cnt[e] = 0;
  if (r >= live(M_dev, M_max)) return;
  __shared__ int sl[16];
  __shared__ float w[16];
  if (threadIdx.x < K) {                         // written kernels back: L2 loads (see k_gemm_grouped)
    sl[threadIdx.x] = __ldcg(slot_of + (size_t)r * K + threadIdx.x);
    w[threadIdx.x] = __ldcg(wt + (size_t)r * K + threadIdx.x);
  }
  __syncthreads();
  for (int c = threadIdx.x * 4; c < d; c += blockDim.x * 4) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int k = 0; k < K; ++k) {
      const float4 v = __ldcg(reinterpret_cast<const float4*>(y + (size_t)sl[k] * d + c));
      acc.x += w[k] * v.x; acc.y += w[k] * v.y; acc.z += w[k] * v.z; acc.w += w[k] * v.w;
    }
    float4* xr = reinterpret_cast<float4*>(x + (size_t)r * d + c);
    float4 o = *xr;
    o.x += acc.x; o.y += acc.y; o.z += acc.z; o.w += acc.w;
    *xr = o;
  }
}

void launch_moe_route(const float* z, int ldz, const int* M_dev, int M_max, int E, int K, int* sel, float* wt, int* cnt,
                      cudaStream_t s) {
  if (M_max <= 0) return;
  launch_pdl(k_moe_route, dim3((M_max + 7) / 8), dim3(256), 0, s, z, ldz, M_dev, M_max, E, K, sel, wt, cnt);
}

void launch_moe_place(const int* sel, const int* cnt, const int* M_dev, int M_max, int E, int K, int* off, int* tok_of,
                      int* slot_of, cudaStream_t s) {
  launch_pdl(k_moe_place, dim3(E), dim3(256), 0, s, sel, cnt, M_dev, M_max, E, K, off, tok_of, slot_of);
}

void launch_moe_gather(const bf16* h, const int* tok_of, const int* M_dev, int M_max, int K, int d, bf16* Ag,
                       cudaStream_t s) {
  if (M_max <= 0) return;
  launch_pdl(k_moe_gather, dim3((M_max * K + 7) / 8), dim3(256), 0, s, h, tok_of, M_dev, M_max, K, d, Ag);
}

void launch_moe_combine(const float* y, const int* slot_of, const float* wt, const int* M_dev, int M_max, int K, int d,
                        float* x, int* cnt, int E, cudaStream_t s) {
  if (M_max <= 0) return;
  launch_pdl(k_moe_combine, dim3(M_max), dim3(256), 0, s, y, slot_of, wt, M_dev, M_max, K, d, x, cnt, E);
}

}  // namespace focus
