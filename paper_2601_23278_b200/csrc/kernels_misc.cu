#include <cstdio>
// Small HBM-bound kernels of the decode step: weight init, step setup (P/M/U masks, ragged row
// maps), embedding gather, RMSNorm, RoPE + paged KV store, SwiGLU, row compaction gather.
#include "common.cuh"

namespace focus {

// ------------------------------------------------------------------ synthetic weights
// w = (2k - 255) * 2^e, k = mix64(((tid << 40) + i) + (seed+1)*golden) >> 56   (DESIGN.md "input
// recipe"; the oracle's generator is synth/gen.py - same recipe, separate code).
// gu_group > 0: logical row r of the gate (gu_off = 0) / up (gu_off = 1) matrix is stored at
// row (r / g) * 2g + gu_off * g + r % g of the fused Wgu (tile-friendly interleave).
__global__ void k_init_weights(bf16* __restrict__ dst, int rows, int cols, uint64_t tid, uint64_t seed,
                               int exp2, int gu_group, int gu_off) {
  const size_t n = (size_t)rows * cols;
  const uint64_t base = (tid << 40) + (seed + 1ull) * kGolden;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const uint64_t u = mix64(base + i);
    const int k = (int)(u >> 56);
    const float v = ldexpf((float)(2 * k - 255), exp2);
    size_t r = i / cols, c = i % cols;
    if (gu_group) r = (r / gu_group) * 2 * gu_group + (size_t)gu_off * gu_group + r % gu_group;
    dst[r * cols + c] = __float2bfloat16_rn(v);
  }
}

void launch_init_weights(bf16* dst, int rows, int cols, uint64_t tid, uint64_t seed, int exp2,
                         int gu_group, int gu_off, cudaStream_t st) {
  k_init_weights<<<148 * 8, 256, 0, st>>>(dst, rows, cols, tid, seed, exp2, gu_group, gu_off);
}

// ------------------------------------------------------------------ step setup
// Per request (Alg.1 input; App.E state P:797-821): P = uncommitted, M = masked & P; t += 1;
// exclusive scan of |P| over the call's request list -> P-row offsets; row maps in
// (list order, j ascending) (SURVEY c.4 COMPACT rule applied to P).  One CTA.
// Profiling only: hold the stream for `ns` of device time so the host enqueues the whole profiled step
// (launches and their timing events) before the device reaches it -- the per-launch event intervals then
// measure device time, not the host's eager launch latency.
__global__ void k_hold(long long ns) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    __nanosleep(1000);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while ((long long)(t - t0) < ns);
}
void launch_hold(long long ns, cudaStream_t s) { k_hold<<<1, 1, 0, s>>>(ns); }

__global__ void __launch_bounds__(1024) k_step_setup(const int* __restrict__ req_list, int n_req,
                                                     focus_req_state* __restrict__ st, int B,
                                                     RowInfo* __restrict__ rowP, int* __restrict__ offP,
                                                     int* __restrict__ tokP, Counters* __restrict__ cnt) {
  pdl_trigger();
  pdl_wait();
  __shared__ int scan[1024];
  __shared__ int carry;
  __shared__ uint64_t sP[1024];
  __shared__ int sslot[1024], soff[1024];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const uint64_t full = full_mask(B);
  for (int base = 0; base < n_req; base += blockDim.x) {
    const int i = base + threadIdx.x;
    int np = 0;
    uint64_t P = 0;
    int slot = -1;
    if (i < n_req) {
      slot = req_list[i];
      focus_req_state& s = st[slot];
      if (s.active && !s.finished) {
        P = full & ~s.committed;
        const uint64_t M = s.masked & P;
        s.t += 1;
        s.P = P;
        s.M = M;
        s.flush = (M == 0ull);
        np = __popcll(P);
      } else {
        s.P = s.M = s.S = 0ull;
        s.flush = 1;
      }
    }
    scan[threadIdx.x] = np;
    __syncthreads();
    for (int off = 1; off < (int)blockDim.x; off <<= 1) {
      const int v = threadIdx.x >= off ? scan[threadIdx.x - off] : 0;
      __syncthreads();
      scan[threadIdx.x] += v;
      __syncthreads();
    }
    const int excl = carry + scan[threadIdx.x] - np;
    if (i < n_req) offP[i] = excl;
    sP[threadIdx.x] = P;
    sslot[threadIdx.x] = slot;
    soff[threadIdx.x] = excl;
    __syncthreads();
    // row maps: one thread per (request, block position), so the token loads are all in flight at once
    const int nb = min((int)blockDim.x, n_req - base);
    for (int e = threadIdx.x; e < nb * B; e += blockDim.x) {
      const int li = e / B, j = e - li * B;
      const uint64_t Pm = sP[li];
      if ((Pm >> j) & 1ull) {
        const int sl = sslot[li];
        const int r = soff[li] + __popcll(Pm & ((1ull << j) - 1ull));
        rowP[r] = RowInfo{sl, j, st[sl].s + j, base + li};
        tokP[r] = st[sl].tok[j];
      }
    }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry += scan[threadIdx.x];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    offP[n_req] = carry;
    cnt->M_P = carry;
    cnt->sum_P += carry;
    cnt->steps += 1;
  }
}

void launch_step_setup(const int* req_list, int n_req, focus_req_state* st, int B, RowInfo* rowP,
                       int* offP, int* tokP, Counters* cnt, cudaStream_t s) {
  launch_pdl(k_step_setup, dim3(1), dim3(1024), 0, s, req_list, n_req, st, B, rowP, offP, tokP, cnt);
}

__device__ __forceinline__ int live_rows(const int* M_dev, int M_max) {
  return M_dev ? min(*M_dev, M_max) : M_max;
}

// ------------------------------------------------------------------ embedding
// x_r = E[tok_r] (fp32 residual stream).  One CTA per row, 16-byte loads.
__global__ void k_embed(const int* __restrict__ tok, const int* __restrict__ M_dev, int M_max,
                        const bf16* __restrict__ E, int d, float* __restrict__ x) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x;
  if (r >= live_rows(M_dev, M_max)) return;
  const bf16* src = E + (size_t)tok[r] * d;
  float* dst = x + (size_t)r * d;
  for (int c = threadIdx.x * 8; c < d; c += blockDim.x * 8) {
    const uint4 u = *reinterpret_cast<const uint4*>(src + c);
    const __nv_bfloat162* p = reinterpret_cast<const __nv_bfloat162*>(&u);
    float4 a, b;
    float2 f0 = __bfloat1622float2(p[0]), f1 = __bfloat1622float2(p[1]);
    float2 f2 = __bfloat1622float2(p[2]), f3 = __bfloat1622float2(p[3]);
    a = make_float4(f0.x, f0.y, f1.x, f1.y);
    b = make_float4(f2.x, f2.y, f3.x, f3.y);
    *reinterpret_cast<float4*>(dst + c) = a;
    *reinterpret_cast<float4*>(dst + c + 4) = b;
  }
}

void launch_embed(const int* tok, const int* M_dev, int M_max, const bf16* E, int d, float* x, cudaStream_t s) {
  if (M_max <= 0) return;
  launch_pdl(k_embed, dim3(M_max), dim3(128), 0, s, tok, M_dev, M_max, E, d, x);
}

// ------------------------------------------------------------------ RMSNorm
// out_r = bf16( x_src(r) / sqrt(mean(x^2) + eps) )   (gains are 1; SURVEY c.1)
__global__ void k_rmsnorm(const float* __restrict__ x, const int* __restrict__ src_map,
                          const int* __restrict__ M_dev, int M_max, int d, float eps,
                          bf16* __restrict__ out) {
  // one row per block; the row stays in registers between the sum of squares and the scaling
  // (one read of x), vector loads/stores, d <= 4 * 256 * kRmsVec
  constexpr int kRmsVec = 8;
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x;
  if (r >= live_rows(M_dev, M_max)) return;
  const int src = src_map ? src_map[r] : r;
  const float* xr = x + (size_t)src * d;
  float4 v[kRmsVec];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < kRmsVec; ++i) {
    const int c = (i * blockDim.x + threadIdx.x) * 4;
    v[i] = c < d ? __ldcg(reinterpret_cast<const float4*>(xr + c)) : make_float4(0.f, 0.f, 0.f, 0.f);
    ss += v[i].x * v[i].x + v[i].y * v[i].y + v[i].z * v[i].z + v[i].w * v[i].w;
  }
  __shared__ float red[32];
  for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  const float inv = 1.0f / sqrtf(red[0] / (float)d + eps);
  bf16* o = out + (size_t)r * d;
#pragma unroll
  for (int i = 0; i < kRmsVec; ++i) {
    const int c = (i * blockDim.x + threadIdx.x) * 4;
    if (c < d) {
      __nv_bfloat162 lo = __floats2bfloat162_rn(v[i].x * inv, v[i].y * inv);
      __nv_bfloat162 hi = __floats2bfloat162_rn(v[i].z * inv, v[i].w * inv);
      uint2 pk;
      pk.x = *reinterpret_cast<uint32_t*>(&lo);
      pk.y = *reinterpret_cast<uint32_t*>(&hi);
      *reinterpret_cast<uint2*>(o + c) = pk;
    }
  }
}

void launch_rmsnorm(const float* x, const int* src_map, const int* M_dev, int M_max, int d, float eps,
                    bf16* out, cudaStream_t s) {
  if (M_max <= 0) return;
  // the register-resident row needs d <= 256 threads * 8 float4 (every SDAR shape: d <= 4096)
  if (d > 256 * 8 * 4 || d % 4) { std::fprintf(stderr, "libfocus: rmsnorm width %d unsupported\n", d); return; }
  launch_pdl(k_rmsnorm, dim3(M_max), dim3(256), 0, s, x, src_map, M_dev, M_max, d, eps, out);
}

// ------------------------------------------------------------------ per-row RoPE factors (transposed)
// The fused QKV epilogue owns one row per thread; with the factors stored [f][row] a warp's load of
// factor f for its 32 consecutive rows is one coalesced 128-B line instead of 32 scattered table rows.
__global__ void k_rope_rows(const RowInfo* __restrict__ rows, const int* __restrict__ M_dev, int M_max,
                            const float* __restrict__ rcos, const float* __restrict__ rsin, float* __restrict__ out,
                            int ld) {
  pdl_trigger();
  pdl_wait();
  const int M = live_rows(M_dev, M_max);
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < 64 * M_max; e += gridDim.x * blockDim.x) {
    const int f = e / M_max, r = e - f * M_max;
    if (r >= M) continue;
    const int p = rows[r].pos;
    out[(size_t)f * ld + r] = rcos[(size_t)p * 64 + f];
    out[(size_t)(64 + f) * ld + r] = rsin[(size_t)p * 64 + f];
  }
}

void launch_rope_rows(const RowInfo* rows, const int* M_dev, int M_max, const float* rcos, const float* rsin,
                      float* out, int ld, cudaStream_t s) {
  if (M_max <= 0) return;
  const int blocks = std::min(4 * num_sms(), (64 * M_max + 255) / 256);
  launch_pdl(k_rope_rows, dim3(blocks), dim3(256), 0, s, rows, M_dev, M_max, rcos, rsin, out, ld);
}

// ------------------------------------------------------------------ RoPE + paged KV store
// q, k rotated (rotate-half pairs (k, k+dh/2), angle pos*theta^(-2k/dh) from a host-built fp64
// table), rounded to bf16; k, v stored at the row's KV slot of the paged pool ("sparse KV fill",
// P:789).  Writing a committed block slot raises the invariant flag.
__global__ void k_rope_store(const float* __restrict__ qkv, const RowInfo* __restrict__ rows,
                             const int* __restrict__ M_dev, int M_max, int n_q_heads,
                             const float* __restrict__ rcos, const float* __restrict__ rsin,
                             const focus_req_state* __restrict__ st, KVView kv, bf16* __restrict__ out,
                             Counters* cnt) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x;
  if (r >= live_rows(M_dev, M_max)) return;
  const RowInfo ri = rows[r];
  const int dh = kv.head_dim, half = dh / 2, hkv = kv.n_kv_heads;
  const int nh = n_q_heads + 2 * hkv;
  const float* in = qkv + (size_t)r * nh * dh;
  bf16* o = out + (size_t)r * nh * dh;
  if (threadIdx.x == 0 && ri.j >= 0 && ((st[ri.slot].committed >> ri.j) & 1ull)) atomicExch(&cnt->invariant, 1);
  const float* cr = rcos + (size_t)ri.pos * half;
  const float* sr = rsin + (size_t)ri.pos * half;
  // rotated heads: q heads and k heads
  for (int e = threadIdx.x; e < (n_q_heads + hkv) * half; e += blockDim.x) {
    const int h = e / half, k = e % half;
    const float x1 = in[h * dh + k], x2 = in[h * dh + k + half];
    const float c = cr[k], sn = sr[k];
    const bf16 y1 = __float2bfloat16_rn(x1 * c - x2 * sn);
    const bf16 y2 = __float2bfloat16_rn(x2 * c + x1 * sn);
    o[h * dh + k] = y1;
    o[h * dh + k + half] = y2;
    if (h >= n_q_heads) {
      const size_t off = kv_offset(kv, ri.slot, ri.pos, h - n_q_heads);
      kv.K[off + k] = y1;
      kv.K[off + k + half] = y2;
    }
  }
  for (int e = threadIdx.x; e < hkv * dh; e += blockDim.x) {
    const int h = e / dh, c = e % dh;
    const bf16 v = __float2bfloat16_rn(in[(n_q_heads + hkv) * dh + e]);
    o[(n_q_heads + hkv) * dh + e] = v;
    kv.V[kv_offset(kv, ri.slot, ri.pos, h) + c] = v;
  }
}

void launch_rope_store(const float* qkv_f32, const RowInfo* rows, const int* M_dev, int M_max, int n_q_heads,
                       const float* rope_cos, const float* rope_sin, const focus_req_state* st, KVView kv,
                       bf16* qkv_out, Counters* cnt, cudaStream_t s) {
  if (M_max <= 0) return;
  launch_pdl(k_rope_store, dim3(M_max), dim3(256), 0, s, qkv_f32, rows, M_dev, M_max, n_q_heads, rope_cos, rope_sin, st, kv,
                                     qkv_out, cnt);
}

// ------------------------------------------------------------------ SwiGLU
// act[r][f] = bf16( silu(g) * u ), g/u read from the interleaved gate|up GEMM output.
__global__ void k_silu_mul(const float* __restrict__ gu, const int* __restrict__ M_dev, int M_max, int d_ff,
                           bf16* __restrict__ act) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x;
  if (r >= live_rows(M_dev, M_max)) return;
  const float* in = gu + (size_t)r * 2 * d_ff;
  for (int f = threadIdx.x; f < d_ff; f += blockDim.x) {
    const int c = (f / kGuGroup) * 2 * kGuGroup + f % kGuGroup;
    const float g = in[c], u = in[c + kGuGroup];
    act[(size_t)r * d_ff + f] = __float2bfloat16_rn(g / (1.0f + expf(-g)) * u);
  }
}

void launch_silu_mul(const float* gu, const int* M_dev, int M_max, int d_ff, bf16* act, cudaStream_t s) {
  if (M_max <= 0) return;
  launch_pdl(k_silu_mul, dim3(M_max), dim3(256), 0, s, gu, M_dev, M_max, d_ff, act);
}

// ------------------------------------------------------------------ compaction gather
// Dense S-rows from P-rows ("Gather"; App.E): residual (fp32) and the layer-1
// query block of the qkv row (bf16).
__global__ void k_gather_rows(const float* __restrict__ x, const bf16* __restrict__ qkv, int qkv_dim, int q_dim,
                              const int* __restrict__ src, const int* __restrict__ M_dev, int M_max, int d,
                              float* __restrict__ x_out, bf16* __restrict__ q_out) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x;
  if (r >= live_rows(M_dev, M_max)) return;
  const int sr = src[r];
  const float4* xi = reinterpret_cast<const float4*>(x + (size_t)sr * d);
  float4* xo = reinterpret_cast<float4*>(x_out + (size_t)r * d);
  for (int c = threadIdx.x; c < d / 4; c += blockDim.x) xo[c] = xi[c];
  if (q_out) {
    const uint4* qi = reinterpret_cast<const uint4*>(qkv + (size_t)sr * qkv_dim);
    uint4* qo = reinterpret_cast<uint4*>(q_out + (size_t)r * q_dim);
    for (int c = threadIdx.x; c < q_dim / 8; c += blockDim.x) qo[c] = qi[c];
  }
}

void launch_gather_rows(const float* x, const bf16* qkv, int qkv_dim, int q_dim, const int* src, const int* M_dev,
                        int M_max, int d, float* x_out, bf16* q_out, cudaStream_t s) {
  if (M_max <= 0) return;
  launch_pdl(k_gather_rows, dim3(M_max), dim3(256), 0, s, x, qkv, qkv_dim, q_dim, src, M_dev, M_max, d, x_out, q_out);
}

}  // namespace focus
