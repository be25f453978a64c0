// Block-diffusion paged attention with the fused Eq.2 importance epilogue (scaffolding SIMT
// version: CUDA-core FMA, online softmax, KV pages streamed through shared memory).
//
// One CTA = (request, query-row chunk, kv head).  Its query rows are G heads x up to 64/G block
// rows (GQA packing).  Keys: context [0, s) + block [s, s+B) (layers 0 / 1, A-K2/A-K3), context +
// block [s, s+R'] (layers >= 2, A-K1), or causal [0, pos] (prefill, A-K5).
// Importance (Eq.2; App.E): the scaled block scores S_ij = q_i.k_j/sqrt(dh), j in the
// block, are kept in shared memory while the key loop passes the block; after the loop each query
// row (i in P, head h) is MaxPool1D'ed along j with -inf outside P (A-I3, A-I5), softmax-normalised
// over P and summed over rows and heads in a fixed order -> one partial I per (request, chunk, kv
// head); the selection kernel adds the partials in a fixed order (deterministic).
#include <math_constants.h>

#include "common.cuh"

namespace focus {

template <int DH>
__global__ void __launch_bounds__(128) k_attention(AttnArgs a) {
  pdl_trigger();
  pdl_wait();
  constexpr int QR = kAttnQRows, KT = kAttnKT;
  constexpr int DPL = DH >= 32 ? DH / 32 : 1;          // head dims per lane in the PV product
  extern __shared__ __align__(16) float smem[];
  float* qs = smem;                                     // [QR][DH]
  float* ks = qs + QR * DH;                             // [KT][DH+1]
  float* vs = ks + KT * (DH + 1);                       // [KT][DH]
  float* sc = vs + KT * DH;                             // [QR][64] block scores (importance)
  float* red = sc + QR * kMaxB;                         // [4][64]

  const int kvh = blockIdx.y;
  const int G = a.n_q_heads / a.kv.n_kv_heads;
  const int rpc = QR / G;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  int slot, r0, nr, kbeg = 0, kend, list_i = 0, chunk = 0, s0 = 0, pos0 = 0;
  uint64_t P = 0;
  bool want_imp = false;
  if (a.ext_mode == 2) {
    slot = a.prefill_slot;
    r0 = blockIdx.x * rpc;
    nr = min(rpc, a.prefill_rows - r0);
    if (nr <= 0) return;
    pos0 = a.prefill_pos0;
    kend = pos0 + r0 + nr;
  } else {
    list_i = blockIdx.x / a.n_chunks;
    chunk = blockIdx.x % a.n_chunks;
    slot = a.req_list[list_i];
    const focus_req_state& s = a.st[slot];
    const int rb = a.row_off[list_i], re = a.row_off[list_i + 1];
    r0 = rb + chunk * rpc;
    nr = min(rpc, re - r0);
    if (nr <= 0) return;
    s0 = s.s;
    P = s.P;
    want_imp = a.imp != nullptr && !s.flush;
    if (a.imp_only) {
      if (!want_imp) return;
      kbeg = s0;
      kend = s0 + a.B;
    } else {
      kend = a.ext_mode == 0 ? s0 + a.B : s0 + s.R_new + 1;
    }
  }
  const int nq = nr * G;

  // Q rows -> smem (fp32)
  for (int e = threadIdx.x; e < QR * DH; e += blockDim.x) {
    const int qi = e / DH, d = e % DH;
    float v = 0.f;
    if (qi < nq) {
      const int row = r0 + qi / G, h = kvh * G + qi % G;
      v = __bfloat162float(a.q[(size_t)row * a.ldq + h * DH + d]);
    }
    qs[e] = v;
  }

  float m[16], l[16], o[16][DPL];
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    m[r] = -CUDART_INF_F;
    l[r] = 0.f;
#pragma unroll
    for (int e = 0; e < DPL; ++e) o[r][e] = 0.f;
  }

  for (int k0 = kbeg; k0 < kend; k0 += KT) {
    __syncthreads();
    for (int e = threadIdx.x; e < KT * DH; e += blockDim.x) {
      const int kk = e / DH, d = e % DH, p = k0 + kk;
      float kv = 0.f, vv = 0.f;
      if (p < kend) {
        const size_t off = kv_offset(a.kv, slot, p, kvh) + d;
        kv = __bfloat162float(a.kv.K[off]);
        if (!a.imp_only) vv = __bfloat162float(a.kv.V[off]);
      }
      ks[kk * (DH + 1) + d] = kv;
      vs[kk * DH + d] = vv;
    }
    __syncthreads();
    const int p = k0 + lane;
    float sv[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const int qi = warp * 16 + r;
      float sdot = -CUDART_INF_F;
      bool valid = qi < nq && p < kend;
      if (a.ext_mode == 2) valid = valid && p <= pos0 + r0 + qi / G;
      if (valid) {
        float acc = 0.f;
        const float* qr = qs + qi * DH;
        const float* kr = ks + lane * (DH + 1);
#pragma unroll 16
        for (int d = 0; d < DH; ++d) acc = fmaf(qr[d], kr[d], acc);
        sdot = acc * a.scale;
        if (want_imp && p >= s0 && p < s0 + a.B) sc[qi * kMaxB + (p - s0)] = sdot;
      }
      sv[r] = sdot;
    }
    if (a.imp_only) continue;
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      if (warp * 16 + r >= nq) continue;   // warp-uniform
      float mt = sv[r];
      for (int off = 16; off; off >>= 1) mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, off));
      const float mn = fmaxf(m[r], mt);
      if (mn == -CUDART_INF_F) continue;
      const float corr = expf(m[r] - mn);
      const float pr = expf(sv[r] - mn);
      float ls = pr;
      for (int off = 16; off; off >>= 1) ls += __shfl_xor_sync(0xffffffffu, ls, off);
      l[r] = l[r] * corr + ls;
      m[r] = mn;
#pragma unroll
      for (int e = 0; e < DPL; ++e) o[r][e] *= corr;
#pragma unroll 8
      for (int kk = 0; kk < KT; ++kk) {
        const float pk = __shfl_sync(0xffffffffu, pr, kk);
#pragma unroll
        for (int e = 0; e < DPL; ++e) {
          const int d = lane * DPL + e;
          if (d < DH) o[r][e] = fmaf(pk, vs[kk * DH + d], o[r][e]);
        }
      }
    }
  }

  if (!a.imp_only) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const int qi = warp * 16 + r;
      if (qi >= nq) continue;
      const int row = r0 + qi / G, h = kvh * G + qi % G;
      const float inv = 1.0f / l[r];
#pragma unroll
      for (int e = 0; e < DPL; ++e) {
        const int d = lane * DPL + e;
        if (d < DH) a.out[(size_t)row * a.ldo + h * DH + d] = __float2bfloat16_rn(o[r][e] * inv);
      }
    }
  }

  if (!want_imp) return;
  __syncthreads();
  // ---- importance epilogue (Eq.2): per query row, pool + softmax over P, column sums.
  const int B = a.B, rad = a.mp_kernel / 2;
  float acc0 = 0.f, acc1 = 0.f;            // positions j = lane, lane + 32
  for (int r = 0; r < 16; ++r) {
    const int qi = warp * 16 + r;
    if (qi >= nq) break;
    float pj[2];
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const int j = lane + 32 * t;
      float v = -CUDART_INF_F;
      if (j < B && ((P >> j) & 1ull)) {
        const int lo = max(0, j - rad), hi = min(B - 1, j + rad);
        for (int jj = lo; jj <= hi; ++jj)
          if ((P >> jj) & 1ull) v = fmaxf(v, sc[qi * kMaxB + jj]);
      }
      pj[t] = v;
    }
    float mx = fmaxf(pj[0], pj[1]);
    for (int off = 16; off; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    const float e0 = pj[0] == -CUDART_INF_F ? 0.f : expf(pj[0] - mx);
    const float e1 = pj[1] == -CUDART_INF_F ? 0.f : expf(pj[1] - mx);
    float z = e0 + e1;
    for (int off = 16; off; off >>= 1) z += __shfl_xor_sync(0xffffffffu, z, off);
    acc0 += e0 / z;
    acc1 += e1 / z;
  }
  red[warp * kMaxB + lane] = acc0;
  red[warp * kMaxB + lane + 32] = acc1;
  __syncthreads();
  if (threadIdx.x < B) {
    const int j = threadIdx.x;
    float v = 0.f;
    for (int w = 0; w < 4; ++w) v += red[w * kMaxB + j];
    a.imp[(((size_t)list_i * a.n_chunks + chunk) * a.kv.n_kv_heads + kvh) * B + j] = v;
  }
}

template <int DH>
static void launch_attn_dh(const AttnArgs& a, cudaStream_t s) {
  constexpr int QR = kAttnQRows, KT = kAttnKT;
  const size_t smem = sizeof(float) * (QR * DH + KT * (DH + 1) + KT * DH + QR * kMaxB + 4 * kMaxB);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_attention<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  const int G = a.n_q_heads / a.kv.n_kv_heads;
  const int rpc = QR / G;
  dim3 grid(a.ext_mode == 2 ? (a.prefill_rows + rpc - 1) / rpc : a.n_req * a.n_chunks, a.kv.n_kv_heads);
  if (grid.x == 0) return;
  launch_pdl(k_attention<DH>, grid, dim3(128), smem, s, a);
}

void launch_attention(const AttnArgs& a, cudaStream_t s) {
  switch (a.kv.head_dim) {
    case 16: launch_attn_dh<16>(a, s); break;
    case 32: launch_attn_dh<32>(a, s); break;
    case 64: launch_attn_dh<64>(a, s); break;
    case 128: launch_attn_dh<128>(a, s); break;
    default: break;
  }
}

}  // namespace focus
