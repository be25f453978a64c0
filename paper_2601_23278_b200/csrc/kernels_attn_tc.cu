// Block-diffusion paged attention on the 5th-generation tensor cores (tcgen05 / TMEM / TMA), with
// the Eq.2 token-importance epilogue fused in (§3.1 Eq.2, App.E).
//
// Work unit = (request i of the call, query-row chunk, kv head, key split).  The unit's query rows
// are the G = Hq/Hkv heads of up to 128/G block rows (GQA packing: one K/V stream serves the whole
// group); they form one M = 128 MMA tile.  Keys (block-diffusion mask):
//   ext_mode 0  context [0, s) + the whole block [s, s+B)          (layer 0, layer-1 suffix; A-K2/A-K3)
//   ext_mode 1  context + block [s, s+R']                          (layers >= 2; A-K1)
//   ext_mode 2  causal prefill (row at position p sees [0, p])      (focus_kv_append; A-K5)
//   imp_only    block keys [s, s+B) only, no output                  (layer-1 importance, A-I8)
// Keys stream in 64-key tiles straight from the paged pool by TMA (no gather copy); a request's key
// range is cut into splits of `split_tiles` tiles so the persistent grid stays busy, and split
// partials (unnormalised O, running max, sum) are merged by the last-arriving split in split order
// (deterministic).
//
// Persistent CTA (one per SM), 384 threads, warp-specialised:
//   warp 0      TMA producer: K and V tiles (64 keys x head_dim, 128-B swizzle) into a 4-stage ring
//   warp 1      MMA issuer: S = Q K^T (M=128, N=64, K=head_dim) into a double-buffered TMEM S tile,
//               then O += P V (M=128, N=head_dim, K=64; V as an MN-major operand) into a
//               double-buffered TMEM O accumulator (one buffer per unit in flight)
//   warp 2      TMEM allocator
//   warp 3      Q loader: cp.async of the unit's q rows into a swizzled smem tile (double-buffered)
//   warps 4-7   softmax: one TMEM lane (= one query row) per thread; online softmax in the log2
//               domain with lazy O rescaling (only when the running max grows by > 8), P -> smem as
//               bf16; records the block-column scores for the importance epilogue
//   warps 8-11  epilogue: O / l -> bf16 output rows (or split partials + fixed-order merge)
// Query rows are spread over the 4 TMEM lane quadrants (row qi -> lane (qi%4)*32 + qi/4) so that the
// ~30-60 real rows of a decode unit use all four SM sub-partitions.
#include <math_constants.h>

#include "tc_ptx.cuh"

namespace focus {
namespace attn {

using namespace tc;

constexpr int KT = 64;            // keys per tile
constexpr int QR = 128;           // query rows per unit (MMA M)
constexpr int ST = 4;             // K/V pipeline stages
constexpr int NTHREADS = 384;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kRescaleThresh = 8.0f;   // log2 units

template <int DH>
struct Cfg {
  static constexpr int NH = DH / 64;                  // 64-column (128-B) halves of head_dim
  static constexpr int HALF_BYTES = QR * 128;         // one half of the Q tile (16 KB)
  static constexpr int Q_BYTES = NH * HALF_BYTES;
  static constexpr int KH_BYTES = KT * 128;           // one half of a K or V tile (8 KB)
  static constexpr int K_BYTES = NH * KH_BYTES;
  static constexpr int STAGE_BYTES = 2 * K_BYTES;     // K + V
  static constexpr int P_BYTES = QR * KT * 2;         // 16 KB
  static constexpr int TMEM_COLS = (2 * DH + 2 * KT) <= 256 ? 256 : 512;
  static constexpr int O_COL = 0;                     // O buffers at [0, DH), [DH, 2DH)
  static constexpr int S_COL = 2 * DH;                // S buffers at [2DH, 2DH+KT), [2DH+KT, 2DH+2KT)
  static constexpr uint32_t IDESC_QK = idesc_bf16(QR, KT, false, false);
  static constexpr uint32_t IDESC_PV = idesc_bf16(QR, DH, false, true);
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_KV = OFF_Q + 2 * Q_BYTES;
  static constexpr int OFF_P = OFF_KV + ST * STAGE_BYTES;
  static constexpr int OFF_BAR = OFF_P + P_BYTES;
  static constexpr int N_BARS = 2 * ST + 2 * 2 + 2 * 2 + 2 + 2 * 2 + 2;
  static constexpr int OFF_STAT = OFF_BAR + 8 * N_BARS + 8;
  static constexpr int OFF_RED = OFF_STAT + 2 * QR * 8;
  static constexpr int OFF_PRE = OFF_RED + 4 * kMaxB * 4;
  static constexpr int SMEM_BYTES = OFF_PRE + 2 * 1028 * 4 + 64 + 1024;
};

struct Unit {
  int i, chunk, kvh, sp, nsplit, slot, r0, nr, nq, kbeg, kend, t_lo, t_hi, s0, pos_base, pair;
  uint64_t P;
  bool want_imp;
};

// Tiles [t0, t1) of request list index i (or the prefill chunk) and its split count.
__device__ __forceinline__ void key_range(const AttnArgs& a, int i, int& kbeg, int& kend, int& s0) {
  const focus_req_state& s = a.st[a.req_list[i]];
  s0 = s.s;
  if (a.imp_only) { kbeg = s.s; kend = s.s + a.B; }
  else { kbeg = 0; kend = a.ext_mode == 0 ? s.s + a.B : s.s + s.R_new + 1; }
}

__device__ __forceinline__ int req_units(const AttnArgs& a, int i, int rpc, int& nsplit) {
  const int rows = a.row_off[i + 1] - a.row_off[i];
  nsplit = 0;
  if (rows <= 0) return 0;
  const focus_req_state& s = a.st[a.req_list[i]];
  if (a.imp_only && (a.imp == nullptr || s.flush)) return 0;
  int kbeg, kend, s0;
  key_range(a, i, kbeg, kend, s0);
  const int nt = (kend + KT - 1) / KT - kbeg / KT;
  nsplit = a.imp_only ? 1 : (nt + a.split_tiles - 1) / a.split_tiles;
  const int nch = (rows + rpc - 1) / rpc;
  return nch * a.kv.n_kv_heads * nsplit;
}

__device__ __forceinline__ Unit decode_unit(const AttnArgs& a, int u, const int* pre, const int* nsp, int n_ent, int G,
                                            int rpc) {
  Unit x;
  const int H = a.kv.n_kv_heads;
  if (a.ext_mode == 2) {
    x.i = 0;
    x.sp = 0;
    x.nsplit = 1;
    x.kvh = u % H;
    x.chunk = u / H;
    x.slot = a.prefill_slot;
    x.r0 = x.chunk * rpc;
    x.nr = min(rpc, a.prefill_rows - x.r0);
    x.kbeg = 0;
    x.kend = a.prefill_pos0 + x.r0 + x.nr;
    x.s0 = 0;
    x.P = 0;
    x.want_imp = false;
    x.pos_base = a.prefill_pos0 + x.r0;
  } else {
    int lo = 0, hi = n_ent - 1;                        // largest i with pre[i] <= u
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (pre[mid] <= u) lo = mid; else hi = mid - 1;
    }
    x.i = lo;
    int rem = u - pre[lo];
    x.nsplit = nsp[lo];
    x.sp = rem % x.nsplit;
    rem /= x.nsplit;
    x.kvh = rem % H;
    x.chunk = rem / H;
    x.slot = a.req_list[x.i];
    const focus_req_state& s = a.st[x.slot];
    const int rb = a.row_off[x.i], re = a.row_off[x.i + 1];
    x.r0 = rb + x.chunk * rpc;
    x.nr = min(rpc, re - x.r0);
    key_range(a, x.i, x.kbeg, x.kend, x.s0);
    x.P = s.P;
    x.want_imp = a.imp != nullptr && !s.flush && x.sp == x.nsplit - 1;
    x.pos_base = 0;
  }
  x.nq = x.nr * G;
  const int t0 = x.kbeg / KT, t1 = (x.kend + KT - 1) / KT;
  x.t_hi = t1 - (x.nsplit - 1 - x.sp) * a.split_tiles;
  x.t_lo = max(t0, x.t_hi - a.split_tiles);
  x.pair = (x.i * a.n_chunks + x.chunk) * H + x.kvh;
  return x;
}

template <int DH, bool IMP_ONLY>
__global__ void __launch_bounds__(NTHREADS, 1)
    k_attn_tc(const __grid_constant__ CUtensorMap mapK, const __grid_constant__ CUtensorMap mapV, AttnArgs a) {
  using C = Cfg<DH>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sQ = smem + C::OFF_Q;
  uint8_t* sKV = smem + C::OFF_KV;
  uint8_t* sP = smem + C::OFF_P;
  uint64_t* bars = (uint64_t*)(smem + C::OFF_BAR);
  uint64_t* kvfull = bars;                 // [ST]
  uint64_t* kvempty = bars + ST;           // [ST]
  uint64_t* qfull = bars + 2 * ST;         // [2]
  uint64_t* qempty = qfull + 2;            // [2]
  uint64_t* sfull = qempty + 2;            // [2]
  uint64_t* sfree = sfull + 2;             // [2]
  uint64_t* pfull = sfree + 2;             // [1]
  uint64_t* pvdone = pfull + 1;            // [1]
  uint64_t* ofull = pvdone + 1;            // [2]
  uint64_t* ofree = ofull + 2;             // [2]
  uint64_t* statfull = ofree + 2;          // [2]
  uint32_t* tmem_sh = (uint32_t*)(bars + C::N_BARS);
  int* flag_sh = (int*)(tmem_sh + 1);
  float2* stat = (float2*)(smem + C::OFF_STAT);   // [2][QR] (m_used, l)
  float* red = (float*)(smem + C::OFF_RED);       // [4][64]
  int* pre = (int*)(smem + C::OFF_PRE);           // [n_ent + 1]
  int* nsp = pre + 1028;                          // [n_ent]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int H = a.kv.n_kv_heads;
  const int G = a.n_q_heads / H;
  const int rpc = QR / G;

  // ---- unit table: per-request unit counts and their exclusive prefix (smem)
  const int n_ent = a.ext_mode == 2 ? 1 : a.n_req;
  if (a.ext_mode == 2) {
    if (threadIdx.x == 0) {
      nsp[0] = 1;
      pre[0] = 0;
      pre[1] = ((a.prefill_rows + rpc - 1) / rpc) * H;
    }
  } else {
    for (int i = threadIdx.x; i < n_ent; i += NTHREADS) {
      int ns;
      const int nu = req_units(a, i, rpc, ns);
      nsp[i] = ns;
      pre[i + 1] = nu;
    }
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < ST; ++i) { mbar_init(&kvfull[i], 1); mbar_init(&kvempty[i], 1); }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&qfull[i], 1); mbar_init(&qempty[i], 1);
      mbar_init(&sfull[i], 1); mbar_init(&sfree[i], 4);
      mbar_init(&ofull[i], 1); mbar_init(&ofree[i], 4);
      mbar_init(&statfull[i], 4);
    }
    mbar_init(pfull, 4);
    mbar_init(pvdone, 1);
    fence_barrier_init();
  }
  if (warp == 1 && lane == 0) {
    prefetch_map(&mapK);
    if (!IMP_ONLY) prefetch_map(&mapV);
  }
  if (warp == 2) tmem_alloc<C::TMEM_COLS>(tmem_sh);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (a.ext_mode != 2 && warp == 0) {             // exclusive scan of unit counts (warp 0)
    const int per = (n_ent + 31) / 32;
    const int b0 = min(n_ent, lane * per), b1 = min(n_ent, b0 + per);
    int loc = 0;
    for (int i = b0; i < b1; ++i) loc += pre[i + 1];
    int inc = loc;
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += v;
    }
    int run = inc - loc;
    for (int i = b0; i < b1; ++i) { const int c = pre[i + 1]; pre[i] = run; run += c; }
    if (lane == 31) pre[n_ent] = inc;
  }
  __syncthreads();
  const int total = pre[n_ent];
  const uint32_t tmem = *tmem_sh;

  if (warp == 0) {
    // ================================================================ TMA producer
    if (lane == 0) {
      const int ps = a.kv.page_size;
      const int pr = min(ps, KT);                  // keys per TMA box
      const size_t layer_rows = (size_t)a.kv_pages * H * ps;
      uint32_t g = 0;
      for (int u = blockIdx.x; u < total; u += gridDim.x) {
        const Unit x = decode_unit(a, u, pre, nsp, n_ent, G, rpc);
        for (int t = x.t_lo; t < x.t_hi; ++t, ++g) {
          const int stage = g % ST;
          mbar_wait(&kvempty[stage], ((g / ST) & 1) ^ 1);
          mbar_expect_tx(&kvfull[stage], IMP_ONLY ? C::K_BYTES : C::STAGE_BYTES);
          uint8_t* dK = sKV + stage * C::STAGE_BYTES;
          uint8_t* dV = dK + C::K_BYTES;
          for (int pc = 0; pc < KT / pr; ++pc) {
            const int pos = t * KT + pc * pr;
            const int pidx = min(pos / ps, a.kv.max_pages - 1);
            const int page = a.kv.page_table[(size_t)x.slot * a.kv.max_pages + pidx];
            const int row = (int)((size_t)a.layer * layer_rows + ((size_t)page * H + x.kvh) * ps + pos % ps);
#pragma unroll
            for (int h = 0; h < C::NH; ++h) {
              tma_load_2d(dK + h * C::KH_BYTES + pc * pr * 128, &mapK, &kvfull[stage], h * 64, row);
              if (!IMP_ONLY) tma_load_2d(dV + h * C::KH_BYTES + pc * pr * 128, &mapV, &kvfull[stage], h * 64, row);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ================================================================ MMA issuer
    if (lane == 0) {
      uint32_t g = 0, it = 0;
      // deferred PV of the previous tile (issued after the next QK so softmax overlaps the tensor pipe)
      bool pend = false;
      uint32_t p_g = 0, p_stage = 0, p_ob = 0, p_it = 0;
      bool p_first = false, p_last = false;
      auto issue_pv = [&]() {
        mbar_wait(pfull, p_g & 1);
        if (p_first) mbar_wait(&ofree[p_ob], ((p_it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + C::O_COL + p_ob * DH;
        const uint32_t pa = smem_u32(sP);
        const uint32_t vb = smem_u32(sKV + p_stage * C::STAGE_BYTES + C::K_BYTES);
#pragma unroll
        for (int kk = 0; kk < KT / 16; ++kk)
          mma_bf16(d, desc_kmajor_sw128(pa + kk * 32), desc_mnmajor_sw128(vb + kk * 16 * 128, C::KH_BYTES),
                   C::IDESC_PV, (p_first && kk == 0) ? 0u : 1u);
        mma_commit(&kvempty[p_stage]);
        mma_commit(pvdone);
        if (p_last) mma_commit(&ofull[p_ob]);
      };
      for (int u = blockIdx.x; u < total; u += gridDim.x, ++it) {
        const Unit x = decode_unit(a, u, pre, nsp, n_ent, G, rpc);
        const uint32_t ob = it & 1;
        mbar_wait(&qfull[ob], (it >> 1) & 1);
        tc_fence_after();
        const uint32_t qa = smem_u32(sQ + ob * C::Q_BYTES);
        for (int t = x.t_lo; t < x.t_hi; ++t, ++g) {
          const uint32_t stage = g % ST, sb = g & 1;
          mbar_wait(&kvfull[stage], (g / ST) & 1);
          mbar_wait(&sfree[sb], ((g >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t kb = smem_u32(sKV + stage * C::STAGE_BYTES);
          const uint32_t d = tmem + C::S_COL + sb * KT;
#pragma unroll
          for (int kk = 0; kk < DH / 16; ++kk) {
            const int h = kk >> 2, w = (kk & 3) * 32;
            mma_bf16(d, desc_kmajor_sw128(qa + h * C::HALF_BYTES + w), desc_kmajor_sw128(kb + h * C::KH_BYTES + w),
                     C::IDESC_QK, kk > 0 ? 1u : 0u);
          }
          mma_commit(&sfull[sb]);
          if (t + 1 == x.t_hi) mma_commit(&qempty[ob]);
          if (IMP_ONLY) {
            mma_commit(&kvempty[stage]);
            continue;
          }
          if (pend) issue_pv();
          pend = true;
          p_g = g; p_stage = stage; p_ob = ob; p_it = it;
          p_first = t == x.t_lo;
          p_last = t + 1 == x.t_hi;
        }
      }
      if (!IMP_ONLY && pend) issue_pv();
    }
  } else if (warp == 3) {
    // ================================================================ Q loader
    uint32_t it = 0;
    for (int u = blockIdx.x; u < total; u += gridDim.x, ++it) {
      const Unit x = decode_unit(a, u, pre, nsp, n_ent, G, rpc);
      const uint32_t ob = it & 1;
      mbar_wait(&qempty[ob], ((it >> 1) & 1) ^ 1);
      uint8_t* q = sQ + ob * C::Q_BYTES;
      constexpr int CPR = DH / 8;                  // 16-B chunks per row
      for (int idx = lane; idx < QR * CPR; idx += 32) {
        const int L = idx / CPR, cc = idx % CPR;
        const int h = cc >> 3, c = cc & 7;
        const int qi = (L & 31) * 4 + (L >> 5);
        uint8_t* dst = q + h * C::HALF_BYTES + sw128_off(L, c);
        if (qi < x.nq) {
          const int row = x.r0 + qi / G, head = x.kvh * G + qi % G;
          const bf16* src = a.q + (size_t)row * a.ldq + head * DH + h * 64 + c * 8;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
        } else {
          *reinterpret_cast<uint4*>(dst) = make_uint4(0, 0, 0, 0);
        }
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(&qfull[ob]);
    }
  } else if (warp >= 4 && warp < 8) {
    // ================================================================ softmax (+ importance)
    const int q4 = warp & 3;
    const int L = q4 * 32 + lane;                  // TMEM lane = smem Q/P row of this thread
    const int qi = lane * 4 + q4;                  // logical query row
    const float sl2 = a.scale * kLog2e;
    uint32_t g = 0, it = 0;
    for (int u = blockIdx.x; u < total; u += gridDim.x, ++it) {
      const Unit x = decode_unit(a, u, pre, nsp, n_ent, G, rpc);
      const uint32_t ob = it & 1;
      const bool active = q4 < x.nq;               // warp-uniform: quadrant has a real row
      const bool real = qi < x.nq;
      const int lim = a.ext_mode == 2 ? x.pos_base + qi / G : x.kend - 1;   // last visible key
      float m_used = -CUDART_INF_F, l = 0.f;
      float sc[kMaxB];
      for (int t = x.t_lo; t < x.t_hi; ++t, ++g) {
        const uint32_t sb = g & 1;
        mbar_wait(&sfull[sb], (g >> 1) & 1);
        tc_fence_after();
        uint32_t r[KT];
        if (active) {
          const uint32_t ta = tmem + ((uint32_t)(q4 * 32) << 16) + C::S_COL + sb * KT;
          tmem_ld32_nowait(ta, r);
          tmem_ld32_nowait(ta + 32, r + 32);
          tmem_wait_ld();
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sfree[sb]);
        const int k0 = t * KT;
        if (x.want_imp && real) {
#pragma unroll
          for (int c = 0; c < KT; ++c) {
            const int j = k0 + c - x.s0;
            if (j >= 0 && j < a.B) sc[j] = __uint_as_float(r[c]) * a.scale;
          }
        }
        if (IMP_ONLY) continue;
        // online softmax (log2 domain), lazy rescale
        float mt = -CUDART_INF_F;
        if (real) {
#pragma unroll
          for (int c = 0; c < KT; ++c) {
            const int p = k0 + c;
            const bool ok = p >= x.kbeg && p <= lim;
            const float v = ok ? __uint_as_float(r[c]) * sl2 : -CUDART_INF_F;
            r[c] = __float_as_uint(v);
            mt = fmaxf(mt, v);
          }
        }
        float alpha = 1.f;
        bool resc = false;
        if (mt > m_used + kRescaleThresh || (m_used == -CUDART_INF_F && mt > -CUDART_INF_F)) {
          const float mn = fmaxf(mt, m_used);
          alpha = exp2f(m_used - mn);             // 0 when m_used = -inf
          m_used = mn;
          resc = true;
        }
        uint32_t pk[KT / 2];
        float rs = 0.f;
        if (real) {
#pragma unroll
          for (int c = 0; c < KT; c += 2) {
            const float p0 = exp2f(__uint_as_float(r[c]) - m_used);
            const float p1 = exp2f(__uint_as_float(r[c + 1]) - m_used);
            const __nv_bfloat162 b2 = __floats2bfloat162_rn(p0, p1);
            const float2 bf = __bfloat1622float2(b2);
            rs += bf.x + bf.y;                      // sum what the tensor core will multiply
            pk[c / 2] = *reinterpret_cast<const uint32_t*>(&b2);
          }
        } else {
#pragma unroll
          for (int c = 0; c < KT / 2; ++c) pk[c] = 0u;
        }
        l = l * alpha + rs;
        if (g > 0) mbar_wait(pvdone, (g - 1) & 1);   // PV of the previous tile done: P free, O stable
        if (active) {
#pragma unroll
          for (int c = 0; c < 8; ++c)
            *reinterpret_cast<uint4*>(sP + sw128_off(L, c)) =
                make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
          const bool any = __any_sync(0xffffffffu, resc && real) && t > x.t_lo;
          if (any) {
            tc_fence_after();
            const float f = (resc && real) ? alpha : 1.f;
#pragma unroll 1
            for (int c0 = 0; c0 < DH; c0 += 32) {
              const uint32_t ta = tmem + ((uint32_t)(q4 * 32) << 16) + C::O_COL + ob * DH + c0;
              float v[32];
              tmem_ld32(ta, v);
#pragma unroll
              for (int e = 0; e < 32; ++e) v[e] *= f;
              tmem_st32(ta, v);
            }
            tmem_wait_st();
          }
        }
        fence_proxy_async();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(pfull);
      }
      if (!IMP_ONLY) {
        // per-row statistics for the epilogue (buffer ob is free once unit it-2's epilogue is done)
        mbar_wait(&ofree[ob], ((it >> 1) & 1) ^ 1);
        stat[ob * QR + L] = make_float2(m_used, l);
        __syncwarp();
        if (lane == 0) mbar_arrive(&statfull[ob]);
      }
      if (x.want_imp) {
        // Eq.2: per query row, MaxPool1D (k = mp_kernel, -inf outside P; A-I3, A-I5) over the block
        // scores, softmax over P, then the sum over rows and heads (fixed order: lanes, then warps).
        const int B = a.B, rad = a.mp_kernel / 2;
        float w[kMaxB];
        float mx = -CUDART_INF_F;
        if (real) {
          for (int j = 0; j < B; ++j) {
            float v = -CUDART_INF_F;
            if ((x.P >> j) & 1ull) {
              const int lo = max(0, j - rad), hi = min(B - 1, j + rad);
              for (int jj = lo; jj <= hi; ++jj)
                if ((x.P >> jj) & 1ull) v = fmaxf(v, sc[jj]);
            }
            w[j] = v;
            mx = fmaxf(mx, v);
          }
          float z = 0.f;
          for (int j = 0; j < B; ++j) {
            const float e = w[j] == -CUDART_INF_F ? 0.f : expf(w[j] - mx);
            w[j] = e;
            z += e;
          }
          for (int j = 0; j < B; ++j) w[j] = w[j] / z;
        }
        for (int j = 0; j < B; ++j) {
          float v = real ? w[j] : 0.f;
          for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
          if (lane == 0) red[q4 * kMaxB + j] = v;
        }
        named_bar(1, 128);
        if (warp == 4 && lane < 32) {
          for (int j = lane; j < B; j += 32) {
            const float v = ((red[j] + red[kMaxB + j]) + red[2 * kMaxB + j]) + red[3 * kMaxB + j];
            a.imp[(size_t)x.pair * B + j] = v;
          }
        }
        named_bar(1, 128);
      }
    }
  } else if (warp >= 8 && !IMP_ONLY) {
    // ================================================================ epilogue
    const int q4 = warp & 3;
    const int L = q4 * 32 + lane;
    const int qi = lane * 4 + q4;
    const int et = threadIdx.x - 256;
    uint32_t it = 0;
    for (int u = blockIdx.x; u < total; u += gridDim.x, ++it) {
      const Unit x = decode_unit(a, u, pre, nsp, n_ent, G, rpc);
      const uint32_t ob = it & 1;
      const bool active = q4 < x.nq, real = qi < x.nq;
      mbar_wait(&ofull[ob], (it >> 1) & 1);
      mbar_wait(&statfull[ob], (it >> 1) & 1);
      tc_fence_after();
      const float2 ml = stat[ob * QR + L];
      float o[DH];
      if (active) {
#pragma unroll
        for (int c0 = 0; c0 < DH; c0 += 32)
          tmem_ld32(tmem + ((uint32_t)(q4 * 32) << 16) + C::O_COL + ob * DH + c0, o + c0);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&ofree[ob]);
      const int row = x.r0 + qi / G, head = x.kvh * G + qi % G;
      if (x.nsplit == 1) {
        if (real) {
          const float inv = 1.0f / ml.y;
          bf16* dst = a.out + (size_t)row * a.ldo + head * DH;
#pragma unroll
          for (int c = 0; c < DH; c += 8) {
            uint4 pk;
            __nv_bfloat162 b0 = __floats2bfloat162_rn(o[c] * inv, o[c + 1] * inv);
            __nv_bfloat162 b1 = __floats2bfloat162_rn(o[c + 2] * inv, o[c + 3] * inv);
            __nv_bfloat162 b2 = __floats2bfloat162_rn(o[c + 4] * inv, o[c + 5] * inv);
            __nv_bfloat162 b3 = __floats2bfloat162_rn(o[c + 6] * inv, o[c + 7] * inv);
            pk.x = *reinterpret_cast<uint32_t*>(&b0); pk.y = *reinterpret_cast<uint32_t*>(&b1);
            pk.z = *reinterpret_cast<uint32_t*>(&b2); pk.w = *reinterpret_cast<uint32_t*>(&b3);
            *reinterpret_cast<uint4*>(dst + c) = pk;
          }
        }
      } else {
        // split partial -> workspace; the last-arriving split merges all partials in split order
        const size_t slot_floats = (size_t)QR * DH + 2 * QR;
        float* base = a.part + (size_t)x.pair * a.max_nsplit * slot_floats;
        if (real) {
          float* po = base + (size_t)x.sp * slot_floats + (size_t)qi * DH;
#pragma unroll
          for (int c = 0; c < DH; c += 4) __stcg(reinterpret_cast<float4*>(po + c), make_float4(o[c], o[c + 1], o[c + 2], o[c + 3]));
          __stcg(reinterpret_cast<float2*>(base + (size_t)x.sp * slot_floats + (size_t)QR * DH + 2 * qi), ml);
        }
        __threadfence();
        named_bar(2, 128);
        if (et == 0) *flag_sh = atomicAdd(&a.sem[x.pair], 1);
        named_bar(2, 128);
        const bool last = *flag_sh == x.nsplit - 1;
        named_bar(2, 128);
        if (last) {
          __threadfence();
          if (real) {
            float m = -CUDART_INF_F;
            for (int s = 0; s < x.nsplit; ++s) {
              const float2 v = __ldcg(reinterpret_cast<const float2*>(base + (size_t)s * slot_floats + (size_t)QR * DH + 2 * qi));
              m = fmaxf(m, v.x);
            }
            float lsum = 0.f;
#pragma unroll
            for (int c = 0; c < DH; ++c) o[c] = 0.f;
            for (int s = 0; s < x.nsplit; ++s) {
              const float2 v = __ldcg(reinterpret_cast<const float2*>(base + (size_t)s * slot_floats + (size_t)QR * DH + 2 * qi));
              const float f = v.x == -CUDART_INF_F ? 0.f : exp2f(v.x - m);
              lsum += v.y * f;
              const float* po = base + (size_t)s * slot_floats + (size_t)qi * DH;
#pragma unroll
              for (int c = 0; c < DH; c += 4) {
                const float4 pv = __ldcg(reinterpret_cast<const float4*>(po + c));
                o[c] += pv.x * f; o[c + 1] += pv.y * f; o[c + 2] += pv.z * f; o[c + 3] += pv.w * f;
              }
            }
            const float inv = 1.0f / lsum;
            bf16* dst = a.out + (size_t)row * a.ldo + head * DH;
#pragma unroll
            for (int c = 0; c < DH; c += 2)
              *reinterpret_cast<__nv_bfloat162*>(dst + c) = __floats2bfloat162_rn(o[c] * inv, o[c + 1] * inv);
          }
          if (et == 0) a.sem[x.pair] = 0;
        }
      }
    }
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_free<C::TMEM_COLS>(tmem);
  }
}

}  // namespace attn

bool attn_tc_supported(int head_dim, int page_size) {
  return (head_dim == 64 || head_dim == 128) && page_size >= 8 && page_size <= 4096 &&
         (page_size & (page_size - 1)) == 0;
}

// KV pool tensor maps: the whole pool (all layers) viewed as [rows][head_dim] bf16.
bool attn_tc_make_maps(const bf16* Kpool, const bf16* Vpool, size_t rows, int head_dim, int page_size,
                       CUtensorMap* mk, CUtensorMap* mv) {
  const uint32_t box_rows = (uint32_t)std::min(page_size, attn::KT);
  return make_tma_2d_bf16(Kpool, rows, head_dim, head_dim, 64, box_rows, mk) &&
         make_tma_2d_bf16(Vpool, rows, head_dim, head_dim, 64, box_rows, mv);
}

template <int DH, bool IMP>
static void launch_tc(const CUtensorMap& mk, const CUtensorMap& mv, const AttnArgs& a, int grid, cudaStream_t s) {
  constexpr int smem = attn::Cfg<DH>::SMEM_BYTES;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn::k_attn_tc<DH, IMP>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  attn::k_attn_tc<DH, IMP><<<grid, attn::NTHREADS, smem, s>>>(mk, mv, a);
}

void launch_attention_tc(const CUtensorMap& mk, const CUtensorMap& mv, const AttnArgs& a, cudaStream_t s) {
  const int G = a.n_q_heads / a.kv.n_kv_heads;
  const int rpc = attn::QR / G;
  int max_units;
  if (a.ext_mode == 2) max_units = ((a.prefill_rows + rpc - 1) / rpc) * a.kv.n_kv_heads;
  else max_units = a.n_req * a.n_chunks * a.kv.n_kv_heads * (a.imp_only ? 1 : a.max_nsplit);
  if (max_units <= 0) return;
  const int grid = std::max(1, std::min(num_sms(), max_units));
  if (a.kv.head_dim == 128) {
    if (a.imp_only) launch_tc<128, true>(mk, mv, a, grid, s); else launch_tc<128, false>(mk, mv, a, grid, s);
  } else {
    if (a.imp_only) launch_tc<64, true>(mk, mv, a, grid, s); else launch_tc<64, false>(mk, mv, a, grid, s);
  }
}

}  // namespace focus
