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
//   warp 0 / 2  TMA producers: K tiles / V tiles (64 keys x head_dim, 128-B swizzle) into a 4-slot K
//               ring (freed when QK^T completes) and a 3-slot V ring (freed when PV completes)
//   warp 1      MMA issuer: S = Q K^T (M=128, N=64, K=head_dim) into a double-buffered TMEM S tile,
//               then O += P V (M=128, N=head_dim, K=64; V as an MN-major operand) into a
//               double-buffered TMEM O accumulator (one buffer per unit in flight)
//   warp 3      TMEM allocator + Q loader: cp.async of the unit's q rows into a swizzled smem tile (double-buffered)
//   warps 4-7   softmax: warp 4+q owns TMEM lane quadrant q and reads its (<= 32) real rows 16 lanes
//               at a time (16x256b shape: 4 threads per row, 16 columns each); online softmax in the
//               log2 domain with lazy O rescaling (only when the running max grows by > 8), P -> a
//               double-buffered smem tile as bf16; block-column scores -> per-CTA scratch for the
//               importance epilogue
//   warps 8-11  epilogue: O / l -> bf16 output rows (or split partials + fixed-order merge)
// Q tile lane L = g * (128/G) + r holds query head g of block row r (G <= 4), so with G = 4 every TMEM
// lane quadrant (SM sub-partition) gets one head's rows and the ~30-60 real rows of a decode unit
// keep all four softmax warps busy.
#include <math_constants.h>

#include "tc_ptx.cuh"

namespace focus {
namespace attn {

using namespace tc;

constexpr int KT = 64;            // keys per tile
constexpr int QR = 128;           // query rows per unit (MMA M)
constexpr int SK = 4;             // K ring slots (released when QK^T completes)
constexpr int SV = 3;             // V ring slots (released when PV completes)
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
  static constexpr int P_BYTES = QR * KT * 2;         // 16 KB
  static constexpr int TMEM_COLS = (2 * DH + 2 * KT) <= 256 ? 256 : 512;
  static constexpr int O_COL = 0;                     // O buffers at [0, DH), [DH, 2DH)
  static constexpr int S_COL = 2 * DH;                // S buffers at [2DH, 2DH+KT), [2DH+KT, 2DH+2KT)
  static constexpr uint32_t IDESC_QK = idesc_bf16(QR, KT, false, false);
  static constexpr uint32_t IDESC_PV = idesc_bf16(QR, DH, false, true);
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + 2 * Q_BYTES;
  static constexpr int OFF_V = OFF_K + SK * K_BYTES;
  static constexpr int OFF_P = OFF_V + SV * K_BYTES;
  static constexpr int OFF_BAR = OFF_P + 2 * P_BYTES;
  static constexpr int N_BARS = 2 * SK + 2 * SV + 9 * 2;
  static constexpr int OFF_STAT = OFF_BAR + 8 * N_BARS + 8;
  static constexpr int OFF_RED = OFF_STAT + 2 * QR * 8;
  static constexpr int OFF_PRE = OFF_RED + 4 * kMaxB * 4;
  static constexpr int SMEM_BYTES = OFF_PRE + 2 * 1028 * 4 + 64 + 1024;
};

// debug trace: role r of this CTA appends clock64 stamps (event kind in the top 8 bits)
struct Tracer {
  unsigned long long* p;
  int n;
  __device__ __forceinline__ Tracer(unsigned long long* base, int role) : p(base ? base + ((size_t)blockIdx.x * 8 + role) * kTraceEv : nullptr), n(0) {}
  __device__ __forceinline__ void ev(int kind) {
    if (p && n < kTraceEv) p[n++] = ((unsigned long long)kind << 56) | (clock64() & ((1ull << 56) - 1));
  }
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
  // tiles split evenly; the last split (which holds the block tiles) gets the larger share
  const int t0 = x.kbeg / KT, nt = (x.kend + KT - 1) / KT - t0;
  x.t_lo = t0 + (x.sp * nt) / x.nsplit;
  x.t_hi = t0 + ((x.sp + 1) * nt) / x.nsplit;
  x.pair = (x.i * a.n_chunks + x.chunk) * H + x.kvh;
  return x;
}

template <int DH, bool IMP_ONLY>
__global__ void __launch_bounds__(NTHREADS, 1)
    k_attn_tc(const __grid_constant__ CUtensorMap mapK, const __grid_constant__ CUtensorMap mapV,
              const __grid_constant__ CUtensorMap mapQ, AttnArgs a) {
  using C = Cfg<DH>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sQ = smem + C::OFF_Q;
  uint8_t* sK = smem + C::OFF_K;
  uint8_t* sV = smem + C::OFF_V;
  uint8_t* sP = smem + C::OFF_P;
  uint64_t* bars = (uint64_t*)(smem + C::OFF_BAR);
  uint64_t* kfull = bars;                  // [SK]
  uint64_t* kempty = kfull + SK;           // [SK]
  uint64_t* vfull = kempty + SK;           // [SV]
  uint64_t* vempty = vfull + SV;           // [SV]
  uint64_t* qfull = vempty + SV;           // [2]
  uint64_t* qempty = qfull + 2;            // [2]
  uint64_t* sfull = qempty + 2;            // [2]
  uint64_t* sfree = sfull + 2;             // [2]
  uint64_t* pfull = sfree + 2;             // [2] (per P buffer)
  uint64_t* pvdone = pfull + 2;            // [2] (per P buffer)
  uint64_t* ofull = pvdone + 2;            // [2]
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
    for (int i = 0; i < SK; ++i) { mbar_init(&kfull[i], 1); mbar_init(&kempty[i], 1); }
    for (int i = 0; i < SV; ++i) { mbar_init(&vfull[i], 1); mbar_init(&vempty[i], 1); }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&qfull[i], 1); mbar_init(&qempty[i], 1);
      mbar_init(&sfull[i], 1); mbar_init(&sfree[i], 4);
      mbar_init(&ofull[i], 1); mbar_init(&ofree[i], 4);
      mbar_init(&statfull[i], 4);
    }
    for (int i = 0; i < 2; ++i) { mbar_init(&pfull[i], 4); mbar_init(&pvdone[i], 1); }
    fence_barrier_init();
  }
  if (warp == 1 && lane == 0) {
    prefetch_map(&mapQ);
    prefetch_map(&mapK);
    if (!IMP_ONLY) prefetch_map(&mapV);
  }
  if (warp == 3) tmem_alloc<C::TMEM_COLS>(tmem_sh);
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
  if (threadIdx.x == 0 && a.trace) a.trace[((size_t)blockIdx.x * 8 + 7) * kTraceEv] = clock64();
  const int total = pre[n_ent];
  const uint32_t tmem = *tmem_sh;

  if (warp == 0 || (warp == 2 && !IMP_ONLY)) {
    // ================================================================ TMA producers
    // warp 0 lane 0 streams K tiles, warp 2 lane 0 streams V tiles (separate rings: K is consumed by
    // QK^T about two tiles before V is consumed by PV, so each ring prefetches its own distance)
    if (lane == 0) {
      const bool isK = warp == 0;
      const int NS = isK ? SK : SV;
      uint64_t* fullb = isK ? kfull : vfull;
      uint64_t* emptyb = isK ? kempty : vempty;
      uint8_t* ring = isK ? sK : sV;
      const CUtensorMap* map = isK ? &mapK : &mapV;
      const int ps = a.kv.page_size;
      const int pr = min(ps, KT);                  // keys per TMA box
      const size_t layer_rows = (size_t)a.kv_pages * H * ps;
      uint32_t g = 0;
      Tracer tr(a.trace, isK ? 0 : 1);
      for (int u = blockIdx.x; u < total; u += gridDim.x) {
        tr.ev(0);
        const Unit x = decode_unit(a, u, pre, nsp, n_ent, G, rpc);
        tr.ev(9);
        for (int t = x.t_lo; t < x.t_hi; ++t, ++g) {
          const int slot = g % NS;
          mbar_wait(&emptyb[slot], ((g / NS) & 1) ^ 1);
          tr.ev(1);
          mbar_expect_tx(&fullb[slot], C::K_BYTES);
          uint8_t* dst = ring + slot * C::K_BYTES;
          for (int pc = 0; pc < KT / pr; ++pc) {
            const int pos = t * KT + pc * pr;
            const int pidx = min(pos / ps, a.kv.max_pages - 1);
            const int page = a.kv.page_table[(size_t)x.slot * a.kv.max_pages + pidx];
            const int row = (int)((size_t)a.layer * layer_rows + ((size_t)page * H + x.kvh) * ps + pos % ps);
#pragma unroll
            for (int h = 0; h < C::NH; ++h) tma_load_2d(dst + h * C::KH_BYTES + pc * pr * 128, map, &fullb[slot], h * 64, row);
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
      uint32_t p_g = 0, p_ob = 0, p_it = 0;
      bool p_first = false, p_last = false;
      auto issue_pv = [&]() {
        const uint32_t pb = p_g & 1;
        mbar_wait(&pfull[pb], (p_g >> 1) & 1);
        if (p_first) mbar_wait(&ofree[p_ob], ((p_it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + C::O_COL + p_ob * DH;
        const uint32_t pa = smem_u32(sP + pb * C::P_BYTES);
        const uint32_t vs = p_g % SV;
        mbar_wait(&vfull[vs], (p_g / SV) & 1);
        tc_fence_after();
        const uint32_t vb = smem_u32(sV + vs * C::K_BYTES);
#pragma unroll
        for (int kk = 0; kk < KT / 16; ++kk)
          mma_bf16(d, desc_kmajor_sw128(pa + kk * 32), desc_mnmajor_sw128(vb + kk * 16 * 128, C::KH_BYTES),
                   C::IDESC_PV, (p_first && kk == 0) ? 0u : 1u);
        mma_commit(&vempty[vs]);
        mma_commit(&pvdone[pb]);
        if (p_last) mma_commit(&ofull[p_ob]);
      };
      Tracer tr(a.trace, 2);
      for (int u = blockIdx.x; u < total; u += gridDim.x, ++it) {
        tr.ev(0);
        const Unit x = decode_unit(a, u, pre, nsp, n_ent, G, rpc);
        tr.ev(9);
        const uint32_t ob = it & 1;
        mbar_wait(&qfull[ob], (it >> 1) & 1);
        tr.ev(2);
        tc_fence_after();
        const uint32_t qa = smem_u32(sQ + ob * C::Q_BYTES);
        for (int t = x.t_lo; t < x.t_hi; ++t, ++g) {
          const uint32_t ks = g % SK, sb = g & 1;
          mbar_wait(&kfull[ks], (g / SK) & 1);
          tr.ev(3);
          mbar_wait(&sfree[sb], ((g >> 1) & 1) ^ 1);
          tr.ev(4);
          tc_fence_after();
          const uint32_t kb = smem_u32(sK + ks * C::K_BYTES);
          const uint32_t d = tmem + C::S_COL + sb * KT;
#pragma unroll
          for (int kk = 0; kk < DH / 16; ++kk) {
            const int h = kk >> 2, w = (kk & 3) * 32;
            mma_bf16(d, desc_kmajor_sw128(qa + h * C::HALF_BYTES + w), desc_kmajor_sw128(kb + h * C::KH_BYTES + w),
                     C::IDESC_QK, kk > 0 ? 1u : 0u);
          }
          mma_commit(&sfull[sb]);
          mma_commit(&kempty[ks]);
          if (t + 1 == x.t_hi) mma_commit(&qempty[ob]);
          if (IMP_ONLY) continue;
          if (pend) { issue_pv(); tr.ev(5); }
          pend = true;
          p_g = g; p_ob = ob; p_it = it;
          p_first = t == x.t_lo;
          p_last = t + 1 == x.t_hi;
        }
      }
      if (!IMP_ONLY && pend) issue_pv();
    }
  } else if (warp == 3) {
    // ================================================================ Q loader (TMA)
    // Q tile lane L holds head g = L / rpc of block row r = L % rpc of the unit: for each head and
    // 64-column half, one box of rpc consecutive q rows (rows past the unit belong to other requests
    // or are zero-filled out of bounds; their outputs are discarded).
    if (lane == 0) {
      uint32_t it = 0;
      Tracer tr(a.trace, 3);
      for (int u = blockIdx.x; u < total; u += gridDim.x, ++it) {
        tr.ev(0);
        const Unit x = decode_unit(a, u, pre, nsp, n_ent, G, rpc);
        tr.ev(9);
        const uint32_t ob = it & 1;
        mbar_wait(&qempty[ob], ((it >> 1) & 1) ^ 1);
        tr.ev(1);
        mbar_expect_tx(&qfull[ob], C::Q_BYTES);
        uint8_t* q = sQ + ob * C::Q_BYTES;
        for (int gq = 0; gq < G; ++gq)
#pragma unroll
          for (int h = 0; h < C::NH; ++h)
            tma_load_2d(q + h * C::HALF_BYTES + gq * rpc * 128, &mapQ, &qfull[ob], (x.kvh * G + gq) * DH + h * 64, x.r0);
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // ================================================================ softmax (+ importance)
    // Warp 4+q owns TMEM lane quadrant q.  Its real rows sit in lanes 0.. of the quadrant; they are
    // read 16 lanes at a time with the 16x256b shape, so 4 threads share a row (16 of the 64 columns
    // each) and every lane of the warp works on a real row.
    const int q4 = warp & 3;
    const int t0 = lane & 3, t1 = lane >> 2;
    const float sl2 = a.scale * kLog2e;
    float* scr = a.imp_scratch + (size_t)blockIdx.x * QR * kMaxB;
    uint32_t g = 0, it = 0;
    Tracer tr(warp == 4 && lane == 0 ? a.trace : nullptr, 4);
    for (int u = blockIdx.x; u < total; u += gridDim.x, ++it) {
      tr.ev(0);
      const Unit x = decode_unit(a, u, pre, nsp, n_ent, G, rpc);
      tr.ev(9);
      const uint32_t ob = it & 1;
      const int rows_q = min(32, max(0, x.nr - (32 * q4) % rpc));  // real rows: a prefix of the quadrant
      const int ngrp = rows_q > 16 ? 2 : (rows_q > 0 ? 1 : 0);      // warp-uniform
      const int lim_min = a.ext_mode == 2 ? x.pos_base : x.kend - 1;
      int lim[2][2];
      bool real[2][2];
#pragma unroll
      for (int gr = 0; gr < 2; ++gr)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int rr = (q4 * 32 + gr * 16 + t1 + 8 * h) % rpc;   // block row of this lane
          real[gr][h] = rr < x.nr;
          lim[gr][h] = a.ext_mode == 2 ? x.pos_base + rr : x.kend - 1;
        }
      float m_used[2][2], l[2][2];
#pragma unroll
      for (int gr = 0; gr < 2; ++gr)
#pragma unroll
        for (int h = 0; h < 2; ++h) { m_used[gr][h] = -CUDART_INF_F; l[gr][h] = 0.f; }
      for (int t = x.t_lo; t < x.t_hi; ++t, ++g) {
        const uint32_t sb = g & 1;
        mbar_wait(&sfull[sb], (g >> 1) & 1);
        tr.ev(1);
        tc_fence_after();
        uint32_t r[2][32];
#pragma unroll
        for (int gr = 0; gr < 2; ++gr)
          if (gr < ngrp)
            tmem_ld16x256_x8(tmem + ((uint32_t)(q4 * 32 + gr * 16) << 16) + C::S_COL + sb * KT, r[gr]);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sfree[sb]);
        const int k0 = t * KT;
        if (x.want_imp) {                          // block-column scores for the Eq.2 epilogue
#pragma unroll
          for (int gr = 0; gr < 2; ++gr)
            if (gr < ngrp)
#pragma unroll
              for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int j = 0; j < 8; ++j)
#pragma unroll
                  for (int e = 0; e < 2; ++e) {
                    const int jb = k0 + 8 * j + 2 * t0 + e - x.s0;
                    if (real[gr][h] && jb >= 0 && jb < a.B)
                      scr[(q4 * 32 + gr * 16 + t1 + 8 * h) * kMaxB + jb] = __uint_as_float(r[gr][4 * j + 2 * h + e]) * a.scale;
                  }
        }
        if (IMP_ONLY) continue;
        const bool full = k0 >= x.kbeg && k0 + KT - 1 <= lim_min;
        const uint32_t pb = g & 1;
        uint32_t pk[2][2][8];
        bool resc_any = false;
        float alpha[2][2];
#pragma unroll
        for (int gr = 0; gr < 2; ++gr) {
          if (gr >= ngrp) continue;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            float mx = -CUDART_INF_F;
            if (!full) {
#pragma unroll
              for (int j = 0; j < 8; ++j)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                  const int c = k0 + 8 * j + 2 * t0 + e;
                  if (c < x.kbeg || c > lim[gr][h]) r[gr][4 * j + 2 * h + e] = __float_as_uint(-CUDART_INF_F);
                }
            }
#pragma unroll
            for (int j = 0; j < 8; ++j)
              mx = fmaxf(mx, fmaxf(__uint_as_float(r[gr][4 * j + 2 * h]), __uint_as_float(r[gr][4 * j + 2 * h + 1])));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
            const float mt = mx * sl2;
            float al = 1.f;
            float mu = m_used[gr][h];
            if (mt > mu + kRescaleThresh || (mu == -CUDART_INF_F && mt > -CUDART_INF_F)) {
              const float mn = fmaxf(mt, mu);
              al = ex2(mu - mn);                   // 0 when mu = -inf
              m_used[gr][h] = mn;
              resc_any |= real[gr][h] && t > x.t_lo;
            }
            alpha[gr][h] = al;
            const float nm = m_used[gr][h] == -CUDART_INF_F ? 0.f : -m_used[gr][h];
            float sum = 0.f;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              float p0 = ex2(fmaf(__uint_as_float(r[gr][4 * j + 2 * h]), sl2, nm));
              float p1 = ex2(fmaf(__uint_as_float(r[gr][4 * j + 2 * h + 1]), sl2, nm));
              if (!real[gr][h]) { p0 = 0.f; p1 = 0.f; }
              sum += p0 + p1;
              const __nv_bfloat162 b2 = __floats2bfloat162_rn(p0, p1);
              pk[gr][h][j] = *reinterpret_cast<const uint32_t*>(&b2);
            }
            l[gr][h] = l[gr][h] * al + sum;
          }
        }
        resc_any = __any_sync(0xffffffffu, resc_any);
        tr.ev(2);
        if (g >= 2) mbar_wait(&pvdone[pb], ((g >> 1) & 1) ^ 1);   // PV of tile g-2 done: P buffer free
        tr.ev(3);
        const uint32_t pbase = smem_u32(sP + pb * C::P_BYTES);
#pragma unroll
        for (int gr = 0; gr < 2; ++gr) {
          if (gr >= ngrp) continue;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int Lr = q4 * 32 + gr * 16 + t1 + 8 * h;
#pragma unroll
            for (int j = 0; j < 8; ++j) sts32(pbase + sw128_off(Lr, j) + 4 * t0, pk[gr][h][j]);
          }
        }
        if (resc_any) {                            // O *= alpha for rows whose running max moved (lazy)
          mbar_wait(&pvdone[(g - 1) & 1], ((g - 1) >> 1) & 1);   // PV of tile g-1 done: O stable
          tc_fence_after();
#pragma unroll
          for (int gr = 0; gr < 2; ++gr) {
            if (gr >= ngrp) continue;
#pragma unroll 1
            for (int c0 = 0; c0 < DH; c0 += 64) {
              const uint32_t ta = tmem + ((uint32_t)(q4 * 32 + gr * 16) << 16) + C::O_COL + ob * DH + c0;
              uint32_t v[32];
              tmem_ld16x256_x8(ta, v);
              tmem_wait_ld();
#pragma unroll
              for (int j = 0; j < 8; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                  for (int e = 0; e < 2; ++e)
                    v[4 * j + 2 * h + e] = __float_as_uint(__uint_as_float(v[4 * j + 2 * h + e]) * alpha[gr][h]);
              tmem_st16x256_x8(ta, v);
            }
          }
          tmem_wait_st();
        }
        fence_proxy_async();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&pfull[pb]);
        tr.ev(4);
      }
      if (!IMP_ONLY) {
        // row sums over the 4 threads of a row; per-row statistics for the epilogue (buffer ob is
        // free once the epilogue of unit it-2 is done)
        mbar_wait(&ofree[ob], ((it >> 1) & 1) ^ 1);
#pragma unroll
        for (int gr = 0; gr < 2; ++gr)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            float ls = l[gr][h];
            ls += __shfl_xor_sync(0xffffffffu, ls, 1);
            ls += __shfl_xor_sync(0xffffffffu, ls, 2);
            if (gr < ngrp && t0 == 0) stat[ob * QR + q4 * 32 + gr * 16 + t1 + 8 * h] = make_float2(m_used[gr][h], ls);
          }
        __syncwarp();
        if (lane == 0) mbar_arrive(&statfull[ob]);
      }
      if (x.want_imp) {
        // Eq.2: per query row, MaxPool1D (k = mp_kernel, -inf outside P; A-I3, A-I5) over the block
        // scores, softmax over P, then the sum over rows and heads (fixed order: lanes, then warps).
        __syncwarp();
        const int B = a.B, rad = a.mp_kernel / 2;
        const int L = q4 * 32 + lane;
        const bool rr = L % rpc < x.nr;
        const float* sc = scr + L * kMaxB;
        float w[kMaxB];
        float mx = -CUDART_INF_F;
        if (rr) {
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
          float v = rr ? w[j] : 0.f;
          for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
          if (lane == 0) red[q4 * kMaxB + j] = v;
        }
        named_bar(1, 128);
        if (warp == 4) {
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
    const int et = threadIdx.x - 256;
    uint32_t it = 0;
    Tracer tr(warp == 8 && lane == 0 ? a.trace : nullptr, 5);
    for (int u = blockIdx.x; u < total; u += gridDim.x, ++it) {
      tr.ev(0);
      const Unit x = decode_unit(a, u, pre, nsp, n_ent, G, rpc);
      tr.ev(9);
      const uint32_t ob = it & 1;
      const bool active = (32 * q4) % rpc < x.nr, real = L % rpc < x.nr;
      const int qi = L;                            // partial-buffer row index
      mbar_wait(&ofull[ob], (it >> 1) & 1);
      mbar_wait(&statfull[ob], (it >> 1) & 1);
      tr.ev(1);
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
      const int row = x.r0 + L % rpc, head = x.kvh * G + L / rpc;
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
  if (warp == 3) {
    tc_fence_after();
    tmem_free<C::TMEM_COLS>(tmem);
  }
}

}  // namespace attn

bool attn_tc_supported(int head_dim, int page_size, int group) {
  return (head_dim == 64 || head_dim == 128) && page_size >= 8 && page_size <= 4096 &&
         (page_size & (page_size - 1)) == 0 && (group == 1 || group == 2 || group == 4);
}

// Query-row tensor map: q buffer [rows][ld] bf16, box = 64 columns x (128 / group) rows.
bool attn_tc_make_qmap(const bf16* q, size_t rows, int ld, int group, CUtensorMap* mq) {
  return make_tma_2d_bf16(q, rows, ld, ld, 64, 128 / group, mq);
}

// KV pool tensor maps: the whole pool (all layers) viewed as [rows][head_dim] bf16.
bool attn_tc_make_maps(const bf16* Kpool, const bf16* Vpool, size_t rows, int head_dim, int page_size,
                       CUtensorMap* mk, CUtensorMap* mv) {
  const uint32_t box_rows = (uint32_t)std::min(page_size, attn::KT);
  return make_tma_2d_bf16(Kpool, rows, head_dim, head_dim, 64, box_rows, mk) &&
         make_tma_2d_bf16(Vpool, rows, head_dim, head_dim, 64, box_rows, mv);
}

template <int DH, bool IMP>
static void launch_tc(const CUtensorMap& mk, const CUtensorMap& mv, const CUtensorMap& mq, const AttnArgs& a, int grid,
                      cudaStream_t s) {
  constexpr int smem = attn::Cfg<DH>::SMEM_BYTES;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn::k_attn_tc<DH, IMP>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  attn::k_attn_tc<DH, IMP><<<grid, attn::NTHREADS, smem, s>>>(mk, mv, mq, a);
}

void launch_attention_tc(const CUtensorMap& mk, const CUtensorMap& mv, const CUtensorMap& mq, const AttnArgs& a,
                         cudaStream_t s) {
  const int G = a.n_q_heads / a.kv.n_kv_heads;
  const int rpc = attn::QR / G;
  int max_units;
  if (a.ext_mode == 2) max_units = ((a.prefill_rows + rpc - 1) / rpc) * a.kv.n_kv_heads;
  else max_units = a.n_req * a.n_chunks * a.kv.n_kv_heads * (a.imp_only ? 1 : a.max_nsplit);
  if (max_units <= 0) return;
  const int grid = std::max(1, std::min(num_sms(), max_units));
  if (a.kv.head_dim == 128) {
    if (a.imp_only) launch_tc<128, true>(mk, mv, mq, a, grid, s); else launch_tc<128, false>(mk, mv, mq, a, grid, s);
  } else {
    if (a.imp_only) launch_tc<64, true>(mk, mv, mq, a, grid, s); else launch_tc<64, false>(mk, mv, mq, a, grid, s);
  }
}

}  // namespace focus
