// Block-diffusion paged attention on the 5th-generation tensor cores (tcgen05 / TMEM / TMA), with
// the Eq.2 token-importance epilogue fused in (§3.1 Eq.2, App.E).
//
// Decode attention here has few query rows per (request, kv head) — the G = Hq/Hkv heads of the
// retained block rows, ~30-60 at the SDAR-8B shapes — and a long key stream, so the kernel is
// "swap-AB": keys sit on the MMA M side and query rows on N,
//     S^T [128 keys x NQ rows] = K_tile [128 x d_h] . Q^T            (tcgen05.mma, A = K, B = Q, K-major)
//     O^T [d_h x NQ]          += V_tile^T [d_h x 128] . P^T          (A = V as MN-major, B = P^T MN-major)
// with NQ = the unit's query rows rounded up to 16 (MMA N), so each softmax thread owns one key and
// every lane does useful work, and the accumulators are tiny (NQ TMEM columns).
//
// Work unit = (request i of the call, query-row chunk, kv head, key split): up to 64 query rows
// (GQA packing: one K/V stream serves the G heads of 64/G block rows).  Keys (block-diffusion mask,
// P:102-103):
//   ext_mode 0  context [0, s) + the whole block [s, s+B)          (layer 0, layer-1 suffix; A-K2/A-K3)
//   ext_mode 1  context + block [s, s+R']                          (layers >= 2; A-K1)
//   ext_mode 2  causal prefill (row at position p sees [0, p])      (focus_kv_append; A-K5)
//   imp_only    block keys [s, s+B) only, no output                  (layer-1 importance, A-I8)
// Keys stream in 128-key tiles straight from the paged pool by TMA (no gather copy).  A request's
// tiles are cut into balanced splits so the persistent grid stays busy; split partials
// (unnormalised O, running max, sum) are merged by the last-arriving split in split order
// (deterministic).
//
// Persistent CTA (one per SM), 384 threads, warp-specialised:
//   warp 0 / 2  TMA producers: K tiles / V tiles (128 keys x 128, 128-B swizzle); 2-slot K ring (freed when
//               QK^T completes), 3-slot V ring (freed when PV completes)
//   warp 1      QK^T issuer (one thread) + Q loader: S^T into one of four TMEM tiles; one Q buffer
//   warp 3      TMEM allocator + PV^T issuer (one thread): O^T += V^T P^T into a double-buffered TMEM
//               accumulator (one per unit in flight) and the row sums L^T += ONES P^T.  Two issuing
//               threads, so a QK^T never waits behind a PV^T's dependencies
//   warps 4-7   softmax, thread = key: online softmax in the log2 domain with a lazy running max
//               (started from the unit's first key's scores; it only moves when a score exceeds it by
//               > 2^8: a one-barrier vote, then a cross-warp exact max and, if a max moved, the O^T / L^T
//               column rescale), P^T -> double-buffered smem as bf16; block-column scores -> scratch and
//               the Eq.2 epilogue (importance-only mode: one tile per unit, scratch and a second Q
//               buffer in the idle V ring)
//   warps 8-11  epilogue, thread = d_h lane of O^T: O/l -> bf16 rows (or split partials + merge)
#include <math_constants.h>
#include <cstdio>

#include "tc_ptx.cuh"

namespace focus {
namespace attn {

using namespace tc;

constexpr int DH = 128;           // head_dim of the tensor-core path
constexpr int KT = 128;           // keys per tile (MMA M)
constexpr int NQM = 64;           // max query rows per unit (MMA N)
constexpr int SK = 2;             // K ring slots (freed as soon as QK^T completes)
constexpr int SV = 3;             // V ring slots (held from landing until PV completes; measured 2 K + 3 V > 3 K + 2 V
                                  // once QK^T had its own issuer and four S^T buffers)
constexpr int UCAP = 24;          // unit descriptors per CTA kept in smem
constexpr int NTHREADS = 384;
constexpr float kLog2e = 1.4426950408889634f;
constexpr int kMaxPoolRad = 2;           // MaxPool1D kernel <= 5 (the host rejects larger)

constexpr int HALF_Q = NQM * 128;               // 8 KB: one 64-column half of the Q tile
constexpr int Q_BYTES = 2 * HALF_Q;             // 16 KB (one buffer: unit u+1's Q loads once unit u's QK^T are done)
constexpr int HALF_KV = KT * 128;               // 16 KB: one 64-column half of a K / V tile
constexpr int KV_BYTES = 2 * HALF_KV;           // 32 KB
constexpr int P_CHUNK = (KT / 8) * 128;         // 2 KB: 8 query rows x 128 keys of P^T
constexpr int P_BYTES = (NQM / 8) * P_CHUNK;    // 16 KB
constexpr int NPB = 2;                          // P^T buffers (measured: one buffer stalls the softmax on PV(g-1))
constexpr int TMEM_COLS = 512;
constexpr int O_COL = 0;                        // O^T buffers [0, 64), [64, 128)
constexpr int NSB = 4;                          // S^T buffers: QK^T runs up to NSB tiles ahead of PV
constexpr int S_COL = 2 * NQM;                  // S^T buffers [128, 192) .. [320, 384)
constexpr int L_COL = (2 + NSB) * NQM;          // row-sum buffers (two): ONES . P^T
static_assert(L_COL + 2 * NQM <= TMEM_COLS, "TMEM columns");
constexpr int MAXS = 16;                        // split partials merged through smem
constexpr int OFF_Q = 0;
constexpr int OFF_K = OFF_Q + Q_BYTES;
constexpr int OFF_V = OFF_K + SK * KV_BYTES;
constexpr int OFF_P = OFF_V + SV * KV_BYTES;
constexpr int OFF_BAR = OFF_P + NPB * P_BYTES;
constexpr int N_BARS = 2 * SK + 2 * SV + 4 + 2 * NSB + 2 * NPB + 6;
constexpr int OFF_MISC = OFF_BAR + 8 * N_BARS + 16;
constexpr int OFF_M = OFF_MISC;                 // float [NQM] running max (log2 units)
constexpr int OFF_ALPHA = OFF_M + NQM * 4;      // float [NQM]
constexpr int OFF_THR = OFF_ALPHA + NQM * 4;    // float [NQM] raw-score rescale threshold (+inf: padding row)
constexpr int OFF_NM = OFF_THR + NQM * 4;       // float [NQM] -m (0 while m = -inf)
constexpr int OFF_STAT = OFF_NM + NQM * 4;      // float [2][NQM] m for the epilogue (split merge)
constexpr int OFF_RED = OFF_STAT + 2 * NQM * 4; // float [4][64]
constexpr int OFF_FLAG = OFF_RED + 4 * 64 * 4;  // float [4] chunk threshold minima (64 B reserved)
constexpr int OFF_ONES = OFF_FLAG + 64;         // 128 B of bf16 ones (A operand of the row-sum MMA)
constexpr int OFF_MERGE = OFF_ONES + 128;       // float [MAXS + 1][NQM] split-merge scales + 1/l
constexpr int OFF_OST = OFF_MERGE + (MAXS + 1) * NQM * 4;   // bf16 [32][DH] output staging: 32 query rows per pass
constexpr int OFF_UTAB = OFF_OST + 2 * 16 * DH * 2;
constexpr int SMEM_BYTES = OFF_UTAB + UCAP * 80 + 1024;
static_assert(SMEM_BYTES <= 227 * 1024 - 64, "attention shared memory");

using Unit = AttnUnit;
static_assert(sizeof(Unit) == 80, "unit descriptor size");

// debug trace: role r of this CTA appends clock64 stamps (event kind in the top 8 bits)
struct Tracer {
  unsigned long long* p;
  int n;
  __device__ __forceinline__ Tracer(unsigned long long* base, int role)
      : p(base ? base + ((size_t)blockIdx.x * 8 + role) * kTraceEv : nullptr), n(0) {}
  __device__ __forceinline__ void ev(int kind) {
    if (p && n < kTraceEv) p[n++] = ((unsigned long long)kind << 56) | (clock64() & ((1ull << 56) - 1));
  }
};

__device__ __forceinline__ void key_range(const AttnArgs& a, int i, int& kbeg, int& kend, int& s0) {
  const focus_req_state& s = a.st[a.req_list[i]];
  s0 = s.s;
  if (a.imp_only) { kbeg = s.s; kend = s.s + a.B; }
  else { kbeg = 0; kend = a.ext_mode == 0 ? s.s + a.B : s.s + s.R_new + 1; }
}

__device__ __forceinline__ int req_units(const AttnArgs& a, int i, int rpc, int tps, int& nsplit) {
  const int rows = a.row_off[i + 1] - a.row_off[i];
  nsplit = 0;
  if (rows <= 0) return 0;
  const focus_req_state& s = a.st[a.req_list[i]];
  if (a.imp_only && (a.imp == nullptr || s.flush)) return 0;
  int kbeg, kend, s0;
  key_range(a, i, kbeg, kend, s0);
  const int nt = (kend + KT - 1) / KT - kbeg / KT;
  nsplit = a.imp_only ? 1 : min(MAXS, (nt + tps - 1) / tps);
  return ((rows + rpc - 1) / rpc) * a.kv.n_kv_heads * nsplit;
}

__device__ Unit decode_unit(const AttnArgs& a, int u, const int* pre, const int* nsp, int n_ent, int G, int rpc) {
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
    x.want_imp = 0;
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
  x.pad = 0;
  return x;
}

// Transposed butterfly over a warp: on entry lane l holds v[0..31] (one value per row); on exit
// lane j holds op-reduce over the 32 lanes of row j.  31 shuffles for 32 rows.
template <bool MAX>
__device__ __forceinline__ float warp_transpose_reduce(float (&v)[32], int lane) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < o; ++i) {
      const float send = up ? v[i] : v[i + o];
      const float keep = up ? v[i + o] : v[i];
      const float recv = __shfl_xor_sync(0xffffffffu, send, o);
      v[i] = MAX ? fmaxf(keep, recv) : keep + recv;
    }
  }
  return v[0];
}

// ---------------------------------------------------------------- softmax warps
struct SoftSmem {
  float* m;          // [NQM] running max (log2 units)
  float* alpha;      // [NQM] rescale factor of the current tile
  float* thr;        // [NQM] raw-score threshold above which the running max must move
  float* nm;         // [NQM] -m (0 while m = -inf)
  float* stat;       // [2][NQM] m of the finished unit (split merge)
  float* red;        // [4][64]
  float* tmin;       // [4] per 16-row chunk: the smallest row threshold (the per-tile check compares with it)
  uint8_t* sP;
  uint64_t *sfull, *sfree, *pfull, *pvdone, *ofree, *statfull;
};
struct SoftThread {
  int L, lane, q4, G;
  uint32_t tmem, lane_base;
  float sl2;
  float* scr;
};

// One unit on the softmax warps (thread = key lane L of each 128-key tile).  NCH = 16-row chunks of
// query rows.  Per tile: (1) does any score exceed its row threshold (running max + 2^8)?  (rare after
// the first tile) -> exact tile max per row, new running max, O^T / L^T column rescale; (2) P^T =
// exp2(s * scale * log2e - m) in bf16 into the P^T buffer.  Row sums come from the tensor core.
template <int NCH, bool CAUSAL, bool IMP_ONLY>
__device__ __forceinline__ void softmax_unit(const AttnArgs& a, const Unit& xr, int it, uint32_t& g,
                                             const SoftThread& th, const SoftSmem& ss, Tracer& tr) {
  const int L = th.L, lane = th.lane, nq = xr.nq;
  const uint32_t ob = it & 1;
  named_bar(1, 128);                               // previous unit's readers of m/thr/nm are done
  if (L < NQM) {
    ss.m[L] = -CUDART_INF_F;
    ss.thr[L] = L < nq ? -CUDART_INF_F : CUDART_INF_F;
    ss.nm[L] = 0.f;
  }
  if (L < NQM / 16) ss.tmin[L] = 16 * L < nq ? -CUDART_INF_F : CUDART_INF_F;
  named_bar(1, 128);
  for (int t = xr.t_lo; t < xr.t_hi; ++t, ++g) {
    const uint32_t sb = g % NSB, pb = g % NPB;
    mbar_wait(&ss.sfull[sb], (g / NSB) & 1);
    tr.ev(1);
    tc_fence_after();
    const int k = t * KT + L;
    const bool kvalid = k >= xr.kbeg && k < xr.kend;
    const uint32_t sbase = th.tmem + th.lane_base + S_COL + sb * NQM;
    uint32_t r[NCH][16];
#pragma unroll
    for (int c = 0; c < NCH; ++c) tmem_ld32x16(sbase + 16 * c, r[c]);
    tmem_wait_ld();
    tr.ev(6);
    tc_fence_before();                             // S^T is in registers: the tile may be overwritten
    __syncwarp();
    if (lane == 0) mbar_arrive(&ss.sfree[sb]);
    if (!IMP_ONLY && t == xr.t_lo) {
      // running-max estimate for the unit's first tile: the scores of its first valid key (one thread
      // holds them for every row; they are handed to the row threads through red[]), instead of an exact
      // tile max.  Correctness does not depend on it: any score above estimate + 2^8 (log2 units) still
      // takes the exact path below.
      const int L0 = max(0, xr.kbeg - t * KT);
      if (L == L0) {
#pragma unroll
        for (int c = 0; c < NCH; ++c)
#pragma unroll
          for (int e = 0; e < 16; ++e) ss.red[16 * c + e] = __uint_as_float(r[c][e]);
      }
      named_bar(1, 128);
      if (L < nq && L < NCH * 16) {
        const float mv = ss.red[L] * th.sl2;
        ss.m[L] = mv;
        ss.nm[L] = -mv;
        ss.thr[L] = (mv + a.rescale_log2) / th.sl2;
      }
      named_bar(1, 128);
      if (L < NCH) {
        float tm = CUDART_INF_F;
#pragma unroll
        for (int e = 0; e < 16; ++e) tm = fminf(tm, ss.thr[16 * L + e]);
        ss.tmin[L] = tm;
      }
      named_bar(1, 128);
    }
    // ---- (1) threshold check: against the chunk's smallest row threshold (conservative: a hit only sends
    // the tile through the exact per-row test below)
    bool need = false;
    if (kvalid && !CAUSAL) {
#pragma unroll
      for (int c = 0; c < NCH; ++c) {             // max tree of the chunk's 16 scores, one compare
        float m8[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) m8[e] = fmaxf(__uint_as_float(r[c][e]), __uint_as_float(r[c][e + 8]));
#pragma unroll
        for (int e = 0; e < 4; ++e) m8[e] = fmaxf(m8[e], m8[e + 4]);
        const float mx = fmaxf(fmaxf(m8[0], m8[2]), fmaxf(m8[1], m8[3]));
        need |= mx > ss.tmin[c];
      }
    } else if (kvalid) {
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
#pragma unroll
        for (int e4 = 0; e4 < 16; e4 += 4) {
          const float4 t4 = *reinterpret_cast<const float4*>(ss.thr + 16 * c + e4);
          const float tv[4] = {t4.x, t4.y, t4.z, t4.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const bool vis = !CAUSAL || k <= xr.pos_base + (16 * c + e4 + e) / th.G;
            need |= vis && __uint_as_float(r[c][e4 + e]) > tv[e];
          }
        }
      }
    }
    if (xr.want_imp && kvalid && k >= xr.s0 && k < xr.s0 + a.B) {   // block-column scores (Eq.2 epilogue)
      // scratch [block column j][query row n]: this thread's column is one contiguous run (vector stores)
      float* col = th.scr + (size_t)(k - xr.s0) * NQM;
#pragma unroll
      for (int c = 0; c < NCH; ++c)
#pragma unroll
        for (int e4 = 0; e4 < 16; e4 += 4)
          *reinterpret_cast<float4*>(col + 16 * c + e4) =
              make_float4(__uint_as_float(r[c][e4]) * a.scale, __uint_as_float(r[c][e4 + 1]) * a.scale,
                          __uint_as_float(r[c][e4 + 2]) * a.scale, __uint_as_float(r[c][e4 + 3]) * a.scale);
    }
    if (IMP_ONLY) continue;
    tr.ev(7);
    const bool any_need = named_bar_or(1, 128, need);   // one barrier: does any key of the tile need it?
    tr.ev(8);
    if (any_need) {
      tr.ev(9);
      // ---- slow path: exact tile max per row (transposed butterfly + 4-warp combine)
#pragma unroll
      for (int rd = 0; rd < (NCH + 1) / 2; ++rd) {
        float v[32];
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          const int c = rd * 2 + cc;
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            bool ok = c < NCH && kvalid;
            if (CAUSAL) ok = ok && k <= xr.pos_base + (16 * c + e) / th.G;
            v[cc * 16 + e] = ok ? __uint_as_float(r[c < NCH ? c : 0][e]) * th.sl2 : -CUDART_INF_F;
          }
        }
        ss.red[th.q4 * 64 + rd * 32 + lane] = warp_transpose_reduce<true>(v, lane);
      }
      named_bar(1, 128);
      bool moved = false;
      if (L < NQM) {
        float al = 1.f;
        if (L < nq && L < NCH * 16) {
          const float mt = fmaxf(fmaxf(ss.red[L], ss.red[64 + L]), fmaxf(ss.red[128 + L], ss.red[192 + L]));
          const float mo = ss.m[L];
          if (mt > mo + a.rescale_log2 || (mo == -CUDART_INF_F && mt > -CUDART_INF_F)) {
            const float mn = fmaxf(mt, mo);
            al = ex2(mo - mn);                     // 0 when mo = -inf
            ss.m[L] = mn;
            ss.nm[L] = -mn;
            ss.thr[L] = (mn + a.rescale_log2) / th.sl2;
            moved = true;
          }
        }
        ss.alpha[L] = al;
      }
      moved = named_bar_or(1, 128, moved);         // did any row's running max move?
      if (L < NQM / 16) {                          // chunk minima of the (possibly) moved thresholds
        float tm = CUDART_INF_F;
#pragma unroll
        for (int e = 0; e < 16; ++e) tm = fminf(tm, ss.thr[16 * L + e]);
        ss.tmin[L] = tm;
      }
      named_bar(1, 128);
      if (t > xr.t_lo && moved) {                  // O^T and L^T columns *= alpha (PV of tile g-1 done)
        mbar_wait(&ss.pvdone[(g - 1) % NPB], ((g - 1) / NPB) & 1);
        tr.ev(10);
        tc_fence_after();
#pragma unroll
        for (int buf = 0; buf < 2; ++buf) {
          const uint32_t base = th.tmem + th.lane_base + (buf == 0 ? O_COL : L_COL) + ob * NQM;
#pragma unroll
          for (int c = 0; c < NCH; ++c) {
            uint32_t q[16];
            tmem_ld32x16(base + 16 * c, q);
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 16; ++e) q[e] = __float_as_uint(__uint_as_float(q[e]) * ss.alpha[16 * c + e]);
            tmem_st32x16(base + 16 * c, q);
          }
        }
        tmem_wait_st();
      }
    }
    // ---- (2) P^T = exp2(s * scale*log2e - m) as bf16 into the MN-major P^T buffer
    tr.ev(2);
    if (g >= NPB) mbar_wait(&ss.pvdone[pb], ((g / NPB) & 1) ^ 1);   // PV of tile g-NPB done: buffer free
    tr.ev(3);
    const uint32_t pdst = smem_u32(ss.sP + pb * P_BYTES) + (L >> 3) * 128 + (L & 7) * 16;
    if (kvalid) {
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        uint32_t pk[8];
#pragma unroll
        for (int e4 = 0; e4 < 16; e4 += 4) {
          const float4 n4 = *reinterpret_cast<const float4*>(ss.nm + 16 * c + e4);
          const float nv[4] = {n4.x, n4.y, n4.z, n4.w};
          float p[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            p[e] = ex2(fmaf(__uint_as_float(r[c][e4 + e]), th.sl2, nv[e]));
            if (CAUSAL && k > xr.pos_base + (16 * c + e4 + e) / th.G) p[e] = 0.f;
          }
          const __nv_bfloat162 b0 = __floats2bfloat162_rn(p[0], p[1]);
          const __nv_bfloat162 b1 = __floats2bfloat162_rn(p[2], p[3]);
          pk[e4 / 2] = *reinterpret_cast<const uint32_t*>(&b0);
          pk[e4 / 2 + 1] = *reinterpret_cast<const uint32_t*>(&b1);
        }
        sts128(pdst + (2 * c) * P_CHUNK, make_uint4(pk[0], pk[1], pk[2], pk[3]));
        sts128(pdst + (2 * c + 1) * P_CHUNK, make_uint4(pk[4], pk[5], pk[6], pk[7]));
      }
    } else {
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        sts128(pdst + (2 * c) * P_CHUNK, make_uint4(0, 0, 0, 0));
        sts128(pdst + (2 * c + 1) * P_CHUNK, make_uint4(0, 0, 0, 0));
      }
    }
    tc_fence_before();
    fence_proxy_async();
    __syncwarp();
    if (lane == 0) mbar_arrive(&ss.pfull[pb]);
    tr.ev(4);
  }
  if (!IMP_ONLY) {
    mbar_wait(&ss.ofree[ob], ((it >> 1) & 1) ^ 1);   // epilogue of unit it-2 is done with stat[ob]
    tr.ev(5);
    if (L < NQM) ss.stat[ob * NQM + L] = ss.m[L];
    __syncwarp();
    if (lane == 0) mbar_arrive(&ss.statfull[ob]);
  }
}

// Eq.2 on the block scores of the unit (scratch rows = query rows n = r*G + g): per row MaxPool1D
// (k = mp_kernel, -inf outside P; A-I3, A-I5), softmax over P, then the sum over rows and heads in a
// fixed order (lanes, then warps) -> one partial per (request, chunk, kv head).
template <int KB>
__device__ __noinline__ void importance_epilogue_t(const AttnArgs& a, const Unit& xr, const SoftThread& th,
                                                   const SoftSmem& ss) {
  named_bar(1, 128);                               // all block scores of the unit are in scratch
  const int B = a.B, rad = a.mp_kernel / 2, L = th.L, lane = th.lane;
  const uint64_t P = xr.P;
  const bool rr = L < xr.nq;
  // the row's B scores in registers (one batch of vector loads: a per-element load chain through the
  // L2 made this epilogue ~22 k cycles per unit), then MaxPool / softmax in registers
  float w[KB];
  if (rr) {
    float sv[KB];                                  // scratch [column j][row]: consecutive rows coalesce
#pragma unroll
    for (int j = 0; j < KB; ++j) sv[j] = j < B ? th.scr[(size_t)j * NQM + L] : 0.f;
    float mx = -CUDART_INF_F;
#pragma unroll
    for (int j = 0; j < KB; ++j) {
      float v = -CUDART_INF_F;
      if (j < B && ((P >> j) & 1ull)) {
#pragma unroll
        for (int d = -kMaxPoolRad; d <= kMaxPoolRad; ++d) {
          const int jj = j + d;
          if (jj >= 0 && jj < KB && d >= -rad && d <= rad && jj < B && ((P >> jj) & 1ull)) v = fmaxf(v, sv[jj]);
        }
      }
      w[j] = v;
      mx = fmaxf(mx, v);
    }
    float z = 0.f;
#pragma unroll
    for (int j = 0; j < KB; ++j) {
      const float e = w[j] == -CUDART_INF_F ? 0.f : __expf(w[j] - mx);
      w[j] = e;
      z += e;
    }
    const float iz = 1.0f / z;
#pragma unroll
    for (int j = 0; j < KB; ++j) w[j] *= iz;
  } else {
#pragma unroll
    for (int j = 0; j < KB; ++j) w[j] = 0.f;
  }
  // column sums over the warp's 32 rows: transposed butterfly (31 shuffles per 32 columns), lane j
  // then holds column 32q + j of this warp, in a fixed order
#pragma unroll
  for (int q = 0; q < KB / 32 + (KB % 32 ? 1 : 0); ++q) {
    float v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = (32 * q + i < KB) ? w[32 * q + i] : 0.f;
    const float cs = warp_transpose_reduce<false>(v, lane);
    if (32 * q + lane < B) ss.red[th.q4 * 64 + 32 * q + lane] = cs;
  }
  named_bar(1, 128);
  if (th.q4 == 0)
    for (int j = lane; j < B; j += 32)
      a.imp[(size_t)xr.pair * B + j] = ((ss.red[j] + ss.red[64 + j]) + ss.red[128 + j]) + ss.red[192 + j];
  named_bar(1, 128);                               // red[] reuse
}

__device__ __forceinline__ void importance_epilogue(const AttnArgs& a, const Unit& xr, const SoftThread& th,
                                                    const SoftSmem& ss) {
  if (a.B <= 16) importance_epilogue_t<16>(a, xr, th, ss);
  else if (a.B <= 32) importance_epilogue_t<32>(a, xr, th, ss);
  else importance_epilogue_t<64>(a, xr, th, ss);
}

// Unit table of CTA `cta` of `ncta` (the attention grid): per-request unit counts, exclusive prefix,
// then the CTA's unit descriptors (whole (request, chunk, kv head) pairs, optionally key-split, or
// stream-K pieces).  Called by all 384 threads of a block; `scratch` is >= 17 KB of shared memory.
// Returns the number of units (same value in every thread).
__device__ int build_units(const AttnArgs& a, int cta, int ncta, int* scratch, Unit* utab) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int H = a.kv.n_kv_heads;
  const int G = a.n_q_heads / H;
  const int rpc = NQM / G;
  int* pre = scratch;
  int* nsp = pre + 1028;
  // ---- unit table: per-request unit counts, exclusive prefix, then this CTA's unit descriptors
  const int n_ent = a.ext_mode == 2 ? 1 : a.n_req;
  int tps = max(2, a.split_tiles);
  int total;
  for (;;) {
    if (a.ext_mode == 2) {
      if (threadIdx.x == 0) { nsp[0] = 1; pre[1] = ((a.prefill_rows + rpc - 1) / rpc) * H; }
    } else {
      for (int i = threadIdx.x; i < n_ent; i += NTHREADS) {
        int ns;
        pre[i + 1] = req_units(a, i, rpc, tps, ns);
        nsp[i] = ns;
      }
    }
    __syncthreads();
    if (warp == 0) {                               // exclusive scan of unit counts
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
    total = pre[n_ent];
    if (total <= UCAP * (int)ncta || a.ext_mode == 2 || a.imp_only || tps >= (1 << 20)) break;
    tps *= 2;                                      // too many units for the descriptor table
    __syncthreads();
  }
  int n_my = total > cta ? min(UCAP, (total - 1 - cta) / ncta + 1) : 0;
  __shared__ int sk_on;
  if (a.stream_k && a.ext_mode != 2 && a.imp == nullptr && !a.imp_only) {
    // ---- stream-K over key tiles: every CTA takes T / grid_eff consecutive tiles of the flattened
    // (request, chunk, kv head, tile) sequence; a pair cut at a CTA boundary becomes split pieces
    // (merged in piece order by the pair's last-arriving piece)
    __syncthreads();
    int* pre2 = nsp + 1028;                        // [n_ent + 1] tile prefix   (P^T buffers, setup only)
    int* ntr = pre2 + 1028;                        // [n_ent] tiles per pair
    int* piece = ntr + 1028;                       // [UCAP][4] (request, pair_local, tile offset, tiles)
    __shared__ int nt_minmax[2], n_pieces;
    if (threadIdx.x == 0) { nt_minmax[0] = 1 << 30; nt_minmax[1] = 0; }
    __syncthreads();
    for (int i = threadIdx.x; i < n_ent; i += NTHREADS) {
      const int rows = a.row_off[i + 1] - a.row_off[i];
      int tiles = 0, nt = 0;
      if (rows > 0) {
        int kbeg, kend, s0;
        key_range(a, i, kbeg, kend, s0);
        nt = (kend + KT - 1) / KT - kbeg / KT;
        tiles = ((rows + rpc - 1) / rpc) * H * nt;
        atomicMin(&nt_minmax[0], nt);
        atomicMax(&nt_minmax[1], nt);
      }
      ntr[i] = nt;
      pre2[i + 1] = tiles;
    }
    __syncthreads();
    if (warp == 0) {
      const int per = (n_ent + 31) / 32;
      const int b0 = min(n_ent, lane * per), b1 = min(n_ent, b0 + per);
      int loc = 0;
      for (int i = b0; i < b1; ++i) loc += pre2[i + 1];
      int inc = loc;
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += v;
      }
      int run = inc - loc;
      for (int i = b0; i < b1; ++i) { const int c = pre2[i + 1]; pre2[i] = run; run += c; }
      if (lane == 31) pre2[n_ent] = inc;
    }
    __syncthreads();
    const long long T = pre2[n_ent];
    const int ntmax = nt_minmax[1], ntmin = max(1, nt_minmax[0]);
    // enough CTAs that a pair is cut into at most MAXS pieces; few enough pieces per CTA for utab
    long long gel = T * (MAXS - 2) / max(1, ntmax);
    if (gel < 1) gel = 1;
    if (gel > (long long)ncta) gel = ncta;
    if (gel > T) gel = T;
    const int ge = (int)gel;
    const bool fits = T > 0 && (T + ge - 1) / ge / ntmin + 2 <= UCAP;
    if (threadIdx.x == 0) sk_on = fits ? 1 : 0;
    if (fits && threadIdx.x == 0) {
      int np = 0;
      if ((int)cta < ge) {
        const long long lo = (long long)cta * T / ge, hi = (long long)(cta + 1) * T / ge;
        int i = 0, l = 0, h = n_ent - 1;             // request whose tiles contain lo
        while (l < h) { const int mid = (l + h + 1) >> 1; if (pre2[mid] <= lo) l = mid; else h = mid - 1; }
        i = l;
        long long pos = lo;
        while (pos < hi && np < UCAP) {
          while (pos >= pre2[i + 1]) ++i;
          const int nt = ntr[i];
          const long long off = pos - pre2[i];
          const int pl = (int)(off / nt), to = (int)(off % nt);
          const int take = (int)min((long long)(nt - to), hi - pos);
          piece[np * 4 + 0] = i; piece[np * 4 + 1] = pl; piece[np * 4 + 2] = to; piece[np * 4 + 3] = take;
          ++np;
          pos += take;
        }
      }
      n_pieces = np;
    }
    __syncthreads();
    if (sk_on) {
      n_my = n_pieces;
      for (int k = threadIdx.x; k < n_my; k += NTHREADS) {
        const int i = piece[k * 4 + 0], pl = piece[k * 4 + 1], to = piece[k * 4 + 2], take = piece[k * 4 + 3];
        const int nt = ntr[i];
        Unit x;
        x.i = i;
        x.chunk = pl / H;
        x.kvh = pl % H;
        x.slot = a.req_list[i];
        const focus_req_state& st = a.st[x.slot];
        const int rb = a.row_off[i], re = a.row_off[i + 1];
        x.r0 = rb + x.chunk * rpc;
        x.nr = min(rpc, re - x.r0);
        x.nq = x.nr * G;
        key_range(a, i, x.kbeg, x.kend, x.s0);
        x.t_lo = x.kbeg / KT + to;
        x.t_hi = x.t_lo + take;
        const long long ps = pre2[i] + (long long)pl * nt, pe = ps + nt - 1;
        const int o0 = (int)(((ps + 1) * ge + T - 1) / T) - 1, o1 = (int)(((pe + 1) * ge + T - 1) / T) - 1;
        x.sp = cta - o0;
        x.nsplit = o1 - o0 + 1;
        x.pos_base = 0;
        x.P = st.P;
        x.want_imp = 0;
        x.pair = (i * a.n_chunks + x.chunk) * H + x.kvh;
        x.pad = 0;
        utab[k] = x;
      }
    }
    __syncthreads();
  } else if (threadIdx.x == 0) {
    sk_on = 0;
  }
  __syncthreads();
  if (!sk_on) {
    // Tail split: whole units round-robin for the R = total / ncta full rounds; the U' = total % ncta
    // units of the last, partial round are each cut into s = ncta / U' key ranges (one piece per CTA)
    // so no CTA ends a whole unit behind the others.  Only for unsplit units of plain attention.
    const int R = total / ncta, Ut = total - R * ncta;
    const int s = (a.tail_split && Ut > 0 && a.ext_mode != 2 && a.imp == nullptr && !a.imp_only) ? min(MAXS, ncta / Ut) : 1;
    if (s >= 2 && R < UCAP) {
      // the piece runs FIRST: its pair's merge (by the last-arriving piece's epilogue warps) then
      // overlaps the CTA's whole units instead of trailing the kernel
      __shared__ int extra;
      if (threadIdx.x == 0) {
        extra = 0;
        if (cta < Ut * s) {
          Unit x = decode_unit(a, R * ncta + cta / s, pre, nsp, n_ent, G, rpc);
          const int t0 = x.kbeg / KT, nt = (x.kend + KT - 1) / KT - t0;
          const int ns = min(s, nt), sp = cta % s;
          if (x.nsplit == 1 && sp < ns) {
            x.sp = sp;
            x.nsplit = ns;
            x.t_lo = t0 + (sp * nt) / ns;
            x.t_hi = t0 + ((sp + 1) * nt) / ns;
            x.want_imp = 0;
            utab[0] = x;
            extra = 1;
          } else if (x.nsplit > 1 && sp == 0) {        // already key-split unit: keep it whole here
            utab[0] = x;
            extra = 1;
          }
        }
      }
      __syncthreads();
      for (int k = threadIdx.x; k < R; k += NTHREADS)
        utab[extra + k] = decode_unit(a, cta + k * ncta, pre, nsp, n_ent, G, rpc);
      n_my = R + extra;
    } else {
      for (int k = threadIdx.x; k < n_my; k += NTHREADS)
        utab[k] = decode_unit(a, cta + k * ncta, pre, nsp, n_ent, G, rpc);
    }
  }
  __syncthreads();
  return n_my;
}

template <bool IMP_ONLY>
__global__ void __launch_bounds__(NTHREADS, 1)
    k_attn_tc(const __grid_constant__ CUtensorMap mapK, const __grid_constant__ CUtensorMap mapV,
              const __grid_constant__ CUtensorMap mapQ, const __grid_constant__ AttnArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sQ = smem + OFF_Q;
  uint8_t* sK = smem + OFF_K;
  uint8_t* sV = smem + OFF_V;
  uint8_t* sP = smem + OFF_P;
  uint64_t* bars = (uint64_t*)(smem + OFF_BAR);
  uint64_t* kfull = bars;                  // [SK]
  uint64_t* kempty = kfull + SK;           // [SK]
  uint64_t* vfull = kempty + SK;           // [SV]
  uint64_t* vempty = vfull + SV;           // [SV]
  uint64_t* qfull = vempty + SV;           // [2]  (the second buffer: importance-only mode)
  uint64_t* qempty = qfull + 2;            // [2]
  uint64_t* sfull = qempty + 2;            // [NSB]
  uint64_t* sfree = sfull + NSB;           // [NSB]  (4 softmax warps)
  uint64_t* pfull = sfree + NSB;           // [NPB]  (4 softmax warps)
  uint64_t* pvdone = pfull + NPB;          // [NPB]
  uint64_t* ofull = pvdone + NPB;          // [2]
  uint64_t* ofree = ofull + 2;             // [2]  (4 epilogue warps)
  uint64_t* statfull = ofree + 2;          // [2]  (4 softmax warps)
  uint32_t* tmem_sh = (uint32_t*)(bars + N_BARS);
  SoftSmem ss;
  ss.m = (float*)(smem + OFF_M);
  ss.alpha = (float*)(smem + OFF_ALPHA);
  ss.thr = (float*)(smem + OFF_THR);
  ss.nm = (float*)(smem + OFF_NM);
  ss.stat = (float*)(smem + OFF_STAT);
  ss.red = (float*)(smem + OFF_RED);
  ss.tmin = (float*)(smem + OFF_FLAG);
  ss.sP = sP;
  ss.sfull = sfull; ss.sfree = sfree; ss.pfull = pfull; ss.pvdone = pvdone; ss.ofree = ofree; ss.statfull = statfull;
  uint16_t* ones = (uint16_t*)(smem + OFF_ONES);
  Unit* utab = (Unit*)(smem + OFF_UTAB);
  int* pre = (int*)sP;                     // setup only (aliases the P^T buffers: 17 KB of scan scratch)
  int* nsp = pre + 1028;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int H = a.kv.n_kv_heads;
  const int G = a.n_q_heads / H;
  const int rpc = NQM / G;

  pdl_trigger();
  if (threadIdx.x == 0 && a.trace) {               // debug: entry clock and global time
    unsigned long long gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    a.trace[((size_t)blockIdx.x * 8 + 7) * kTraceEv + 1] = clock64();
    a.trace[((size_t)blockIdx.x * 8 + 7) * kTraceEv + 2] = gt;
  }
  if (threadIdx.x < 64) ones[threadIdx.x] = 0x3F80;   // bf16 1.0
  // V ring zeroed once: boxes past a unit's last key are not loaded, so the V rows they would have filled
  // must hold finite values (P = 0 there, and 0 * finite = 0 in the PV MMA).  Stale K rows only reach
  // S^T entries of keys outside the unit, which the softmax never reads (P = 0 is written for them).
  for (int i = threadIdx.x; i < SV * KV_BYTES / 16; i += NTHREADS)
    reinterpret_cast<uint4*>(sV)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    for (int i = 0; i < SK; ++i) { mbar_init(&kfull[i], 1); mbar_init(&kempty[i], 1); }
    for (int i = 0; i < SV; ++i) { mbar_init(&vfull[i], 1); mbar_init(&vempty[i], 1); }
    for (int i = 0; i < NSB; ++i) { mbar_init(&sfull[i], 1); mbar_init(&sfree[i], 4); }
    for (int i = 0; i < NPB; ++i) { mbar_init(&pfull[i], 4); mbar_init(&pvdone[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&qfull[i], 1); mbar_init(&qempty[i], 1); }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&ofull[i], 1); mbar_init(&ofree[i], 4);
      mbar_init(&statfull[i], 4);
    }
    fence_barrier_init();
  }
  fence_proxy_async();                             // the ones block is read by the tensor core
  if (warp == 1 && lane == 0) {
    prefetch_map(&mapQ);
    prefetch_map(&mapK);
    if (!IMP_ONLY) prefetch_map(&mapV);
  }
  if (warp == 3) tmem_alloc<TMEM_COLS>(tmem_sh);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0 && lane == 0 && a.plan_n != nullptr && a.pre_pf_tiles > 0 && !IMP_ONLY) {
    // Start-up: the first K/V tiles of this CTA's first unit are prefetched into L2 BEFORE the grid
    // dependency wait, so they stream while the previous kernel (the QKV GEMM) drains; the TMA loads
    // after the wait then hit L2 instead of paying the full loaded-HBM latency (~4 us for the first
    // tile when every CTA starts at once).  The plan / page-table reads here may see data of an
    // unfinished earlier kernel; a prefetch is only a hint, so a stale address costs a wasted fetch and
    // never a wrong result (everything that is consumed is read after pdl_wait below).
    const int n0 = a.plan_n[blockIdx.x];
    if (n0 > 0) {
      const Unit& x0 = static_cast<const Unit*>(a.plan_units)[(size_t)blockIdx.x * UCAP];
      const int H = a.kv.n_kv_heads, ps = a.kv.page_size, pr = min(ps, KT);
      const size_t layer_rows = (size_t)a.kv_pages * H * ps;
      const int t_end = min(x0.t_hi, x0.t_lo + a.pre_pf_tiles);
      if (x0.slot >= 0 && x0.slot < a.max_slots && x0.kvh >= 0 && x0.kvh < H && x0.t_hi - x0.t_lo < (1 << 16))
        for (int t = max(x0.t_lo, 0); t < t_end; ++t)
          for (int pc = 0; pc < KT / pr; ++pc) {
            const int pos = t * KT + pc * pr;
            if (pos >= x0.s0) break;                     // context keys only (the block's are being written)
            const int pidx = max(0, min(pos / ps, a.kv.max_pages - 1));
            const int page = a.kv.page_table[(size_t)x0.slot * a.kv.max_pages + pidx];
            const int row = (int)((size_t)a.layer * layer_rows + ((size_t)page * H + x0.kvh) * ps + pos % ps);
            tma_prefetch_2d(&mapK, 0, row);
            tma_prefetch_2d(&mapK, 64, row);
            tma_prefetch_2d(&mapV, 0, row);
            tma_prefetch_2d(&mapV, 64, row);
          }
    }
  }
  pdl_wait();                                       // plan tables, q rows, KV pages come from earlier kernels
  __shared__ int n_my_sh;
  __shared__ int merge_flag;
  int n_my;
  if (a.plan_n) {                                  // precomputed once per step by k_attn_plan
    if (threadIdx.x == 0) n_my_sh = a.plan_n[blockIdx.x];
    __syncthreads();
    n_my = n_my_sh;
    for (int k = threadIdx.x; k < n_my; k += NTHREADS)
      utab[k] = static_cast<const Unit*>(a.plan_units)[(size_t)blockIdx.x * UCAP + k];
  } else {
    n_my = build_units(a, blockIdx.x, gridDim.x, pre, utab);
  }
  __syncthreads();
  if (a.debug_check && threadIdx.x == 0 && a.ext_mode != 2) {
    const int rows = a.row_off[a.n_req];
    for (int k = 0; k < n_my; ++k) {
      const Unit& x = utab[k];
      const bool bad = x.i < 0 || x.i >= a.n_req || x.kvh < 0 || x.kvh >= H || x.nq <= 0 || x.nq > NQM ||
                       x.sp < 0 || x.sp >= x.nsplit || x.nsplit > a.max_nsplit || x.nsplit > MAXS || x.t_lo >= x.t_hi ||
                       x.pair < 0 || x.pair >= a.n_req * a.n_chunks * H || x.r0 < 0 || x.r0 + x.nr > rows ||
                       x.t_lo < x.kbeg / KT || x.t_hi > (x.kend + KT - 1) / KT;
      if (bad) {
        printf("attn unit check: cta %d unit %d/%d i %d kvh %d nq %d nr %d r0 %d rows %d sp %d/%d t %d-%d keys %d-%d pair %d\n",
               blockIdx.x, k, n_my, x.i, x.kvh, x.nq, x.nr, x.r0, rows, x.sp, x.nsplit, x.t_lo, x.t_hi, x.kbeg, x.kend, x.pair);
        __trap();
      }
    }
  }
  if (threadIdx.x == 0 && a.trace) a.trace[((size_t)blockIdx.x * 8 + 7) * kTraceEv] = clock64();
  const uint32_t tmem = *tmem_sh;

  if (warp == 0 || (warp == 2 && !IMP_ONLY)) {
    // ================================================================ TMA producers (K / V)
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
      Tracer tr(a.trace, isK ? 0 : 1);
      uint32_t g = 0;
      auto prefetch_tile = [&](const Unit& x, int t) {
        for (int pc = 0; pc < KT / pr; ++pc) {
          const int pos = t * KT + pc * pr;
          const int pidx = min(pos / ps, a.kv.max_pages - 1);
          const int page = a.kv.page_table[(size_t)x.slot * a.kv.max_pages + pidx];
          const int row = (int)((size_t)a.layer * layer_rows + ((size_t)page * H + x.kvh) * ps + pos % ps);
          tma_prefetch_2d(map, 0, row);
          tma_prefetch_2d(map, 64, row);
        }
      };
      const int pf = a.l2_prefetch;                // tiles past the ring to warm in L2
      const uint64_t pol = l2_policy_evict_first();  // the KV stream is read once per layer and step
      for (int k = 0; k < n_my; ++k) {
        const Unit& x = utab[k];
        tr.ev(0);
        for (int t = x.t_lo; t < min(x.t_hi, x.t_lo + NS + pf); ++t)
          if (t >= x.t_lo + NS) prefetch_tile(x, t);
        for (int t = x.t_lo; t < x.t_hi; ++t, ++g) {
          const int slot = g % NS;
          if (pf > 0 && t + NS + pf < x.t_hi) prefetch_tile(x, t + NS + pf);
          // only the boxes that hold keys of [kbeg, kend): the tail of a unit's last tile (and the head
          // of an importance-only tile) is not streamed; those smem rows keep finite data (the rings
          // are zeroed at kernel start) and the softmax masks their keys (P = 0)
          const int pc0 = a.page_skip ? max(0, (x.kbeg - t * KT) / pr) : 0;
          const int pc1 = a.page_skip ? min(KT / pr, (x.kend - t * KT + pr - 1) / pr) : KT / pr;
          // (measured: issuing the page-table lookups before the slot wait doubled the per-tile time of
          // the C3 layers; the lookups stay after the wait)
          mbar_wait(&emptyb[slot], ((g / NS) & 1) ^ 1);
          tr.ev(1);
          mbar_expect_tx(&fullb[slot], (uint32_t)(pc1 - pc0) * pr * 256);
          uint8_t* dst = ring + slot * KV_BYTES;
          for (int pc = pc0; pc < pc1; ++pc) {
            const int pos = t * KT + pc * pr;
            const int pidx = min(pos / ps, a.kv.max_pages - 1);
            const int page = a.kv.page_table[(size_t)x.slot * a.kv.max_pages + pidx];
            const int row = (int)((size_t)a.layer * layer_rows + ((size_t)page * H + x.kvh) * ps + pos % ps);
            if (a.kv_hint) {
              tma_load_2d_hint(dst + pc * pr * 128, map, &fullb[slot], 0, row, pol);
              tma_load_2d_hint(dst + HALF_KV + pc * pr * 128, map, &fullb[slot], 64, row, pol);
            } else {
              tma_load_2d(dst + pc * pr * 128, map, &fullb[slot], 0, row);
              tma_load_2d(dst + HALF_KV + pc * pr * 128, map, &fullb[slot], 64, row);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ================================================================ QK^T issuer + Q loader
    // S^T(t) = K_t . Q^T into one of NSB TMEM tiles, up to NSB tiles ahead of the softmax; the K ring
    // slot is released as soon as its QK^T completes.  This thread issues no PV^T (warp 3 does), so a
    // QK^T never waits behind the softmax.  Q: unit u's Q tile (one 3-D TMA box per 64-column half: row
    // n = r*G + g holds head kvh*G + g of block row r0 + r; rows past the unit belong to other requests or
    // are zero-filled out of bounds and their results are discarded) goes into buffer u % NQB once the
    // QK^T MMAs of unit u - NQB have completed.  One buffer for attention (the softmax still has up to NSB
    // S^T tiles of the previous unit queued then); two in the importance-only mode, whose units are one
    // tile each (the idle V ring holds the second).
    if (lane == 0) {
      Tracer tr(a.trace, 2);
      constexpr int NQB = IMP_ONLY ? 2 : 1;
      auto qbuf = [&](int b) { return b == 0 ? sQ : sV; };
      auto load_q = [&](int u) {
        const Unit& x = utab[u];
        const int b = u % NQB;
        mbar_expect_tx(&qfull[b], Q_BYTES);
        tma_load_3d(qbuf(b), &mapQ, &qfull[b], 0, x.kvh * G, x.r0);
        tma_load_3d(qbuf(b) + HALF_Q, &mapQ, &qfull[b], 64, x.kvh * G, x.r0);
      };
      for (int u = 0; u < NQB && u < n_my; ++u) load_q(u);
      uint32_t qg = 0;
      for (int qu = 0; qu < n_my; ++qu) {
        const Unit& x = utab[qu];
        const int qb = qu % NQB;
        mbar_wait(&qfull[qb], (qu / NQB) & 1);
        tr.ev(2);
        const int NQ = (x.nq + 15) & ~15;
        const uint32_t idesc_qk = idesc_bf16(KT, NQ, false, false);
        const uint32_t qa = smem_u32(qbuf(qb));
        for (int qt = x.t_lo; qt < x.t_hi; ++qt, ++qg) {
          const uint32_t ks = qg % SK, sb = qg % NSB;
          mbar_wait(&kfull[ks], (qg / SK) & 1);
          tr.ev(3);
          mbar_wait(&sfree[sb], ((qg / NSB) & 1) ^ 1);
          tr.ev(4);
          tc_fence_after();
          const uint32_t kb = smem_u32(sK + ks * KV_BYTES);
          const uint32_t d = tmem + S_COL + sb * NQM;
#pragma unroll
          for (int kk = 0; kk < DH / 16; ++kk) {
            const int h = kk >> 2, w = (kk & 3) * 32;
            mma_bf16(d, desc_kmajor_sw128(kb + h * HALF_KV + w), desc_kmajor_sw128(qa + h * HALF_Q + w), idesc_qk,
                     kk > 0 ? 1u : 0u);
          }
          mma_commit(&sfull[sb]);
          mma_commit(&kempty[ks]);
        }
        mma_commit(&qempty[qb]);
        if (qu + NQB < n_my) {                     // this buffer's next unit
          mbar_wait(&qempty[qb], (qu / NQB) & 1);
          load_q(qu + NQB);
        }
      }
    }
  } else if (warp == 3) {
    // ================================================================ PV^T issuer
    // O^T += V_t^T . P_t^T and the row sums L^T += ONES . P_t^T (every lane holds l_n) into the unit's
    // double-buffered TMEM accumulator
    if (lane == 0 && !IMP_ONLY) {
      Tracer tr(a.trace, 3);
      uint32_t pg = 0;
      const uint64_t ones_desc = desc_kmajor_noswz(smem_u32(ones), 0, 0);
      for (int pu = 0; pu < n_my; ++pu) {
        const Unit& x = utab[pu];
        const uint32_t ob = pu & 1;
        const int NQ = (x.nq + 15) & ~15;
        const uint32_t idesc_pv = idesc_bf16(DH, NQ, true, true);
        const uint32_t idesc_l = idesc_bf16(128, NQ, false, true);
        const uint32_t dO = tmem + O_COL + ob * NQM;
        const uint32_t dl = tmem + L_COL + ob * NQM;
        for (int pt = x.t_lo; pt < x.t_hi; ++pt, ++pg) {
          const uint32_t pb = pg % NPB, vs = pg % SV;
          const bool first = pt == x.t_lo;
          mbar_wait(&pfull[pb], (pg / NPB) & 1);
          tr.ev(5);
          if (first) mbar_wait(&ofree[ob], ((pu >> 1) & 1) ^ 1);
          mbar_wait(&vfull[vs], (pg / SV) & 1);
          tr.ev(6);
          tc_fence_after();
          const uint32_t vb = smem_u32(sV + vs * KV_BYTES);
          const uint32_t pa = smem_u32(sP + pb * P_BYTES);
#pragma unroll
          for (int kk = 0; kk < KT / 16; ++kk) {
            const uint64_t pdesc = desc_mnmajor_noswz(pa + kk * 256, 128, P_CHUNK);
            const uint32_t acc = (first && kk == 0) ? 0u : 1u;
            mma_bf16(dO, desc_mnmajor_sw128(vb + kk * 16 * 128, HALF_KV), pdesc, idesc_pv, acc);
            mma_bf16(dl, ones_desc, pdesc, idesc_l, acc);
          }
          mma_commit(&vempty[vs]);
          mma_commit(&pvdone[pb]);
          if (pt + 1 == x.t_hi) mma_commit(&ofull[ob]);
        }
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // ================================================================ softmax (+ importance)
    SoftThread th;
    th.L = threadIdx.x - 128;                      // key lane of the tile (= TMEM lane of S^T)
    th.lane = lane;
    th.q4 = warp & 3;
    th.tmem = tmem;
    th.lane_base = (uint32_t)(th.q4 * 32) << 16;
    th.sl2 = a.scale * kLog2e;
    th.G = G;
    // block-score scratch [64 rows][64 columns]: the idle V ring (past the second Q buffer) in the
    // importance-only mode, a per-CTA global slice otherwise (layer 0, where the V ring is busy)
    th.scr = IMP_ONLY ? reinterpret_cast<float*>(sV + Q_BYTES) : a.imp_scratch + (size_t)blockIdx.x * NQM * kMaxB;
    Tracer tr(th.L == 0 ? a.trace : nullptr, 4);
    uint32_t g = 0;
    const bool causal = a.ext_mode == 2;
    for (int it = 0; it < n_my; ++it) {
      const Unit& xr = utab[it];
      const int nch = (xr.nq + 15) >> 4;           // 16-row chunks (1..4)
      tr.ev(0);
      if (causal) {
        switch (nch) {
          case 1: softmax_unit<1, true, IMP_ONLY>(a, xr, it, g, th, ss, tr); break;
          case 2: softmax_unit<2, true, IMP_ONLY>(a, xr, it, g, th, ss, tr); break;
          case 3: softmax_unit<3, true, IMP_ONLY>(a, xr, it, g, th, ss, tr); break;
          default: softmax_unit<4, true, IMP_ONLY>(a, xr, it, g, th, ss, tr); break;
        }
      } else {
        switch (a.nch_fixed ? 4 : nch) {
          case 1: softmax_unit<1, false, IMP_ONLY>(a, xr, it, g, th, ss, tr); break;
          case 2: softmax_unit<2, false, IMP_ONLY>(a, xr, it, g, th, ss, tr); break;
          case 3: softmax_unit<3, false, IMP_ONLY>(a, xr, it, g, th, ss, tr); break;
          default: softmax_unit<4, false, IMP_ONLY>(a, xr, it, g, th, ss, tr); break;
        }
      }
      if (xr.want_imp) importance_epilogue(a, xr, th, ss);
    }
  } else if (warp >= 8 && !IMP_ONLY) {
    // ================================================================ epilogue (thread = d_h lane)
    const int d = threadIdx.x - 256;
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    Tracer tr(d == 0 ? a.trace : nullptr, 5);
    // Output rows leave through shared memory, 32 query rows (two 16-row chunks) at a time: element
    // (query row n = r*G + g, lane d) of pass p goes to ost[(n - 32p) * DH + d], i.e. block row r's G heads
    // are one contiguous G*DH*2-byte run matching the output row [r0 + r][kvh*G*DH, (kvh+1)*G*DH); one
    // bulk async copy per block row then writes it (instead of 2-byte scattered stores from every thread).
    __nv_bfloat16* ost = reinterpret_cast<__nv_bfloat16*>(smem + OFF_OST);
    auto pass_begin = [&]() {                      // all 128 threads: the previous pass's stores have read ost
      if (d == 0) bulk_wait_read0();
      named_bar(2, 128);
    };
    auto pass_flush = [&](const Unit& xr, int p) {   // all 128 threads: rows [32p, 32p + 32) of the unit
      fence_proxy_async();
      named_bar(2, 128);
      if (d == 0) {
        const int r1 = min((32 * p + 32) / G, xr.nq / G);
        for (int r = 32 * p / G; r < r1; ++r)
          bulk_store_s2g(a.out + (size_t)(xr.r0 + r) * a.ldo + (size_t)xr.kvh * G * DH,
                         smem_u32(ost + (size_t)(r * G - 32 * p) * DH), (uint32_t)(G * DH * 2));
        bulk_commit();
      }
    };
    for (int it = 0; it < n_my; ++it) {
      const Unit& xr = utab[it];
      const int nq = xr.nq, nch = (nq + 15) >> 4;
      const uint32_t ob = it & 1;
      tr.ev(0);
      mbar_wait(&ofull[ob], (it >> 1) & 1);
      mbar_wait(&statfull[ob], (it >> 1) & 1);
      tr.ev(1);
      tc_fence_after();
      if (xr.nsplit == 1) {
        // O * (1/l) -> bf16 staging (MUFU reciprocal: ~1 ulp of fp32 before the bf16 rounding), 32 query rows
        // per pass, one bulk store per block row
#pragma unroll 1
        for (int p = 0; 2 * p < nch; ++p) {
          const bool two = 2 * p + 1 < nch;
          uint32_t r[32], rl[32];
          tmem_ld32x16(tmem + lane_base + O_COL + ob * NQM + 32 * p, r);
          tmem_ld32x16(tmem + lane_base + L_COL + ob * NQM + 32 * p, rl);
          if (two) {
            tmem_ld32x16(tmem + lane_base + O_COL + ob * NQM + 32 * p + 16, r + 16);
            tmem_ld32x16(tmem + lane_base + L_COL + ob * NQM + 32 * p + 16, rl + 16);
          }
          tmem_wait_ld();
          tr.ev(3);
          if (2 * p + 2 >= nch) {                  // the accumulator is in registers: free it early
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&ofree[ob]);
          }
          pass_begin();
          tr.ev(4);
#pragma unroll
          for (int e = 0; e < 32; ++e)
            if ((e < 16 || two) && 32 * p + e < nq)
              ost[e * DH + d] = __float2bfloat16_rn(__uint_as_float(r[e]) * rcp_approx(__uint_as_float(rl[e])));
          tr.ev(5);
          pass_flush(xr, p);
          tr.ev(6);
        }
        tr.ev(2);
      } else {
        // split piece: partial (unnormalised O^T rows, running max, row sum) -> workspace; the
        // last-arriving piece of the pair merges all partials in split order (flash-decoding style):
        // O = sum_s 2^(m_s - m) O_s / sum_s 2^(m_s - m) l_s.  Every piece reads the partials back from
        // global memory, so the arithmetic does not depend on which piece arrives last.
        const size_t slot_floats = (size_t)NQM * DH + 2 * NQM;
        float* base = a.part + (size_t)xr.pair * a.max_nsplit * slot_floats;
        float* po = base + (size_t)xr.sp * slot_floats;
#pragma unroll 1
        for (int c = 0; c < nch; ++c) {
          uint32_t r[16], rl[16];
          tmem_ld32x16(tmem + lane_base + O_COL + ob * NQM + 16 * c, r);
          tmem_ld32x16(tmem + lane_base + L_COL + ob * NQM + 16 * c, rl);
          tmem_wait_ld();
          float ld = 0.f;
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            if (16 * c + e < nq) __stcg(po + (16 * c + e) * DH + d, __uint_as_float(r[e]));
            if (16 * c + e == d) ld = __uint_as_float(rl[e]);
          }
          if (d >= 16 * c && d < 16 * c + 16 && d < nq)
            __stcg(reinterpret_cast<float2*>(po + NQM * DH) + d, make_float2(ss.stat[ob * NQM + d], ld));
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&ofree[ob]);
        __threadfence();
        named_bar(2, 128);
        if (d == 0) merge_flag = atomicAdd(&a.sem[xr.pair], 1);
        named_bar(2, 128);
        if (merge_flag == xr.nsplit - 1) {               // last piece: merge
          __threadfence();
          pass_begin();                                  // (also: the previous merge's readers of fsc are done)
          const int ns = xr.nsplit;
          float* fsc = reinterpret_cast<float*>(smem + OFF_MERGE);   // [MAXS][NQM] scales, [MAXS][..] 1/l
          if (d < nq) {
            float2 ml[MAXS];
#pragma unroll
            for (int s2 = 0; s2 < MAXS; ++s2)          // all statistics loads in flight at once
              if (s2 < ns) ml[s2] = __ldcg(reinterpret_cast<const float2*>(base + (size_t)s2 * slot_floats + NQM * DH) + d);
            float m = -CUDART_INF_F;
#pragma unroll
            for (int s2 = 0; s2 < MAXS; ++s2)
              if (s2 < ns) m = fmaxf(m, ml[s2].x);
            float lsum = 0.f;
#pragma unroll
            for (int s2 = 0; s2 < MAXS; ++s2)
              if (s2 < ns) {
                const float f = ml[s2].x == -CUDART_INF_F ? 0.f : ex2(ml[s2].x - m);
                fsc[s2 * NQM + d] = f;
                lsum += ml[s2].y * f;
              }
            fsc[MAXS * NQM + d] = 1.0f / lsum;
          }
          named_bar(2, 128);
#pragma unroll 1
          for (int n0 = 0; n0 < nq; n0 += 16) {
            float acc[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) acc[e] = 0.f;
#pragma unroll 2
            for (int s2 = 0; s2 < ns; ++s2) {
              const float* ps = base + (size_t)s2 * slot_floats + d;
              float v[16];
#pragma unroll
              for (int e = 0; e < 16; ++e) v[e] = n0 + e < nq ? __ldcg(ps + (n0 + e) * DH) : 0.f;
#pragma unroll
              for (int e = 0; e < 16; ++e) acc[e] += v[e] * fsc[s2 * NQM + n0 + e];
            }
            if (n0 % 32 == 0 && n0 > 0) {              // rows [n0 - 32, n0) staged: write them, reuse ost
              pass_flush(xr, n0 / 32 - 1);
              pass_begin();
            }
#pragma unroll
            for (int e = 0; e < 16; ++e)
              if (n0 + e < nq) ost[(n0 % 32 + e) * DH + d] = __float2bfloat16_rn(acc[e] * fsc[MAXS * NQM + n0 + e]);
          }
          pass_flush(xr, (nq - 1) / 32);
          if (d == 0) a.sem[xr.pair] = 0;                 // re-arm for the next launch
        }
        tr.ev(2);
      }
    }
    if (d == 0) bulk_wait0();                        // output rows written before the CTA retires
  }
  __syncthreads();
  if (warp == 3) {
    tc_fence_after();
    tmem_free<TMEM_COLS>(tmem);
  }
  if (threadIdx.x == 0 && a.trace) {
    unsigned long long gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    a.trace[((size_t)blockIdx.x * 8 + 7) * kTraceEv + 3] = clock64();
    a.trace[((size_t)blockIdx.x * 8 + 7) * kTraceEv + 4] = gt;
  }
}

// Unit table of one attention launch shape (CTA b of the attention grid = block b here), computed
// once per step instead of in the prologue of every attention launch (34 launches share the plan of
// layers >= 2).
__global__ void __launch_bounds__(NTHREADS) k_attn_plan(const __grid_constant__ AttnArgs a) {
  pdl_trigger();
  pdl_wait();
  __shared__ __align__(16) int scratch[4400];
  __shared__ Unit ut[UCAP];
  const int n = build_units(a, blockIdx.x, gridDim.x, scratch, ut);
  Unit* out = static_cast<Unit*>(a.plan_units);
  for (int k = threadIdx.x; k < n; k += NTHREADS) out[(size_t)blockIdx.x * UCAP + k] = ut[k];
  if (threadIdx.x == 0) a.plan_n[blockIdx.x] = n;
}

}  // namespace attn

bool attn_tc_supported(int head_dim, int page_size, int group) {
  return head_dim == attn::DH && page_size >= 8 && page_size <= 4096 && (page_size & (page_size - 1)) == 0 &&
         (group == 1 || group == 2 || group == 4);
}

int attn_tc_rows_per_chunk(int group) { return attn::NQM / group; }

// Query-row tensor map: q buffer [rows][ld] bf16 viewed as {head_dim, heads, rows}; box = 64 columns x
// G heads x (64 / G) rows, so one box fills a 64-column half of the unit's Q tile (row n = r*G + g).
bool attn_tc_make_qmap(const bf16* q, size_t rows, int ld, int n_heads, int group, CUtensorMap* mq) {
  return make_tma_3d_bf16(q, attn::DH, n_heads, rows, (uint64_t)attn::DH * 2, (uint64_t)ld * 2, 64, group,
                          attn::NQM / group, mq);
}

// KV pool tensor maps: the whole pool (all layers) viewed as [rows][head_dim] bf16.
bool attn_tc_make_maps(const bf16* Kpool, const bf16* Vpool, size_t rows, int head_dim, int page_size,
                       CUtensorMap* mk, CUtensorMap* mv) {
  const uint32_t box_rows = (uint32_t)std::min(page_size, attn::KT);
  return make_tma_2d_bf16(Kpool, rows, head_dim, head_dim, 64, box_rows, mk) &&
         make_tma_2d_bf16(Vpool, rows, head_dim, head_dim, 64, box_rows, mv);
}

template <bool IMP>
static void launch_tc(const CUtensorMap& mk, const CUtensorMap& mv, const CUtensorMap& mq, const AttnArgs& a, int grid,
                      cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn::k_attn_tc<IMP>, cudaFuncAttributeMaxDynamicSharedMemorySize, attn::SMEM_BYTES);
    attr = true;
  }
  launch_pdl(attn::k_attn_tc<IMP>, dim3(grid), dim3(attn::NTHREADS), attn::SMEM_BYTES, s, mk, mv, mq, a);
}

int attn_tc_grid(const AttnArgs& a);
static int attn_grid(const AttnArgs& a) { return attn_tc_grid(a); }
int attn_tc_grid(const AttnArgs& a) {
  const int G = a.n_q_heads / a.kv.n_kv_heads;
  const int rpc = attn::NQM / G;
  int max_units;
  if (a.ext_mode == 2) max_units = ((a.prefill_rows + rpc - 1) / rpc) * a.kv.n_kv_heads;
  else max_units = a.n_req * a.n_chunks * a.kv.n_kv_heads * (a.imp_only ? 1 : a.max_nsplit);
  return max_units <= 0 ? 0 : std::max(1, std::min(num_sms(), max_units));
}

int attn_tc_plan_capacity() { return attn::UCAP; }

// Plan the unit table of a decode attention launch shape into a.plan_units / a.plan_n; the launches
// that use it must have the same request list, row offsets and split settings.
bool launch_attention_plan(const AttnArgs& a, cudaStream_t s) {
  const int g = attn_grid(a);
  if (g <= 0 || !a.plan_units || !a.plan_n || a.ext_mode == 2) return false;
  launch_pdl(attn::k_attn_plan, dim3(g), dim3(attn::NTHREADS), 0, s, a);
  return true;
}

void launch_attention_tc(const CUtensorMap& mk, const CUtensorMap& mv, const CUtensorMap& mq, const AttnArgs& a,
                         cudaStream_t s) {
  const int grid = attn_grid(a);
  if (grid <= 0) return;
  if (a.imp_only) {
    launch_tc<true>(mk, mv, mq, a, grid, s);
  } else {
    launch_tc<false>(mk, mv, mq, a, grid, s);
  }
}

}  // namespace focus
