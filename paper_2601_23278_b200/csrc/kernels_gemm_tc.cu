// tcgen05 / TMEM / TMA GEMM for sm_100a:  acc[M x N] (fp32) = A[M x K] . W[N x K]^T, with epilogues
//   GEMM_STORE / GEMM_ADD  C = acc / C += acc (fp32; residual add for the O and down projections)
//   GEMM_SWIGLU            act = bf16(silu(gate) * up) from the interleaved gate|up tile (no fp32 round trip)
//   GEMM_QKV_ROPE          q|k|v = bf16(RoPE(acc)) + paged KV store of k and v (head_dim 128)
// A = activations (bf16, K-major rows), W = weights (bf16, [N][K] row-major = K-major).
//
// Default path: k_gemm_pair (below), CTA pairs on 256-row tiles with tcgen05.mma.cta_group::2.
// k_gemm_tc is the one-CTA-per-tile variant (FOCUS_GEMM_PAIR=0, and the stream-K / multicast
// experiments).  Persistent, warp-specialised (one CTA per SM, 256 threads):
//   warp 0      TMA producer: A tile 128 x 64 and W tile 256 x 64 per stage (128B swizzle), 4 stages
//   warp 1      MMA issuer: one elected thread issues tcgen05.mma.cta_group::1.kind::f16
//               (M=128, N=256, K=16) x 4 per stage into a TMEM accumulator; tcgen05.commit releases
//               the smem stage and, after the last k-block, signals the epilogue
//   warp 2      TMEM allocator (512 columns = two 128 x 256 fp32 accumulators, double-buffered)
//   warps 4..7  epilogue: tcgen05.ld 32x32b -> registers -> the mode's emitter (thread = output row),
//               stores staged through shared memory so they leave as whole 128-B lines
// Work units = (m tile, n tile, k split) with m fastest (CTAs sharing a weight tile run together and
// hit L2).  M is read from device memory (ragged row counts of the FOCUS step) and the split-K factor
// is chosen on device from the live tile count; split-K partials are reduced by the last-arriving
// split in a fixed order (deterministic).
#include <mutex>
#include <unordered_map>

#include <math_constants.h>

#include "tc_ptx.cuh"

namespace focus {

namespace tc {

constexpr int BM = 128, BK = 64;
constexpr int A_BYTES = BM * BK * 2;               // 16 KB
constexpr int EPI_SMEM = 4 * 32 * 128;             // epilogue staging: 4 warps x 32 rows x 128 B
// per tile width BN (128 or 256): W tile bytes, pipeline depth (192 KB of stages), shared memory
template <int BN>
struct GT {
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (192 * 1024) / STAGE_BYTES;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + EPI_SMEM + 1024 /*align*/ + 256 /*barriers*/;
};
constexpr int NUM_THREADS = 256;
constexpr int TMEM_COLS = 512;


// Hybrid data-parallel + stream-K schedule.  Tiles are ordered m-fastest.  The first dp_tiles tiles
// (whole waves of `grid` tiles) run data-parallel round-robin (tile = b + wave*grid: CTAs running
// together cover the m-tiles of the same weight tiles, which then stream from HBM once); the k-blocks
// of the remaining tiles are cut into `grid` equal contiguous ranges (stream-K).  A tile whose
// k-blocks span several CTAs is computed in pieces (one per CTA, in k order); each piece writes an
// fp32 partial to its CTA's slot (slot 0: its first stream-K segment, slot 1: its last) and the
// last-arriving piece reduces the partials in piece order (deterministic) and runs the epilogue.
// Every CTA derives the same schedule from the live M.
struct Sched {
  int m_tiles, n_tiles, kb, tiles, dp_tiles, sk_tiles, dp_mine;
  long long W, w_lo, w_hi;                          // stream-K work and this CTA's range
  int cs, rank, cluster, n_clusters, m_groups;     // clusters of cs CTAs share one weight tile (multicast)
};
__device__ __forceinline__ long long range_start(long long W, int b, int grid) { return (long long)b * W / grid; }
// CTA whose stream-K range contains work position x
__device__ __forceinline__ int owner(long long W, long long x, int grid) {
  return (int)(((x + 1) * grid + W - 1) / W) - 1;
}
template <int BN, int CS>
__device__ __forceinline__ Sched make_sched(int M, int N, int K, int policy) {
  Sched s;
  s.m_tiles = (M + BM - 1) / BM;
  s.n_tiles = (N + BN - 1) / BN;
  s.kb = K / BK;
  s.tiles = s.m_tiles * s.n_tiles;
  s.cs = CS;
  s.rank = CS > 1 ? (int)cluster_ctarank() : 0;
  s.cluster = blockIdx.x / CS;
  s.n_clusters = gridDim.x / CS;
  s.m_groups = (s.m_tiles + CS - 1) / CS;
  if (CS > 1) {
    // cluster-granular data-parallel units (weight tile nt, m-group): CTA rank r takes m-tile
    // mg * CS + r (past the live rows it computes discarded rows so the multicast stays in lockstep)
    const int units = s.n_tiles * s.m_groups;
    s.dp_tiles = units;
    s.sk_tiles = 0;
    s.dp_mine = units > s.cluster ? (units - 1 - s.cluster) / s.n_clusters + 1 : 0;
    s.W = 0;
    s.w_lo = s.w_hi = 0;
    return s;
  }
  const int grid = gridDim.x;
  // policy 0: hybrid, 1: all stream-K, 2: all data-parallel
  s.dp_tiles = policy == 1 ? 0 : (policy == 2 ? s.tiles : (s.tiles / grid) * grid);
  s.sk_tiles = s.tiles - s.dp_tiles;
  s.dp_mine = s.dp_tiles > (int)blockIdx.x ? (s.dp_tiles - 1 - (int)blockIdx.x) / grid + 1 : 0;
  s.W = (long long)s.sk_tiles * s.kb;
  s.w_lo = range_start(s.W, blockIdx.x, grid);
  s.w_hi = range_start(s.W, blockIdx.x + 1, grid);
  return s;
}
struct Seg {
  int tile, mt, nt, kb0, kb1, piece, npieces, slot, mine;   // slot = CTA where the tile's SK work starts
};
// i-th segment of this CTA: data-parallel tiles first, then stream-K segments starting at work w
__device__ __forceinline__ Seg dp_seg(const Sched& s, int i) {
  Seg g;
  g.kb0 = 0;
  g.kb1 = s.kb;
  g.piece = 0;
  g.npieces = 1;
  g.slot = 0;
  g.mine = 0;
  if (s.cs > 1) {
    const int u = s.cluster + i * s.n_clusters;
    g.nt = u / s.m_groups;
    g.mt = (u % s.m_groups) * s.cs + s.rank;
    g.tile = g.nt * s.m_tiles + g.mt;
  } else {
    g.tile = blockIdx.x + i * gridDim.x;
    g.mt = g.tile % s.m_tiles;
    g.nt = g.tile / s.m_tiles;
  }
  return g;
}
__device__ __forceinline__ Seg sk_seg(const Sched& s, long long w) {
  Seg g;
  const int lt = (int)(w / s.kb);
  g.tile = s.dp_tiles + lt;
  g.kb0 = (int)(w % s.kb);
  g.kb1 = (int)min((long long)s.kb, g.kb0 + (s.w_hi - w));
  g.mt = g.tile % s.m_tiles;
  g.nt = g.tile / s.m_tiles;
  const long long t0 = (long long)lt * s.kb;
  const int o0 = owner(s.W, t0, gridDim.x), o1 = owner(s.W, t0 + s.kb - 1, gridDim.x);
  g.piece = blockIdx.x - o0;
  g.npieces = o1 - o0 + 1;
  g.slot = o0;
  g.mine = (int)(s.w_lo / s.kb) == lt ? 0 : 1;
  return g;
}
// iterate this CTA's segments: for (SegIter it(sc); it.valid(); it.next()) { const Seg& g = it.g; ... }
struct SegIter {
  const Sched& s;
  int i;
  long long w;
  Seg g;
  __device__ __forceinline__ explicit SegIter(const Sched& sc) : s(sc), i(0), w(sc.w_lo) { load(); }
  __device__ __forceinline__ bool valid() const { return i < s.dp_mine || w < s.w_hi; }
  __device__ __forceinline__ void load() {
    if (i < s.dp_mine) g = dp_seg(s, i);
    else if (w < s.w_hi) g = sk_seg(s, w);
  }
  __device__ __forceinline__ void next() {
    if (i < s.dp_mine) ++i;
    else w += g.kb1 - g.kb0;
    load();
  }
};

// ---------------------------------------------------------------- epilogue emitters
// The accumulator arrives thread = row (tcgen05.ld 32x32b).  Stores go through a per-warp 32 x 128 B
// shared staging buffer (16-B chunks XOR-swizzled by row & 7: conflict-free both ways) and leave it
// row-contiguous: 8 lanes per row, 4 rows per instruction, so every warp store writes whole 128-B lines
// instead of 32 rows x 16 B.
constexpr int EPI_BUF = 32 * 128;                       // bytes per epilogue warp
__device__ __forceinline__ uint32_t epi_slot(uint32_t buf, int r, int j) { return buf + r * 128 + ((j ^ (r & 7)) << 4); }
__device__ __forceinline__ uint4 f4_bits(const float* v) {
  return make_uint4(__float_as_uint(v[0]), __float_as_uint(v[1]), __float_as_uint(v[2]), __float_as_uint(v[3]));
}
__device__ __forceinline__ uint32_t pack_bf2(float a, float b) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}

// `chunk(c0, v)` yields 32 consecutive fp32 accumulator columns [c0, c0+32) of this thread's row of the
// tile (TMEM or merged split partials); it must be called uniformly by the whole warp.  row0 = the
// warp's first tile row (this thread's row = row0 + lane), rows >= M are not written.
// part / nparts: the tile's columns are split into nparts equal groups (of 32-column chunks, SwiGLU
// 64-column pairs, RoPE half-head pairs) and this warp emits group `part` (two warps per TMEM lane
// quarter share a tile when nparts = 2).
// 192-wide QKV tiles (see k_gemm_pair): weight rows (relative to head 3j) of the 32-row boxes of
// [tile parity][pair rank][box]
__device__ __constant__ int kQkv192Rows[12] = {0, 32, 64, 96, 128, 192, 160, 224, 256, 288, 320, 352};
// RoPE step st of QKV tile nt: accumulator columns lo (dims d0..d0+31) and hi (d0+64..d0+95) of `head`
template <int BN>
__device__ __forceinline__ void qkv_step(int nt, int st, int& lo, int& hi, int& head, int& d0) {
  if constexpr (BN == 192) {
    const int j3 = 3 * (nt >> 1);
    if ((nt & 1) == 0) {
      lo = st == 2 ? 128 : 32 * st;  hi = st == 2 ? 160 : 32 * st + 64;  head = j3 + (st == 2);  d0 = st == 1 ? 32 : 0;
    } else {
      lo = st == 0 ? 0 : 32 + 32 * st;  hi = st == 0 ? 32 : 96 + 32 * st;  head = j3 + 1 + (st > 0);  d0 = st == 2 ? 32 : (st == 0 ? 32 : 0);
    }
  } else {
    const int hh = st >> 1;
    d0 = (st & 1) * 32;
    lo = hh * 128 + d0;
    hi = lo + 64;
    head = nt * (BN / 128) + hh;
  }
}

template <int MODE, int BN, typename Chunk>
__device__ __forceinline__ void epilogue_tile(Chunk&& chunk, int row0, int M, int nt, int N, float* __restrict__ C,
                                              int ldc, const GemmEpi& epi, uint32_t buf, int part = 0,
                                              int nparts = 1) {
  const int lane = threadIdx.x & 31;
  const int rr = lane >> 3, jj = lane & 7;              // read-back: row 4i + rr, 16-B chunk jj
  if constexpr (MODE == GEMM_STORE || MODE == GEMM_ADD) {
    const bool vec_ok = (ldc % 4) == 0 && (((uintptr_t)C) & 15) == 0;
    // LM head: the confidence statistics of this thread's row over each 64-column group (columns in
    // ascending order; ties keep the lowest id).  conf = 1 / sum exp(z - max) (A-CF1), mask id excluded.
    const bool vocab = MODE == GEMM_STORE && epi.vpart != nullptr;
    VocabPartial vp{-CUDART_INF_F, 0.f, 0x7fffffff, 0};
#pragma unroll 1
    for (int c0 = part * (BN / nparts); c0 < (part + 1) * (BN / nparts); c0 += 32) {
      float v[32];
      chunk(c0, v);
      if (vocab) {
        const int cb = nt * BN + c0;
        float m = -CUDART_INF_F;
        int im = 0x7fffffff;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const bool ok = cb + i < N && cb + i != epi.mask_id;
          if (ok && v[i] > m) { m = v[i]; im = cb + i; }
        }
        float sum = 0.f;
        if (m != -CUDART_INF_F) {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (cb + i < N && cb + i != epi.mask_id) sum += __expf(v[i] - m);
        }
        if ((c0 & 32) == 0) {
          vp = VocabPartial{m, sum, im, 0};
        } else if (m != -CUDART_INF_F) {            // second half of the 64-column group
          if (vp.m == -CUDART_INF_F) {
            vp = VocabPartial{m, sum, im, 0};
          } else {
            const float mm = fmaxf(vp.m, m);
            vp.s = vp.s * __expf(vp.m - mm) + sum * __expf(m - mm);
            vp.idx = m > vp.m ? im : vp.idx;        // equal maxima: the first group's id is lower
            vp.m = mm;
          }
        }
        if ((c0 & 32) != 0 || c0 + 32 >= (part + 1) * (BN / nparts)) {
          const int row = row0 + lane;
          if (row < M && (cb & ~63) < N) epi.vpart[(size_t)row * epi.vp_ld + (cb >> 6)] = vp;
        }
        if (C == nullptr) continue;                    // logits not stored (no debug taps)
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) sts128(epi_slot(buf, lane, j), f4_bits(v + 4 * j));
      __syncwarp();
      const int col = nt * BN + c0 + 4 * jj;
      const bool col_vec = col + 4 <= N && vec_ok;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int r = 4 * i + rr, row = row0 + r;
        const uint4 x = lds128(epi_slot(buf, r, jj));
        if (row < M && col < N) {
          float* dst = C + (size_t)row * ldc + col;
          const float e[4] = {__uint_as_float(x.x), __uint_as_float(x.y), __uint_as_float(x.z), __uint_as_float(x.w)};
          if (col_vec) {
            if (MODE == GEMM_ADD)   // residual += acc as a vector reduction at L2 (one contributor per
                                    // element, so the result is exactly fl(x + acc)); no load round trip
              asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "f"(e[0]), "f"(e[1]), "f"(e[2]),
                           "f"(e[3])
                           : "memory");
            else
              *reinterpret_cast<float4*>(dst) = make_float4(e[0], e[1], e[2], e[3]);
          } else {
            for (int t = 0; t < 4 && col + t < N; ++t) dst[t] = MODE == GEMM_ADD ? dst[t] + e[t] : e[t];
          }
        }
      }
      __syncwarp();
    }
  } else if constexpr (MODE == GEMM_SWIGLU) {
    // tile nt = gate rows [128 nt, 128 nt + 128) | up rows (W_gu interleaved by kGuGroup = BN / 2):
    // act[row][128 nt + c] = bf16(silu(gate_c) * up_c); two 32-column groups (64 bf16 = 128 B) per staging
    static_assert(BN == 2 * kGuGroup, "gate/up interleave must match the tile");
#pragma unroll 1
    for (int c0 = part * (kGuGroup / nparts); c0 < (part + 1) * (kGuGroup / nparts); c0 += 64) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float gv[32], uv[32];
        chunk(c0 + 32 * h, gv);
        chunk(c0 + 32 * h + kGuGroup, uv);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          uint32_t w[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int i = 8 * j + 2 * e;
            // silu(g) * u = g * u / (1 + 2^(-g log2 e)): MUFU ex2 + rcp (relative error ~1e-7, far below
            // the bf16 rounding of the result)
            const float a0 = __fdividef(gv[i] * uv[i], 1.0f + exp2f(-1.4426950408889634f * gv[i]));
            const float a1 = __fdividef(gv[i + 1] * uv[i + 1], 1.0f + exp2f(-1.4426950408889634f * gv[i + 1]));
            w[e] = pack_bf2(a0, a1);
          }
          sts128(epi_slot(buf, lane, 4 * h + j), make_uint4(w[0], w[1], w[2], w[3]));
        }
      }
      __syncwarp();
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int r = 4 * i + rr, row = row0 + r;
        const uint4 x = lds128(epi_slot(buf, r, jj));
        if (row < M) *reinterpret_cast<uint4*>(epi.out + (size_t)row * epi.ldo + nt * kGuGroup + c0 + 8 * jj) = x;
      }
      __syncwarp();
    }
  } else {
    // GEMM_QKV_ROPE (head_dim 128): the tile holds BN/128 heads of the fused q|k|v output.  q and k heads
    // are rotated (rotate-half pairs (c, c+64), angle pos * theta^(-2c/dh) from the fp64-built table),
    // rounded to bf16 and written to the qkv rows; k and v heads are also stored at the row's paged
    // KV slot (the "sparse KV fill").  Writing a committed block slot raises the invariant flag.
    const int row = row0 + lane;
    RowInfo ri{0, -1, 0, 0};
    if (row < M) ri = epi.rows[row];
    if (row < M && ri.j >= 0 && ((epi.st[ri.slot].committed >> ri.j) & 1ull)) atomicExch(&epi.cnt->invariant, 1);
    const int hkv = epi.kv.n_kv_heads;
    // this row's paged KV slot (kv head 0), looked up once per tile: the store loop below then has no
    // dependent page-table load per 16-B chunk
    const unsigned long long kv_row = row < M ? (unsigned long long)kv_offset(epi.kv, ri.slot, ri.pos, 0) : 0ull;
    const size_t kv_head_stride = (size_t)epi.kv.page_size * epi.kv.head_dim;
    // (head, 32-column half-pair) steps of the tile, split evenly between the parts
    constexpr int kSteps = BN == 192 ? 3 : (BN / 128) * 2;
#pragma unroll 1
    for (int st = part * kSteps / nparts; st < (part + 1) * kSteps / nparts; ++st) {
      int lo_col, hi_col, head, c0;                      // head: 0..Hq-1 q, then k, then v
      qkv_step<BN>(nt, st, lo_col, hi_col, head, c0);
      const bool is_v = head >= epi.n_q_heads + hkv;
      const bool is_k = !is_v && head >= epi.n_q_heads;
      const int kvh = head - epi.n_q_heads - (is_v ? hkv : 0);
      {
        float lo[32], hi[32];
        chunk(lo_col, lo);
        chunk(hi_col, hi);
        if (!is_v && row < M) {
          const float* cr = epi.ropeT + (size_t)c0 * epi.rope_ld + row;          // [f][row]: coalesced
          const float* sr = cr + (size_t)64 * epi.rope_ld;
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float cc = __ldg(cr + (size_t)i * epi.rope_ld), ss = __ldg(sr + (size_t)i * epi.rope_ld);
            const float y1 = lo[i] * cc - hi[i] * ss;
            const float y2 = hi[i] * cc + lo[i] * ss;
            lo[i] = y1;
            hi[i] = y2;
          }
        }
        // staged row: chunks 0..3 = bf16 cols [c0, c0+32), chunks 4..7 = cols [c0+64, c0+96)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          sts128(epi_slot(buf, lane, j),
                 make_uint4(pack_bf2(lo[8 * j], lo[8 * j + 1]), pack_bf2(lo[8 * j + 2], lo[8 * j + 3]),
                            pack_bf2(lo[8 * j + 4], lo[8 * j + 5]), pack_bf2(lo[8 * j + 6], lo[8 * j + 7])));
          sts128(epi_slot(buf, lane, 4 + j),
                 make_uint4(pack_bf2(hi[8 * j], hi[8 * j + 1]), pack_bf2(hi[8 * j + 2], hi[8 * j + 3]),
                            pack_bf2(hi[8 * j + 4], hi[8 * j + 5]), pack_bf2(hi[8 * j + 6], hi[8 * j + 7])));
        }
        __syncwarp();
        const int col = c0 + (jj < 4 ? 8 * jj : 64 + 8 * (jj - 4));
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int r = 4 * i + rr, rw = row0 + r;
          const uint4 x = lds128(epi_slot(buf, r, jj));
          const unsigned long long kvo = __shfl_sync(0xffffffffu, kv_row, r);
          if (rw < M) {
            *reinterpret_cast<uint4*>(epi.out + (size_t)rw * epi.ldo + head * 128 + col) = x;
            if (is_k || is_v)
              *reinterpret_cast<uint4*>((is_v ? epi.kv.V : epi.kv.K) + kvo + (size_t)kvh * kv_head_stride + col) = x;
          }
        }
        __syncwarp();
      }
    }
  }
}

template <int MODE, int BN, int CS>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    k_gemm_tc(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, float* __restrict__ C,
              int ldc, int N, int K, const int* __restrict__ M_dev, int M_max, float* __restrict__ ws,
              int* __restrict__ sem, int policy, const GemmEpi epi) {
  constexpr int STAGES = GT<BN>::STAGES, B_BYTES = GT<BN>::B_BYTES, STAGE_BYTES = GT<BN>::STAGE_BYTES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;                                   // STAGES x A_BYTES
  uint8_t* sB = smem + STAGES * A_BYTES;                // STAGES x B_BYTES
  const uint32_t epi_buf = smem_u32(smem + STAGES * STAGE_BYTES) + (uint32_t)(((threadIdx.x >> 5) & 3) * 32 * 128);
  uint64_t* bars = (uint64_t*)(smem + STAGES * STAGE_BYTES + EPI_SMEM);
  uint64_t* full = bars;                                // [STAGES]
  uint64_t* empty = bars + STAGES;                      // [STAGES]
  uint64_t* tfull = bars + 2 * STAGES;                  // [2]
  uint64_t* tempty = bars + 2 * STAGES + 2;             // [2]
  uint32_t* tmem_base_sh = (uint32_t*)(bars + 2 * STAGES + 4);
  int* flag_sh = (int*)(tmem_base_sh + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  pdl_trigger();
  const int pf = policy >> 8;                           // L2 prefetch distance in k-blocks
  constexpr uint16_t cmask = (uint16_t)((1u << CS) - 1u);

  if (warp == 0 && lane == 0) {
    // empty[s] completes when the MMA of every CTA of the cluster has consumed stage s (each CTA's
    // commit multicasts an arrival), so any CTA may then multicast its W slice into all of them
    for (int i = 0; i < STAGES; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], CS); }
    for (int i = 0; i < 2; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], 4); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&mapA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&mapB) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_base_sh)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  if (CS > 1) cluster_sync();                           // peers' barriers initialised before any multicast
  tc_fence_after();
  const uint32_t tmem = *tmem_base_sh;
  pdl_wait();                                           // the A rows / live M come from earlier kernels
  const int M = M_dev ? min(*M_dev, M_max) : M_max;
  const Sched sc = make_sched<BN, CS>(M, N, K, policy & 0xff);

  if (warp == 0) {
    // ---------------- TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (SegIter si(sc); si.valid(); si.next()) {
        const Seg& g = si.g;
        // warm L2 with the first k-blocks of the segment beyond the smem ring
        for (int kb = g.kb0 + STAGES; kb < min(g.kb1, g.kb0 + STAGES + pf); ++kb) {
          tma_prefetch_2d(&mapA, kb * BK, g.mt * BM);
          tma_prefetch_2d(&mapB, kb * BK, g.nt * BN + (CS > 1 ? sc.rank * (BN / CS) : 0));
        }
        for (int kb = g.kb0; kb < g.kb1; ++kb) {
          // L2 prefetch `pf` k-blocks past the ring, so the TMA loads below hit L2 instead of HBM
          if (pf > 0 && kb + STAGES + pf < g.kb1) {
            tma_prefetch_2d(&mapA, (kb + STAGES + pf) * BK, g.mt * BM);
            tma_prefetch_2d(&mapB, (kb + STAGES + pf) * BK, g.nt * BN + (CS > 1 ? sc.rank * (BN / CS) : 0));
          }
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], STAGE_BYTES);
          tma_load_2d(sA + stage * A_BYTES, &mapA, &full[stage], kb * BK, g.mt * BM);
          if (CS == 1) {
            tma_load_2d(sB + stage * B_BYTES, &mapB, &full[stage], kb * BK, g.nt * BN);
          } else {                                      // my 1/CS slice of the W tile, to every CTA
            constexpr int SL = BN / CS;
            tma_load_2d_mc(sB + stage * B_BYTES + sc.rank * SL * 128, &mapB, &full[stage], kb * BK,
                           g.nt * BN + sc.rank * SL, cmask);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16(BM, BN, false, false);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (SegIter si(sc); si.valid(); si.next(), ++it) {
        const Seg& g = si.g;
        const int kb0 = g.kb0, kb1 = g.kb1;
        const int acc = it & 1;
        mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(acc * BN);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + stage * A_BYTES), b0 = smem_u32(sB + stage * B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            mma_bf16(d, desc_kmajor_sw128(a0 + k * 32), desc_kmajor_sw128(b0 + k * 32), idesc, (kb > kb0 || k > 0) ? 1u : 0u);
          if (CS == 1) mma_commit(&empty[stage]);
          else mma_commit_mc(&empty[stage], cmask);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        mma_commit(&tfull[acc]);
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: warp q = warp-4 owns TMEM lanes [32q, 32q+32) (thread = output row)
    const int q = warp - 4;
    const int et = threadIdx.x - 128;                   // 0..127
    int it = 0;
    for (SegIter si(sc); si.valid(); si.next(), ++it) {
      const Seg& g = si.g;
      const int nt = g.nt;
      const int acc = it & 1;
      mbar_wait(&tfull[acc], (it >> 1) & 1);
      tc_fence_after();
      const int row = g.mt * BM + q * 32 + lane;
      const bool row_ok = row < M;
      const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN);
      if (g.npieces == 1) {
        // accumulator chunks straight from TMEM (warp-collective loads)
        auto chunk = [&](int c0, float* v) { tmem_ld32(taddr + c0, v); };
        epilogue_tile<MODE, BN>(chunk, row - lane, M, nt, N, C, ldc, epi, epi_buf);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
      } else {
        // piece of a tile split across CTAs: write the partial, the last-arriving piece reduces all
        // partials in piece (= k) order
        float* my = ws + ((size_t)blockIdx.x * 2 + g.mine) * (BM * BN) + (size_t)(q * 32 + lane) * BN;
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 32) {
          float v[32];
          tmem_ld32(taddr + c0, v);
#pragma unroll
          for (int i = 0; i < 32; i += 4)
            __stcg(reinterpret_cast<float4*>(my + c0 + i), make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]));
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
        __threadfence();
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (et == 0) *flag_sh = atomicAdd(&sem[g.slot], 1);
        asm volatile("bar.sync 1, 128;" ::: "memory");
        const bool last = *flag_sh == g.npieces - 1;
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (last) {
          __threadfence();
          // piece p was written by CTA slot+p: into its slot 1 if p == 0 and the tile is not that CTA's
          // first segment, else into its slot 0
          const int w0 = (int)(range_start(sc.W, g.slot, gridDim.x) / sc.kb) == g.tile - sc.dp_tiles ? 0 : 1;
          const size_t row_off = (size_t)(q * 32 + lane) * BN;
          auto piece_ptr = [&](int p) {
            return ws + ((size_t)(g.slot + p) * 2 + (p == 0 ? w0 : 0)) * (BM * BN) + row_off;
          };
          auto chunk = [&](int c0, float* v) {
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
              float4 s4 = __ldcg(reinterpret_cast<const float4*>(piece_ptr(0) + c0 + i));
              for (int p = 1; p < g.npieces; ++p) {
                const float4 t = __ldcg(reinterpret_cast<const float4*>(piece_ptr(p) + c0 + i));
                s4.x += t.x; s4.y += t.y; s4.z += t.z; s4.w += t.w;
              }
              v[i] = s4.x; v[i + 1] = s4.y; v[i + 2] = s4.z; v[i + 3] = s4.w;
            }
          };
          epilogue_tile<MODE, BN>(chunk, row - lane, M, nt, N, C, ldc, epi, epi_buf);
          asm volatile("bar.sync 1, 128;" ::: "memory");
          if (et == 0) sem[g.slot] = 0;
        }
      }
    }
  }
  __syncthreads();
  if (CS > 1) cluster_sync();                           // no CTA leaves while peers may still signal it
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

// ---------------------------------------------------------------- CTA-pair variant (cta_group::2)
// A (2,1,1) cluster computes a 256 x BN tile: CTA r stages A rows [256 mp + 128 r, +128) and W rows
// [BN nt + BN/2 r, +BN/2) in its own shared memory (both loads complete on the leader's `full`
// barrier), the leader's MMA thread issues tcgen05.mma.cta_group::2 (M=256, N=BN, K=16) which reads
// both CTAs' operands, and each CTA's TMEM receives its own 128 rows x BN columns.  Per CTA and
// k-block this moves (128 + BN/2) x 64 operand elements instead of (128 + BN) x 64 for the same MMA
// work, i.e. a quarter less L2->SM traffic at BN = 256 and a deeper pipeline (6 stages instead of 4).
// KA k-atoms (64 columns each) per pipeline stage: each operand of a stage is ONE 3-D TMA box
// {64, rows, KA} (measured: a CTA's TMA throughput is set by boxes per stage more than by bytes per box,
// so fewer, larger boxes per stage feed the tensor core faster).
template <int BN, int KA>
struct GP {
  static constexpr int A_STAGE = BM * BK * 2 * KA;
  static constexpr int B_ATOM = (BN / 2) * BK * 2;
  static constexpr int B_STAGE = B_ATOM * KA;
  static constexpr int STAGE_BYTES = A_STAGE + B_STAGE;
  static constexpr int STAGES = (192 * 1024) / STAGE_BYTES;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 2 * EPI_SMEM + 1024 + 256;   // + staging of warps 0-3
};

__device__ __forceinline__ void tma_load_3d_pair(void* dst, const CUtensorMap* map, uint32_t bar_cluster, int x, int y,
                                                 int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(bar_cluster), "r"(x), "r"(y), "r"(z)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_pair_hint(void* dst, const CUtensorMap* map, uint32_t bar_cluster, int x,
                                                      int y, int z, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], "
      "[%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(bar_cluster), "r"(x), "r"(y), "r"(z), "l"(pol)
      : "memory");
}

// development trace (scripts/gemm_bench.cu): per CTA, 3 roles x 256 clock64 stamps (producer after each
// empty wait, MMA after each full wait, epilogue after each tfull wait / at the end); null = off
__device__ long long* g_gemm_trace = nullptr;
constexpr int kGemmTraceEv = 256;

__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* map, int x, int y, int z) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global [%0, {%1, %2, %3}];" ::"l"((uint64_t)map), "r"(x), "r"(y), "r"(z)
               : "memory");
}

// m_hint: expected live rows (host estimate).  Before waiting on the producing kernel (PDL), the
// producer prefetches into L2 the weight boxes of the first stages of the unit it expects to run
// first; weights are never written by earlier kernels, and a wrong guess only costs a wasted prefetch.
template <int MODE, int BN, int KA>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    k_gemm_pair(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, float* __restrict__ C,
                int ldc, int N, int K, const int* __restrict__ M_dev, int M_max, const GemmEpi epi, int m_hint,
                float* __restrict__ ws, int* __restrict__ sem, int flags) {
  const int sk = flags & 1;                             // bit 0: stream-K schedule
  const bool hints = (flags & 2) != 0;                  // bit 1: L2 hints (weights evict-first, activations evict-last)
  const int nsplit = ((flags >> 3) & 3) + 1;            // bits 3-4: k-ranges per unit (ordered split-K)
  using G = GP<BN, KA>;
  constexpr int STAGES = G::STAGES, STAGE_BYTES = G::STAGE_BYTES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * G::A_STAGE;
  // epilogue staging: warps 4-7 use the first 16 KB, warps 0-3 (last-tile helpers) the second
  const uint32_t epi_buf = smem_u32(smem + STAGES * STAGE_BYTES) + (uint32_t)(((threadIdx.x >> 5) & 3) * 32 * 128) +
                           (threadIdx.x < 128 ? (uint32_t)EPI_SMEM : 0u);
  uint64_t* bars = (uint64_t*)(smem + STAGES * STAGE_BYTES + 2 * EPI_SMEM);
  uint64_t* full = bars;                                // [STAGES]  (leader's are the live ones)
  uint64_t* empty = bars + STAGES;                      // [STAGES]  (both CTAs, by the leader's commit)
  uint64_t* tfull = bars + 2 * STAGES;                  // [2]       (both CTAs, by the leader's commit)
  uint64_t* tempty = bars + 2 * STAGES + 2;             // [2]       (leader's: 8 epilogue warps of the pair)
  uint32_t* tmem_base_sh = (uint32_t*)(bars + 2 * STAGES + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  pdl_trigger();
  const uint32_t rank = cluster_ctarank();
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < STAGES; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], 8); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    prefetch_map(&mapA);
    prefetch_map(&mapB);
  }
  if (warp == 2) {   // the same warp of both CTAs allocates the pair's TMEM (same destination offset)
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_base_sh)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (warp == 0 && lane == 0 && m_hint > 0 && !sk) {
    const int mph = (m_hint + 2 * BM - 1) / (2 * BM);
    const int u = blockIdx.x >> 1;
    if (u < mph * ((N + BN - 1) / BN)) {
      const int nt = u / mph;
      const int pf = min(K / (BK * KA), STAGES);
      for (int ks = 0; ks < pf; ++ks) tma_prefetch_3d(&mapB, 0, nt * BN + (int)rank * (BN / 2), ks * KA);
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_base_sh;
  pdl_wait();
  const int M = M_dev ? min(*M_dev, M_max) : M_max;
  const int m_pairs = (M + 2 * BM - 1) / (2 * BM);
  const int units = m_pairs * ((N + BN - 1) / BN);
  const int pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;
  const int ks_n = K / (BK * KA);                      // pipeline stages per tile
  long long* trace = g_gemm_trace ? g_gemm_trace + (size_t)blockIdx.x * 3 * kGemmTraceEv : nullptr;
  int tn = 0;
  auto stamp = [&](int role) {
    if (trace && tn < kGemmTraceEv - 1) trace[role * kGemmTraceEv + 1 + tn++] = clock64();
  };
  if (trace && threadIdx.x == 0) trace[0] = clock64();

  // Work of this pair: data-parallel (sk = 0: whole units pair, pair + n_pairs, ...) or stream-K
  // (sk = 1: the flattened (unit, stage) sequence cut into n_pairs equal contiguous ranges).  A unit
  // cut by a range boundary is computed in pieces; the piece holding its first stages (run last by
  // its pair) finalises it: it adds the later pieces' fp32 partials (run first by the following
  // pairs, written to their CTA's workspace slot) in pair order, then runs the epilogue.  Every pair
  // writes at most one partial (its first segment), so slot = CTA.
  const long long W = (long long)units * ks_n;
  const long long w_lo = sk ? (long long)pair * W / n_pairs : 0, w_hi = sk ? (long long)(pair + 1) * W / n_pairs : 0;
  auto owner = [&](long long x) { return (int)(((x + 1) * n_pairs + W - 1) / W) - 1; };
  auto empty_range = [&](int qq) { return (long long)qq * W / n_pairs == (long long)(qq + 1) * W / n_pairs; };
  struct PSeg { int u, k0, k1, h; };
  // segment i of this pair (valid while the returned u < units)
  // Ordered split-K (flags bit 2, GEMM_ADD, one wave): pair p computes half p & 1 of the k-blocks of
  // unit p >> 1; half 0 adds its partial to the residual first and raises the unit's flag, half 1
  // waits for the flag before adding its own, so the result is fl(fl(x + acc_0) + acc_1) on every run.
  // (the split depends only on the GEMM's shape, never on the live row count, so every row's result
  // is the same whatever the batch: the ordered ranges are data-parallel segments (unit, range) in
  // increasing order, and a range only waits on the previous range of its unit, a smaller segment,
  // so the persistent pairs cannot deadlock)
  const bool split2 = MODE == GEMM_ADD && (flags & 4) && !sk && ks_n >= 4 * nsplit;
  // k-range boundaries of the ordered split: range h = [kb(h), kb(h + 1)); every range but the last
  // gives up ks_n / 32 k-blocks to the last, so the adds of the earlier ranges overlap its tail
  auto kb = [&](int h) { return h == 0 ? 0 : h == nsplit ? ks_n : h * ks_n / nsplit - ks_n / 32 * h / (nsplit - 1); };
  // a pair with a single data-parallel unit (the decode shapes' QKV / O / down GEMMs) emits it with 8
  // warps: warps 0-3 are idle by then and the epilogue is not overlapped with any MMA
  const bool joint = !sk && !split2;
  const int n_mine = (!sk && !split2 && pair < units) ? (units - pair + n_pairs - 1) / n_pairs : 0;
  auto seg_at = [&](int i, long long& w) -> PSeg {
    PSeg g;
    g.h = 0;
    if (split2) {
      const int j = pair + i * n_pairs;
      if (j >= nsplit * units) { g.u = units; g.k0 = g.k1 = 0; return g; }
      g.u = j / nsplit;
      g.h = j % nsplit;
      g.k0 = kb(g.h);
      g.k1 = kb(g.h + 1);
      return g;
    }
    if (!sk) { g.u = pair + i * n_pairs; g.k0 = 0; g.k1 = ks_n; return g; }
    if (w >= w_hi) { g.u = units; g.k0 = g.k1 = 0; return g; }
    g.u = (int)(w / ks_n);
    g.k0 = (int)(w % ks_n);
    g.k1 = (int)min((long long)ks_n, g.k0 + (w_hi - w));
    w += g.k1 - g.k0;
    return g;
  };

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t full_l = mapa_shared(smem_u32(full), 0);
      const uint64_t pol_a = l2_policy_evict_last(), pol_b = l2_policy_evict_first();
      int stage = 0;
      uint32_t phase = 0;
      long long w = w_lo;
      for (int i = 0;; ++i) {
        const PSeg g = seg_at(i, w);
        if (g.u >= units) break;
        const int mp = g.u % m_pairs, nt = g.u / m_pairs;
        for (int ks = g.k0; ks < g.k1; ++ks) {
          mbar_wait(&empty[stage], phase ^ 1);
          stamp(0);
          if (rank == 0) mbar_expect_tx(&full[stage], 2 * STAGE_BYTES);
          const uint32_t fb = full_l + stage * 8;
          if (MODE == GEMM_QKV_ROPE && BN == 192) {
            // 192-wide QKV tile = 1.5 heads, gathered so every RoPE pair (d, d + 64) stays in the tile:
            // even tiles n = 2j: head 3j + head 3j+1 dims [0,32) and [64,96); odd tiles: head 3j+1 dims
            // [32,64) and [96,128) + head 3j+2.  Weight rows in 32-row boxes, 3 per CTA of the pair.
            const int base = 384 * (nt >> 1);
            const int seg = ((nt & 1) * 2 + (int)rank) * 3;
#pragma unroll
            for (int i = 0; i < 3; ++i)
              tma_load_3d_pair_hint(sB + stage * G::B_STAGE + i * 32 * 128, &mapB, fb, 0, base + kQkv192Rows[seg + i],
                                    ks * KA, pol_b);
            tma_load_3d_pair_hint(sA + stage * G::A_STAGE, &mapA, fb, 0, mp * 2 * BM + (int)rank * BM, ks * KA, pol_a);
          } else if (hints) {
            tma_load_3d_pair_hint(sA + stage * G::A_STAGE, &mapA, fb, 0, mp * 2 * BM + (int)rank * BM, ks * KA, pol_a);
            tma_load_3d_pair_hint(sB + stage * G::B_STAGE, &mapB, fb, 0, nt * BN + (int)rank * (BN / 2), ks * KA, pol_b);
          } else {
            tma_load_3d_pair(sA + stage * G::A_STAGE, &mapA, fb, 0, mp * 2 * BM + (int)rank * BM, ks * KA);
            tma_load_3d_pair(sB + stage * G::B_STAGE, &mapB, fb, 0, nt * BN + (int)rank * (BN / 2), ks * KA);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0 && lane == 0) {
      constexpr uint32_t idesc = idesc_bf16(2 * BM, BN, false, false);
      int stage = 0;
      uint32_t phase = 0;
      long long w = w_lo;
      for (int it = 0;; ++it) {
        const PSeg g = seg_at(it, w);
        if (g.u >= units) break;
        const int acc = it & 1;
        mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(acc * BN);
        for (int ks = g.k0; ks < g.k1; ++ks) {
          mbar_wait(&full[stage], phase);
          stamp(1);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + stage * G::A_STAGE), b0 = smem_u32(sB + stage * G::B_STAGE);
#pragma unroll
          for (int ka = 0; ka < KA; ++ka)
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              mma_bf16_pair(d, desc_kmajor_sw128(a0 + ka * A_BYTES + k * 32), desc_kmajor_sw128(b0 + ka * G::B_ATOM + k * 32),
                            idesc, (ks > g.k0 || ka > 0 || k > 0) ? 1u : 0u);
          mma_commit_pair(&empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        mma_commit_pair(&tfull[acc]);
      }
    }
  } else if (warp == 3) {
    if constexpr (MODE == GEMM_QKV_ROPE) {
      // L2 prefetch of the next attention launch's context K/V (see GemmEpi::pf_units): attention CTA
      // c's first units, pf_tiles key tiles each, spread over this GEMM's CTAs.  Context pages are
      // complete (committed in earlier steps); the plan comes from this step's k_attn_plan, which
      // completed before this kernel's griddepcontrol.wait returned.
      if (lane == 0 && epi.pf_units != nullptr && epi.pf_tiles > 0) {
        const KVView& kv = epi.kv;
        const uint32_t page_bytes = (uint32_t)kv.page_size * kv.head_dim * 2;
        const int tile_keys = 128;
        for (int c = blockIdx.x; c < epi.pf_grid; c += gridDim.x) {
          const int n = min(epi.pf_n[c], epi.pf_ucap);
          int budget = epi.pf_tiles;
          for (int k = 0; k < n && budget > 0; ++k) {
            const AttnUnit& u = epi.pf_units[(size_t)c * epi.pf_ucap + k];
            for (int t = u.t_lo; t < u.t_hi && budget > 0; ++t, --budget) {
              const int k0 = t * tile_keys, k1 = min(k0 + tile_keys, u.s0);   // context keys only
              for (int pos = k0; pos < k1; pos += kv.page_size) {
                const int page = kv.page_table[(size_t)u.slot * kv.max_pages + pos / kv.page_size];
                const size_t off = (((size_t)page * kv.n_kv_heads + u.kvh) * kv.page_size) * kv.head_dim;
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(kv.K + off), "r"(page_bytes) : "memory");
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(kv.V + off), "r"(page_bytes) : "memory");
              }
            }
          }
        }
      }
    }
  } else if (warp >= 4) {
    const int q = warp - 4;
    const int rl = q * 32 + lane;                        // this thread's row within the CTA's 128
    const uint32_t tempty_l = mapa_shared(smem_u32(tempty), 0);
    float* my_part = ws + (size_t)blockIdx.x * BM * BN;  // column-major [BN][128]: coalesced by row
    long long w = w_lo;
    for (int it = 0;; ++it) {
      const PSeg g = seg_at(it, w);
      if (g.u >= units) break;
      const int mp = g.u % m_pairs, nt = g.u / m_pairs;
      const int acc = it & 1;
      mbar_wait(&tfull[acc], (it >> 1) & 1);
      if (threadIdx.x == 128) stamp(2);
      tc_fence_after();
      const int row = mp * 2 * BM + (int)rank * BM + rl;
      const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN);
      if (g.k0 > 0 && !split2) {
        // later piece of a cut unit: fp32 partial -> this CTA's slot, then flag it for the finaliser
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 32) {
          float v[32];
          tmem_ld32(taddr + c0, v);
#pragma unroll
          for (int i = 0; i < 32; ++i) __stcg(my_part + (size_t)(c0 + i) * BM + rl, v[i]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(tempty_l + acc * 8);
        __threadfence();
        named_bar(1, 128);
        if (threadIdx.x == 128) asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(sem + blockIdx.x), "r"(1) : "memory");
      } else {
        // whole unit, or the first piece: add the partials of the pieces that follow (pairs
        // pair+1 .. owner(last stage of the unit), same CTA rank), in pair order
        const int q1 = (g.k1 < ks_n && !split2) ? owner((long long)(g.u + 1) * ks_n - 1) : pair;
        int* sflag = sem + 2048 + 2 * g.u + (int)rank;   // ordered split-K flag of this unit's rows
        const int hsplit = split2 ? g.h : 0;
        if (split2 && hsplit > 0) {                      // range h: ranges 0..h-1 have added theirs
          if (threadIdx.x == 128) {
            int f = 0;
            do {
              asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(f) : "l"(sflag) : "memory");
            } while (f != hsplit);
            // the flags re-arm themselves: the last range is the flag's last reader in this launch, so
            // every launch (and every replay of a captured graph) starts from 0 whatever units an
            // earlier launch of a different row count touched
            if (hsplit == nsplit - 1) *(volatile int*)sflag = 0;
          }
          named_bar(1, 128);
        }
        if (q1 > pair) {
          if (threadIdx.x == 128)
            for (int qq = pair + 1; qq <= q1; ++qq) {
              if (empty_range(qq)) continue;              // (W < n_pairs: some pairs own no stage)
              int f = 0;
              do {
                asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(f) : "l"(sem + 2 * qq + (int)rank) : "memory");
              } while (f == 0);
            }
          named_bar(1, 128);
        }
        auto chunk = [&](int c0, float* v) {
          tmem_ld32(taddr + c0, v);
          for (int qq = pair + 1; qq <= q1; ++qq) {
            if (empty_range(qq)) continue;
            const float* pp = ws + (size_t)(2 * qq + (int)rank) * BM * BN + (size_t)c0 * BM + rl;
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] += __ldcg(pp + (size_t)i * BM);
          }
        };
        const bool shared_tile = joint && n_mine == 1;
        epilogue_tile<MODE, BN>(chunk, row - lane, M, nt, N, C, ldc, epi, epi_buf, 0, shared_tile ? 2 : 1);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(tempty_l + acc * 8);
        if (split2 && hsplit < nsplit - 1) {             // residual updated -> release the next range
          __threadfence();
          named_bar(1, 128);
          if (threadIdx.x == 128)
            asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(sflag), "r"(hsplit + 1) : "memory");
        }
        if (q1 > pair) {
          named_bar(1, 128);                             // every thread has read the partials
          if (threadIdx.x == 128)
            for (int qq = pair + 1; qq <= q1; ++qq)
              if (!empty_range(qq)) sem[2 * qq + (int)rank] = 0;   // re-arm
        }
      }
      if (threadIdx.x == 128) stamp(2);
    }
  }
  if (warp < 4 && joint && n_mine == 1) {
    // warps 0-3: second column half of this pair's last unit (TMEM lane quarter = warp)
    __syncwarp();
    const int it = n_mine - 1, u = pair + it * n_pairs;
    const int mp = u % m_pairs, nt = u / m_pairs;
    const int acc = it & 1;
    // follow every accumulator hand-off in order: a parity wait only identifies a phase while the
    // barrier is less than two phases ahead, and these warps arrive here long before the last unit
    for (int i = 0; i < n_mine; ++i) mbar_wait(&tfull[i & 1], (i >> 1) & 1);
    __syncwarp();                                       // converged for the .sync.aligned TMEM loads
    tc_fence_after();
    const int q = warp;
    const int row = mp * 2 * BM + (int)rank * BM + q * 32 + lane;
    const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN);
    auto chunk = [&](int c0, float* v) { tmem_ld32(taddr + c0, v); };
    epilogue_tile<MODE, BN>(chunk, row - lane, M, nt, N, C, ldc, epi, epi_buf, 1, 2);
    tc_fence_before();
  }
  __syncthreads();
  cluster_sync();                                       // no CTA leaves while its peer may still signal it
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

// ---------------------------------------------------------------------------- host side
struct MapKey {
  const void* p;
  int rows, cols, ld, box_rows, ka;
  bool operator==(const MapKey& o) const {
    return p == o.p && rows == o.rows && cols == o.cols && ld == o.ld && box_rows == o.box_rows && ka == o.ka;
  }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    return std::hash<const void*>()(k.p) ^ ((size_t)k.rows * 1000003u) ^ ((size_t)k.cols * 7919u) ^
           ((size_t)k.ld << 20) ^ (size_t)k.box_rows ^ ((size_t)k.ka << 40);
  }
};


// ====================================================================================== swap-AB decode GEMM
// Few live rows (M_max <= 256, SWIGLU <= 64: the decode shapes of C2, ...): the weight rows go on the MMA M
// side and the tokens on N ("swap-AB"),  acc^T[128 features x M tokens] = W_tile[128 x K] . A^T.  The MMA
// N and the activation boxes follow the LIVE row count (32-row TMA boxes), so no tensor-core work or L2
// traffic is spent on padding rows.  Each CTA computes one 128-feature tile (SWIGLU: the gate and the up
// tile of the same 128 features, two accumulators) over one of CS contiguous K ranges, so every SM
// streams weights even when the GEMM has few feature tiles.  The CS CTAs of a tile form a thread-block
// cluster and reduce through distributed shared memory: after its last MMA each CTA parks its fp32
// partial [acc][token][feature] in its own drained pipeline buffers; after a cluster barrier CTA r sums,
// for its slice [r M / CS, (r + 1) M / CS) of the tokens, the CS partials in K-range order (deterministic:
// CS depends on N, K and the SM count only, never on M) and runs the mode's epilogue, thread = feature:
//   ADD       x[t][f] += acc (one writer per element; 32 consecutive features per warp store)
//   STORE     logits C[t][f] (when C) and per (token, 64-feature group) vocab statistics (epi.vpart)
//   SWIGLU    act[t][f] = bf16(silu(gate) * up)
//   QKV_ROPE  tile = one q/k/v head: RoPE pairs (d, d+64) exchanged through shared memory, bf16 q|k|v
//             rows and the paged KV store
// so the reduction and the epilogue are spread over the cluster instead of trailing on one CTA.
namespace swp {
constexpr int THREADS = 256;
constexpr int ABOX = 32;                                         // activation rows per TMA box
// layout of the grouped expert GEMM (k_gemm_grouped)
template <int NT, bool GU>
struct SL {
  static constexpr int NW = GU ? 2 : 1;                          // weight tiles (accumulators) per CTA
  static constexpr int W_BYTES = NW * 128 * BK * 2;              // 16 / 32 KB
  static constexpr int ACT_BYTES = NT * BK * 2;
  static constexpr int STAGE = W_BYTES + ACT_BYTES;
  static constexpr int STAGES = (160 * 1024) / STAGE > 8 ? 8 : (160 * 1024) / STAGE;
  static constexpr int XCH = 32 * 128 * 4;                       // exchange buffer: 32 tokens x 128 features
  static constexpr int SMEM = STAGES * STAGE + XCH + 1024 + 256;
  static constexpr int COLS = NW * NT;
  static constexpr int TCOLS = COLS <= 32 ? 32 : COLS <= 64 ? 64 : COLS <= 128 ? 128 : 256;
};
// layout of the cluster-reduced swap-AB GEMM (k_gemm_swap): NT = token capacity (>= M_max)
template <int NT, bool GU>
struct SC {
  static constexpr int NW = GU ? 2 : 1;
  static constexpr int W_BYTES = NW * 128 * BK * 2;
  static constexpr int ACT_BYTES = NT * BK * 2;
  static constexpr int STAGE = W_BYTES + ACT_BYTES;
  static constexpr int STAGES = (180 * 1024) / STAGE > 8 ? 8 : (180 * 1024) / STAGE;
  static constexpr int RED = NW * NT * 128 * 4;                  // parked partial, aliases the drained stages
  // + the epilogue's chunk buffer [NW][32][128] fp32 (also in the drained stages)
  static_assert(RED + NW * 32 * 128 * 4 <= STAGES * STAGE, "the partial fits the pipeline buffers");
  static constexpr int XCH = 32 * 128 * 4;
  static constexpr int RS = 128 * 33 * 4 + 32 * 8;               // QKV: RoPE rows [128][33] + 32 KV offsets
  static constexpr int SMEM = STAGES * STAGE + XCH + RS + 1024 + 256;
  static_assert(SMEM <= 227 * 1024, "shared memory");
  static constexpr int COLS = NW * NT;
  static constexpr int TCOLS = COLS <= 32 ? 32 : COLS <= 64 ? 64 : COLS <= 128 ? 128 : 256;
};
}  // namespace swp

template <int MODE, int NT>
__global__ void __launch_bounds__(swp::THREADS, 1)
    k_gemm_swap(const __grid_constant__ CUtensorMap mapW, const __grid_constant__ CUtensorMap mapA, float* __restrict__ C,
                int ldc, int N, int K, const int* __restrict__ M_dev, int M_max, const GemmEpi epi) {
  constexpr bool GU = MODE == GEMM_SWIGLU;
  using L = swp::SC<NT, GU>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  float* red = (float*)smem;                            // after the last MMA: this CTA's partial
  float* xch = (float*)(smem + L::STAGES * L::STAGE);
  float* rs = (float*)(smem + L::STAGES * L::STAGE + L::XCH);     // QKV: RoPE rows [128][33] of a chunk
  size_t* kvs = reinterpret_cast<size_t*>(rs + 128 * 33);         // QKV: KV element offsets of a chunk
  uint64_t* bars = (uint64_t*)(smem + L::STAGES * L::STAGE + L::XCH + L::RS);
  uint64_t* full = bars;                                // [STAGES]
  uint64_t* empty = bars + L::STAGES;                   // [STAGES]
  uint64_t* tfull = bars + 2 * L::STAGES;               // [1]
  uint32_t* tmem_sh = (uint32_t*)(tfull + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int CS = (int)cluster_nctarank();
  const int rank = (int)cluster_ctarank();              // = K range
  const int tile = blockIdx.x / CS;
  const int kbt = K / BK, kb0 = rank * kbt / CS, kb1 = (rank + 1) * kbt / CS;
  const int wrow0 = tile * 128 * L::NW;                 // first weight row of the tile (SWIGLU: gate, then up)
  // development trace (gemm_set_trace): global-timer stamps per CTA
  long long* trace = g_gemm_trace ? g_gemm_trace + (size_t)blockIdx.x * 3 * kGemmTraceEv : nullptr;
  auto stamp = [&](int e) {
    if (trace) {
      unsigned long long gt;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
      trace[e] = (long long)gt;
    }
  };
  if (threadIdx.x == 0) stamp(0);
  pdl_trigger();
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < L::STAGES; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    mbar_init(&tfull[0], 1);
    fence_barrier_init();
    prefetch_map(&mapW);
    prefetch_map(&mapA);
  }
  if (warp == 2) tmem_alloc<L::TCOLS>(tmem_sh);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_sh;
  if (threadIdx.x == 0) stamp(1);
  if (warp == 0) {
    if (lane == 0) {
      // the weight tiles do not depend on earlier kernels: the first stages' weight loads are issued
      // before the grid dependency wait (they overlap the previous kernel's tail); the NT activation rows
      // after it (a fixed count: waiting for the live row count here would put a global load behind the
      // weight stream, ~2 us)
      const uint64_t pol = l2_policy_evict_first();
      const int pre = min(kb1 - kb0, L::STAGES);
      for (int i = 0; i < pre; ++i) {
        uint8_t* st = smem + i * L::STAGE;
        mbar_expect_tx_only(&full[i], L::W_BYTES);
        tma_load_2d_hint(st, &mapW, &full[i], (kb0 + i) * BK, wrow0, pol);
        if (GU) tma_load_2d_hint(st + 128 * BK * 2, &mapW, &full[i], (kb0 + i) * BK, wrow0 + 128, pol);
      }
      stamp(8);
      pdl_wait();
      stamp(9);
      constexpr int nb = NT / swp::ABOX;
      constexpr uint32_t a_bytes = (uint32_t)L::ACT_BYTES;
      for (int i = 0; i < pre; ++i) {
        uint8_t* sa = smem + i * L::STAGE + L::W_BYTES;
        mbar_expect_tx(&full[i], a_bytes);
        for (int b = 0; b < nb; ++b) tma_load_2d(sa + b * swp::ABOX * 128, &mapA, &full[i], (kb0 + i) * BK, b * swp::ABOX);
      }
      int stage = pre % L::STAGES;
      uint32_t phase = pre == L::STAGES ? 1u : 0u;
      for (int kb = kb0 + pre; kb < kb1; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* st = smem + stage * L::STAGE;
        mbar_expect_tx(&full[stage], L::W_BYTES + a_bytes);
        tma_load_2d_hint(st, &mapW, &full[stage], kb * BK, wrow0, pol);
        if (GU) tma_load_2d_hint(st + 128 * BK * 2, &mapW, &full[stage], kb * BK, wrow0 + 128, pol);
        for (int b = 0; b < nb; ++b)
          tma_load_2d(st + L::W_BYTES + b * swp::ABOX * 128, &mapA, &full[stage], kb * BK, b * swp::ABOX);
        if (++stage == L::STAGES) { stage = 0; phase ^= 1; }
      }
      stamp(7);
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16(128, NT, false, false);
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        const uint32_t w0 = smem_u32(smem + stage * L::STAGE), a0 = w0 + L::W_BYTES;
#pragma unroll
        for (int k = 0; k < BK / 16; ++k) {
          const uint32_t acc = (kb > kb0 || k > 0) ? 1u : 0u;
          mma_bf16(tmem, desc_kmajor_sw128(w0 + k * 32), desc_kmajor_sw128(a0 + k * 32), idesc, acc);
          if (GU) mma_bf16(tmem + NT, desc_kmajor_sw128(w0 + 128 * BK * 2 + k * 32), desc_kmajor_sw128(a0 + k * 32), idesc, acc);
        }
        mma_commit(&empty[stage]);
        if (++stage == L::STAGES) { stage = 0; phase ^= 1; }
      }
      mma_commit(&tfull[0]);
    }
  }
  // QKV: stage the RoPE rows (lane = token, rows r0 .. r0 + nr of ropeT, coalesced) and, with kv, the
  // KV element offsets and committed-slot check of the 32-token chunk at t0 (one warp per call)
  const bool qkv_v = MODE == GEMM_QKV_ROPE && tile >= epi.n_q_heads + epi.kv.n_kv_heads;
  const bool qkv_kv = MODE == GEMM_QKV_ROPE && tile >= epi.n_q_heads;
  auto stage_qkv = [&](int t0, int te, int r0, int nr, bool kv) {
    const int t = min(t0 + lane, te - 1);
    if (!qkv_v) {
      float tmp[64];
#pragma unroll
      for (int i = 0; i < 64; ++i)
        if (i < nr) tmp[i] = __ldcg(epi.ropeT + (size_t)(r0 + i) * epi.rope_ld + t);
#pragma unroll
      for (int i = 0; i < 64; ++i)
        if (i < nr) rs[(r0 + i) * 33 + lane] = tmp[i];
    }
    if (kv && qkv_kv) {
      const int kvh = tile - epi.n_q_heads - (qkv_v ? epi.kv.n_kv_heads : 0);
      const RowInfo ri = epi.rows[t];
      kvs[lane] = kv_offset(epi.kv, ri.slot, ri.pos, kvh);
      if (t0 + lane < te && ri.j >= 0 && ((epi.st[ri.slot].committed >> ri.j) & 1ull))
        atomicExch(&epi.cnt->invariant, 1);
    }
  };
  if (MODE == GEMM_QKV_ROPE && (warp == 2 || warp == 3)) {
    // idle during the main loop: stage the epilogue's first chunk (barrier 2 hands it over)
    pdl_wait();
    const int Ms = M_dev ? min(__ldcg(M_dev), M_max) : M_max;
    const int lo = rank * Ms / CS, hi = (rank + 1) * Ms / CS;
    if (lo < hi) {
      stage_qkv(lo, hi, (warp - 2) * 64, 64, warp == 2);
      asm volatile("bar.arrive 2, 192;" ::: "memory");
    }
  }
  const int f = threadIdx.x - 128, q = warp - 4;        // epilogue warps 4..7: thread = feature f of the tile
  const uint32_t tb = tmem + ((uint32_t)(q * 32) << 16);
  int M = 0, t_lo = 0, t_hi = 0;
  if (warp >= 4) {
    pdl_wait();
    M = M_dev ? min(__ldcg(M_dev), M_max) : M_max;
    t_lo = rank * M / CS;
    t_hi = (rank + 1) * M / CS;
    mbar_wait(&tfull[0], 0);
    tc_fence_after();
    if (threadIdx.x == 128) stamp(2);
    if (CS > 1) {                                       // park the partial (every MMA has drained the stages)
      const int mp = (M + 31) & ~31;
#pragma unroll 1
      for (int c = 0; c < L::NW * NT; c += 32) {
        const int acc = c / NT, t0 = c % NT;
        if (t0 >= mp) continue;
        float v[32];
        tmem_ld32(tb + c, v);
#pragma unroll
        for (int i = 0; i < 32; ++i) red[(size_t)(acc * NT + t0 + i) * 128 + f] = v[i];
      }
    }
  }
  if (threadIdx.x == 128) stamp(3);
  if (CS > 1) {                                         // every partial of the cluster is parked
    __syncwarp();
    cluster_sync();
  }
  if (threadIdx.x == 128) stamp(4);
  if (warp >= 4) {
    // Per 32-token chunk [t0, t0 + 32) of the slice: the CS parked partials are summed in K-range order
    // by all 128 threads (thread = 4 features of every 4th token: 16-B DSMEM loads, all of one peer in
    // flight at once) into this CTA's chunk buffer red2 [acc][32][128]; get() then hands thread f its
    // 32 token values (CS = 1: straight from TMEM)
    float* red2 = (float*)(smem + L::RED);
    auto reduce_chunk = [&](int t0) {
      named_bar(1, 128);                                // the previous chunk's readers of red2 are done
      const int r = f >> 5, c4 = f & 31;
      float4 acc4[L::NW][8];
#pragma unroll
      for (int a = 0; a < L::NW; ++a)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc4[a][j] = make_float4(0.f, 0.f, 0.f, 0.f);
      const uint32_t mine = smem_u32(red + 4 * c4);
      constexpr int PU = GU ? 2 : 4;                    // peers whose loads are in flight together
#pragma unroll 1
      for (int p0 = 0; p0 < CS; p0 += PU) {
        float4 w[PU][L::NW][8];
#pragma unroll
        for (int pp = 0; pp < PU; ++pp) {
          const uint32_t base = mapa_shared(mine, (uint32_t)min(p0 + pp, CS - 1));
#pragma unroll
          for (int a = 0; a < L::NW; ++a)
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const int t = t0 + r + 4 * j;
              w[pp][a][j] = (t < t_hi && p0 + pp < CS) ? ld_dsmem_f32x4(base + (uint32_t)((a * NT + t) * 128) * 4u)
                                                       : make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
#pragma unroll
        for (int pp = 0; pp < PU; ++pp)                 // in K-range order
#pragma unroll
          for (int a = 0; a < L::NW; ++a)
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              acc4[a][j].x += w[pp][a][j].x; acc4[a][j].y += w[pp][a][j].y;
              acc4[a][j].z += w[pp][a][j].z; acc4[a][j].w += w[pp][a][j].w;
            }
      }
#pragma unroll
      for (int a = 0; a < L::NW; ++a)
#pragma unroll
        for (int j = 0; j < 8; ++j)
          *reinterpret_cast<float4*>(red2 + (size_t)(a * 32 + r + 4 * j) * 128 + 4 * c4) = acc4[a][j];
      named_bar(1, 128);
    };
    auto get = [&](int acc, int t0, float* v) {
      if (CS == 1) {
        tmem_ld32(tb + acc * NT + t0, v);
        return;
      }
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = red2[(size_t)(acc * 32 + i) * 128 + f];
    };
    const int feat = tile * 128 + f;                    // output feature (SWIGLU: act column)
    const int te = t_hi;
#pragma unroll 1
    for (int t0 = t_lo; t0 < te; t0 += 32) {            // warp-uniform bounds
      float v[32];
      if (CS > 1) reduce_chunk(t0);
      if (threadIdx.x == 128 && t0 == t_lo) stamp(11);
      get(0, t0, v);
      if constexpr (MODE == GEMM_ADD) {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (t0 + i < te)
            asm volatile("red.global.add.f32 [%0], %1;" ::"l"(C + (size_t)(t0 + i) * ldc + feat), "f"(v[i]) : "memory");
      } else if constexpr (MODE == GEMM_SWIGLU) {
        float u[32];
        get(1, t0, u);
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (t0 + i < te) {
            const float a = __fdividef(v[i] * u[i], 1.0f + exp2f(-1.4426950408889634f * v[i]));
            epi.out[(size_t)(t0 + i) * epi.ldo + feat] = __float2bfloat16_rn(a);
          }
      } else if constexpr (MODE == GEMM_STORE) {
        if (C != nullptr) {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (t0 + i < te && feat < N) C[(size_t)(t0 + i) * ldc + feat] = v[i];
        }
        if (epi.vpart != nullptr) {
          // per token: (max, sum exp(z - max), lowest argmax) over this warp's 32 features, then the
          // two warps of each 64-feature group combined through shared memory
          float* xm = xch;                               // [4 warps][32 tokens] max, sum, idx
          const bool ok = feat < N && feat != epi.mask_id;
#pragma unroll 1
          for (int i = 0; i < 32; ++i) {
            const float z = ok ? v[i] : -CUDART_INF_F;
            float m = z;
            for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
            const unsigned hit = __ballot_sync(0xffffffffu, z == m && m != -CUDART_INF_F);
            float e = (m == -CUDART_INF_F || !ok) ? 0.f : __expf(z - m);
            for (int o = 16; o; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
            if (lane == 0) {
              xm[(q * 32 + i) * 4 + 0] = m;
              xm[(q * 32 + i) * 4 + 1] = e;
              xm[(q * 32 + i) * 4 + 2] = __int_as_float(hit ? tile * 128 + q * 32 + __ffs(hit) - 1 : 0x7fffffff);
            }
          }
          named_bar(1, 128);
          if ((q & 1) == 0) {                            // warps 0 and 2: lane i = token t0 + i
            const int i = lane, t = t0 + i;
            const float* a = xm + (q * 32 + i) * 4;
            const float* b = xm + ((q + 1) * 32 + i) * 4;
            VocabPartial r;
            const float ma = a[0], mb = b[0];
            r.m = fmaxf(ma, mb);
            if (r.m == -CUDART_INF_F) { r.s = 0.f; r.idx = 0x7fffffff; }
            else {
              r.s = (ma == -CUDART_INF_F ? 0.f : a[1] * __expf(ma - r.m)) + (mb == -CUDART_INF_F ? 0.f : b[1] * __expf(mb - r.m));
              r.idx = ma >= mb ? __float_as_int(a[2]) : __float_as_int(b[2]);   // equal maxima: warp q's ids are lower
            }
            r.pad = 0;
            const int g = (tile * 128 + q * 32) >> 6;
            if (t < te && g < epi.vp_ld) epi.vpart[(size_t)t * epi.vp_ld + g] = r;
          }
          named_bar(1, 128);
        }
      } else {   // GEMM_QKV_ROPE: tile = head
        const int head = tile;
        const int hkv = epi.kv.n_kv_heads;
        const bool is_v = head >= epi.n_q_heads + hkv;
        const bool is_k = !is_v && head >= epi.n_q_heads;
#pragma unroll
        for (int i = 0; i < 32; ++i) xch[i * 128 + f] = v[i];
        named_bar(1, 128);
        const int kf = f & 63;
        // the chunk's RoPE rows and KV offsets: the first chunk was staged by warps 2-3 during the main
        // loop (barrier 2), later chunks are staged here (32 rows per warp)
        if (t0 == t_lo) {
          named_bar(2, 192);
        } else {
          stage_qkv(t0, te, q * 32, 32, q == 0);
          named_bar(1, 128);
        }
        float cc[32], sn[32];
        if (!is_v) {
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            cc[i] = rs[kf * 33 + i];
            sn[i] = rs[(64 + kf) * 33 + i];
          }
        }
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int t = t0 + i;
          if (t < te) {
            float y = v[i];
            if (!is_v) {
              const float other = xch[i * 128 + (f ^ 64)];
              y = f < 64 ? v[i] * cc[i] - other * sn[i] : v[i] * cc[i] + other * sn[i];
            }
            const __nv_bfloat16 b = __float2bfloat16_rn(y);
            epi.out[(size_t)t * epi.ldo + head * 128 + f] = b;
            if (is_k || is_v) (is_v ? epi.kv.V : epi.kv.K)[kvs[i] + f] = b;
          }
        }
        named_bar(1, 128);                               // xch reuse by the next chunk
      }
    }
  }
  if (threadIdx.x == 128) stamp(5);
  if (CS > 1) {                                         // the peers have read this CTA's partial
    __syncwarp();
    cluster_sync();
  }
  if (threadIdx.x == 128) stamp(6);
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_free<L::TCOLS>(tmem);
  }
}

// Grouped swap-AB GEMM over experts (MoE FFN, readings A-M5/A-M6): expert e owns the rows
// [off[e], off[e+1]) of the gathered activations A (the tokens routed to e, in row order) and the
// weight rows [e * wrows, (e + 1) * wrows) of W; CTA (e, tile) computes the features
// [tile * 128, tile * 128 + 128) of expert e (SWIGLU: its gate and up tiles, 256 weight rows) for all
// of e's rows, NT at a time (one TMEM accumulator, handed between the MMA issuer and the epilogue per
// chunk).  An expert with no tokens costs its CTAs one barrier setup and no weight traffic.
//   SWIGLU  act[p][f] = bf16(silu(gate) * up)   (p = gathered row)
//   STORE   C[p][f] = acc (fp32)
template <int MODE, int NT>
__global__ void __launch_bounds__(swp::THREADS, 1)
    k_gemm_grouped(const __grid_constant__ CUtensorMap mapW, const __grid_constant__ CUtensorMap mapA,
                   float* __restrict__ C, int ldc, int K, const int* __restrict__ off, int wrows, int tiles,
                   const GemmEpi epi) {
  constexpr bool GU = MODE == GEMM_SWIGLU;
  using L = swp::SL<NT, GU>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = (uint64_t*)(smem + L::STAGES * L::STAGE + L::XCH);
  uint64_t* full = bars;                                // [STAGES]
  uint64_t* empty = bars + L::STAGES;                   // [STAGES]
  uint64_t* tfull = bars + 2 * L::STAGES;               // [1]
  uint64_t* tempty = tfull + 1;                         // [1] (4 epilogue warps)
  uint32_t* tmem_sh = (uint32_t*)(tempty + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int e = blockIdx.x / tiles, tile = blockIdx.x % tiles;
  pdl_trigger();
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < L::STAGES; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    mbar_init(&tfull[0], 1);
    mbar_init(&tempty[0], 4);
    fence_barrier_init();
    prefetch_map(&mapW);
    prefetch_map(&mapA);
  }
  if (warp == 2) tmem_alloc<L::TCOLS>(tmem_sh);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_sh;
  pdl_wait();                                           // the expert offsets and rows come from earlier kernels
  // (L2 loads: the offsets were written two kernels back, and under programmatic dependent launch an L1
  // line of an earlier co-resident grid may still hold the previous layer's values)
  const int r0 = __ldcg(off + e), n = __ldcg(off + e + 1) - r0;
  const int chunks = n > 0 ? (n + NT - 1) / NT : 0;
  const int kbt = K / BK;
  const int wrow0 = e * wrows + tile * 128 * L::NW;
  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol = l2_policy_evict_first();
      int stage = 0;
      uint32_t phase = 0;
      for (int c = 0; c < chunks; ++c)
        for (int kb = 0; kb < kbt; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* st = smem + stage * L::STAGE;
          mbar_expect_tx(&full[stage], L::STAGE);
          tma_load_2d_hint(st, &mapW, &full[stage], kb * BK, wrow0, pol);
          if (GU) tma_load_2d_hint(st + 128 * BK * 2, &mapW, &full[stage], kb * BK, wrow0 + 128, pol);
          tma_load_2d(st + L::W_BYTES, &mapA, &full[stage], kb * BK, r0 + c * NT);
          if (++stage == L::STAGES) { stage = 0; phase ^= 1; }
        }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16(128, NT, false, false);
      int stage = 0;
      uint32_t phase = 0;
      for (int c = 0; c < chunks; ++c) {
        mbar_wait(&tempty[0], (c & 1) ^ 1);             // the epilogue has read the previous chunk
        tc_fence_after();
        for (int kb = 0; kb < kbt; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t w0 = smem_u32(smem + stage * L::STAGE), a0 = w0 + L::W_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint32_t acc = (kb > 0 || k > 0) ? 1u : 0u;
            mma_bf16(tmem, desc_kmajor_sw128(w0 + k * 32), desc_kmajor_sw128(a0 + k * 32), idesc, acc);
            if (GU) mma_bf16(tmem + NT, desc_kmajor_sw128(w0 + 128 * BK * 2 + k * 32), desc_kmajor_sw128(a0 + k * 32), idesc, acc);
          }
          mma_commit(&empty[stage]);
          if (++stage == L::STAGES) { stage = 0; phase ^= 1; }
        }
        mma_commit(&tfull[0]);
      }
    }
  } else if (warp >= 4) {
    const int f = threadIdx.x - 128, q = warp - 4;
    const uint32_t tb = tmem + ((uint32_t)(q * 32) << 16);
    const int feat = tile * 128 + f;
    for (int c = 0; c < chunks; ++c) {
      mbar_wait(&tfull[0], c & 1);
      tc_fence_after();
      const int nc = min(NT, n - c * NT);               // rows of this chunk
#pragma unroll 1
      for (int t0 = 0; t0 < NT; t0 += 32) {
        if (t0 >= nc) break;
        float v[32];
        tmem_ld32(tb + t0, v);
        if constexpr (GU) {
          float u[32];
          tmem_ld32(tb + NT + t0, u);
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (t0 + i < nc) {
              const float a = __fdividef(v[i] * u[i], 1.0f + exp2f(-1.4426950408889634f * v[i]));
              epi.out[(size_t)(r0 + c * NT + t0 + i) * epi.ldo + feat] = __float2bfloat16_rn(a);
            }
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (t0 + i < nc) __stcg(C + (size_t)(r0 + c * NT + t0 + i) * ldc + feat, v[i]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[0]);
    }
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_free<L::TCOLS>(tmem);
  }
}

// ka = 0: 2-D map [rows][cols], box box_rows x 64.  ka >= 1: 3-D view {64, rows, cols / 64} of the same
// matrix (k-atom stride 128 B), box {64, box_rows, ka} = ka consecutive SW128 K-major tiles.
bool get_map(const void* ptr, int rows, int cols, int ld, int box_rows, CUtensorMap* out, int ka = 0) {
  static std::mutex mu;
  static std::unordered_map<MapKey, CUtensorMap, MapKeyHash> cache;
  std::lock_guard<std::mutex> g(mu);
  const MapKey k{ptr, rows, cols, ld, box_rows, ka};
  auto it = cache.find(k);
  if (it != cache.end()) { *out = it->second; return true; }
  CUtensorMap m;
  const bool ok = ka == 0 ? make_tma_2d_bf16(ptr, rows, cols, ld, BK, box_rows, &m)
                          : make_tma_3d_bf16(ptr, BK, rows, cols / BK, (uint64_t)ld * 2, BK * 2, BK, box_rows, ka, &m);
  if (!ok) return false;
  cache.emplace(k, m);
  *out = m;
  return true;
}

}  // namespace tc

static int g_backend = -1;

int gemm_backend() {
  if (g_backend < 0) {
    const char* e = getenv("FOCUS_GEMM");
    g_backend = (e && e[0] == 's') ? 0 : 1;     // FOCUS_GEMM=simt forces the scaffolding path
  }
  return g_backend;
}

void gemm_set_backend(int b) { g_backend = b; }

// development hook: route the pair kernel's clock64 trace to `buf` (3 * 256 int64 per CTA) or off (null)
void gemm_set_trace(long long* buf) { cudaMemcpyToSymbol(tc::g_gemm_trace, &buf, sizeof(buf)); }

template <int MODE, int BN, int CS>
static void launch_k(int grid, int smem, cudaStream_t s, const CUtensorMap& ma, const CUtensorMap& mb, float* C, int ldc,
                     int N, int K, const int* M_dev, int M_max, const GemmWs& ws, int policy, const GemmEpi& e) {
  using namespace tc;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_gemm_tc<MODE, BN, CS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(NUM_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  cudaLaunchKernelEx(&cfg, k_gemm_tc<MODE, BN, CS>, ma, mb, C, ldc, N, K, M_dev, M_max, ws.ptr, ws.sem, policy, e);
}

template <int BN, int CS>
static bool launch_bn(const bf16* A, int lda, int a_rows, const bf16* W, int N, int K, float* C, int ldc,
                      const int* M_dev, int M_max, GemmMode mode, const GemmWs& ws, cudaStream_t s, const GemmEpi* epi) {
  using namespace tc;
  if ((mode == GEMM_SWIGLU || mode == GEMM_QKV_ROPE) && (!epi || N % BN)) return false;
  if (mode == GEMM_SWIGLU && BN != 2 * kGuGroup) return false;
  if (mode == GEMM_QKV_ROPE && (epi->kv.head_dim != 128 || BN % 128)) return false;
  CUtensorMap ma, mb;
  if (!get_map(A, a_rows, K, lda, BM, &ma) || !get_map(W, N, K, K, BN / CS, &mb)) return false;
  constexpr int SMEM = GT<BN>::SMEM_BYTES;
  // grid: one CTA per SM (a multiple of the cluster size), never more CTAs than k-blocks of work at
  // the smallest live M (one m-tile), and at most as many as the partial workspace and semaphores allow
  const long long w_min = (long long)((N + BN - 1) / BN) * (K / BK) * CS;
  int grid = (int)std::min<long long>(num_sms(), std::max<long long>(1, w_min));
  grid = std::max(1, std::min<int>(grid, (int)std::min<size_t>(ws.sem_count, ws.bytes / (sizeof(float) * BM * BN * 2))));
  grid = std::max(CS, grid / CS * CS);
  static int policy0 = -1;
  if (policy0 < 0) {   // default: data-parallel tiles (measured fastest at the decode shapes)
    const char* e = getenv("FOCUS_GEMM_SCHED");
    policy0 = (e && e[0] == 's') ? 1 : (e && e[0] == 'h') ? 0 : 2;
  }
  int policy = policy0;
  static int pf = -1;
  if (pf < 0) {
    const char* e = getenv("FOCUS_GEMM_PF");
    pf = e ? std::max(0, std::min(64, atoi(e))) : 0;   // measured: prefetch does not help
  }
  policy = (policy & 0xff) | (pf << 8);
  const GemmEpi e = epi ? *epi : GemmEpi{};
  switch (mode) {
    case GEMM_ADD: launch_k<GEMM_ADD, BN, CS>(grid, SMEM, s, ma, mb, C, ldc, N, K, M_dev, M_max, ws, policy, e); break;
    case GEMM_SWIGLU:
      if constexpr (BN == 2 * kGuGroup)
        launch_k<GEMM_SWIGLU, BN, CS>(grid, SMEM, s, ma, mb, C, ldc, N, K, M_dev, M_max, ws, policy, e);
      break;
    case GEMM_QKV_ROPE:
      launch_k<GEMM_QKV_ROPE, BN, CS>(grid, SMEM, s, ma, mb, C, ldc, N, K, M_dev, M_max, ws, policy, e);
      break;
    default: launch_k<GEMM_STORE, BN, CS>(grid, SMEM, s, ma, mb, C, ldc, N, K, M_dev, M_max, ws, policy, e);
  }
  return true;
}

template <int MODE, int BN, int KA>
static void launch_pair_k(int grid, cudaStream_t s, const CUtensorMap& ma, const CUtensorMap& mb, float* C, int ldc,
                          int N, int K, const int* M_dev, int M_max, const GemmEpi& e, int m_hint, const GemmWs& ws,
                          int sk) {
  using namespace tc;
  constexpr int SMEM = GP<BN, KA>::SMEM_BYTES;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_gemm_pair<MODE, BN, KA>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    attr = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(NUM_THREADS);
  cfg.dynamicSmemBytes = SMEM;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  cudaLaunchKernelEx(&cfg, k_gemm_pair<MODE, BN, KA>, ma, mb, C, ldc, N, K, M_dev, M_max, e, m_hint, ws.ptr, ws.sem, sk);
}

template <int BN, int KA>
static bool launch_pair(const bf16* A, int lda, int a_rows, const bf16* W, int N, int K, float* C, int ldc,
                        const int* M_dev, int M_max, GemmMode mode, const GemmWs& ws, cudaStream_t s, const GemmEpi* epi,
                        int m, int split = 1) {
  using namespace tc;
  if ((mode == GEMM_SWIGLU || mode == GEMM_QKV_ROPE) && (!epi || N % BN)) return false;
  if (mode == GEMM_SWIGLU && BN != 2 * kGuGroup) return false;
  if constexpr (BN == 192) {                        // 1.5-head QKV tiles only (RoPE pairs kept in the tile)
    if (mode != GEMM_QKV_ROPE || KA != 1 || N % 384) return false;
  }
  if (mode == GEMM_QKV_ROPE && (epi->kv.head_dim != 128 || (BN % 128 && BN != 192))) return false;
  CUtensorMap ma, mb;
  if (K % (BK * KA)) return false;
  if (!get_map(A, a_rows, K, lda, BM, &ma, KA) || !get_map(W, N, K, K, BN == 192 ? 32 : BN / 2, &mb, KA)) return false;
  // one pair per unit, at most one CTA per SM (opt-in stream-K: every SM busy, units cut at pair
  // boundaries).  The grid comes from the row-count upper bound M_max (persistent pairs; pairs without a unit at the live
  // count exit): the launch must not depend on the host's row-count estimate, which only picks the
  // tile width, or a graph captured at a small estimate would starve a step with many rows
  const long long units = (long long)((M_max + 2 * BM - 1) / (2 * BM)) * ((N + BN - 1) / BN);
  const int np = num_sms() / 2;
  // opt-in (FOCUS_GEMM_PSK=1, read per call): measured slower at the C3 shapes -- the fp32 partial
  // write + read of the cut units costs more than the idle SMs of the ragged last wave
  const char* sk_e = getenv("FOCUS_GEMM_PSK");
  int sk = (sk_e && sk_e[0] == '1') ? 1 : 0;
  if (ws.ptr == nullptr || ws.sem == nullptr || ws.sem_count < (size_t)2 * np ||
      ws.bytes < (size_t)2 * np * BM * BN * sizeof(float))
    sk = 0;
  const bool split2_ok = split > 1 && mode == GEMM_ADD && !sk && ws.sem != nullptr &&
                         ws.sem_count >= 2048 + 2 * ((size_t)M_max + 2 * BM - 1) / (2 * BM) * ((N + BN - 1) / BN);
  const int grid = sk ? 2 * np
                      : (int)std::max<long long>(2, std::min<long long>(np, split2_ok ? split * units : units) * 2);
  const GemmEpi e = epi ? *epi : GemmEpi{};
  static int pf_on = -1;
  if (pf_on < 0) {
    const char* ev = getenv("FOCUS_GEMM_WPF");      // opt-in weight L2 prefetch before the PDL wait
    pf_on = (ev && ev[0] == '1') ? 1 : 0;   // measured: no gain in the step (default off)
  }
  const int pf_hint = pf_on ? m : 0;
  static int hint_on = -1;
  if (hint_on < 0) {
    const char* eh = getenv("FOCUS_GEMM_L2HINT");      // L2 eviction hints on the operand streams
    hint_on = (eh && eh[0] == '0') ? 0 : 1;
  }
  sk |= hint_on << 1;
  // GEMM_ADD, 256-wide tiles, one wave even with two k-halves per unit: ordered split-K (see kernel)
  // (the per-unit flags hold h while range h may add; the last range resets them to 0, so nothing
  // launch-specific is baked into a captured graph)
  if (split2_ok) sk |= 4 | ((split - 1) << 3);

  if constexpr (BN == 192) {
    launch_pair_k<GEMM_QKV_ROPE, BN, KA>(grid, s, ma, mb, C, ldc, N, K, M_dev, M_max, e, pf_hint, ws, sk);
    return true;
  }
  switch (mode) {
    case GEMM_ADD: launch_pair_k<GEMM_ADD, BN, KA>(grid, s, ma, mb, C, ldc, N, K, M_dev, M_max, e, pf_hint, ws, sk); break;
    case GEMM_SWIGLU:
      if constexpr (BN == 2 * kGuGroup) launch_pair_k<GEMM_SWIGLU, BN, KA>(grid, s, ma, mb, C, ldc, N, K, M_dev, M_max, e, pf_hint, ws, sk);
      break;
    case GEMM_QKV_ROPE: launch_pair_k<GEMM_QKV_ROPE, BN, KA>(grid, s, ma, mb, C, ldc, N, K, M_dev, M_max, e, pf_hint, ws, sk); break;
    default: launch_pair_k<GEMM_STORE, BN, KA>(grid, s, ma, mb, C, ldc, N, K, M_dev, M_max, e, pf_hint, ws, sk);
  }
  return true;
}

// m_est: expected live row count (host estimate, e.g. last step's counter) used only to pick the tile
// width: 128-wide tiles when 256-wide tiles would leave more than ~half of the SMs idle.
// Tile configuration of a tensor-core GEMM of shape (N, K, mode) at an expected live row count m:
// the ONLY host decision that depends on the row-count estimate (grids come from M_max).  The
// whole-step graph cache keys on these choices, so a captured graph is replayed exactly when the
// eager sequence would launch the same kernels.
enum { GC_SPLIT = 1, GC_128x2, GC_256x2, GC_128x1, GC_256x1, GC_SINGLE_128, GC_SINGLE_256, GC_SWAP, GC_QKV192 };

// swap-AB decode GEMM (see k_gemm_swap): M_max <= 256 (SWIGLU: 64) live rows, 128-aligned feature tiles,
// and few enough tiles that a cluster of >= 2 K ranges per tile fits one wave (the LM head's ~1 200
// tiles stay on the CTA-pair kernel).  Default on (FOCUS_GEMM_SWAP=0: off; read per call, the tests
// switch it per context).  The cluster size depends on N, K and the SM count only.
static bool swap_enabled() {
  const char* e = getenv("FOCUS_GEMM_SWAP");
  return !(e && e[0] == '0');
}
static int swap_nt(int M_max) { return M_max <= 32 ? 32 : M_max <= 64 ? 64 : M_max <= 128 ? 128 : 256; }
// K ranges per tile: as many as fill the SMs with one CTA each, >= 2 k-blocks per range, <= 16 (the
// non-portable cluster limit)
static int swap_cs(int tiles, int kbt) {
  static int cap = -1;
  if (cap < 0) {   // FOCUS_GEMM_SWAP_CS: cap on the cluster size (development: 1 = no K split)
    const char* e = getenv("FOCUS_GEMM_SWAP_CS");
    cap = e ? std::max(1, std::min(16, atoi(e))) : 16;
  }
  return std::max(1, std::min(std::min(cap, kbt / 2), num_sms() / std::max(1, tiles)));
}
static bool swap_shape_ok(int N, int K, GemmMode mode, int M_max) {
  const int nw = mode == GEMM_SWIGLU ? 2 : 1;
  if (!swap_enabled() || M_max < 1 || M_max > (nw == 2 ? 64 : 256) || K % tc::BK || N % (128 * nw)) return false;
  return N / (128 * nw) <= num_sms() / 2;
}
static bool swap_applies(int N, int K, GemmMode mode, int M_max, const GemmEpi* epi) {
  if (!swap_shape_ok(N, K, mode, M_max)) return false;
  if ((mode == GEMM_SWIGLU || mode == GEMM_QKV_ROPE) && !epi) return false;
  if (mode == GEMM_QKV_ROPE && epi->kv.head_dim != 128) return false;
  return true;
}

template <int MODE, int NT>
static void launch_swap_k(int tiles, int cs, cudaStream_t s, const CUtensorMap& mw, const CUtensorMap& ma, float* C,
                          int ldc, int N, int K, const int* M_dev, int M_max, const GemmEpi& e) {
  using namespace tc;
  constexpr int SMEM = swp::SC<NT, MODE == GEMM_SWIGLU>::SMEM;
  auto kern = k_gemm_swap<MODE, NT>;
  static bool attr = false;
  static int fits[17];                                  // largest co-resident cluster count per size (0: unknown)
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(swp::THREADS);
  cfg.dynamicSmemBytes = SMEM;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  // the largest cluster size <= cs whose `tiles` clusters are co-resident (clusters live inside one GPC)
  for (; cs > 1; --cs) {
    if (fits[cs] == 0) {
      at[0].val.clusterDim.x = cs;
      cfg.gridDim = dim3(tiles * cs);
      cfg.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) {
        (void)cudaGetLastError();
        n = -1;                                         // unknown: trust the SM count
      }
      fits[cs] = n == 0 ? -2 : n;
    }
    if (fits[cs] == -1 || fits[cs] >= tiles) break;
  }
  at[0].val.clusterDim.x = cs;
  cfg.gridDim = dim3(tiles * cs);
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  cudaLaunchKernelEx(&cfg, kern, mw, ma, C, ldc, N, K, M_dev, M_max, e);
}

template <int NT>
static bool launch_swap_nt(const bf16* A, int lda, int a_rows, const bf16* W, int N, int K, float* C, int ldc,
                           const int* M_dev, int M_max, GemmMode mode, cudaStream_t s, const GemmEpi* epi) {
  using namespace tc;
  CUtensorMap mw, ma;
  if (!get_map(W, N, K, K, 128, &mw) || !get_map(A, a_rows, K, lda, swp::ABOX, &ma)) return false;
  const int nw = mode == GEMM_SWIGLU ? 2 : 1;
  const int tiles = N / (128 * nw);
  const int cs = swap_cs(tiles, K / BK);
  const GemmEpi e = epi ? *epi : GemmEpi{};
  switch (mode) {
    case GEMM_ADD: launch_swap_k<GEMM_ADD, NT>(tiles, cs, s, mw, ma, C, ldc, N, K, M_dev, M_max, e); break;
    case GEMM_SWIGLU:
      if constexpr (NT <= 64) launch_swap_k<GEMM_SWIGLU, NT>(tiles, cs, s, mw, ma, C, ldc, N, K, M_dev, M_max, e);
      break;
    case GEMM_QKV_ROPE: launch_swap_k<GEMM_QKV_ROPE, NT>(tiles, cs, s, mw, ma, C, ldc, N, K, M_dev, M_max, e); break;
    default: launch_swap_k<GEMM_STORE, NT>(tiles, cs, s, mw, ma, C, ldc, N, K, M_dev, M_max, e);
  }
  return true;
}

static bool launch_gemm_swap(const bf16* A, int lda, int a_rows, const bf16* W, int N, int K, float* C, int ldc,
                             const int* M_dev, int M_max, GemmMode mode, const GemmWs&, cudaStream_t s,
                             const GemmEpi* epi) {
  switch (swap_nt(M_max)) {
    case 32: return launch_swap_nt<32>(A, lda, a_rows, W, N, K, C, ldc, M_dev, M_max, mode, s, epi);
    case 64: return launch_swap_nt<64>(A, lda, a_rows, W, N, K, C, ldc, M_dev, M_max, mode, s, epi);
    case 128: return launch_swap_nt<128>(A, lda, a_rows, W, N, K, C, ldc, M_dev, M_max, mode, s, epi);
    default: return launch_swap_nt<256>(A, lda, a_rows, W, N, K, C, ldc, M_dev, M_max, mode, s, epi);
  }
}
static int split_parts(int K) {
  // ordered split into S k-ranges (at least 8 k-blocks each, S units in one wave): two ranges for deep
  // K at the C3 shapes.  S up to 4 (FOCUS_GEMM_SPLIT_MAX) was measured slower on the C2 shapes (O
  // 0.53 -> 0.93 ms/step: the ordered chain of residual adds costs more than the extra SMs give)
  static int s_cap = -1, s2_env = -1, s2_mink = -1;
  if (s_cap < 0) {
    const char* e = getenv("FOCUS_GEMM_SPLIT_MAX");
    s_cap = e ? std::max(2, std::min(4, atoi(e))) : 2;
    // GEMM_ADD whose 256-wide units fit one wave twice over: 256-wide tiles with ordered split-K
    // (FOCUS_GEMM_SPLIT2=0: off) instead of 128-wide tiles, halving the activation re-reads
    e = getenv("FOCUS_GEMM_SPLIT2");
    s2_env = (e && e[0] == '0') ? 0 : 1;
    // (measured at M = 428: down, K = 12288, 57 -> 53 us; O, K = 4096, 29 -> 33 us, so only for deep K)
    e = getenv("FOCUS_GEMM_SPLIT2_MINK");
    s2_mink = e ? std::max(256, atoi(e)) : 8192;
  }
  if (!s2_env || K < s2_mink) return 1;
  const int sp = std::min(s_cap, K / tc::BK / 8);
  return sp >= 2 ? sp : 1;
}

static int env_flag(const char* name, int& cache) {
  if (cache < 0) cache = getenv(name) != nullptr ? 1 : 0;
  return cache;
}


// Grouped expert GEMM of an MoE layer (k_gemm_grouped): A = gathered rows [a_rows][K] (tokens routed to
// each expert, expert-contiguous, offsets off[E + 1] on the device), W = E experts x wrows rows of K.
// SWIGLU: wrows = 2 d_expert (gate/up interleaved by 128 rows), out act [rows][d_expert] bf16;
// STORE: wrows = N (feature rows per expert), out C [rows][ldc] fp32.
bool launch_gemm_grouped(const bf16* A, int a_rows, const bf16* W, int n_experts, int wrows, int K, float* C, int ldc,
                         const int* off, int M_max_rows, GemmMode mode, const GemmEpi* epi, cudaStream_t s) {
  using namespace tc;
  if (K % BK || wrows % 128 || (mode == GEMM_SWIGLU && (wrows % 256 || !epi))) return false;
  const int NT = M_max_rows <= 32 ? 32 : 64;            // rows per chunk (an expert's rows loop in chunks)
  CUtensorMap mw, ma;
  if (!get_map(W, n_experts * wrows, K, K, 128, &mw) || !get_map(A, a_rows, K, K, NT, &ma)) return false;
  const int tiles = mode == GEMM_SWIGLU ? wrows / 256 : wrows / 128;
  const GemmEpi e = epi ? *epi : GemmEpi{};
  const int grid = n_experts * tiles;
  auto go = [&](auto kern, int smem) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    launch_pdl(kern, dim3(grid), dim3(swp::THREADS), smem, s, mw, ma, C, ldc, K, off, wrows, tiles, e);
  };
  if (mode == GEMM_SWIGLU) {
    if (NT == 32) go(k_gemm_grouped<GEMM_SWIGLU, 32>, swp::SL<32, true>::SMEM);
    else go(k_gemm_grouped<GEMM_SWIGLU, 64>, swp::SL<64, true>::SMEM);
  } else {
    if (NT == 32) go(k_gemm_grouped<GEMM_STORE, 32>, swp::SL<32, false>::SMEM);
    else go(k_gemm_grouped<GEMM_STORE, 64>, swp::SL<64, false>::SMEM);
  }
  return true;
}

int gemm_tc_choice(int N, int K, GemmMode mode, int M_max, int m_est, bool allow_swap) {
  using namespace tc;
  if (allow_swap && swap_shape_ok(N, K, mode, M_max)) return GC_SWAP;
  const int m = m_est > 0 ? std::min(m_est, M_max) : M_max;
  static int bn256 = -1, bn128 = -1, pair_env = -1, ka_env = -1;
  const bool force256 = env_flag("FOCUS_GEMM_BN256", bn256) != 0;
  if (pair_env < 0) {   // CTA-pair tiles by default; FOCUS_GEMM_PAIR=0: one CTA per tile
    const char* e = getenv("FOCUS_GEMM_PAIR");
    pair_env = !(e && e[0] == '0');
  }
  if (pair_env) {
    const long long units256 = (long long)((m + 2 * BM - 1) / (2 * BM)) * ((N + 255) / 256);
    const bool narrow2 = mode != GEMM_SWIGLU && !force256 &&
                         (4 * units256 <= (num_sms() * 11) / 10 || env_flag("FOCUS_GEMM_BN128", bn128));
    // k-atoms per stage (measured at the C3 shapes): 2 for 128-wide tiles (4 stages of 48 KB), 1 for
    // 256-wide tiles (6 stages of 32 KB); FOCUS_GEMM_KA=1|2 forces one
    if (ka_env < 0) {
      const char* e = getenv("FOCUS_GEMM_KA");
      ka_env = (e && (e[0] == '1' || e[0] == '2')) ? e[0] - '0' : 0;
    }
    const int ka = ka_env ? ka_env : (narrow2 ? 2 : 1);
    // the split decision uses the GEMM's shape only (K), never the row count, so results are batch
    // invariant
    if (mode == GEMM_ADD && ka_env == 0 && split_parts(K) >= 2) return GC_SPLIT;
    // QKV: 192-wide (1.5-head) tiles when 256-wide tiles leave a partial wave that 192-wide ones fill
    // better (C3 S rows: 48 -> 64 units on 74 pairs); FOCUS_GEMM_QKV192=0: off
    static int q192 = -1;
    if (q192 < 0) q192 = (getenv("FOCUS_GEMM_QKV192") && getenv("FOCUS_GEMM_QKV192")[0] == '0') ? 0 : 1;
    if (q192 && mode == GEMM_QKV_ROPE && ka_env == 0 && !force256 && N % 384 == 0) {
      const long long mpairs = (m + 2 * BM - 1) / (2 * BM), np = num_sms() / 2;
      const long long u192 = mpairs * (N / 192);
      if (units256 < np && u192 <= np && u192 > units256) return GC_QKV192;
    }
    if (ka == 2 && K % (2 * BK) == 0) return narrow2 ? GC_128x2 : GC_256x2;
    return narrow2 ? GC_128x1 : GC_256x1;
  }
  const long long tiles256 = (long long)((m + BM - 1) / BM) * ((N + 255) / 256);
  const bool narrow = mode != GEMM_SWIGLU && 2 * tiles256 <= (num_sms() * 11) / 10 && !force256;
  return narrow ? GC_SINGLE_128 : GC_SINGLE_256;
}

// m_est: expected live row count (host estimate, e.g. last step's counter) used only to pick the tile
// width: 128-wide tiles when 256-wide tiles would leave more than ~half of the SMs idle.
bool launch_gemm_tc(const bf16* A, int lda, int a_rows, const bf16* W, int N, int K, float* C, int ldc, const int* M_dev,
                    int M_max, GemmMode mode, const GemmWs& ws, cudaStream_t s, const GemmEpi* epi, int m_est) {
  using namespace tc;
  if (M_max <= 0) return true;
  if (K % BK || lda % 8 || a_rows < 1) return false;
  const int m = m_est > 0 ? std::min(m_est, M_max) : M_max;
  if (!ws.no_swap && swap_applies(N, K, mode, M_max, epi) &&
      launch_gemm_swap(A, lda, a_rows, W, N, K, C, ldc, M_dev, M_max, mode, ws, s, epi))
    return true;
  switch (gemm_tc_choice(N, K, mode, M_max, m_est, false)) {
    case GC_SPLIT: return launch_pair<256, 1>(A, lda, a_rows, W, N, K, C, ldc, M_dev, M_max, mode, ws, s, epi, m, split_parts(K));
    case GC_128x2: return launch_pair<128, 2>(A, lda, a_rows, W, N, K, C, ldc, M_dev, M_max, mode, ws, s, epi, m);
    case GC_256x2: return launch_pair<256, 2>(A, lda, a_rows, W, N, K, C, ldc, M_dev, M_max, mode, ws, s, epi, m);
    case GC_128x1: return launch_pair<128, 1>(A, lda, a_rows, W, N, K, C, ldc, M_dev, M_max, mode, ws, s, epi, m);
    case GC_256x1: return launch_pair<256, 1>(A, lda, a_rows, W, N, K, C, ldc, M_dev, M_max, mode, ws, s, epi, m);
    case GC_QKV192: return launch_pair<192, 1>(A, lda, a_rows, W, N, K, C, ldc, M_dev, M_max, mode, ws, s, epi, m);
    default: break;
  }
  // opt-in (FOCUS_GEMM_PAIR=0): one CTA per tile; (FOCUS_GEMM_MC=1) clusters of 4 CTAs (the 4 m-tiles
  // of a weight tile) share W by TMA multicast when the live row count fills them.  Measured no
  // faster at the C3 shapes (at cluster size <= 4 the L2 already serves the duplicate requests once)
  const bool narrow = gemm_tc_choice(N, K, mode, M_max, m_est, false) == GC_SINGLE_128;
  const int m_tiles = (m + BM - 1) / BM;
  const bool cluster4 = getenv("FOCUS_GEMM_MC") != nullptr && m_tiles % 4 == 0;
  if (narrow) {
    if (cluster4) return launch_bn<128, 4>(A, lda, a_rows, W, N, K, C, ldc, M_dev, M_max, mode, ws, s, epi);
    return launch_bn<128, 1>(A, lda, a_rows, W, N, K, C, ldc, M_dev, M_max, mode, ws, s, epi);
  }
  if (cluster4) return launch_bn<256, 4>(A, lda, a_rows, W, N, K, C, ldc, M_dev, M_max, mode, ws, s, epi);
  return launch_bn<256, 1>(A, lda, a_rows, W, N, K, C, ldc, M_dev, M_max, mode, ws, s, epi);
}

}  // namespace focus
