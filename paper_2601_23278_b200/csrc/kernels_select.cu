// Decodable-token selection (Alg.1 Phase 2-3; §4.2; App.E)
// fused with the compaction plan (App.E).  One CTA of 32 warps; warp w handles the
// requests w, w+32, ... of the call (one uint64 mask per request, lane = block positions lane and
// lane+32).  Then one thread per request scans |S| and |S cap M| and writes the dense row maps.
//
// Bit-exact contract with the oracle (DESIGN.md A-S4, A-B3, A-E1): dI = fl32(I1 - I0) with I summed
// over the partials in a fixed order; mu, sigma in binary64, two-pass, ascending positions,
// explicit _rn intrinsics (no FMA contraction); K_hist = ceil(num*T / (den*N)) in int64; top-K by
// rank with (dI descending, j ascending), +0 == -0.
#include "common.cuh"

namespace focus {

__global__ void __launch_bounds__(1024) k_select_plan(SelectArgs a) {
  pdl_trigger();
  pdl_wait();
  __shared__ float dl[32][kMaxB];
  __shared__ int nS_sh[1024], nL_sh[1024];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int B = a.B;
  const uint64_t full = full_mask(B);

  for (int i = warp; i < a.n_req; i += 32) {
    const int slot = a.req_list[i];
    focus_req_state& st = a.st[slot];
    const bool live = st.active && !st.finished;
    const uint64_t P = live ? st.P : 0ull, M = live ? st.M : 0ull, U = P & ~M;
    uint64_t S = 0ull;
    int K = 0, ns = 0, kh = 0;
    if (live && M == 0ull) {
      S = P;                                            // flush step: re-forward U, no selection
    } else if (live) {
      // dI per position (fixed-order partial sums)
      float d[2];
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int j = lane + 32 * t;
        float i0 = 0.f, i1 = 0.f;
        if (j < B) {
          // partials of the chunks that hold rows (chunk-major, kv head minor), in that fixed order
          const int n_parts = ((__popcll(P) + a.attn_rpc - 1) / a.attn_rpc) * a.n_kv_heads;
          const size_t base = (size_t)i * a.n_chunks * a.n_kv_heads;
          // L2 loads: I0 was written several kernels back (layer-0 attention); under programmatic
          // dependent launch only the immediate predecessor's writes are guaranteed through L1.  Loaded
          // 8 partials at a time (all in flight), added in the fixed order p = 0, 1, ...
          for (int p0 = 0; p0 < n_parts; p0 += 8) {
            float v0[8], v1[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const bool ok = p0 + q < n_parts;
              v0[q] = ok ? __ldcg(a.I0p + (base + p0 + q) * B + j) : 0.f;
              v1[q] = ok ? __ldcg(a.I1p + (base + p0 + q) * B + j) : 0.f;
            }
#pragma unroll
            for (int q = 0; q < 8; ++q)
              if (p0 + q < n_parts) { i0 = __fadd_rn(i0, v0[q]); i1 = __fadd_rn(i1, v1[q]); }
          }
        }
        d[t] = __fsub_rn(i1, i0);
        dl[warp][j] = d[t];
      }
      __syncwarp();
      // Eq.5 statistics over masked positions (A-S1..A-S4)
      double th = 0.0;
      int n = 0;
      if (lane == 0) {
        double s = 0.0;
        for (int j = 0; j < B; ++j)
          if ((M >> j) & 1ull) { s = __dadd_rn(s, (double)dl[warp][j]); ++n; }
        const double mu = __ddiv_rn(s, (double)n);
        double acc = 0.0;
        for (int j = 0; j < B; ++j)
          if ((M >> j) & 1ull) {
            const double dv = __dsub_rn((double)dl[warp][j], mu);
            acc = __dadd_rn(acc, __dmul_rn(dv, dv));
          }
        th = __dadd_rn(mu, __dsqrt_rn(__ddiv_rn(acc, (double)n)));
      }
      th = __shfl_sync(0xffffffffu, th, 0);
      n = __popcll(M);
      const bool m0 = (M >> lane) & 1ull, m1 = lane + 32 < 64 && ((M >> (lane + 32)) & 1ull);
      ns = __popc(__ballot_sync(0xffffffffu, m0 && (double)d[0] >= th)) +
           __popc(__ballot_sync(0xffffffffu, m1 && (double)d[1] >= th));
      // Eq.4 budget
      if (a.strategy == FOCUS_STRATEGY_FOCUS) {
        long long T = st.token_sum, N = st.total_steps;
        if (N <= 0) { T = 1; N = 1; }
        const long long num = (long long)a.alpha_num * T, den = (long long)a.alpha_den * N;
        kh = (int)((num + den - 1) / den);
        K = min(B, max(kh, ns));
      } else if (a.strategy == FOCUS_STRATEGY_NONE) {
        K = B;
      } else {
        K = a.fixed_k;
      }
      const int Kp = min(K, n);
      // TopK_Indices by rank (Alg.1)
      uint64_t C = 0ull;
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int j = lane + 32 * t;
        bool cand = false;
        if (j < B && ((M >> j) & 1ull)) {
          int rank = 0;
          const float dj = dl[warp][j];
          uint64_t uj = 0;
          if (a.strategy == FOCUS_STRATEGY_FIXED_RANDOM)
            uj = mix64((((uint64_t)slot << 32) | ((uint64_t)(st.t & 0xFFFFFF) << 8) | (uint64_t)j) +
                       (a.seed + 1ull) * kGolden);
          for (int q = 0; q < B; ++q) {
            if (q == j || !((M >> q) & 1ull)) continue;
            const float dq = dl[warp][q];
            bool before;
            if (a.strategy == FOCUS_STRATEGY_FIXED_BOTTOM) {
              before = dq < dj || (dq == dj && q < j);
            } else if (a.strategy == FOCUS_STRATEGY_FIXED_RANDOM) {
              const uint64_t uq = mix64((((uint64_t)slot << 32) | ((uint64_t)(st.t & 0xFFFFFF) << 8) | (uint64_t)q) +
                                        (a.seed + 1ull) * kGolden);
              before = uq < uj || (uq == uj && q < j);
            } else {
              before = dq > dj || (dq == dj && q < j);
            }
            rank += before;
          }
          cand = rank < Kp;
        }
        const uint32_t b = __ballot_sync(0xffffffffu, cand);
        C |= t == 0 ? (uint64_t)b : ((uint64_t)b << 32);
      }
      // AR-context preservation, placeholder integrity, uncached decoded (A-E2..A-E4)
      S = C | ((C >> 1) & ~st.committed);
      const int mx = S ? 63 - __clzll((long long)S) : -1;
      const uint64_t below = mx > 0 ? ((1ull << mx) - 1ull) : 0ull;
      uint64_t aboveR;
      if (st.R < 0) aboveR = ~0ull;
      else if (st.R >= 63) aboveR = 0ull;
      else aboveR = ~((2ull << st.R) - 1ull);
      S |= (a.placeholder_mode == FOCUS_PLACEHOLDER_UNPROCESSED_ONLY ? (M & aboveR) : M) & below;
      S |= U;
      if (S == 0ull && lane == 0) atomicExch(&a.cnt->invariant, 1);   // minimum retention (unreachable)
    }
    S &= full;
    if (lane == 0) {
      st.S = S;
      st.K = K;
      st.n_sigma = ns;
      st.k_hist = kh;
      const int mxS = S ? 63 - __clzll((long long)S) : -1;
      st.R_new = live ? max(st.R, mxS) : st.R;
      nS_sh[i] = __popcll(S);
      nL_sh[i] = __popcll(S & M);
    }
  }
  __syncthreads();

  // ---- compaction plan: exclusive scans over the request list (one thread per request)
  __shared__ int scanS[1024], scanL[1024];
  __shared__ int carryS, carryL;
  if (threadIdx.x == 0) { carryS = 0; carryL = 0; }
  __syncthreads();
  for (int base = 0; base < a.n_req; base += 1024) {
    const int i = base + threadIdx.x;
    const int ns = i < a.n_req ? nS_sh[i] : 0, nl = i < a.n_req ? nL_sh[i] : 0;
    scanS[threadIdx.x] = ns;
    scanL[threadIdx.x] = nl;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {
      const int vs = threadIdx.x >= off ? scanS[threadIdx.x - off] : 0;
      const int vl = threadIdx.x >= off ? scanL[threadIdx.x - off] : 0;
      __syncthreads();
      scanS[threadIdx.x] += vs;
      scanL[threadIdx.x] += vl;
      __syncthreads();
    }
    if (i < a.n_req) {
      const int oS = carryS + scanS[threadIdx.x] - ns, oL = carryL + scanL[threadIdx.x] - nl;
      a.offS[i] = oS;
      a.offL[i] = oL;
      const int slot = a.req_list[i];
      const focus_req_state& st = a.st[slot];
      int rs = oS, rl = oL;
      for (uint64_t m = st.S; m; m &= m - 1) {
        const int j = __ffsll((long long)m) - 1;
        const RowInfo ri{slot, j, st.s + j, i};
        a.rowS[rs] = ri;
        a.srcP[rs] = a.offP[i] + __popcll(st.P & ((1ull << j) - 1ull));
        if ((st.M >> j) & 1ull) {
          a.rowL[rl] = ri;
          a.srcL[rl] = rs;
          ++rl;
        }
        ++rs;
      }
    }
    __syncthreads();
    if (threadIdx.x == 1023) { carryS += scanS[1023]; carryL += scanL[1023]; }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    a.offS[a.n_req] = carryS;
    a.offL[a.n_req] = carryL;
    a.cnt->M_S = carryS;
    a.cnt->M_L = carryL;
    a.cnt->sum_S += carryS;
    a.cnt->sum_L += carryL;
  }
}

void launch_select_plan(const SelectArgs& a, cudaStream_t s) {
  launch_pdl(k_select_plan, dim3(1), dim3(1024), 0, s, a);
}

}  // namespace focus
