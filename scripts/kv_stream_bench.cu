// Memory side of the decode attention in isolation: a persistent grid (one CTA per SM) streams paged
// K/V tiles (128 keys x 128 dims bf16, 32 KB each for K and V) with TMA into per-CTA rings, and a
// consumer thread frees each slot after an emulated per-tile compute delay.  Measures the achieved
// HBM rate for ring depths, page-table access and pool layouts.  Development tool:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/kv_stream_bench.cu -o gpurun_out/kvb -lcuda
//   gpurun_out/kvb SK SV DELAY PTMODE LAYOUT [KEYS] [UNITS]
//     PTMODE 0: page-table entry loaded from global after the slot wait (as k_attn_tc)
//            1: the unit's row indices staged in registers of the producer warp (shuffled per tile)
//     LAYOUT 0: [page][head][64 keys][128 dims] (two 64-column boxes per page, 128 of every 256 B)
//            1: [page][head][half][64 keys][64 dims] (each box one contiguous 8 KB run)
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <random>
#include <vector>

#define CK(x)                                                                                         \
  do {                                                                                                \
    cudaError_t e_ = (x);                                                                             \
    if (e_ != cudaSuccess) { fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_)); exit(1); }      \
  } while (0)

constexpr int KT = 128, PS = 64, H = 8, SLOT = 32768, MAXSLOT = 6;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(su32(b)),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, uint64_t* bar, int x, int y, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, %4}], "
      "[%2], %5;" ::"r"(su32(dst)),
      "l"((uint64_t)m), "r"(su32(bar)), "r"(x), "r"(y), "l"(pol)
      : "memory");
}

struct Args {
  const int* pt;      // [req][max_pages]
  int max_pages, n_units, keys, sk, sv, delay, ptmode, layout;
};

__global__ void __launch_bounds__(96, 1) k_stream(const __grid_constant__ CUtensorMap mK,
                                                  const __grid_constant__ CUtensorMap mV, Args a) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[2][MAXSLOT], empty[2][MAXSLOT];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < MAXSLOT; ++s)
      for (int k = 0; k < 2; ++k) { mbar_init(&full[k][s], 1); mbar_init(&empty[k][s], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int nt = (a.keys + KT - 1) / KT;
  if (warp < 2) {                                   // producers: warp 0 K, warp 1 V
    const bool isK = warp == 0;
    const int NS = isK ? a.sk : a.sv;
    const CUtensorMap* m = isK ? &mK : &mV;
    uint8_t* ring = sm + (isK ? 0 : a.sk * SLOT);
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    uint32_t g = 0;
    for (int u = blockIdx.x; u < a.n_units; u += gridDim.x) {
      const int req = u / H, head = u % H;
      int myrow = 0;                                // PTMODE 1: lane p holds page p's base row
      if (a.ptmode == 1 && lane < a.max_pages) {
        const int page = a.pt[req * a.max_pages + lane];
        myrow = a.layout == 0 ? (page * H + head) * PS : (page * H + head) * 2 * PS;
      }
      __syncwarp();
      for (int t = 0; t < nt; ++t, ++g) {
        const int s = g % NS;
        mbar_wait(&empty[isK][s], ((g / NS) & 1) ^ 1);
        int rows[2];
#pragma unroll
        for (int pc = 0; pc < 2; ++pc) {
          const int p = (t * KT) / PS + pc;
          if (a.ptmode == 1) rows[pc] = __shfl_sync(0xffffffffu, myrow, p & 31);
          else if (lane == 0) {
            const int page = a.pt[req * a.max_pages + p];
            rows[pc] = a.layout == 0 ? (page * H + head) * PS : (page * H + head) * 2 * PS;
          }
        }
        if (lane == 0) {
          mbar_expect_tx(&full[isK][s], SLOT);
          uint8_t* dst = ring + s * SLOT;
          for (int pc = 0; pc < 2; ++pc) {
            if (a.layout == 0) {
              tma2d(dst + pc * PS * 128, m, &full[isK][s], 0, rows[pc], pol);
              tma2d(dst + 16384 + pc * PS * 128, m, &full[isK][s], 64, rows[pc], pol);
            } else {
              tma2d(dst + pc * PS * 128, m, &full[isK][s], 0, rows[pc], pol);
              tma2d(dst + 16384 + pc * PS * 128, m, &full[isK][s], 0, rows[pc] + PS, pol);
            }
          }
        }
        __syncwarp();
      }
    }
  } else if (lane == 0) {                           // consumer
    uint32_t g = 0;
    for (int u = blockIdx.x; u < a.n_units; u += gridDim.x)
      for (int t = 0; t < nt; ++t, ++g) {
        mbar_wait(&full[1][g % a.sk], (g / a.sk) & 1);
        const long long t0 = clock64();
        while (clock64() - t0 < a.delay) {}
        mbar_arrive(&empty[1][g % a.sk]);
        mbar_wait(&full[0][g % a.sv], (g / a.sv) & 1);
        mbar_arrive(&empty[0][g % a.sv]);
      }
  }
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  if (argc < 6) { fprintf(stderr, "usage: kvb SK SV DELAY PTMODE LAYOUT [KEYS] [UNITS]\n"); return 2; }
  Args a{};
  a.sk = atoi(argv[1]); a.sv = atoi(argv[2]); a.delay = atoi(argv[3]); a.ptmode = atoi(argv[4]); a.layout = atoi(argv[5]);
  a.keys = argc > 6 ? atoi(argv[6]) : 1280;
  a.n_units = argc > 7 ? atoi(argv[7]) : 512;
  const int n_req = (a.n_units + H - 1) / H;
  a.max_pages = (a.keys + PS - 1) / PS + 2;
  if (a.max_pages > 32 && a.ptmode == 1) { fprintf(stderr, "PTMODE 1 needs <= 32 pages\n"); return 2; }
  const size_t pages = (size_t)n_req * a.max_pages;
  const size_t rows = pages * H * PS;             // rows of 128 dims
  void *K, *V;
  CK(cudaMalloc(&K, rows * 256));
  CK(cudaMalloc(&V, rows * 256));
  CK(cudaMemset(K, 0, rows * 256));
  CK(cudaMemset(V, 0, rows * 256));
  std::vector<int> perm(pages);
  std::iota(perm.begin(), perm.end(), 0);
  std::shuffle(perm.begin(), perm.end(), std::mt19937(7));
  int* pt;
  CK(cudaMalloc(&pt, pages * 4));
  CK(cudaMemcpy(pt, perm.data(), pages * 4, cudaMemcpyHostToDevice));
  a.pt = pt;
  EncFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
  CUtensorMap mK, mV;
  for (int w = 0; w < 2; ++w) {
    const cuuint64_t gdim[2] = {(cuuint64_t)(a.layout == 0 ? 128 : 64), (cuuint64_t)(a.layout == 0 ? rows : 2 * rows)};
    const cuuint64_t gstr[1] = {(cuuint64_t)(a.layout == 0 ? 256 : 128)};
    const cuuint32_t box[2] = {64, 64}, es[2] = {1, 1};
    CUresult r = enc(w ? &mV : &mK, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w ? V : K, gdim, gstr, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { fprintf(stderr, "encode failed %d\n", (int)r); return 1; }
  }
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  const int smem = (a.sk + a.sv) * SLOT + 1024;
  CK(cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (int i = 0; i < 3; ++i) k_stream<<<nsm, 96, smem>>>(mK, mV, a);
  CK(cudaDeviceSynchronize());
  const int iters = 20;
  float best = 1e30f, sum = 0.f;
  for (int i = 0; i < iters; ++i) {
    CK(cudaEventRecord(e0));
    k_stream<<<nsm, 96, smem>>>(mK, mV, a);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    best = std::min(best, ms);
    sum += ms;
  }
  const int nt = (a.keys + KT - 1) / KT;
  const double bytes = (double)a.n_units * nt * 2 * SLOT;
  printf("SK %d SV %d delay %d ptmode %d layout %d keys %d units %d: %.1f MB, best %.1f us (%.0f GB/s), mean %.1f us (%.0f GB/s)\n",
         a.sk, a.sv, a.delay, a.ptmode, a.layout, a.keys, a.n_units, bytes / 1e6, best * 1e3, bytes / best / 1e6,
         sum / iters * 1e3, bytes / (sum / iters) / 1e6);
  return 0;
}
