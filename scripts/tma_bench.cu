// TMA streaming microbenchmark (development tool): how fast can CTAs pull K-major SW128 tiles the way
// the GEMM producer does, as a function of CTA count, boxes per stage, pipeline depth and whether the
// source is HBM-fresh or L2-resident.  No MMA: the consumer releases each stage as soon as it lands.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I include scripts/tma_bench.cu \
//        -o /tmp/tma_bench -Lpaper_2601_23278_b200 -lfocus -Xlinker -rpath=$PWD/paper_2601_23278_b200
#include <cstdio>
#include <cstdlib>

#include "../paper_2601_23278_b200/csrc/tc_ptx.cuh"

using namespace focus;
using namespace focus::tc;

// CTA b streams row band (b % bands) of [rows][K]: for kb in 0..K/64: `boxes` boxes of box_rows x 64
// (stacked rows), stage = boxes * box_rows * 128 B
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)), "l"((uint64_t)src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// wait variants: 0 try_wait (no hint), 1 test_wait spin, 2 try_wait with a 20 ns suspend hint
template <int WM>
__device__ __forceinline__ void wait_v(uint64_t* bar, uint32_t parity) {
  if constexpr (WM == 0) {
    mbar_wait(bar, parity);
  } else if constexpr (WM == 1) {
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\nmbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
            smem_u32(bar)), "r"(parity)
        : "memory");
  } else {
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 20;\n@!p bra W_%=;\n}\n" ::"r"(
            smem_u32(bar)), "r"(parity)
        : "memory");
  }
}

// linear = true: the band's tiles are pre-packed contiguously ([band][kb][boxes*box_rows*128 B]) and
// each box is one 1-D bulk copy instead of a 2-D tensor box
template <int WM>
__global__ void __launch_bounds__(64, 1) k_stream(const __grid_constant__ CUtensorMap map, const uint8_t* lin, int K,
                                                  int box_rows, int boxes, int stages, int bands, int reps, int linear, long long* cyc) {
  const long long t0 = clock64();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int stage_bytes = boxes * box_rows * 128;
  uint64_t* full = (uint64_t*)(smem + stages * stage_bytes);
  uint64_t* empty = full + stages;
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int kbn = K / 64;
  const int band = blockIdx.x % bands;
  if (threadIdx.x == 0) {
    int st = 0;
    uint32_t ph = 0;
    long long tw = 0, ti = 0;
    for (int r = 0; r < reps; ++r)
      for (int kb = 0; kb < kbn; ++kb) {
        const long long a0 = clock64();
        wait_v<WM>(&empty[st], ph ^ 1);
        const long long a1 = clock64();
        tw += a1 - a0;
        mbar_expect_tx(&full[st], stage_bytes);
        for (int b = 0; b < boxes; ++b)
          if (linear)
            bulk_load(smem + st * stage_bytes + b * box_rows * 128,
                      lin + ((size_t)band * kbn + kb) * stage_bytes + (size_t)b * box_rows * 128, box_rows * 128, &full[st]);
          else
            tma_load_2d(smem + st * stage_bytes + b * box_rows * 128, &map, &full[st], kb * 64,
                      (band * boxes + b) * box_rows);
        ti += clock64() - a1;
        if (++st == stages) { st = 0; ph ^= 1; }
      }
    if (blockIdx.x == 0) { cyc[1] = tw; cyc[2] = ti; }
  } else if (threadIdx.x == 32) {
    int st = 0;
    uint32_t ph = 0;
    for (int r = 0; r < reps; ++r)
      for (int kb = 0; kb < kbn; ++kb) {
        wait_v<WM>(&full[st], ph);
        mbar_arrive(&empty[st]);
        if (++st == stages) { st = 0; ph ^= 1; }
      }
    if (blockIdx.x == 0) cyc[0] = clock64() - t0;
  }
}

// plain vectorised streaming read (reference for achievable HBM read bandwidth)
__global__ void k_ldg(const uint4* __restrict__ p, size_t n, uint4* sink) {
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x * 4) {
    uint4 v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const size_t k = i + (size_t)j * gridDim.x * blockDim.x;
      v[j] = k < n ? __ldcs(p + k) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) { acc.x ^= v[j].x; acc.y ^= v[j].y; acc.z ^= v[j].z; acc.w ^= v[j].w; }
  }
  if (acc.x == 0x12345678) sink[0] = acc;
}

int main() {
  const int K = 4096;
  const long long rows = 24576 * 2;                     // 402 MB source (HBM-fresh when bands differ)
  bf16* W;
  cudaMalloc(&W, rows * K * 2);
  cudaMemset(W, 1, rows * K * 2);
  void* flush;
  cudaMalloc(&flush, (size_t)256 << 20);
  long long* cyc;
  cudaMalloc(&cyc, 24);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaFuncSetAttribute(k_stream<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_stream<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_stream<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  struct Cfg { int ctas, box_rows, boxes, stages; bool l2; int lin = 0; int wm = 0; };
  const Cfg cfgs[] = {
      {1, 128, 1, 4, false},   {1, 128, 1, 8, false},   {1, 128, 1, 12, false},  {1, 128, 2, 6, false},
      {1, 256, 1, 6, false},   {48, 128, 1, 6, false},  {48, 128, 2, 6, false},  {48, 128, 1, 12, false},
      {96, 128, 1, 6, false},  {96, 128, 1, 12, false}, {96, 128, 2, 3, false},  {96, 128, 2, 6, false},
      {148, 128, 1, 6, false}, {148, 128, 1, 12, false},{148, 128, 2, 6, false}, {148, 256, 1, 6, false},
      {1, 128, 1, 6, true},    {1, 128, 1, 12, true},   {48, 128, 1, 6, true},   {96, 128, 1, 6, true},
      {148, 128, 1, 6, true},  {148, 128, 1, 12, true}, {148, 128, 2, 6, true},
      {1, 256, 1, 6, true},    {148, 256, 1, 6, true},  {148, 128, 4, 3, true},  {148, 64, 4, 6, true},
      // pre-packed contiguous tiles, 1-D bulk copies
      {1, 128, 1, 6, false, 1},   {1, 128, 2, 6, false, 1},   {48, 128, 2, 6, false, 1},  {96, 128, 2, 6, false, 1},
      {148, 128, 1, 6, false, 1}, {148, 128, 2, 6, false, 1}, {148, 128, 1, 12, false, 1},
      {1, 128, 1, 6, true, 1},    {148, 128, 1, 6, true, 1},  {148, 128, 2, 6, true, 1},  {148, 128, 4, 3, true, 1},
      // wait variants
      {1, 128, 1, 6, true, 0, 1},   {1, 128, 1, 12, true, 0, 1},  {148, 128, 1, 6, true, 0, 1}, {148, 128, 2, 6, true, 0, 1},
      {1, 128, 1, 6, false, 0, 1},  {148, 128, 1, 6, false, 0, 1}, {148, 128, 2, 6, false, 0, 1},
      {1, 128, 1, 6, true, 0, 2},   {148, 128, 1, 6, true, 0, 2},  {148, 128, 2, 6, false, 0, 2},
  };
  printf("%2s %3s %5s %5s %5s %6s %3s  %9s %9s %8s %9s %8s %8s\n", "wm", "lin", "ctas", "rows", "boxes", "stages", "L2", "us", "GB/s", "GB/s/SM", "cyc/stage", "wait/st", "issue/st");
  for (const Cfg& c : cfgs) {
    CUtensorMap map;
    if (!make_tma_2d_bf16(W, rows, K, K, 64, c.box_rows, &map)) { printf("map failed\n"); return 1; }
    const int stage_bytes = c.boxes * c.box_rows * 128;
    const int smem = c.stages * stage_bytes + 1024 + 2 * c.stages * 8;
    if (smem > 200 * 1024) continue;
    // HBM-fresh: every CTA its own band (distinct rows), one pass; L2: 8 bands shared, 4 passes
    const int bands = c.l2 ? 2 : c.ctas, reps = c.l2 ? 4 : 1;
    float best = 1e30f;
    for (int r = 0; r < 4; ++r) {
      cudaMemset(flush, r, (size_t)256 << 20);
      auto fn = c.wm == 0 ? k_stream<0> : c.wm == 1 ? k_stream<1> : k_stream<2>;
      if (c.l2) fn<<<c.ctas, 64, smem>>>(map, (const uint8_t*)W, K, c.box_rows, c.boxes, c.stages, bands, 1, c.lin, cyc);   // warm
      cudaEventRecord(e0);
      fn<<<c.ctas, 64, smem>>>(map, (const uint8_t*)W, K, c.box_rows, c.boxes, c.stages, bands, reps, c.lin, cyc);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    long long hcs[3] = {0, 0, 0};
    cudaMemcpy(hcs, cyc, 24, cudaMemcpyDeviceToHost);
    const long long hc = hcs[0];
    const double bytes = (double)c.ctas * reps * (K / 64) * stage_bytes;
    printf("%2d %3d %5d %5d %5d %6d %3s  %9.1f %9.0f %8.1f %9.0f %8.0f %8.0f\n", c.wm, c.lin, c.ctas, c.box_rows, c.boxes, c.stages, c.l2 ? "yes" : "no",
           best * 1e3, bytes / (best * 1e-3) / 1e9, bytes / (best * 1e-3) / 1e9 / c.ctas, (double)hc / (reps * (K / 64)), (double)hcs[1] / (reps * (K / 64)), (double)hcs[2] / (reps * (K / 64)));
  }
  {
    const size_t n = (size_t)rows * K * 2 / 16;
    uint4* sink;
    cudaMalloc(&sink, 16);
    for (int blocks : {148, 296, 592, 1184}) {
      float best = 1e30f;
      for (int r = 0; r < 4; ++r) {
        cudaMemset(flush, r, (size_t)256 << 20);
        cudaEventRecord(e0);
        k_ldg<<<blocks, 512>>>((const uint4*)W, n, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
      }
      printf("ldg blocks %5d x 512: %.1f us  %.0f GB/s\n", blocks, best * 1e3, n * 16.0 / (best * 1e-3) / 1e9);
    }
  }
  // TMA with several CTAs per SM (smaller pipelines each), HBM-fresh
  {
    struct C2 { int ctas, boxes, stages; };
    for (C2 c : {C2{296, 1, 3}, C2{296, 1, 6}, C2{384, 1, 3}, C2{384, 1, 2}}) {
      CUtensorMap map;
      make_tma_2d_bf16(W, rows, K, K, 64, 128, &map);
      const int stage_bytes = c.boxes * 128 * 128;
      const int smem = c.stages * stage_bytes + 1024 + 2 * c.stages * 8;
      float best = 1e30f;
      for (int r = 0; r < 4; ++r) {
        cudaMemset(flush, r, (size_t)256 << 20);
        cudaEventRecord(e0);
        k_stream<0><<<c.ctas, 64, smem>>>(map, (const uint8_t*)W, K, 128, c.boxes, c.stages, c.ctas, 1, 0, cyc);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
      }
      const double bytes = (double)c.ctas * (K / 64) * stage_bytes;
      printf("multi-CTA/SM: ctas %d boxes %d stages %d smem %d: %.1f us  %.0f GB/s\n", c.ctas, c.boxes, c.stages, smem,
             best * 1e3, bytes / (best * 1e-3) / 1e9);
    }
  }
  printf("status: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
