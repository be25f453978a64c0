// Scaffolding GEMM (CUDA-core FMA, 128x128 tiles): C = A . W^T with fp32 accumulation.
// Correctness reference for the ragged device-sized M path; the tcgen05 GEMM (kernels_gemm_tc.cu)
// replaces it on the hot path.
#include "common.cuh"

namespace focus {

template <int MODE>
__global__ void __launch_bounds__(256) k_gemm_simt(const bf16* __restrict__ A, int lda, const bf16* __restrict__ W,
                                                   int N, int K, float* __restrict__ C, int ldc,
                                                   const int* __restrict__ M_dev, int M_max) {
  pdl_trigger();
  pdl_wait();
  const int M = M_dev ? min(*M_dev, M_max) : M_max;
  const int m0 = blockIdx.y * 128, n0 = blockIdx.x * 128;
  if (m0 >= M) return;
  __shared__ __align__(16) float As[16][132];
  __shared__ __align__(16) float Ws[16][132];
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  const int lr = tid / 2, lk = (tid % 2) * 8;
  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
  for (int k0 = 0; k0 < K; k0 += 16) {
    uint4 ua = make_uint4(0, 0, 0, 0), uw = make_uint4(0, 0, 0, 0);
    if (m0 + lr < M) ua = *reinterpret_cast<const uint4*>(A + (size_t)(m0 + lr) * lda + k0 + lk);
    if (n0 + lr < N) uw = *reinterpret_cast<const uint4*>(W + (size_t)(n0 + lr) * K + k0 + lk);
    const bf16* pa = reinterpret_cast<const bf16*>(&ua);
    const bf16* pw = reinterpret_cast<const bf16*>(&uw);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      As[lk + e][lr] = __bfloat162float(pa[e]);
      Ws[lk + e][lr] = __bfloat162float(pw[e]);
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      const float4 a0 = *reinterpret_cast<const float4*>(&As[kk][ty * 4]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[kk][64 + ty * 4]);
      const float4 b0 = *reinterpret_cast<const float4*>(&Ws[kk][tx * 4]);
      const float4 b1 = *reinterpret_cast<const float4*>(&Ws[kk][64 + tx * 4]);
      const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int r = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + i - 4);
    if (r >= M) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int c = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + j - 4);
      if (c >= N) continue;
      float* p = C + (size_t)r * ldc + c;
      if (MODE == GEMM_ADD) *p += acc[i][j];
      else *p = acc[i][j];
    }
  }
}

void launch_gemm_simt(const bf16* A, int lda, const bf16* W, int N, int K, float* C, int ldc, const int* M_dev,
                      int M_max, GemmMode mode, cudaStream_t s) {
  if (M_max <= 0) return;
  dim3 grid((N + 127) / 128, (M_max + 127) / 128);
  if (mode == GEMM_ADD)
    launch_pdl(k_gemm_simt<GEMM_ADD>, grid, dim3(256), 0, s, A, lda, W, N, K, C, ldc, M_dev, M_max);
  else
    launch_pdl(k_gemm_simt<GEMM_STORE>, grid, dim3(256), 0, s, A, lda, W, N, K, C, ldc, M_dev, M_max);
}

}  // namespace focus
