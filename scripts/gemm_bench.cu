// Stand-alone timing of libfocus's tensor-core GEMM launcher (focus::launch_gemm_tc) at one decode
// shape, cold weights (L2 flushed before every launch), CUDA events per launch; optional per-CTA
// global-timer phase trace of the swap-AB kernel (focus::gemm_set_trace).  Development tool:
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I include -I paper_2601_23278_b200/csrc \
//        scripts/gemm_bench.cu -o gpurun_out/gemm_bench -L paper_2601_23278_b200 -lfocus -lcuda \
//        -Xlinker -rpath=$PWD/paper_2601_23278_b200
//   gpurun_out/gemm_bench MODE N K M [M_max] [iters]      MODE: add | store | swiglu | qkv
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"

using namespace focus;
namespace focus {
bool launch_gemm_tc(const bf16* A, int lda, int a_rows, const bf16* W, int N, int K, float* C, int ldc, const int* M_dev,
                    int M_max, GemmMode mode, const GemmWs& ws, cudaStream_t s, const GemmEpi* epi, int m_est);
void gemm_set_trace(long long* buf);
}

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) { fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_)); exit(1); } \
  } while (0)

__global__ void fill_bf16(bf16* p, size_t n, uint64_t seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = __float2bfloat16_rn(((int)(mix64(seed + i) & 0xffff) - 32768) / 32768.f * 0.05f);
}
__global__ void flush(float* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] += 1.f;
}

int main(int argc, char** argv) {
  if (argc < 5) { fprintf(stderr, "usage: gemm_bench MODE N K M [M_max] [iters]\n"); return 2; }
  const char* ms = argv[1];
  const int N = atoi(argv[2]), K = atoi(argv[3]), M = atoi(argv[4]);
  const int M_max = argc > 5 ? atoi(argv[5]) : M;
  const int iters = argc > 6 ? atoi(argv[6]) : 20;
  GemmMode mode = !strcmp(ms, "add") ? GEMM_ADD : !strcmp(ms, "swiglu") ? GEMM_SWIGLU
                : !strcmp(ms, "qkv") ? GEMM_QKV_ROPE : GEMM_STORE;
  const int a_rows = std::max(M_max, 128);
  bf16 *A, *W, *out;
  float *C, *fl, *ropeT;
  int* Mdev;
  CK(cudaMalloc(&A, (size_t)a_rows * K * 2));
  CK(cudaMalloc(&W, (size_t)N * K * 2));
  CK(cudaMalloc(&C, (size_t)a_rows * N * 4));
  CK(cudaMalloc(&out, (size_t)a_rows * N * 2));
  CK(cudaMalloc(&Mdev, 4));
  const size_t nfl = 64ull << 20;                       // 256 MB: > L2
  CK(cudaMalloc(&fl, nfl * 4));
  fill_bf16<<<1024, 256>>>(A, (size_t)a_rows * K, 1);
  fill_bf16<<<1024, 256>>>(W, (size_t)N * K, 2);
  CK(cudaMemset(C, 0, (size_t)a_rows * N * 4));
  CK(cudaMemcpy(Mdev, &M, 4, cudaMemcpyHostToDevice));
  GemmWs ws{};
  CK(cudaMalloc(&ws.ptr, 64ull << 20));
  ws.bytes = 64ull << 20;
  CK(cudaMalloc(&ws.sem, 16384 * 4));
  CK(cudaMemset(ws.sem, 0, 16384 * 4));
  ws.sem_count = 16384;
  GemmEpi epi{};
  epi.out = out;
  epi.ldo = mode == GEMM_SWIGLU ? N / 2 : N;
  // QKV: 128-dim heads, 8 kv heads, one request slot, pages of 64
  const int hd = 128, hkv = 8, page = 64, max_pages = 64;
  RowInfo* rows;
  int* pt;
  focus_req_state* st;
  Counters* cnt;
  bf16 *Kc, *Vc;
  CK(cudaMalloc(&rows, a_rows * sizeof(RowInfo)));
  CK(cudaMalloc(&ropeT, 128ull * a_rows * 4));
  CK(cudaMalloc(&pt, max_pages * 4));
  CK(cudaMalloc(&st, sizeof(focus_req_state) * 4));
  CK(cudaMalloc(&cnt, sizeof(Counters)));
  CK(cudaMalloc(&Kc, (size_t)max_pages * hkv * page * hd * 2));
  CK(cudaMalloc(&Vc, (size_t)max_pages * hkv * page * hd * 2));
  {
    std::vector<RowInfo> hr(a_rows);
    for (int i = 0; i < a_rows; ++i) hr[i] = RowInfo{0, i % 16, 1024 + i % (max_pages * page - 1024), 0};
    CK(cudaMemcpy(rows, hr.data(), a_rows * sizeof(RowInfo), cudaMemcpyHostToDevice));
    std::vector<int> hp(max_pages);
    for (int i = 0; i < max_pages; ++i) hp[i] = max_pages - 1 - i;
    CK(cudaMemcpy(pt, hp.data(), max_pages * 4, cudaMemcpyHostToDevice));
    CK(cudaMemset(st, 0, sizeof(focus_req_state) * 4));
    CK(cudaMemset(cnt, 0, sizeof(Counters)));
    CK(cudaMemset(ropeT, 0, 128ull * a_rows * 4));
  }
  epi.rows = rows;
  epi.ropeT = ropeT;
  epi.rope_ld = a_rows;
  epi.st = st;
  epi.kv = KVView{Kc, Vc, pt, max_pages, page, hkv, hd};
  epi.n_q_heads = N / hd - 2 * hkv;
  epi.cnt = cnt;
  cudaStream_t s;
  CK(cudaStreamCreate(&s));
  auto run = [&]() {
    if (!launch_gemm_tc(A, K, a_rows, W, N, K, C, N, Mdev, M_max, mode, ws, s, &epi, M)) {
      fprintf(stderr, "launch_gemm_tc refused the shape\n");
      exit(1);
    }
  };
  for (int i = 0; i < 3; ++i) run();
  CK(cudaStreamSynchronize(s));
  CK(cudaGetLastError());
  std::vector<float> t;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const bool hot = getenv("GEMM_BENCH_HOT") != nullptr;   // weights L2-resident (no flush)
  for (int i = 0; i < iters; ++i) {
    if (!hot) flush<<<1184, 256, 0, s>>>(fl, nfl);
    cudaEventRecord(e0, s);
    run();
    cudaEventRecord(e1, s);
    CK(cudaEventSynchronize(e1));
    float ms_ = 0;
    cudaEventElapsedTime(&ms_, e0, e1);
    t.push_back(ms_ * 1e3f);
  }
  std::sort(t.begin(), t.end());
  const double wbytes = (double)N * K * 2;
  printf("%s mode %s N %d K %d M %d M_max %d: median %.2f us (min %.2f)  weights %.1f MB -> %.0f GB/s\n", hot ? "hot " : "cold", ms, N, K, M, M_max,
         t[t.size() / 2], t[0], wbytes / 1e6, wbytes / (t[t.size() / 2] * 1e3));
  // phase trace of one launch
  long long* tr;
  const int maxc = 1024;
  CK(cudaMalloc(&tr, (size_t)maxc * 3 * 256 * 8));
  CK(cudaMemset(tr, 0, (size_t)maxc * 3 * 256 * 8));
  gemm_set_trace(tr);
  flush<<<1184, 256, 0, s>>>(fl, nfl);
  run();
  CK(cudaStreamSynchronize(s));
  gemm_set_trace(nullptr);
  std::vector<long long> h((size_t)maxc * 3 * 256);
  CK(cudaMemcpy(h.data(), tr, h.size() * 8, cudaMemcpyDeviceToHost));
  long long t0 = 0;
  int nc = 0;
  for (int c = 0; c < maxc; ++c) {
    const long long v = h[(size_t)c * 768];
    if (v) { t0 = t0 ? std::min(t0, v) : v; ++nc; }
  }
  if (nc) {
    const char* nm[12] = {"entry", "setup", "tfull", "parked", "bar1", "epi", "bar2", "loads", "w_issued", "pdl_wait", "M_read", "reduced"};
    printf("trace: %d CTAs; per event (us after first entry): min / median / max\n", nc);
    for (int e = 0; e < 12; ++e) {
      std::vector<double> v;
      for (int c = 0; c < maxc; ++c)
        if (h[(size_t)c * 768] && h[(size_t)c * 768 + e]) v.push_back((h[(size_t)c * 768 + e] - t0) / 1e3);
      if (v.empty()) continue;
      std::sort(v.begin(), v.end());
      printf("  %-7s %8.2f %8.2f %8.2f\n", nm[e], v[0], v[v.size() / 2], v.back());
    }
  }
  return 0;
}
