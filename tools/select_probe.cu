// Microbenchmark of select_fast (csrc/select.cuh) on one 512-thread CTA:
// cycles per two-stage top-p of K log-masses, outside the plan kernel.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_2602_05191_b200/csrc \
//        tools/select_probe.cu -o tools/select_probe && tools/select_probe 4094
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "select.cuh"

using namespace dp;
#ifndef PROBE_NB
#define PROBE_NB 2048
#endif
constexpr int kT = 512, kNB = PROBE_NB, kCap = 4096;

__global__ void __launch_bounds__(kT, 1) probe(const double* lm_g, int K, int reps, long long* cyc, int* out) {
  extern __shared__ __align__(16) unsigned char sm[];
  double* lmall = reinterpret_cast<double*>(sm);
  unsigned long long* um = reinterpret_cast<unsigned long long*>(lmall + kCap);
  unsigned* hm = reinterpret_cast<unsigned*>(um + kCap);
  int* hc = reinterpret_cast<int*>(hm + 2 * kNB);
  int* cur = hc + kNB + 4;
  int* clist = cur + kNB;
  uint8_t* stown = reinterpret_cast<uint8_t*>(clist + kCap);
  __shared__ SelFastShared S;
  double M = -1e300;
  for (int i = threadIdx.x; i < K; i += kT) lmall[i] = lm_g[i];
  __syncthreads();
  for (int i = 0; i < K; ++i) M = fmax(M, lmall[i]);
  long long total = 0;
  int n1 = 0, n2 = 0;
  for (int r = 0; r < reps; ++r) {
    select_fast_zero<kT, kNB>(hm, hc, &S);
    __syncthreads();
    volatile int sink = stown[0];  // a shared load that waits for the barrier
    (void)sink;
    const long long t0 = clock64();
    if (K <= 2 * kT)
      select_fast<kT, kNB, 2>(K, M, lmall, 0.95, 0.7, um, hm, hc, cur, clist, stown, &S, n1, n2);
    else
      select_fast<kT, kNB, kCap / kT>(K, M, lmall, 0.95, 0.7, um, hm, hc, cur, clist, stown, &S, n1, n2);
    volatile int sink2 = stown[K - 1];
    (void)sink2;
    const long long t1 = clock64();
    if (r > 0) total += t1 - t0;  // the first pass warms the instruction cache
  }
  if (threadIdx.x == 0) {
    *cyc = total / (reps - 1);
    out[0] = n1;
    out[1] = n2;
  }
}

int main(int argc, char** argv) {
  const int K = argc > 1 ? atoi(argv[1]) : 4094;
  std::mt19937_64 g(1);
  std::normal_distribution<double> nd(0.0, 3.0);
  std::vector<double> lm(K);
  for (auto& x : lm) x = nd(g);
  for (int i = 0; i < K / 30; ++i) lm[g() % K] += 12.0;
  double* d_lm;
  long long* d_c;
  int* d_o;
  cudaMalloc(&d_lm, K * 8);
  cudaMalloc(&d_c, 8);
  cudaMalloc(&d_o, 8);
  cudaMemcpy(d_lm, lm.data(), K * 8, cudaMemcpyHostToDevice);
  const size_t smem = kCap * 8 + kCap * 8 + 2 * kNB * 4 + (kNB + 4) * 4 + kNB * 4 + kCap * 4 + kCap + 64;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  probe<<<1, kT, smem>>>(d_lm, K, 20, d_c, d_o);
  long long c;
  int o[2];
  cudaMemcpy(&c, d_c, 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(o, d_o, 8, cudaMemcpyDeviceToHost);
  long long pr[16] = {};
#ifdef SEL_PROBE
  cudaMemcpyFromSymbol(pr, g_sel_probe, sizeof(pr));
#endif
  const char* nm[] = {"hist", "bins-load+warpscan", "warp0 scan", "bins write/b1", "cand", "rank", "cut2", "states"};
  for (int i = 0; i < 8; ++i)
    if (pr[i] && pr[i + 1]) printf("  %-22s %6lld cycles\n", nm[i], pr[i + 1] - pr[i]);
  printf("K %d: select_fast %lld cycles (%.2f us at 1.965 GHz), n1 %d n2 %d  [%s]\n", K, c, c / 1965.0, o[0], o[1],
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
