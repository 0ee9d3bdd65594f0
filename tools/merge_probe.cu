// Probe: cost of the "last CTA merges the partials" pattern (profiling aid).
// 148 CTAs write a 2 KB partial each (+ fence + atomic); the last CTA of
// each group of 20 reads its group's partials (16 float4 per lane in flight).
#include <cstdio>
#include <cuda_runtime.h>
__device__ unsigned long long ts[148][4];
__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__global__ void __launch_bounds__(256) probe(float4* part, int* ctr, float* out, int hint) {
  __shared__ int last;
  const int grp = blockIdx.x / 20, slot = blockIdx.x % 20, n = min(20, (int)gridDim.x - grp * 20);
  // a little work so CTAs finish at different times
  float x = threadIdx.x;
  for (int i = 0; i < 2000 + (blockIdx.x % 7) * 300; ++i) x = x * 1.0000001f + 1e-7f;
  const unsigned long long t0 = gt();
  if (threadIdx.x < 128) part[((size_t)grp * 20 + slot) * 128 + threadIdx.x] = make_float4(x, x, x, x);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(&ctr[grp], 1) == n - 1;
  }
  __syncthreads();
  const unsigned long long t1 = gt();
  if (!last) return;
  __threadfence();
  const unsigned long long t2 = gt();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float4 acc = make_float4(0, 0, 0, 0);
  float4 v[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const int p = warp + u * 8;
    v[u] = p < n * 4 ? __ldcg(&part[((size_t)grp * 20 + p / 4) * 128 + (p % 4) * 32 + lane]) : make_float4(0, 0, 0, 0);
  }
#pragma unroll
  for (int u = 0; u < 16; ++u) { acc.x += v[u].x; acc.y += v[u].y; }
  const unsigned long long t3 = gt();
  out[grp * 256 + threadIdx.x] = acc.x + acc.y;
  if (threadIdx.x == 0) { ts[grp][0] = t1 - t0; ts[grp][1] = t2 - t1; ts[grp][2] = t3 - t2; ctr[grp] = 0; }
}
int main() {
  float4* part; int* ctr; float* out;
  cudaMalloc(&part, 148 * 20 * 128 * 16); cudaMalloc(&ctr, 64 * 4); cudaMalloc(&out, 1 << 20);
  cudaMemset(ctr, 0, 256);
  for (int rep = 0; rep < 4; ++rep) {
    probe<<<148, 256>>>(part, ctr, out, 0);
    cudaDeviceSynchronize();
    unsigned long long h[148][4];
    cudaMemcpyFromSymbol(h, ts, sizeof(h));
    printf("rep %d: write+fence+atomic %.2f us | acquire fence %.2f us | 16 x float4 loads/lane %.2f us\n", rep,
           h[0][0] / 1e3, h[0][1] / 1e3, h[0][2] / 1e3);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
