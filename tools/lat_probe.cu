// Latency probe (profiling aid): %globaltimer deltas around a few primitive
// sequences inside one CTA, to calibrate the plan kernel's phase costs.
#include <cstdio>
#include <cuda_runtime.h>

__device__ unsigned long long ts[64];
__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void probe(const float* __restrict__ buf, float* out, int n) {
  float acc = 0.f;
  unsigned long long t0 = gt();
  acc += __ldg(&buf[threadIdx.x]);  // 1 load
  __syncthreads();
  unsigned long long t1 = gt();
#pragma unroll
  for (int i = 0; i < 32; ++i) acc += __ldg(&buf[(threadIdx.x + i * 64) % n]);  // 32 independent loads
  __syncthreads();
  unsigned long long t2 = gt();
  // dependent chain of 8 loads
  int idx = threadIdx.x;
  for (int i = 0; i < 8; ++i) idx = ((int)__ldg(&buf[idx % n]) + idx + 1) % n;
  acc += idx;
  __syncthreads();
  unsigned long long t3 = gt();
  // 64 DFMA dependent chain
  double x = acc;
  for (int i = 0; i < 64; ++i) x = fma(x, 1.0000001, 1e-9);
  acc += (float)x;
  __syncthreads();
  unsigned long long t4 = gt();
  // 100 __syncthreads
  for (int i = 0; i < 100; ++i) __syncthreads();
  unsigned long long t5 = gt();
  // dependent chain of 16 DMMA
  double c0 = acc, c1 = 0.0, a = 1.0, b = 1.0;
  for (int i = 0; i < 16; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
  acc += (float)(c0 + c1);
  __syncthreads();
  unsigned long long t6 = gt();
  if (threadIdx.x == 0) {
    ts[0] = t1 - t0; ts[1] = t2 - t1; ts[2] = t3 - t2; ts[3] = t4 - t3; ts[4] = t5 - t4; ts[5] = t6 - t5;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  const int n = 1 << 20;
  float* buf;
  float* out;
  cudaMalloc(&buf, n * 4);
  cudaMemset(buf, 0, n * 4);
  cudaMalloc(&out, 1 << 20);
  for (int rep = 0; rep < 3; ++rep) {
    probe<<<1, 512>>>(buf, out, n);
    cudaDeviceSynchronize();
    unsigned long long h[6];
    cudaMemcpyFromSymbol(h, ts, sizeof(h));
    printf("rep %d: 1 load %.2f us | 32 indep loads %.2f | 8 dependent loads %.2f | 64 dep DFMA %.2f | 100 syncthreads %.2f | 16 dep DMMA %.2f\n",
           rep, h[0] / 1e3, h[1] / 1e3, h[2] / 1e3, h[3] / 1e3, h[4] / 1e3, h[5] / 1e3);
  }
  return 0;
}
