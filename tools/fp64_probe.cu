// DFMA / FFMA / exp(double) throughput probe (profiling aid).
#include <cstdio>
#include <cuda_runtime.h>
template <typename T>
__global__ void fma_k(T* out, int iters, T a, T b) {
  T x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
    x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
    x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void exp_k(double* out, int iters) {
  double x = threadIdx.x * 1e-3, s = 0;
  for (int i = 0; i < iters; ++i) { s += exp(x); x += 1e-7; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void lat_k(double* out, int iters, double a, double b) {  // dependent DFMA chain latency
  double x = threadIdx.x;
  for (int i = 0; i < iters; ++i) x = fma(x, a, b);
  out[blockIdx.x * blockDim.x + threadIdx.x] = x;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d; cudaMalloc(&d, sms * 1024 * 8 * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms; const int it = 20000;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0); fma_k<double><<<sms * 4, 256>>>(d, it, 1.0000001, 1e-9); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep) printf("DFMA  %.1f TFLOP/s  (%.1f /clk/SM @1.965GHz)\n", 2.0 * 8 * it * sms * 4 * 256 / (ms * 1e-3) / 1e12, 8.0 * it * sms * 4 * 256 / (ms * 1e-3) / 1.965e9 / sms);
    cudaEventRecord(e0); fma_k<float><<<sms * 4, 256>>>((float*)d, it, 1.0000001f, 1e-9f); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep) printf("FFMA  %.1f TFLOP/s  (%.1f /clk/SM)\n", 2.0 * 8 * it * sms * 4 * 256 / (ms * 1e-3) / 1e12, 8.0 * it * sms * 4 * 256 / (ms * 1e-3) / 1.965e9 / sms);
    cudaEventRecord(e0); exp_k<<<sms * 4, 256>>>(d, 2000); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep) printf("exp(double) %.2f Gexp/s (%.2f /clk/SM)\n", 2000.0 * sms * 4 * 256 / (ms * 1e-3) / 1e9, 2000.0 * sms * 4 * 256 / (ms * 1e-3) / 1.965e9 / sms);
    cudaEventRecord(e0); lat_k<<<1, 32>>>(d, 100000, 1.0000001, 1e-9); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep) printf("DFMA dependent latency %.1f cycles\n", ms * 1e-3 * 1.965e9 / 100000);
  }
  return 0;
}
