// peaks.cu — microbenchmarks for the rooflines of the sweep:
//   FP32 FFMA issue-limited throughput (scalar and packed f32x2), L2 random 32-B gather
//   bandwidth over an L2-resident table, HBM copy.  Prints one JSON object.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bench/peaks bench/peaks.cu
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int ITERS = 4096;

__global__ void ffma_kernel(float* out, float a, float b) {
  float x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3f + k;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fmaf(x[k], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 1234.5f) out[0] = s;
}

__device__ __forceinline__ unsigned long long ffma2(unsigned long long x, unsigned long long a,
                                                    unsigned long long b) {
  unsigned long long d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(x), "l"(a), "l"(b));
  return d;
}

__global__ void ffma2_kernel(float* out, float a, float b) {
  unsigned long long x[8];
  float2 af = make_float2(a, a), bf = make_float2(b, b);
  unsigned long long A = *reinterpret_cast<unsigned long long*>(&af);
  unsigned long long B = *reinterpret_cast<unsigned long long*>(&bf);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    float2 v = make_float2(threadIdx.x * 1e-3f + k, k + 0.5f);
    x[k] = *reinterpret_cast<unsigned long long*>(&v);
  }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = ffma2(x[k], A, B);
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) { float2 v = *reinterpret_cast<float2*>(&x[k]); s += v.x + v.y; }
  if (s == 1234.5f) out[0] = s;
}

// random 32-B sector gathers (one float4 pair per lane per load) from a table of n_sect sectors
__global__ void gather_kernel(const float4* __restrict__ tab, uint32_t mask, int iters,
                              float* out) {
  uint32_t h = (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u + 12345u;
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
    h = h * 1664525u + 1013904223u;
    uint32_t s = (h >> 4) & mask;
    float4 v = __ldg(tab + 2 * s);
    float4 w = __ldg(tab + 2 * s + 1);
    acc += v.x + w.w;
  }
  if (acc == 1234.5f) out[0] = acc;
}

__global__ void copy_kernel(const float4* __restrict__ a, float4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  CK(cudaSetDevice(dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  float* out;
  CK(cudaMalloc(&out, 4));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  const int grid = sms * 8, block = 256;
  // FFMA
  ffma_kernel<<<grid, block>>>(out, 0.999f, 1e-3f);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) ffma_kernel<<<grid, block>>>(out, 0.999f, 1e-3f);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms, e0, e1);
  double ffma_tf = 5.0 * grid * block * (double)ITERS * 8 * 2 / (ms * 1e-3) / 1e12;
  // FFMA2
  ffma2_kernel<<<grid, block>>>(out, 0.999f, 1e-3f);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) ffma2_kernel<<<grid, block>>>(out, 0.999f, 1e-3f);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms, e0, e1);
  double ffma2_tf = 5.0 * grid * block * (double)ITERS * 8 * 4 / (ms * 1e-3) / 1e12;
  // L2 gather over a 16 MiB table
  const uint32_t n_sect = (16u << 20) / 32;
  float4* tab;
  CK(cudaMalloc(&tab, (size_t)n_sect * 32));
  CK(cudaMemset(tab, 0, (size_t)n_sect * 32));
  const int giters = 2048;
  gather_kernel<<<grid, block>>>(tab, n_sect - 1, giters, out);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  gather_kernel<<<grid, block>>>(tab, n_sect - 1, giters, out);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms, e0, e1);
  double gather_gbs = (double)grid * block * giters * 32 / (ms * 1e-3) / 1e9;
  // HBM copy 2 GiB
  size_t n4 = (size_t)1 << 27;
  float4 *a, *b;
  CK(cudaMalloc(&a, n4 * 16));
  CK(cudaMalloc(&b, n4 * 16));
  CK(cudaMemset(a, 0, n4 * 16));
  copy_kernel<<<sms * 16, 512>>>(a, b, n4);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  for (int r = 0; r < 3; ++r) copy_kernel<<<sms * 16, 512>>>(a, b, n4);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms, e0, e1);
  double copy_gbs = 3.0 * 2 * n4 * 16 / (ms * 1e-3) / 1e9;
  printf("{\"sms\": %d, \"clock_mhz_attr\": %d, \"ffma_tflops\": %.2f, \"ffma2_tflops\": %.2f, "
         "\"l2_gather_32B_GBps\": %.1f, \"hbm_copy_GBps\": %.1f}\n",
         sms, clk / 1000, ffma_tf, ffma2_tf, gather_gbs, copy_gbs);
  return 0;
}
