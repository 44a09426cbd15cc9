// fma_rates.cu — FMA-pipe issue rates of the instruction forms the sweep uses:
// scalar FFMA / FMUL / FADD with all-register operands vs a constant-bank operand, and the
// packed FFMA2 / FMUL2 / FADD2.  Each thread runs 8 independent chains (latency hidden), the
// grid fills every SM with 16 warps.  Prints warp-instructions per SMSP-cycle and TFLOP/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fma_rates bench/fma_rates.cu
#include <cuda_runtime.h>
#include <stdio.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int ITERS = 2048;
constexpr int CH = 8;

#define KERNEL_SCALAR(name, ASM)                                                   \
  __global__ void name(float* out, float c) {                                      \
    float x[CH], y[CH], z[CH];                                                     \
    for (int k = 0; k < CH; ++k) {                                                 \
      x[k] = threadIdx.x * 1e-3f + k; y[k] = 1.0f + 1e-7f * k + threadIdx.x * 1e-9f; \
      z[k] = 1e-6f * k * threadIdx.x;                                              \
    }                                                                              \
    for (int it = 0; it < ITERS; ++it) {                                           \
      _Pragma("unroll") for (int k = 0; k < CH; ++k) { ASM; }                      \
    }                                                                              \
    float s = 0.f;                                                                 \
    for (int k = 0; k < CH; ++k) s += x[k] + y[k] + z[k];                          \
    if (s == 1234.5f) out[0] = s;                                                  \
  }

KERNEL_SCALAR(ffma_rrr, asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[k]) : "f"(y[k]), "f"(z[k])))
KERNEL_SCALAR(ffma_rrc, asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[k]) : "f"(y[k]), "f"(c)))
KERNEL_SCALAR(ffma_rri, asm volatile("fma.rn.f32 %0, %0, %1, 0f3F800000;" : "+f"(x[k]) : "f"(y[k])))
KERNEL_SCALAR(fmul_rr, asm volatile("mul.rn.f32 %0, %0, %1;" : "+f"(x[k]) : "f"(y[k])))
KERNEL_SCALAR(fadd_rr, asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(x[k]) : "f"(z[k])))
// accumulate pattern of the H path: acc += a*b with a, b changing registers
KERNEL_SCALAR(ffma_acc, asm volatile("fma.rn.f32 %0, %1, %2, %0;" : "+f"(x[k]) : "f"(y[k]), "f"(z[(k + 1) % CH])))

#define KERNEL_PACKED(name, ASM)                                                   \
  __global__ void name(float* out, float c) {                                      \
    unsigned long long x[CH], y[CH], z[CH];                                        \
    for (int k = 0; k < CH; ++k) {                                                 \
      float2 a = make_float2(threadIdx.x * 1e-3f + k, k + 0.5f);                   \
      float2 b = make_float2(1.0f + 1e-7f * k, 1.0f - 1e-7f * k);                  \
      float2 d = make_float2(1e-6f * k * threadIdx.x, c);                          \
      x[k] = *reinterpret_cast<unsigned long long*>(&a);                           \
      y[k] = *reinterpret_cast<unsigned long long*>(&b);                           \
      z[k] = *reinterpret_cast<unsigned long long*>(&d);                           \
    }                                                                              \
    for (int it = 0; it < ITERS; ++it) {                                           \
      _Pragma("unroll") for (int k = 0; k < CH; ++k) { ASM; }                      \
    }                                                                              \
    float s = 0.f;                                                                 \
    for (int k = 0; k < CH; ++k) {                                                 \
      float2 v = *reinterpret_cast<float2*>(&x[k]); s += v.x + v.y;                \
    }                                                                              \
    if (s == 1234.5f) out[0] = s;                                                  \
  }

KERNEL_PACKED(ffma2_rrr, asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[k]) : "l"(y[k]), "l"(z[k])))
KERNEL_PACKED(fmul2_rr, asm volatile("mul.rn.f32x2 %0, %0, %1;" : "+l"(x[k]) : "l"(y[k])))
KERNEL_PACKED(fadd2_rr, asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(x[k]) : "l"(z[k])))

// half scalar FFMA (rrr), half FFMA2 (rrr), interleaved
__global__ void mix_ffma_ffma2(float* out, float c) {
  float x[CH], y[CH], z[CH];
  unsigned long long X[CH], Y[CH], Z[CH];
  for (int k = 0; k < CH; ++k) {
    x[k] = threadIdx.x * 1e-3f + k; y[k] = 1.0f + 1e-7f * k; z[k] = 1e-6f * k * threadIdx.x;
    float2 a = make_float2(x[k], k + 0.5f), b = make_float2(y[k], y[k]), d = make_float2(z[k], c);
    X[k] = *reinterpret_cast<unsigned long long*>(&a);
    Y[k] = *reinterpret_cast<unsigned long long*>(&b);
    Z[k] = *reinterpret_cast<unsigned long long*>(&d);
  }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int k = 0; k < CH; ++k) {
      asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[k]) : "f"(y[k]), "f"(z[k]));
      asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(X[k]) : "l"(Y[k]), "l"(Z[k]));
    }
  }
  float s = 0.f;
  for (int k = 0; k < CH; ++k) {
    float2 v = *reinterpret_cast<float2*>(&X[k]);
    s += x[k] + v.x + v.y;
  }
  if (s == 1234.5f) out[0] = s;
}

// scalar FFMA (rrr) interleaved with an ALU op (IADD3) — does the ALU pipe dual-issue?
__global__ void mix_ffma_iadd(float* out, float c) {
  float x[CH], y[CH], z[CH];
  unsigned int u[CH];
  for (int k = 0; k < CH; ++k) {
    x[k] = threadIdx.x * 1e-3f + k; y[k] = 1.0f + 1e-7f * k; z[k] = 1e-6f * k * threadIdx.x;
    u[k] = threadIdx.x * 7 + k;
  }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int k = 0; k < CH; ++k) {
      asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[k]) : "f"(y[k]), "f"(z[k]));
      asm volatile("add.u32 %0, %0, %1;" : "+r"(u[k]) : "r"(u[(k + 3) % CH]));
    }
  }
  float s = 0.f;
  for (int k = 0; k < CH; ++k) s += x[k] + (float)u[k];
  if (s == 1234.5f) out[0] = s + c;
}

int main() {
  int sms = 0, clk_khz = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
  float* out;
  CK(cudaMalloc(&out, 16));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  struct K { const char* name; void (*fn)(float*, float); int ops_per_chain; int flops_per_op; };
  K ks[] = {
      {"ffma_rrr", ffma_rrr, 1, 2},   {"ffma_rrc", ffma_rrc, 1, 2}, {"ffma_rri", ffma_rri, 1, 2},
      {"fmul_rr", fmul_rr, 1, 1},     {"fadd_rr", fadd_rr, 1, 1},   {"ffma_acc", ffma_acc, 1, 2},
      {"ffma2_rrr", ffma2_rrr, 1, 4}, {"fmul2_rr", fmul2_rr, 1, 2}, {"fadd2_rr", fadd2_rr, 1, 2},
      {"mix_ffma_ffma2", mix_ffma_ffma2, 2, 3}, {"mix_ffma_iadd", mix_ffma_iadd, 2, 1},
  };
  const int threads = 256, blocks = sms * 4;  // 32 warps per SM
  printf("{\"sms\": %d, \"clock_mhz_attr\": %.0f, \"results\": [\n", sms, clk_khz / 1e3);
  for (size_t i = 0; i < sizeof(ks) / sizeof(ks[0]); ++i) {
    for (int rep = 0; rep < 2; ++rep) ks[i].fn<<<blocks, threads>>>(out, 1.0f);
    CK(cudaEventRecord(a));
    const int reps = 5;
    for (int rep = 0; rep < reps; ++rep) ks[i].fn<<<blocks, threads>>>(out, 1.0f);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, a, b));
    const double warp_instr = (double)reps * blocks * (threads / 32) * ITERS * CH * ks[i].ops_per_chain;
    const double smsp_cycles_at_1965 = ms * 1e-3 * 1.965e9 * sms * 4;
    const double flops = (double)reps * blocks * threads * ITERS * CH * ks[i].flops_per_op;
    printf("  {\"kernel\": \"%s\", \"ms\": %.4f, \"warp_instr_per_smsp_cycle_at_1965\": %.3f, "
           "\"tflops\": %.2f}%s\n", ks[i].name, ms / reps, warp_instr / smsp_cycles_at_1965,
           flops / (ms * 1e-3) / 1e12, i + 1 < sizeof(ks) / sizeof(ks[0]) ? "," : "");
  }
  printf("]}\n");
  return 0;
}
