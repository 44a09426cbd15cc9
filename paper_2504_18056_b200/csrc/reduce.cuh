// reduce.cuh — deterministic block reductions and the "last block finishes" pattern.
// Every reduction tree is fixed by the launch shape, so results are bitwise reproducible
// (no float atomics on any result path).
#pragma once
#include <cuda_runtime.h>

namespace mcs {

template <typename T, typename Op>
__device__ __forceinline__ T warp_reduce(T v, Op op) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

template <typename T>
struct NoDeduce { using type = T; };

// block-wide reduction; result valid in every thread.  blockDim.x multiple of 32, <= 1024.
template <typename T, typename Op>
__device__ T block_reduce(T v, Op op, typename NoDeduce<T>::type ident) {
  __shared__ T sh[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_reduce(v, op);
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  const int nw = blockDim.x >> 5;
  T x = (lane < nw) ? sh[lane] : ident;
  x = warp_reduce(x, op);
  return x;
}

// Returns true in every thread of the last block to arrive; resets the counter.
__device__ __forceinline__ bool last_block(unsigned int* counter) {
  __shared__ bool am_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int v = atomicAdd(counter, 1u);
    am_last = (v == gridDim.x - 1);
    if (am_last) *counter = 0u;
  }
  __syncthreads();
  if (am_last) __threadfence();
  return am_last;
}

struct MaxOp {
  template <typename T>
  __device__ __forceinline__ T operator()(T a, T b) const { return a > b ? a : b; }
};
struct SumOp {
  template <typename T>
  __device__ __forceinline__ T operator()(T a, T b) const { return a + b; }
};

}  // namespace mcs
