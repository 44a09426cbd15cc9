// weights.cu — a5: importance weights (Eq.11) as a max-subtracted log-sum-exp in
// fp64 (R22); a6: dead-particle pruning + respawn (R17-R21); a7: representative
// (P:206).
//
//   m = max L (from a3), e_i = exp(L_i - m), S = sum e (fixed tree), w_i = e_i / S
//   dead_i = (l_i - max l < rel_floor) or (w_i < posterior_floor)            (R17)
//   survivors' rungs q_i = floor(e_i 2^32), dead rungs 0; C = inclusive scan (exact uint64)
//   n(c) = clamp(ceil((c D 2^32 - U Q) / (Q 2^32)), 0, D)  in signed 128-bit  (R18)
//   the r-th dead slot (ascending) takes donor min{j : n(C_j) > r}
//   clone T_t, every T_k and L (R19, R20); re-normalise; representative = argmax w, ties low.
#include <cub/cub.cuh>

#include "mcs_internal.cuh"
#include "reduce.cuh"

namespace mcs {

struct Rung {
  unsigned long long C;
  unsigned int d;
  unsigned int pad;
};
struct RungSum {
  __host__ __device__ Rung operator()(const Rung& a, const Rung& b) const {
    Rung r;
    r.C = a.C + b.C;
    r.d = a.d + b.d;
    r.pad = 0;
    return r;
  }
};

constexpr int kWT = 256;

__global__ void __launch_bounds__(kWT) exp_sum_kernel(const double* __restrict__ L, int N,
                                                      const double* __restrict__ m_ptr,
                                                      double* __restrict__ e,
                                                      double* __restrict__ partials,
                                                      double* __restrict__ S_out,
                                                      unsigned int* counter) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const double m = *m_ptr;
  double v = 0.0;
  if (i < N) {
    v = exp(L[i] - m);
    e[i] = v;
  }
  const double bs = block_reduce(v, SumOp(), 0.0);
  if (threadIdx.x == 0) partials[blockIdx.x] = bs;
  if (last_block(counter)) {
    double s = 0.0;
    for (int k = threadIdx.x; k < (int)gridDim.x; k += blockDim.x) s += partials[k];
    s = block_reduce(s, SumOp(), 0.0);
    if (threadIdx.x == 0) *S_out = s;
  }
}

__global__ void dead_kernel(const double* __restrict__ e, const double* __restrict__ l, int N,
                            const Scalars* __restrict__ sc, double rel_floor, double post_floor,
                            double* __restrict__ w, uint8_t* __restrict__ flags,
                            Rung* __restrict__ rung) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const double wi = e[i] / sc->S;
  w[i] = wi;
  const bool dead = (l[i] - sc->lstar < rel_floor) || (wi < post_floor);
  if (dead) flags[i] |= 8;
  Rung r;
  r.C = dead ? 0ull : (unsigned long long)floor(e[i] * 4294967296.0);
  r.d = dead ? 1u : 0u;
  r.pad = 0;
  rung[i] = r;
}

__global__ void rung_from_inputs_kernel(const double* __restrict__ e,
                                        const uint8_t* __restrict__ dead, int N,
                                        Rung* __restrict__ rung) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  Rung r;
  r.C = dead[i] ? 0ull : (unsigned long long)floor(e[i] * 4294967296.0);
  r.d = dead[i] ? 1u : 0u;
  r.pad = 0;
  rung[i] = r;
}

__global__ void totals_kernel(const Rung* __restrict__ scan, int N, Scalars* sc) {
  const Rung last = scan[N - 1];
  sc->Q = last.C;
  sc->D = (long long)last.d;
  sc->status = (last.d > 0 && last.C == 0ull) ? (int)MCS_E_DEGENERATE : 0;
}

__device__ __forceinline__ long long draws_below(unsigned long long c, long long D,
                                                 unsigned long long Q, unsigned int U) {
  const __int128 num = (__int128)c * (__int128)D * ((__int128)1 << 32) - (__int128)U * (__int128)Q;
  const __int128 den = (__int128)Q * ((__int128)1 << 32);
  __int128 q = num / den;
  if (num > 0 && q * den != num) q += 1;  // ceil for den > 0
  if (q < 0) q = 0;
  if (q > D) q = D;
  return (long long)q;
}

__global__ void ncum_kernel(const Rung* __restrict__ scan, int N, const Scalars* __restrict__ sc,
                            unsigned int U, long long* __restrict__ ncum) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  if (sc->D == 0 || sc->Q == 0) return;
  ncum[i] = draws_below(scan[i].C, sc->D, sc->Q, U);
}

__global__ void assign_kernel(const Rung* __restrict__ rung, const Rung* __restrict__ scan, int N,
                              const Scalars* __restrict__ sc,
                              const long long* __restrict__ ncum, int32_t* __restrict__ donor) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  if (!rung[i].d || sc->D == 0 || sc->Q == 0) {
    donor[i] = -1;
    return;
  }
  const long long r = (long long)scan[i].d - 1;  // rank among dead slots (ascending)
  int lo = 0, hi = N - 1;                        // first j with ncum[j] > r
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (ncum[mid] > r) hi = mid; else lo = mid + 1;
  }
  donor[i] = lo;
}

__global__ void clone_kernel(const int32_t* __restrict__ donor, int N, int K, int capK, int capN,
                             float* __restrict__ pose, float* __restrict__ kfpose,
                             double* __restrict__ L) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int KK = K + 1;
  if (t >= (long long)N * KK) return;
  const int i = (int)(t / KK), k = (int)(t - (long long)i * KK);
  const int d = donor[i];
  if (d < 0) return;
  if (k == K) {
#pragma unroll
    for (int e = 0; e < 12; ++e) pose[(size_t)e * capN + i] = pose[(size_t)e * capN + d];
    L[i] = L[d];
  } else {
    const float4* src = reinterpret_cast<const float4*>(kfpose + ((size_t)d * capK + k) * 12);
    float4* dst = reinterpret_cast<float4*>(kfpose + ((size_t)i * capK + k) * 12);
    dst[0] = src[0];
    dst[1] = src[1];
    dst[2] = src[2];
  }
}

__global__ void __launch_bounds__(kWT) max_kernel(const double* __restrict__ L, int N,
                                                  double* __restrict__ partials,
                                                  double* __restrict__ out,
                                                  unsigned int* counter) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const double v = i < N ? L[i] : -INFINITY;
  const double bm = block_reduce(v, MaxOp(), -INFINITY);
  if (threadIdx.x == 0) partials[blockIdx.x] = bm;
  if (last_block(counter)) {
    double m = -INFINITY;
    for (int k = threadIdx.x; k < (int)gridDim.x; k += blockDim.x) m = fmax(m, partials[k]);
    m = block_reduce(m, MaxOp(), -INFINITY);
    if (threadIdx.x == 0) *out = m;
  }
}

// argmax with ties -> lowest index, on (value, index) pairs
__device__ __forceinline__ void better(double& w, int& i, double w2, int i2) {
  if (w2 > w || (w2 == w && i2 < i)) { w = w2; i = i2; }
}

__device__ void block_argmax(double& w, int& idx) {
  __shared__ double sw[32];
  __shared__ int si[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double w2 = __shfl_xor_sync(0xffffffffu, w, o);
    const int i2 = __shfl_xor_sync(0xffffffffu, idx, o);
    better(w, idx, w2, i2);
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) { sw[wid] = w; si[wid] = idx; }
  __syncthreads();
  const int nw = blockDim.x >> 5;
  w = lane < nw ? sw[lane] : -INFINITY;
  idx = lane < nw ? si[lane] : 0x7fffffff;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double w2 = __shfl_xor_sync(0xffffffffu, w, o);
    const int i2 = __shfl_xor_sync(0xffffffffu, idx, o);
    better(w, idx, w2, i2);
  }
}

__global__ void __launch_bounds__(kWT) weight_argmax_kernel(const double* __restrict__ e, int N,
                                                            const double* __restrict__ S_ptr,
                                                            double* __restrict__ w,
                                                            double* __restrict__ pw,
                                                            int32_t* __restrict__ pi,
                                                            Scalars* sc, int base_index,
                                                            unsigned int* counter) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  double wi = -INFINITY;
  int idx = 0x7fffffff;
  if (i < N) {
    wi = e[i] / *S_ptr;
    w[i] = wi;
    idx = i;
  }
  block_argmax(wi, idx);
  if (threadIdx.x == 0) { pw[blockIdx.x] = wi; pi[blockIdx.x] = idx; }
  if (last_block(counter)) {
    double bw = -INFINITY;
    int bi = 0x7fffffff;
    for (int k = threadIdx.x; k < (int)gridDim.x; k += blockDim.x) better(bw, bi, pw[k], pi[k]);
    block_argmax(bw, bi);
    if (threadIdx.x == 0) {
      sc->rep = base_index + bi;
      sc->wbest = bw;
    }
  }
}

size_t cub_temp_needed(int n) {
  size_t b = 0;
  cub::DeviceScan::InclusiveScan(nullptr, b, (Rung*)nullptr, (Rung*)nullptr, RungSum(), n);
  return b;
}

static void ladder_and_assign(mcs_ctx* c, Rung* rung, int N, uint32_t U, int32_t* donor) {
  cudaStream_t st = c->stream;
  Rung* scan = reinterpret_cast<Rung*>(c->d_ladder_scan);
  size_t tb = c->cub_temp_bytes;
  cub::DeviceScan::InclusiveScan(c->d_cub_temp, tb, rung, scan, RungSum(), N, st);
  const int g = (N + kWT - 1) / kWT;
  totals_kernel<<<1, 1, 0, st>>>(scan, N, c->d_scal);
  ncum_kernel<<<g, kWT, 0, st>>>(scan, N, c->d_scal, U, c->d_ncum);
  assign_kernel<<<g, kWT, 0, st>>>(rung, scan, N, c->d_scal, c->d_ncum, donor);
}

void launch_weights_resample(mcs_ctx* c, uint32_t U) {
  cudaStream_t st = c->stream;
  const int N = c->N;
  const int g = (N + kWT - 1) / kWT;
  Scalars* sc = c->d_scal;
  double* p0 = c->d_partials;
  // a5: e = exp(L - m), S   (m, l* reduced by a3)
  exp_sum_kernel<<<g, kWT, 0, st>>>(c->d_L, N, &sc->m, c->d_e, p0, &sc->S, &sc->counter[1]);
  // a6: dead set, ladder, counts, donors, clones
  Rung* rung = reinterpret_cast<Rung*>(c->d_ladder);
  dead_kernel<<<g, kWT, 0, st>>>(c->d_e, c->d_l, N, sc, c->cfg.loglik_rel_floor,
                                 c->cfg.posterior_floor, c->d_w, c->d_flags, rung);
  ladder_and_assign(c, rung, N, U, c->d_donor);
  const long long tot = (long long)N * (c->K + 1);
  clone_kernel<<<(int)((tot + 255) / 256), 256, 0, st>>>(c->d_donor, N, c->K, c->capK, c->capN,
                                                         c->d_pose, c->d_kfpose, c->d_L);
  // re-normalise on the new L, then a7
  max_kernel<<<g, kWT, 0, st>>>(c->d_L, N, p0, &sc->m2, &sc->counter[2]);
  exp_sum_kernel<<<g, kWT, 0, st>>>(c->d_L, N, &sc->m2, c->d_e, p0, &sc->S2, &sc->counter[3]);
  weight_argmax_kernel<<<g, kWT, 0, st>>>(c->d_e, N, &sc->S2, c->d_w, p0, c->d_ipartials, sc,
                                          c->cfg.rank * 0, &sc->counter[4]);
}

void launch_resample_only(mcs_ctx* c, const double* d_e, const uint8_t* d_dead, int n,
                          uint32_t U, int32_t* d_donor) {
  Rung* rung = reinterpret_cast<Rung*>(c->d_ladder);
  rung_from_inputs_kernel<<<(n + kWT - 1) / kWT, kWT, 0, c->stream>>>(d_e, d_dead, n, rung);
  ladder_and_assign(c, rung, n, U, d_donor);
}

}  // namespace mcs
