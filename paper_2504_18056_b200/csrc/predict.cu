// predict.cu — NEXT rows of SURVEY §8(f): the prediction step (Eq.1, with the elevator
// heuristic's vertical random walk) and the keyframe-insertion overlap test.
//
// Prediction, one thread per particle (global index g):
//   z = 8 standard normals: Philox4x32-10 (key = seed, counter = (block, g, frame)) -> uniforms
//       u = (x + 1) 2^-32 in (0, 1] -> fp64 Box-Muller (R31)
//   delta = chol(cov) z[0:6];  T <- round_fp32( Newton( T dT exp(delta) ) );  t_z += sigma_v z[6]
// Overlap, one thread per scan point: the pinned fp32 key path of the sweep (R27) under the
// odometry relative pose, then one table lookup; an integer count (deterministic).
#include "mcs_internal.cuh"
#include "reduce.cuh"
#include "se3.cuh"

namespace mcs {

__device__ __forceinline__ void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c[0]), lo0 = 0xD2511F53u * c[0];
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c[2]), lo1 = 0xCD9E8D57u * c[2];
    const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

__global__ void predict_kernel(float* __restrict__ pose, int capN, int N, long long gbase,
                               const double* __restrict__ dT, const double* __restrict__ Lc,
                               unsigned long long seed, unsigned long long frame, double vsig) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const long long g = gbase + i;
  uint32_t x[8];
#pragma unroll
  for (int b = 0; b < 2; ++b) {
    uint32_t c[4] = {(uint32_t)b, (uint32_t)g, (uint32_t)frame, (uint32_t)(frame >> 32)};
    philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
#pragma unroll
    for (int k = 0; k < 4; ++k) x[4 * b + k] = c[k];
  }
  double z[8];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const double u1 = ((double)x[2 * k] + 1.0) * 0x1.0p-32;
    const double u2 = ((double)x[2 * k + 1] + 1.0) * 0x1.0p-32;
    const double rr = sqrt(-2.0 * log(u1));
    double sn, cs;
    sincos(2.0 * M_PI * u2, &sn, &cs);
    z[2 * k] = rr * cs;
    z[2 * k + 1] = rr * sn;
  }
  double delta[6];
#pragma unroll
  for (int a = 0; a < 6; ++a) {
    double s = 0.0;
#pragma unroll
    for (int b = 0; b <= a; ++b) s += Lc[6 * a + b] * z[b];
    delta[a] = s;
  }
  double T[12], TdT[12], E[12], TE[12];
#pragma unroll
  for (int e = 0; e < 12; ++e) T[e] = (double)pose[(size_t)e * capN + i];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      double s = (b == 3) ? T[4 * a + 3] : 0.0;
#pragma unroll
      for (int c = 0; c < 3; ++c) s += T[4 * a + c] * dT[4 * c + b];
      TdT[4 * a + b] = s;
    }
  se3_exp_d(delta, E);
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      double s = (b == 3) ? TdT[4 * a + 3] : 0.0;
#pragma unroll
      for (int c = 0; c < 3; ++c) s += TdT[4 * a + c] * E[4 * c + b];
      TE[4 * a + b] = s;
    }
  double RtR[9];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      double s = 0.0;
#pragma unroll
      for (int c = 0; c < 3; ++c) s += TE[4 * c + a] * TE[4 * c + b];
      RtR[3 * a + b] = s;
    }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      double s = 0.0;
#pragma unroll
      for (int c = 0; c < 3; ++c) s += TE[4 * a + c] * (((c == b) ? 3.0 : 0.0) - RtR[3 * c + b]);
      pose[(size_t)(4 * a + b) * capN + i] = (float)(0.5 * s);
    }
    double ta = TE[4 * a + 3];
    if (a == 2) ta += vsig * z[6];  // elevator heuristic: world-frame vertical walk
    pose[(size_t)(4 * a + 3) * capN + i] = (float)ta;
  }
}

// 6x6 Cholesky of the odometry twist covariance (one thread; all-zero -> zero factor)
__global__ void chol6_kernel(const double* __restrict__ cov, double* __restrict__ Lc,
                             int* __restrict__ bad) {
  bool zero = true;
  for (int k = 0; k < 36; ++k) zero = zero && cov[k] == 0.0;
  for (int k = 0; k < 36; ++k) Lc[k] = 0.0;
  if (zero) return;
  for (int j = 0; j < 6; ++j) {
    double d = cov[6 * j + j];
    for (int k = 0; k < j; ++k) d -= Lc[6 * j + k] * Lc[6 * j + k];
    if (!(d > 0.0)) { *bad = 1; return; }
    Lc[6 * j + j] = sqrt(d);
    for (int r = j + 1; r < 6; ++r) {
      double s = cov[6 * r + j];
      for (int k = 0; k < j; ++k) s -= Lc[6 * r + k] * Lc[6 * j + k];
      Lc[6 * r + j] = s / Lc[6 * j + j];
    }
  }
}

// inputs staged in d_buf: [0..12) dT (fp64), [12..48) cov, [48..84) chol factor
mcs_status launch_predict(mcs_ctx* c, double* d_buf, int* d_bad, unsigned long long seed,
                          unsigned long long frame, double vsig) {
  chol6_kernel<<<1, 1, 0, c->stream>>>(d_buf + 12, d_buf + 48, d_bad);
  int bad = 0;
  if (cudaMemcpyAsync(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, c->stream) != cudaSuccess ||
      cudaStreamSynchronize(c->stream) != cudaSuccess)
    return MCS_E_CUDA;
  if (bad) return MCS_E_INVALID_ARG;
  if (c->N > 0)
    predict_kernel<<<(c->N + 127) / 128, 128, 0, c->stream>>>(c->d_pose, c->capN, c->N, c->gbase,
                                                              d_buf, d_buf + 48, seed, frame, vsig);
  return cudaGetLastError() == cudaSuccess ? MCS_OK : MCS_E_CUDA;
}

__global__ void overlap_kernel(const float* __restrict__ mean3, int S, const float* __restrict__ rel,
                               const KfMeta* __restrict__ kmeta, int kf, float inv_r,
                               unsigned long long* __restrict__ count) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  int hit = 0;
  if (j < S) {
    const KfMeta m = kmeta[kf];
    const float mx = mean3[3 * j], my = mean3[3 * j + 1], mz = mean3[3 * j + 2];
    float q[3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
      q[a] = __fmaf_rn(rel[4 * a + 2], mz,
                       __fmaf_rn(rel[4 * a + 1], my, __fmaf_rn(rel[4 * a + 0], mx, rel[4 * a + 3])));
    const unsigned int dx = (unsigned)(__float2int_rd(__fmul_rn(q[0], inv_r)) - m.ox);
    const unsigned int dy = (unsigned)(__float2int_rd(__fmul_rn(q[1], inv_r)) - m.oy);
    const unsigned int dz = (unsigned)(__float2int_rd(__fmul_rn(q[2], inv_r)) - m.oz);
    if (dx < m.ex && dy < m.ey && dz < m.ez) {
      const unsigned int key = local_key(dx, dy, dz);
      unsigned int h = slot_hash(key, m.shift) & m.mask;
      while (true) {
        const unsigned int k = __float_as_uint(m.slots[4 * (size_t)h].x);
        if (k == key) { hit = 1; break; }
        if (k == kEmptyKey32) break;
        h = (h + 1) & m.mask;
      }
    }
  }
  const int bs = block_reduce(hit, SumOp(), 0);
  if (threadIdx.x == 0 && bs) atomicAdd(count, (unsigned long long)bs);
}

mcs_status launch_overlap(mcs_ctx* c, const float* d_mean3, int S, const float* d_rel, int kf,
                          unsigned long long* d_count, unsigned long long* h_count) {
  if (cudaMemsetAsync(d_count, 0, sizeof(unsigned long long), c->stream) != cudaSuccess)
    return MCS_E_CUDA;
  overlap_kernel<<<(S + 255) / 256, 256, 0, c->stream>>>(d_mean3, S, d_rel, c->d_kf_meta, kf,
                                                         1.0f / c->cfg.voxel_resolution, d_count);
  if (cudaMemcpyAsync(h_count, d_count, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                      c->stream) != cudaSuccess ||
      cudaStreamSynchronize(c->stream) != cudaSuccess)
    return MCS_E_CUDA;
  return MCS_OK;
}

}  // namespace mcs
