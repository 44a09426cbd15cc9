// sweep.cu — a2 ★: the fused transform -> hash lookup -> residual -> reduce sweep
// (Eqs.2-4; Eq.6).
//
// One thread per (particle, neighbour slot) work item; the whole CTA walks the scan in
// lock-step, so every lane of a warp reads the SAME scan point from shared memory (a
// broadcast, no bank conflicts) while probing its own keyframe table.  Per point j:
//   q = kT mu_j            pinned fp32 key path (R27) -> cell = floorf(q / r) -> probe
//   unmatched -> skip (R8)
//   e = mu' - q            C = Sigma' + R Sigma_j R^T      Omega = C^-1 (cofactors)
//   l -= e^T Omega e       n += 1
//   H~ += K^T Omega K,  b~ += K^T Omega e,   K = [-I, [m]x],  m = R mu_j
// K is the Jacobian in the rotated frame: J = de/d(delta) = [-R, R[mu]x] = K blockdiag(R, R)
// (R2), so the per-slot rotation back to the body frame happens once in a3, not per point.
// Accumulators are fp32 registers in a fixed point order: bitwise reproducible.
#include "mcs_internal.cuh"

namespace mcs {

constexpr int kSweepThreads = 128;
constexpr int kChunk = 256;  // scan points per shared-memory stage (12 KB)

__device__ __forceinline__ int probe(const unsigned long long* __restrict__ keys, uint32_t shift,
                                     uint32_t mask, unsigned long long key) {
  uint32_t h = (uint32_t)((key * kHashMul) >> shift);
  while (true) {
    unsigned long long k = __ldg(keys + h);
    if (k == key) return (int)h;
    if (k == kEmptyKey) return -1;
    h = (h + 1) & mask;
  }
}

__global__ void __launch_bounds__(kSweepThreads)
    sweep_kernel(const float4* __restrict__ items, const int32_t* __restrict__ order,
                 int n_items, const float4* __restrict__ scan, int S,
                 const KfMeta* __restrict__ kmeta, float inv_r, float* __restrict__ part) {
  __shared__ float4 s_pt[kChunk * 3];
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int item = t < n_items ? order[t] : -1;
  float4 r0 = make_float4(0, 0, 0, 0), r1 = r0, r2 = r0, inf = r0;
  if (item >= 0) {
    r0 = items[4 * (size_t)item + 0];
    r1 = items[4 * (size_t)item + 1];
    r2 = items[4 * (size_t)item + 2];
    inf = items[4 * (size_t)item + 3];
  }
  const int kf = item >= 0 ? __float_as_int(inf.x) : -1;
  const bool active = kf >= 0;
  const bool hb = active && (__float_as_int(inf.z) & 1);
  const unsigned long long* keys = nullptr;
  const float4* pay = nullptr;
  uint32_t shift = 0, mask = 0;
  if (active) {
    keys = kmeta[kf].keys;
    pay = kmeta[kf].payload;
    shift = kmeta[kf].shift;
    mask = kmeta[kf].mask;
  }
  const float R00 = r0.x, R01 = r0.y, R02 = r0.z, tx = r0.w;
  const float R10 = r1.x, R11 = r1.y, R12 = r1.z, ty = r1.w;
  const float R20 = r2.x, R21 = r2.y, R22 = r2.z, tz = r2.w;

  float l = 0.f;
  int n = 0;
  float h[21];
  float bv[6];
#pragma unroll
  for (int k = 0; k < 21; ++k) h[k] = 0.f;
#pragma unroll
  for (int k = 0; k < 6; ++k) bv[k] = 0.f;

  for (int base = 0; base < S; base += kChunk) {
    const int cnt = min(kChunk, S - base);
    __syncthreads();
    for (int k = threadIdx.x; k < cnt * 3; k += kSweepThreads) s_pt[k] = scan[3 * base + k];
    __syncthreads();
    if (!active) continue;
    for (int j = 0; j < cnt; ++j) {
      const float4 A = s_pt[3 * j + 0];
      // pinned fp32 key path (R27)
      const float qx = __fmaf_rn(R02, A.z, __fmaf_rn(R01, A.y, __fmaf_rn(R00, A.x, tx)));
      const float qy = __fmaf_rn(R12, A.z, __fmaf_rn(R11, A.y, __fmaf_rn(R10, A.x, ty)));
      const float qz = __fmaf_rn(R22, A.z, __fmaf_rn(R21, A.y, __fmaf_rn(R20, A.x, tz)));
      const float fx = floorf(__fmul_rn(qx, inv_r));
      const float fy = floorf(__fmul_rn(qy, inv_r));
      const float fz = floorf(__fmul_rn(qz, inv_r));
      if (!(fx >= (float)kCellMin && fx <= (float)kCellMax && fy >= (float)kCellMin &&
            fy <= (float)kCellMax && fz >= (float)kCellMin && fz <= (float)kCellMax))
        continue;
      const int slot = probe(keys, shift, mask, pack_cell((int)fx, (int)fy, (int)fz));
      if (slot < 0) continue;  // unmatched: skipped
      const float4 P0 = __ldg(pay + 3 * slot + 0);
      const float4 P1 = __ldg(pay + 3 * slot + 1);
      const float4 P2 = __ldg(pay + 3 * slot + 2);
      const float4 B = s_pt[3 * j + 1];
      const float4 Cc = s_pt[3 * j + 2];
      // e = mu' - kT mu   (Eq.4)
      const float ex = P0.x - qx, ey = P0.y - qy, ez = P0.z - qz;
      // m = R mu (rotated scan point)
      const float mx = R00 * A.x + R01 * A.y + R02 * A.z;
      const float my = R10 * A.x + R11 * A.y + R12 * A.z;
      const float mz = R20 * A.x + R21 * A.y + R22 * A.z;
      // C = Sigma' + R Sigma R^T  (Eq.4)
      const float s00 = A.w, s01 = B.x, s02 = B.y, s11 = B.z, s12 = B.w, s22 = Cc.x;
      const float a00 = R00 * s00 + R01 * s01 + R02 * s02;
      const float a01 = R00 * s01 + R01 * s11 + R02 * s12;
      const float a02 = R00 * s02 + R01 * s12 + R02 * s22;
      const float a10 = R10 * s00 + R11 * s01 + R12 * s02;
      const float a11 = R10 * s01 + R11 * s11 + R12 * s12;
      const float a12 = R10 * s02 + R11 * s12 + R12 * s22;
      const float a20 = R20 * s00 + R21 * s01 + R22 * s02;
      const float a21 = R20 * s01 + R21 * s11 + R22 * s12;
      const float a22 = R20 * s02 + R21 * s12 + R22 * s22;
      const float c00 = P0.w + a00 * R00 + a01 * R01 + a02 * R02;
      const float c01 = P1.x + a00 * R10 + a01 * R11 + a02 * R12;
      const float c02 = P1.y + a00 * R20 + a01 * R21 + a02 * R22;
      const float c11 = P1.z + a10 * R10 + a11 * R11 + a12 * R12;
      const float c12 = P1.w + a10 * R20 + a11 * R21 + a12 * R22;
      const float c22 = P2.x + a20 * R20 + a21 * R21 + a22 * R22;
      // Omega = C^-1 by cofactors
      const float k00 = c11 * c22 - c12 * c12;
      const float k01 = c02 * c12 - c01 * c22;
      const float k02 = c01 * c12 - c02 * c11;
      const float k11 = c00 * c22 - c02 * c02;
      const float k12 = c01 * c02 - c00 * c12;
      const float k22 = c00 * c11 - c01 * c01;
      const float det = c00 * k00 + c01 * k01 + c02 * k02;
      const float id = __frcp_rn(det);
      const float o00 = k00 * id, o01 = k01 * id, o02 = k02 * id;
      const float o11 = k11 * id, o12 = k12 * id, o22 = k22 * id;
      // w = Omega e ; l -= e^T Omega e  (Eq.3)
      const float w0 = o00 * ex + o01 * ey + o02 * ez;
      const float w1 = o01 * ex + o11 * ey + o12 * ez;
      const float w2 = o02 * ex + o12 * ey + o22 * ez;
      l -= ex * w0 + ey * w1 + ez * w2;
      ++n;
      if (hb) {
        // H~ = K^T Omega K = [[Omega, -Omega M], [-M^T Omega, M^T Omega M]], M = [m]x
        // P = Omega M
        const float p00 = o01 * mz - o02 * my, p01 = o02 * mx - o00 * mz, p02 = o00 * my - o01 * mx;
        const float p10 = o11 * mz - o12 * my, p11 = o12 * mx - o01 * mz, p12 = o01 * my - o11 * mx;
        const float p20 = o12 * mz - o22 * my, p21 = o22 * mx - o02 * mz, p22 = o02 * my - o12 * mx;
        h[0] += o00; h[1] += o01; h[2] += o02;
        h[3] -= p00; h[4] -= p01; h[5] -= p02;
        h[6] += o11; h[7] += o12;
        h[8] -= p10; h[9] -= p11; h[10] -= p12;
        h[11] += o22;
        h[12] -= p20; h[13] -= p21; h[14] -= p22;
        // M^T Omega M = -M P:  (M P)[0][b] = -mz P1b + my P2b, [1][b] = mz P0b - mx P2b,
        //                       [2][b] = -my P0b + mx P1b
        h[15] += mz * p10 - my * p20;  // (3,3)
        h[16] += mz * p11 - my * p21;  // (3,4)
        h[17] += mz * p12 - my * p22;  // (3,5)
        h[18] += mx * p21 - mz * p01;  // (4,4)
        h[19] += mx * p22 - mz * p02;  // (4,5)
        h[20] += my * p02 - mx * p12;  // (5,5)
        // b~ = K^T Omega e = [-w ; w x m]
        bv[0] -= w0; bv[1] -= w1; bv[2] -= w2;
        bv[3] += w1 * mz - w2 * my;
        bv[4] += w2 * mx - w0 * mz;
        bv[5] += w0 * my - w1 * mx;
      }
    }
  }
  if (!active || item < 0) return;
  float4* o = reinterpret_cast<float4*>(part + (size_t)item * kSlotFloats);
  o[0] = make_float4(l, __int_as_float(n), h[0], h[1]);
  o[1] = make_float4(h[2], h[3], h[4], h[5]);
  o[2] = make_float4(h[6], h[7], h[8], h[9]);
  o[3] = make_float4(h[10], h[11], h[12], h[13]);
  o[4] = make_float4(h[14], h[15], h[16], h[17]);
  o[5] = make_float4(h[18], h[19], h[20], bv[0]);
  o[6] = make_float4(bv[1], bv[2], bv[3], bv[4]);
  o[7] = make_float4(bv[5], 0.f, 0.f, 0.f);
}

void launch_sweep(mcs_ctx* c, int S) {
  const int n_items = c->cfg.neighbor_count * c->N;
  const int grid = (n_items + kSweepThreads - 1) / kSweepThreads;
  sweep_kernel<<<grid, kSweepThreads, 0, c->stream>>>(c->d_items, c->d_order, n_items, c->d_scan,
                                                      S, c->d_kf_meta,
                                                      1.0f / c->cfg.voxel_resolution, c->d_part);
}

}  // namespace mcs
