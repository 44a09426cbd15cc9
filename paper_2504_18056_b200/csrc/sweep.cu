// sweep.cu — a2 ★: the fused transform -> hash lookup -> residual -> reduce sweep
// (Eqs.2-4; Eq.6).
//
// One thread per (particle, neighbour slot) work item; items are sorted by a pose-coherence
// key in a1, and the whole CTA walks the scan in lock-step, so every lane of a warp reads the
// SAME scan point from shared memory (a broadcast) and lanes with similar poses probe the same
// table slots (coalesced gathers).  Per point j:
//   q = kT mu_j            pinned fp32 key path (R27) -> cell = floor(q / r) -> bbox-local key
//   unmatched -> skip (R8)
//   e = mu' - q            C = Sigma' + R Sigma_j R^T      Omega = C^-1 (adjugate / det)
//   l -= e^T Omega e       n += 1
//   H~ += K^T Omega K,  b~ += K^T Omega e,   K = [-I, [m]x],  m = R mu_j = q - t
// K is the Jacobian in the rotated frame: J = de/d(delta) = [-R, R[mu]x] = K blockdiag(R, R)
// (R2), so the per-slot rotation back to the body frame happens once in a3, not per point.
// The table probe of point j+1 (key + payload, one 48-byte slot) is issued before the math of
// point j, so the L2 gather latency hides behind ~140 FP32 instructions.
// Accumulators are fp32 registers in a fixed point order: bitwise reproducible.
#include "mcs_internal.cuh"

namespace mcs {

constexpr int kSweepThreads = 128;
constexpr int kChunk = 256;  // scan points per shared-memory stage (12 KB)

struct Probe {
  float4 s0, s1, s2;   // slot payload (first probe position, speculatively loaded)
  float qx, qy, qz;    // pinned fp32 transform of the point
  unsigned int key;    // bbox-local key; kEmptyKey32 = out of the keyframe bbox
  unsigned int h;      // slot index of the first probe
};

__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
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
  KfMeta m;
  if (active) {
    m = kmeta[kf];
  } else {
    m.slots = nullptr;
    m.ox = m.oy = m.oz = 0;
    m.ex = m.ey = m.ez = 0;
    m.shift = 31;
    m.mask = 0;
  }
  const float R00 = r0.x, R01 = r0.y, R02 = r0.z, tx = r0.w;
  const float R10 = r1.x, R11 = r1.y, R12 = r1.z, ty = r1.w;
  const float R20 = r2.x, R21 = r2.y, R22 = r2.z, tz = r2.w;

  // issue the first probe of point j (no wait on the loads)
  auto issue = [&](int j) {
    Probe p;
    const float4 A = s_pt[3 * j];
    p.qx = __fmaf_rn(R02, A.z, __fmaf_rn(R01, A.y, __fmaf_rn(R00, A.x, tx)));
    p.qy = __fmaf_rn(R12, A.z, __fmaf_rn(R11, A.y, __fmaf_rn(R10, A.x, ty)));
    p.qz = __fmaf_rn(R22, A.z, __fmaf_rn(R21, A.y, __fmaf_rn(R20, A.x, tz)));
    // floor(q / r) (pinned: exact power-of-two scaling, R27), then bbox-local coordinates
    const unsigned int dx = (unsigned)(__float2int_rd(__fmul_rn(p.qx, inv_r)) - m.ox);
    const unsigned int dy = (unsigned)(__float2int_rd(__fmul_rn(p.qy, inv_r)) - m.oy);
    const unsigned int dz = (unsigned)(__float2int_rd(__fmul_rn(p.qz, inv_r)) - m.oz);
    const bool in = (dx < m.ex) & (dy < m.ey) & (dz < m.ez);
    p.key = in ? local_key(dx, dy, dz) : kEmptyKey32;
    p.h = slot_hash(p.key, m.shift) & m.mask;
    if (in) {
      const float4* s = m.slots + 4 * (size_t)p.h;
      p.s0 = __ldg(s);
      p.s1 = __ldg(s + 1);
      p.s2 = __ldg(s + 2);
    } else {
      p.s0 = make_float4(0.f, 0.f, 0.f, __uint_as_float(kEmptyKey32));
      p.s1 = p.s0;
      p.s2 = p.s0;
    }
    return p;
  };

  float l = 0.f;
  int n = 0;
  float h[21];
  float bv[6];
#pragma unroll
  for (int k = 0; k < 21; ++k) h[k] = 0.f;
#pragma unroll
  for (int k = 0; k < 6; ++k) bv[k] = 0.f;

  // resolve a probe: first-probe hit, empty slot (miss), or continue linear probing
  auto resolve = [&](Probe& p) -> bool {
    if (p.key == kEmptyKey32) return false;
    const unsigned int k0 = __float_as_uint(p.s0.w);
    if (k0 == p.key) return true;
    if (k0 == kEmptyKey32) return false;
    unsigned int hh = p.h;
    while (true) {
      hh = (hh + 1) & m.mask;
      const float4* sl = m.slots + 4 * (size_t)hh;
      const float4 t0 = __ldg(sl);
      const unsigned int kk = __float_as_uint(t0.w);
      if (kk == p.key) {
        p.s0 = t0;
        p.s1 = __ldg(sl + 1);
        p.s2 = __ldg(sl + 2);
        return true;
      }
      if (kk == kEmptyKey32) return false;
    }
  };

  // Eqs.3-4 and Eq.6 for one matched (item, point)
  auto accumulate = [&](int j, const Probe& p) {
    const float4 A = s_pt[3 * j];
    const float4 B = s_pt[3 * j + 1];
    const float4 Cc = s_pt[3 * j + 2];
    const float4 P0 = p.s0, P1 = p.s1, P2 = p.s2;
    // e = mu' - kT mu   (Eq.4);  m = R mu = q - t
    const float ex = P0.x - p.qx, ey = P0.y - p.qy, ez = P0.z - p.qz;
    const float mx = p.qx - tx, my = p.qy - ty, mz = p.qz - tz;
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
    const float c00 = fmaf(a00, R00, fmaf(a01, R01, fmaf(a02, R02, P1.x)));
    const float c01 = fmaf(a00, R10, fmaf(a01, R11, fmaf(a02, R12, P1.y)));
    const float c02 = fmaf(a00, R20, fmaf(a01, R21, fmaf(a02, R22, P1.z)));
    const float c11 = fmaf(a10, R10, fmaf(a11, R11, fmaf(a12, R12, P1.w)));
    const float c12 = fmaf(a10, R20, fmaf(a11, R21, fmaf(a12, R22, P2.x)));
    const float c22 = fmaf(a20, R20, fmaf(a21, R21, fmaf(a22, R22, P2.y)));
    // Omega = C^-1 = adj(C) / det(C)
    const float k00 = c11 * c22 - c12 * c12;
    const float k01 = c02 * c12 - c01 * c22;
    const float k02 = c01 * c12 - c02 * c11;
    const float k11 = c00 * c22 - c02 * c02;
    const float k12 = c01 * c02 - c00 * c12;
    const float k22 = c00 * c11 - c01 * c01;
    const float id = rcp_approx(fmaf(c00, k00, fmaf(c01, k01, c02 * k02)));
    const float o00 = k00 * id, o01 = k01 * id, o02 = k02 * id;
    const float o11 = k11 * id, o12 = k12 * id, o22 = k22 * id;
    // w = Omega e ; l -= e^T Omega e  (Eq.3)
    const float w0 = o00 * ex + o01 * ey + o02 * ez;
    const float w1 = o01 * ex + o11 * ey + o12 * ez;
    const float w2 = o02 * ex + o12 * ey + o22 * ez;
    l = fmaf(-ex, w0, fmaf(-ey, w1, fmaf(-ez, w2, l)));
    ++n;
    if (hb) {
      // H~ = K^T Omega K = [[Omega, -Omega M], [-M^T Omega, M^T Omega M]], M = [m]x; P = Omega M
      const float p00 = o01 * mz - o02 * my, p01 = o02 * mx - o00 * mz, p02 = o00 * my - o01 * mx;
      const float p10 = o11 * mz - o12 * my, p11 = o12 * mx - o01 * mz, p12 = o01 * my - o11 * mx;
      const float p20 = o12 * mz - o22 * my, p21 = o22 * mx - o02 * mz, p22 = o02 * my - o12 * mx;
      h[0] += o00; h[1] += o01; h[2] += o02;
      h[3] -= p00; h[4] -= p01; h[5] -= p02;
      h[6] += o11; h[7] += o12;
      h[8] -= p10; h[9] -= p11; h[10] -= p12;
      h[11] += o22;
      h[12] -= p20; h[13] -= p21; h[14] -= p22;
      // M^T Omega M = -M P
      h[15] = fmaf(mz, p10, fmaf(-my, p20, h[15]));  // (3,3)
      h[16] = fmaf(mz, p11, fmaf(-my, p21, h[16]));  // (3,4)
      h[17] = fmaf(mz, p12, fmaf(-my, p22, h[17]));  // (3,5)
      h[18] = fmaf(mx, p21, fmaf(-mz, p01, h[18]));  // (4,4)
      h[19] = fmaf(mx, p22, fmaf(-mz, p02, h[19]));  // (4,5)
      h[20] = fmaf(my, p02, fmaf(-mx, p12, h[20]));  // (5,5)
      // b~ = K^T Omega e = [-w ; w x m]
      bv[0] -= w0; bv[1] -= w1; bv[2] -= w2;
      bv[3] = fmaf(w1, mz, fmaf(-w2, my, bv[3]));
      bv[4] = fmaf(w2, mx, fmaf(-w0, mz, bv[4]));
      bv[5] = fmaf(w0, my, fmaf(-w1, mx, bv[5]));
    }
  };

  for (int base = 0; base < S; base += kChunk) {
    const int cnt = min(kChunk, S - base);
    __syncthreads();
    for (int k = threadIdx.x; k < cnt * 3; k += kSweepThreads) s_pt[k] = scan[3 * base + k];
    __syncthreads();
    if (!active) continue;
    // two probe buffers in flight alternately: the slot of point j+1 is requested before the
    // math of point j (no register copies between iterations)
    Probe pa = issue(0), pb;
    for (int j = 0; j < cnt; j += 2) {
      const bool ha = resolve(pa);
      if (j + 1 < cnt) pb = issue(j + 1);
      if (ha) accumulate(j, pa);
      if (j + 1 >= cnt) break;
      const bool hb2 = resolve(pb);
      if (j + 2 < cnt) pa = issue(j + 2);
      if (hb2) accumulate(j + 1, pb);
    }
  }
  if (!active) return;
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
