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
// R Sigma_j R^T uses the per-scan spectral form of Sigma_j (prepare_scan_kernel below).
// Accumulators are fp32 registers in a fixed point order: bitwise reproducible.
#include "mcs_internal.cuh"

namespace mcs {

#ifndef MCS_SWEEP_THREADS
#define MCS_SWEEP_THREADS 128
#endif
#ifndef MCS_SWEEP_CHUNK
#define MCS_SWEEP_CHUNK 256
#endif
#ifndef MCS_SWEEP_MINBLOCKS
#define MCS_SWEEP_MINBLOCKS 4
#endif
constexpr int kSweepThreads = MCS_SWEEP_THREADS;
constexpr int kChunk = MCS_SWEEP_CHUNK;  // scan points per shared-memory stage (48 B each)

struct Probe {
  float4 s0, s1, s2;   // slot payload at the first probe position (speculatively loaded)
  float qx, qy, qz;    // pinned fp32 transform of the point
  unsigned int key;    // bbox-local key; kEmptyKey32 = outside the keyframe bbox
  unsigned int h;      // slot index of the first probe
};

__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

__device__ __forceinline__ void ld_slot(const float4* sl, float4& s0, float4& s1, float4& s2) {
  asm volatile("ld.global.nc.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(s0.x), "=f"(s0.y), "=f"(s0.z), "=f"(s0.w) : "l"(sl));
  asm volatile("ld.global.nc.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(s1.x), "=f"(s1.y), "=f"(s1.z), "=f"(s1.w) : "l"(sl + 1));
  asm volatile("ld.global.nc.v2.f32 {%0, %1}, [%2];" : "=f"(s2.x), "=f"(s2.y) : "l"(sl + 2));
  s2.z = 0.f;
  s2.w = 0.f;
}

// floor(x) as the bits of x + 1.5*2^23 rounded toward -inf: exact for |x| < 2^22, and every
// other finite x maps far outside any keyframe bbox after the offset.
constexpr float kMagic = 12582912.0f;

__global__ void __launch_bounds__(kSweepThreads, MCS_SWEEP_MINBLOCKS)
    sweep_kernel(const float4* __restrict__ items, const int32_t* __restrict__ order,
                 int n_items, const float4* __restrict__ scan, int S,
                 const KfMeta* __restrict__ kmeta, float inv_r, double* __restrict__ part) {
  __shared__ float4 s_pt[kChunk * 3];
  // two-level accumulation: fp32 registers within a stage, fp64 totals per thread in shared
  // memory across stages (the fp32 running sums over a whole 4,096-point scan lose ~1e-5
  // relative, which an ill-conditioned H turns into >1e-5 m of pose error)
  __shared__ double s_acc[28][kSweepThreads];
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
  const unsigned int offx = (unsigned)__float_as_int(kMagic) + (unsigned)m.ox;
  const unsigned int offy = (unsigned)__float_as_int(kMagic) + (unsigned)m.oy;
  const unsigned int offz = (unsigned)__float_as_int(kMagic) + (unsigned)m.oz;
  const float R00 = r0.x, R01 = r0.y, R02 = r0.z, tx = r0.w;
  const float R10 = r1.x, R11 = r1.y, R12 = r1.z, ty = r1.w;
  const float R20 = r2.x, R21 = r2.y, R22 = r2.z, tz = r2.w;

  // transform, cell, key and the (unconditional) first-probe loads of point j
  auto issue = [&](int j) {
    Probe p;
    const float4 A = s_pt[3 * j];
    p.qx = __fmaf_rn(R02, A.z, __fmaf_rn(R01, A.y, __fmaf_rn(R00, A.x, tx)));
    p.qy = __fmaf_rn(R12, A.z, __fmaf_rn(R11, A.y, __fmaf_rn(R10, A.x, ty)));
    p.qz = __fmaf_rn(R22, A.z, __fmaf_rn(R21, A.y, __fmaf_rn(R20, A.x, tz)));
    // floor(q / r) (exact power-of-two scaling, R27) -> bbox-local cell coordinates
    const unsigned int dx =
        (unsigned)__float_as_int(__fadd_rd(__fmul_rn(p.qx, inv_r), kMagic)) - offx;
    const unsigned int dy =
        (unsigned)__float_as_int(__fadd_rd(__fmul_rn(p.qy, inv_r), kMagic)) - offy;
    const unsigned int dz =
        (unsigned)__float_as_int(__fadd_rd(__fmul_rn(p.qz, inv_r), kMagic)) - offz;
    const bool in = (dx < m.ex) & (dy < m.ey) & (dz < m.ez);
    p.key = in ? local_key(dx, dy, dz) : kEmptyKey32;
    p.h = slot_hash(p.key, m.shift) & m.mask;
    const float4* sl = m.slots + 4 * (size_t)p.h;
    if (active) {
      // volatile: the compiler may not sink these loads towards their use (that would undo the
      // prefetch); the payload is consumed one point later
      ld_slot(sl, p.s0, p.s1, p.s2);
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

  // first probe: 1 = hit, 0 = empty slot or out-of-bbox point (miss), 2 = keep probing
  auto first_check = [&](const Probe& p) -> int {
    const unsigned int k0 = __float_as_uint(p.s0.w);
    if (k0 == p.key) return p.key != kEmptyKey32 ? 1 : 0;
    if (k0 == kEmptyKey32 || p.key == kEmptyKey32) return 0;
    return 2;
  };
  // continue linear probing (rare): loads into fresh registers q.s*, waited on inside this
  // path, so the common path never inherits a pending scoreboard from it
  auto probe_on = [&](Probe& q) -> bool {
    unsigned int hh = q.h;
    while (true) {
      hh = (hh + 1) & m.mask;
      const float4* sl = m.slots + 4 * (size_t)hh;
      const float4 t0 = __ldg(sl);
      const unsigned int kk = __float_as_uint(t0.w);
      if (kk == q.key) {
        q.s0 = t0;
        q.s1 = __ldg(sl + 1);
        q.s2 = __ldg(sl + 2);
        return true;
      }
      if (kk == kEmptyKey32) return false;
    }
  };

  // Eqs.3-4 and Eq.6 for one matched (item, point)
  auto accumulate = [&](int j, const Probe& p) {
    const float4 A = s_pt[3 * j];      // {mu, lambda3}
    const float4 U = s_pt[3 * j + 1];  // {u, 0}
    const float4 V = s_pt[3 * j + 2];  // {v, 0}   Sigma_j = lambda3 I + u u^T + v v^T
    const float4 P0 = p.s0, P1 = p.s1, P2 = p.s2;
    // e = mu' - kT mu   (Eq.4);  m = R mu = q - t
    const float ex = P0.x - p.qx, ey = P0.y - p.qy, ez = P0.z - p.qz;
    const float mx = p.qx - tx, my = p.qy - ty, mz = p.qz - tz;
    // C = Sigma' + R Sigma R^T = Sigma' + lambda3 I + (Ru)(Ru)^T + (Rv)(Rv)^T  (Eq.4)
    const float ux = R00 * U.x + R01 * U.y + R02 * U.z;
    const float uy = R10 * U.x + R11 * U.y + R12 * U.z;
    const float uz = R20 * U.x + R21 * U.y + R22 * U.z;
    const float vx = R00 * V.x + R01 * V.y + R02 * V.z;
    const float vy = R10 * V.x + R11 * V.y + R12 * V.z;
    const float vz = R20 * V.x + R21 * V.y + R22 * V.z;
    const float c00 = fmaf(ux, ux, fmaf(vx, vx, P1.x + A.w));
    const float c01 = fmaf(ux, uy, fmaf(vx, vy, P1.y));
    const float c02 = fmaf(ux, uz, fmaf(vx, vz, P1.z));
    const float c11 = fmaf(uy, uy, fmaf(vy, vy, P1.w + A.w));
    const float c12 = fmaf(uy, uz, fmaf(vy, vz, P2.x));
    const float c22 = fmaf(uz, uz, fmaf(vz, vz, P2.y + A.w));
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

#pragma unroll
  for (int k = 0; k < 28; ++k) s_acc[k][threadIdx.x] = 0.0;
  auto flush = [&]() {
    s_acc[0][threadIdx.x] += (double)l;
    l = 0.f;
#pragma unroll
    for (int k = 0; k < 21; ++k) {
      s_acc[1 + k][threadIdx.x] += (double)h[k];
      h[k] = 0.f;
    }
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      s_acc[22 + k][threadIdx.x] += (double)bv[k];
      bv[k] = 0.f;
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
      const int ra = first_check(pa);
      if (j + 1 < cnt) pb = issue(j + 1);
      if (ra == 1) {
        accumulate(j, pa);
      } else if (ra == 2) {
        Probe q;
        q.qx = pa.qx; q.qy = pa.qy; q.qz = pa.qz; q.key = pa.key; q.h = pa.h;
        if (probe_on(q)) accumulate(j, q);
      }
      if (j + 1 >= cnt) break;
      const int rb = first_check(pb);
      if (j + 2 < cnt) pa = issue(j + 2);
      if (rb == 1) {
        accumulate(j + 1, pb);
      } else if (rb == 2) {
        Probe q;
        q.qx = pb.qx; q.qy = pb.qy; q.qz = pb.qz; q.key = pb.key; q.h = pb.h;
        if (probe_on(q)) accumulate(j + 1, q);
      }
    }
    flush();
  }
  if (!active) return;
  double* o = part + (size_t)item * kSlotWords;
  o[0] = s_acc[0][threadIdx.x];
  o[1] = (double)n;
#pragma unroll
  for (int k = 0; k < 21; ++k) o[2 + k] = s_acc[1 + k][threadIdx.x];
#pragma unroll
  for (int k = 0; k < 6; ++k) o[23 + k] = s_acc[22 + k][threadIdx.x];
}

// Scan preparation (once per update): Sigma_j = lambda3 I + u u^T + v v^T with u, v the two
// leading eigenvectors scaled by sqrt(lambda_k - lambda3) — the spectral decomposition,
// exact up to rounding for any symmetric Sigma (fp64 cyclic Jacobi, then rounded).  The sweep
// then forms R Sigma R^T as lambda3 I + (Ru)(Ru)^T + (Rv)(Rv)^T (33 FP32 ops instead of 45).
__global__ void prepare_scan_kernel(const float* __restrict__ mean3,
                                    const float* __restrict__ cov6, int S,
                                    float4* __restrict__ out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= S) return;
  const float* c = cov6 + 6 * j;
  double a[3][3] = {{c[0], c[1], c[2]}, {c[1], c[3], c[4]}, {c[2], c[4], c[5]}};
  double v[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  for (int sweep = 0; sweep < 12; ++sweep) {
    const double off = a[0][1] * a[0][1] + a[0][2] * a[0][2] + a[1][2] * a[1][2];
    const double dg = a[0][0] * a[0][0] + a[1][1] * a[1][1] + a[2][2] * a[2][2];
    if (off <= 1e-36 * dg) break;
    for (int pq = 0; pq < 3; ++pq) {
      const int p = pq == 2 ? 1 : 0, q = pq == 0 ? 1 : 2;
      if (a[p][q] == 0.0) continue;
      const double theta = (a[q][q] - a[p][p]) / (2.0 * a[p][q]);
      const double tt = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
      const double cs = 1.0 / sqrt(tt * tt + 1.0), sn = tt * cs;
      for (int k = 0; k < 3; ++k) {  // A <- J^T A J
        const double akp = a[k][p], akq = a[k][q];
        a[k][p] = cs * akp - sn * akq;
        a[k][q] = sn * akp + cs * akq;
      }
      for (int k = 0; k < 3; ++k) {
        const double apk = a[p][k], aqk = a[q][k];
        a[p][k] = cs * apk - sn * aqk;
        a[q][k] = sn * apk + cs * aqk;
      }
      for (int k = 0; k < 3; ++k) {  // V <- V J
        const double vkp = v[k][p], vkq = v[k][q];
        v[k][p] = cs * vkp - sn * vkq;
        v[k][q] = sn * vkp + cs * vkq;
      }
    }
  }
  // order eigenvalues: l0 >= l1 >= l2
  int i0 = 0, i1 = 1, i2 = 2;
  double lam[3] = {a[0][0], a[1][1], a[2][2]};
  if (lam[i0] < lam[i1]) { int t = i0; i0 = i1; i1 = t; }
  if (lam[i1] < lam[i2]) { int t = i1; i1 = i2; i2 = t; }
  if (lam[i0] < lam[i1]) { int t = i0; i0 = i1; i1 = t; }
  const double l3 = lam[i2];
  const double su = sqrt(fmax(lam[i0] - l3, 0.0)), sv = sqrt(fmax(lam[i1] - l3, 0.0));
  const float* m = mean3 + 3 * j;
  out[3 * j + 0] = make_float4(m[0], m[1], m[2], (float)l3);
  out[3 * j + 1] = make_float4((float)(su * v[0][i0]), (float)(su * v[1][i0]),
                               (float)(su * v[2][i0]), 0.f);
  out[3 * j + 2] = make_float4((float)(sv * v[0][i1]), (float)(sv * v[1][i1]),
                               (float)(sv * v[2][i1]), 0.f);
}

void launch_prepare_scan(const float* mean3, const float* cov6, int S, float4* out,
                         cudaStream_t st) {
  prepare_scan_kernel<<<(S + 127) / 128, 128, 0, st>>>(mean3, cov6, S, out);
}

void launch_sweep(mcs_ctx* c, int S) {
  const int n_items = c->cfg.neighbor_count * c->N;
  const int grid = (n_items + kSweepThreads - 1) / kSweepThreads;
  sweep_kernel<<<grid, kSweepThreads, 0, c->stream>>>(c->d_items, c->d_order, n_items, c->d_scan,
                                                      S, c->d_kf_meta,
                                                      1.0f / c->cfg.voxel_resolution, c->d_part);
}

}  // namespace mcs
