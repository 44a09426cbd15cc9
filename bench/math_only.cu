// math_only.cu — the sweep's per-matched-point arithmetic (sweep.cu `accumulate`: transform,
// C = Sigma' + R Sigma R^T via the spectral form, adjugate inverse, l, H~ 21, b~ 6) in a loop
// with no gathers and every lane matched: the FMA-pipe-bound rate of the instruction mix, to
// compare with the sweep's measured cycles per warp-point.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/math_only bench/math_only.cu
#include <cuda_runtime.h>
#include <stdio.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ float2 bc(float a) { return make_float2(a, a); }
__device__ __forceinline__ float2 sw(float2 a) { return make_float2(a.y, a.x); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 neg2(float2 a) { return make_float2(-a.x, -a.y); }
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

constexpr int kPts = 256;
__constant__ float4 c_pts[kPts * 4];  // variant B/C: the scan in the constant bank (uniform regs)

template <int kH, int kConst, int kMinB = 4>
__global__ void __launch_bounds__(128, kMinB) math_kernel(const float4* __restrict__ scan, int reps,
                                                      float* out, const float* __restrict__ pl) {
  __shared__ float4 sp[kPts * 3];
  for (int k = threadIdx.x; k < kPts * 3; k += blockDim.x) sp[k] = scan[k];
  __syncthreads();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  // per-lane pose and payload from memory (nothing constant-folds)
  const float* pv = pl + 32 * (t & 1023);
  const float R00 = pv[0], R01 = pv[1], R02 = pv[2], tx = pv[3];
  const float2 Ryz0 = make_float2(pv[4], pv[8]), Ryz1 = make_float2(pv[5], pv[9]),
               Ryz2 = make_float2(pv[6], pv[10]);
  const float2 tyz = make_float2(pv[7], pv[11]), ntyz = neg2(tyz);
  const float4 P0 = make_float4(0.f, pv[12], pv[13], pv[14]);
  const float4 P1 = make_float4(pv[15], pv[16], pv[17], pv[18]);
  const float4 P2 = make_float4(pv[19], pv[20], 0.f, 0.f);
  float l = 0.f, h[21], bv[6];
#pragma unroll
  for (int k = 0; k < 21; ++k) h[k] = 0.f;
#pragma unroll
  for (int k = 0; k < 6; ++k) bv[k] = 0.f;
  for (int r = 0; r < reps; ++r) {
#pragma unroll 2
    for (int j = 0; j < kPts; ++j) {
      const float4 A = kConst ? c_pts[4 * j] : sp[3 * j];
      const float4 U = kConst ? c_pts[4 * j + 1] : sp[3 * j + 1];
      const float4 V = kConst ? c_pts[4 * j + 2] : sp[3 * j + 2];
      const float qx = __fmaf_rn(R02, A.z, __fmaf_rn(R01, A.y, __fmaf_rn(R00, A.x, tx)));
      const float2 qyz = fma2(Ryz2, bc(A.z), fma2(Ryz1, bc(A.y), fma2(Ryz0, bc(A.x), tyz)));
      const float ex = P0.y - qx;
      const float2 eyz = fma2(qyz, bc(-1.f), make_float2(P0.z, P0.w));
      const float mx = qx - tx;
      const float2 myz = add2(qyz, ntyz);
      const float my = myz.x, mz = myz.y;
      const float ux = fmaf(R02, U.z, fmaf(R01, U.y, R00 * U.x));
      const float2 uyz = fma2(Ryz2, bc(U.z), fma2(Ryz1, bc(U.y), mul2(Ryz0, bc(U.x))));
      const float vx = fmaf(R02, V.z, fmaf(R01, V.y, R00 * V.x));
      const float2 vyz = fma2(Ryz2, bc(V.z), fma2(Ryz1, bc(V.y), mul2(Ryz0, bc(V.x))));
      const float c00 = fmaf(ux, ux, fmaf(vx, vx, P2.x + A.w));
      const float2 c1122 = fma2(uyz, uyz, fma2(vyz, vyz, add2(make_float2(P1.x, P1.y), bc(A.w))));
      const float2 c0102 = fma2(bc(ux), uyz, fma2(bc(vx), vyz, make_float2(P1.z, P1.w)));
      const float c12 = fmaf(uyz.x, uyz.y, fmaf(vyz.x, vyz.y, P2.y));
      const float k00 = fmaf(c1122.x, c1122.y, -c12 * c12);
      const float2 c0201 = sw(c0102);
      const float2 k1122 = fma2(bc(c00), sw(c1122), mul2(c0201, neg2(c0201)));
      const float2 k0102 = fma2(bc(c12), c0201, mul2(c0102, neg2(sw(c1122))));
      const float k12 = fmaf(c0102.x, c0102.y, -c00 * c12);
      const float id = rcp_approx(fmaf(c00, k00, fmaf(c0102.x, k0102.x, c0102.y * k0102.y)));
      const float o00 = k00 * id, o12 = k12 * id;
      const float2 o1122 = mul2(k1122, bc(id)), o0102 = mul2(k0102, bc(id));
      const float o01 = o0102.x, o02 = o0102.y, o11 = o1122.x, o22 = o1122.y;
      const float ey = eyz.x, ez = eyz.y;
      const float w0 = fmaf(o00, ex, fmaf(o01, ey, o02 * ez));
      const float2 w12 = fma2(bc(ex), o0102, fma2(o1122, eyz, mul2(bc(o12), sw(eyz))));
      const float w1 = w12.x, w2 = w12.y;
      l = fmaf(-ex, w0, fmaf(-ey, w1, fmaf(-ez, w2, l)));
      if (kH) {
        const float p00 = o01 * mz - o02 * my, p01 = o02 * mx - o00 * mz, p02 = o00 * my - o01 * mx;
        const float p10 = o11 * mz - o12 * my, p11 = o12 * mx - o01 * mz, p12 = o01 * my - o11 * mx;
        const float p20 = o12 * mz - o22 * my, p21 = o22 * mx - o02 * mz, p22 = o02 * my - o12 * mx;
        h[0] += o00; h[1] += o01; h[2] += o02;
        h[3] -= p00; h[4] -= p01; h[5] -= p02;
        h[6] += o11; h[7] += o12;
        h[8] -= p10; h[9] -= p11; h[10] -= p12;
        h[11] += o22;
        h[12] -= p20; h[13] -= p21; h[14] -= p22;
        h[15] = fmaf(mz, p10, fmaf(-my, p20, h[15]));
        h[16] = fmaf(mz, p11, fmaf(-my, p21, h[16]));
        h[17] = fmaf(mz, p12, fmaf(-my, p22, h[17]));
        h[18] = fmaf(mx, p21, fmaf(-mz, p01, h[18]));
        h[19] = fmaf(mx, p22, fmaf(-mz, p02, h[19]));
        h[20] = fmaf(my, p02, fmaf(-mx, p12, h[20]));
        bv[0] -= w0; bv[1] -= w1; bv[2] -= w2;
        bv[3] = fmaf(w1, mz, fmaf(-w2, my, bv[3]));
        bv[4] = fmaf(w2, mx, fmaf(-w0, mz, bv[4]));
        bv[5] = fmaf(w0, my, fmaf(-w1, mx, bv[5]));
      }
    }
  }
  float acc = l;
#pragma unroll
  for (int k = 0; k < 21; ++k) acc += h[k];
#pragma unroll
  for (int k = 0; k < 6; ++k) acc += bv[k];
  if (acc == 1234.5f) out[0] = acc;
}


// v17 candidate: body frame (H, b accumulated in the particle's body frame: the per-point
// coefficients [mu]x are warp-uniform), plane-form covariances Sigma_j = alpha I - a n n^T
// (uniform) and Sigma' = alpha' I - a' n' n'^T (gathered): C^b = beta I - a' u u^T - a n n^T
// with u = R^T n', inverted in closed form (Woodbury, 2x2).  Scan point record in the constant
// bank: {mu, 1/a} {n, alpha} {mu products: xx yy zz xy} {xz yz, -, -}
__global__ void __launch_bounds__(128, 4) v17_kernel(int reps, float* out,
                                                     const float* __restrict__ pl) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const float* pv = pl + 32 * (t & 1023);
  const float R00 = pv[0], R01 = pv[1], R02 = pv[2], tx = pv[3];
  const float R10 = pv[4], R11 = pv[5], R12 = pv[6], ty = pv[7];
  const float R20 = pv[8], R21 = pv[9], R22 = pv[10], tz = pv[11];
  // payload {key, mu'} {n', alpha'} {1/a', -}
  const float mpx = pv[12], mpy = pv[13], mpz = pv[14];
  const float npx = pv[21], npy = pv[22], npz = pv[23], alp = pv[24], iap = pv[25];
  float l = 0.f, h[21], bv[6];
#pragma unroll
  for (int k = 0; k < 21; ++k) h[k] = 0.f;
#pragma unroll
  for (int k = 0; k < 6; ++k) bv[k] = 0.f;
  for (int r = 0; r < reps; ++r) {
#pragma unroll 2
    for (int j = 0; j < kPts; ++j) {
      const float4 A = c_pts[4 * j], Nn = c_pts[4 * j + 1], Pm = c_pts[4 * j + 2],
                   Pn = c_pts[4 * j + 3];
      const float mx = A.x, my = A.y, mz = A.z, ia = A.w;
      const float nx = Nn.x, ny = Nn.y, nz = Nn.z, al = Nn.w;
      // q = kT mu (pinned chain, uniform mu)
      const float qx = __fmaf_rn(R02, mz, __fmaf_rn(R01, my, __fmaf_rn(R00, mx, tx)));
      const float qy = __fmaf_rn(R12, mz, __fmaf_rn(R11, my, __fmaf_rn(R10, mx, ty)));
      const float qz = __fmaf_rn(R22, mz, __fmaf_rn(R21, my, __fmaf_rn(R20, mx, tz)));
      const float ex = mpx - qx, ey = mpy - qy, ez = mpz - qz;
      // body frame: e^b = R^T e, u = R^T n'
      const float bx = fmaf(R20, ez, fmaf(R10, ey, R00 * ex));
      const float by = fmaf(R21, ez, fmaf(R11, ey, R01 * ex));
      const float bz = fmaf(R22, ez, fmaf(R12, ey, R02 * ex));
      const float ux = fmaf(R20, npz, fmaf(R10, npy, R00 * npx));
      const float uy = fmaf(R21, npz, fmaf(R11, npy, R01 * npx));
      const float uz = fmaf(R22, npz, fmaf(R12, npy, R02 * npx));
      const float cc = fmaf(uz, nz, fmaf(uy, ny, ux * nx));
      const float ss = fmaf(uz, bz, fmaf(uy, by, ux * bx));
      const float tt = fmaf(nz, bz, fmaf(ny, by, nx * bx));
      const float beta = al + alp;
      const float m11 = fmaf(beta, iap, -1.f), m22 = fmaf(beta, ia, -1.f);
      const float det = fmaf(m11, m22, -cc * cc);
      const float f = rcp_approx(beta * det);
      const float ib = f * det, n11 = f * m22, n12 = f * cc, n22 = f * m11;
      const float z1x = fmaf(n12, nx, n11 * ux), z1y = fmaf(n12, ny, n11 * uy),
                  z1z = fmaf(n12, nz, n11 * uz);
      const float z2x = fmaf(n22, nx, n12 * ux), z2y = fmaf(n22, ny, n12 * uy),
                  z2z = fmaf(n22, nz, n12 * uz);
      const float o00 = fmaf(z1x, ux, fmaf(z2x, nx, ib));
      const float o11 = fmaf(z1y, uy, fmaf(z2y, ny, ib));
      const float o22 = fmaf(z1z, uz, fmaf(z2z, nz, ib));
      const float o01 = fmaf(z1x, uy, z2x * ny), o02 = fmaf(z1x, uz, z2x * nz),
                  o12 = fmaf(z1y, uz, z2y * nz);
      const float w0 = fmaf(z2x, tt, fmaf(z1x, ss, ib * bx));
      const float w1 = fmaf(z2y, tt, fmaf(z1y, ss, ib * by));
      const float w2 = fmaf(z2z, tt, fmaf(z1z, ss, ib * bz));
      l = fmaf(-bx, w0, fmaf(-by, w1, fmaf(-bz, w2, l)));
      // H^b = K^T Omega^b K, K = [-I, [mu]x] (uniform mu); P = Omega^b [mu]x
      const float p00 = o01 * mz - o02 * my, p01 = o02 * mx - o00 * mz, p02 = o00 * my - o01 * mx;
      const float p10 = o11 * mz - o12 * my, p11 = o12 * mx - o01 * mz, p12 = o01 * my - o11 * mx;
      const float p20 = o12 * mz - o22 * my, p21 = o22 * mx - o02 * mz, p22 = o02 * my - o12 * mx;
      h[0] += o00; h[1] += o01; h[2] += o02;
      h[3] -= p00; h[4] -= p01; h[5] -= p02;
      h[6] += o11; h[7] += o12;
      h[8] -= p10; h[9] -= p11; h[10] -= p12;
      h[11] += o22;
      h[12] -= p20; h[13] -= p21; h[14] -= p22;
      h[15] = fmaf(mz, p10, fmaf(-my, p20, h[15]));
      h[16] = fmaf(mz, p11, fmaf(-my, p21, h[16]));
      h[17] = fmaf(mz, p12, fmaf(-my, p22, h[17]));
      h[18] = fmaf(mx, p21, fmaf(-mz, p01, h[18]));
      h[19] = fmaf(mx, p22, fmaf(-mz, p02, h[19]));
      h[20] = fmaf(my, p02, fmaf(-mx, p12, h[20]));
      bv[0] -= w0; bv[1] -= w1; bv[2] -= w2;
      bv[3] = fmaf(w1, mz, fmaf(-w2, my, bv[3]));
      bv[4] = fmaf(w2, mx, fmaf(-w0, mz, bv[4]));
      bv[5] = fmaf(w0, my, fmaf(-w1, mx, bv[5]));
      (void)Pm; (void)Pn;
    }
  }
  float acc = l;
#pragma unroll
  for (int k = 0; k < 21; ++k) acc += h[k];
#pragma unroll
  for (int k = 0; k < 6; ++k) acc += bv[k];
  if (acc == 1234.5f) out[0] = acc;
}


// v18 candidate: rotated (keyframe) frame as the current sweep, plane-form covariances:
// C = beta I - a' u u^T - a v v^T with u = n' (gathered, unrotated) and v = R n (n uniform),
// Omega by the closed-form 2x2 Woodbury inverse; H~, b~ with K = [-I, [m]x] as now.
template <int kSrcConst>
__global__ void __launch_bounds__(128, 4) v18_kernel(const float4* __restrict__ scan, int reps,
                                                     float* out, const float* __restrict__ pl) {
  __shared__ float4 sp[kPts * 2];
  for (int k = threadIdx.x; k < kPts * 2; k += blockDim.x) sp[k] = scan[k];
  __syncthreads();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const float* pv = pl + 32 * (t & 1023);
  const float R00 = pv[0], R01 = pv[1], R02 = pv[2], tx = pv[3];
  const float R10 = pv[4], R11 = pv[5], R12 = pv[6], ty = pv[7];
  const float R20 = pv[8], R21 = pv[9], R22 = pv[10], tz = pv[11];
  const float mpx = pv[12], mpy = pv[13], mpz = pv[14];
  const float ux = pv[21], uy = pv[22], uz = pv[23], alp = pv[24], iap = pv[25];
  float l = 0.f, h[21], bv[6];
#pragma unroll
  for (int k = 0; k < 21; ++k) h[k] = 0.f;
#pragma unroll
  for (int k = 0; k < 6; ++k) bv[k] = 0.f;
  for (int r = 0; r < reps; ++r) {
#pragma unroll 2
    for (int j = 0; j < kPts; ++j) {
      const float4 A = kSrcConst ? c_pts[4 * j] : sp[2 * j];
      const float4 Nn = kSrcConst ? c_pts[4 * j + 1] : sp[2 * j + 1];
      const float Mx = A.x, My = A.y, Mz = A.z, ia = A.w;
      const float nx = Nn.x, ny = Nn.y, nz = Nn.z, al = Nn.w;
      const float qx = __fmaf_rn(R02, Mz, __fmaf_rn(R01, My, __fmaf_rn(R00, Mx, tx)));
      const float qy = __fmaf_rn(R12, Mz, __fmaf_rn(R11, My, __fmaf_rn(R10, Mx, ty)));
      const float qz = __fmaf_rn(R22, Mz, __fmaf_rn(R21, My, __fmaf_rn(R20, Mx, tz)));
      const float ex = mpx - qx, ey = mpy - qy, ez = mpz - qz;
      const float mx = qx - tx, my = qy - ty, mz = qz - tz;
      const float vx = fmaf(R02, nz, fmaf(R01, ny, R00 * nx));
      const float vy = fmaf(R12, nz, fmaf(R11, ny, R10 * nx));
      const float vz = fmaf(R22, nz, fmaf(R21, ny, R20 * nx));
      const float cc = fmaf(uz, vz, fmaf(uy, vy, ux * vx));
      const float ss = fmaf(uz, ez, fmaf(uy, ey, ux * ex));
      const float tt = fmaf(vz, ez, fmaf(vy, ey, vx * ex));
      const float beta = al + alp;
      const float m11 = fmaf(beta, iap, -1.f), m22 = fmaf(beta, ia, -1.f);
      const float det = fmaf(m11, m22, -cc * cc);
      const float f = rcp_approx(beta * det);
      const float ib = f * det, n11 = f * m22, n12 = f * cc, n22 = f * m11;
      const float z1x = fmaf(n12, vx, n11 * ux), z1y = fmaf(n12, vy, n11 * uy),
                  z1z = fmaf(n12, vz, n11 * uz);
      const float z2x = fmaf(n22, vx, n12 * ux), z2y = fmaf(n22, vy, n12 * uy),
                  z2z = fmaf(n22, vz, n12 * uz);
      const float o00 = fmaf(z1x, ux, fmaf(z2x, vx, ib));
      const float o11 = fmaf(z1y, uy, fmaf(z2y, vy, ib));
      const float o22 = fmaf(z1z, uz, fmaf(z2z, vz, ib));
      const float o01 = fmaf(z1x, uy, z2x * vy), o02 = fmaf(z1x, uz, z2x * vz),
                  o12 = fmaf(z1y, uz, z2y * vz);
      const float w0 = fmaf(z2x, tt, fmaf(z1x, ss, ib * ex));
      const float w1 = fmaf(z2y, tt, fmaf(z1y, ss, ib * ey));
      const float w2 = fmaf(z2z, tt, fmaf(z1z, ss, ib * ez));
      l = fmaf(-ex, w0, fmaf(-ey, w1, fmaf(-ez, w2, l)));
      const float p00 = o01 * mz - o02 * my, p01 = o02 * mx - o00 * mz, p02 = o00 * my - o01 * mx;
      const float p10 = o11 * mz - o12 * my, p11 = o12 * mx - o01 * mz, p12 = o01 * my - o11 * mx;
      const float p20 = o12 * mz - o22 * my, p21 = o22 * mx - o02 * mz, p22 = o02 * my - o12 * mx;
      h[0] += o00; h[1] += o01; h[2] += o02;
      h[3] -= p00; h[4] -= p01; h[5] -= p02;
      h[6] += o11; h[7] += o12;
      h[8] -= p10; h[9] -= p11; h[10] -= p12;
      h[11] += o22;
      h[12] -= p20; h[13] -= p21; h[14] -= p22;
      h[15] = fmaf(mz, p10, fmaf(-my, p20, h[15]));
      h[16] = fmaf(mz, p11, fmaf(-my, p21, h[16]));
      h[17] = fmaf(mz, p12, fmaf(-my, p22, h[17]));
      h[18] = fmaf(mx, p21, fmaf(-mz, p01, h[18]));
      h[19] = fmaf(mx, p22, fmaf(-mz, p02, h[19]));
      h[20] = fmaf(my, p02, fmaf(-mx, p12, h[20]));
      bv[0] -= w0; bv[1] -= w1; bv[2] -= w2;
      bv[3] = fmaf(w1, mz, fmaf(-w2, my, bv[3]));
      bv[4] = fmaf(w2, mx, fmaf(-w0, mz, bv[4]));
      bv[5] = fmaf(w0, my, fmaf(-w1, mx, bv[5]));
    }
  }
  float acc = l;
#pragma unroll
  for (int k = 0; k < 21; ++k) acc += h[k];
#pragma unroll
  for (int k = 0; k < 6; ++k) acc += bv[k];
  if (acc == 1234.5f) out[0] = acc;
}


// v19 candidate: body frame with the GENERAL covariance model (no plane approximation):
// Sigma' = lambda3' I + u' u'^T + v' v'^T (spectral form, gathered), Sigma_j general (uniform,
// constant bank): C^b = Sigma_j + lambda3' I + (R^T u')(R^T u')^T + (R^T v')(R^T v')^T,
// Omega^b = adj / det; H^b, b^b with K_b = [-I, [mu]x] (uniform mu).
template <int kSrcConst>
__global__ void __launch_bounds__(128, 4) v19_kernel(const float4* __restrict__ scan, int reps,
                                                     float* out, const float* __restrict__ pl) {
  __shared__ float4 sp[kPts * 3];
  for (int k = threadIdx.x; k < kPts * 3; k += blockDim.x) sp[k] = scan[k];
  __syncthreads();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const float* pv = pl + 32 * (t & 1023);
  const float R00 = pv[0], R01 = pv[1], R02 = pv[2], tx = pv[3];
  const float R10 = pv[4], R11 = pv[5], R12 = pv[6], ty = pv[7];
  const float R20 = pv[8], R21 = pv[9], R22 = pv[10], tz = pv[11];
  const float mpx = pv[12], mpy = pv[13], mpz = pv[14];
  const float upx = pv[15], upy = pv[16], upz = pv[17], vpx = pv[18], vpy = pv[19], vpz = pv[20];
  const float l3p = pv[24];
  float l = 0.f, h[21], bv[6];
#pragma unroll
  for (int k = 0; k < 21; ++k) h[k] = 0.f;
#pragma unroll
  for (int k = 0; k < 6; ++k) bv[k] = 0.f;
  for (int r = 0; r < reps; ++r) {
#pragma unroll 2
    for (int j = 0; j < kPts; ++j) {
      const float4 A = kSrcConst ? c_pts[4 * j] : sp[3 * j];
      const float4 S0 = kSrcConst ? c_pts[4 * j + 1] : sp[3 * j + 1];
      const float4 S1 = kSrcConst ? c_pts[4 * j + 2] : sp[3 * j + 2];
      const float mx = A.x, my = A.y, mz = A.z;
      // Sigma_j = {xx, xy, xz, yy} {yz, zz}
      const float qx = __fmaf_rn(R02, mz, __fmaf_rn(R01, my, __fmaf_rn(R00, mx, tx)));
      const float qy = __fmaf_rn(R12, mz, __fmaf_rn(R11, my, __fmaf_rn(R10, mx, ty)));
      const float qz = __fmaf_rn(R22, mz, __fmaf_rn(R21, my, __fmaf_rn(R20, mx, tz)));
      const float ex = mpx - qx, ey = mpy - qy, ez = mpz - qz;
      const float bx = fmaf(R20, ez, fmaf(R10, ey, R00 * ex));
      const float by = fmaf(R21, ez, fmaf(R11, ey, R01 * ex));
      const float bz = fmaf(R22, ez, fmaf(R12, ey, R02 * ex));
      const float ux = fmaf(R20, upz, fmaf(R10, upy, R00 * upx));
      const float uy = fmaf(R21, upz, fmaf(R11, upy, R01 * upx));
      const float uz = fmaf(R22, upz, fmaf(R12, upy, R02 * upx));
      const float vx = fmaf(R20, vpz, fmaf(R10, vpy, R00 * vpx));
      const float vy = fmaf(R21, vpz, fmaf(R11, vpy, R01 * vpx));
      const float vz = fmaf(R22, vpz, fmaf(R12, vpy, R02 * vpx));
      const float c00 = fmaf(ux, ux, fmaf(vx, vx, S0.x + l3p));
      const float c11 = fmaf(uy, uy, fmaf(vy, vy, S0.w + l3p));
      const float c22 = fmaf(uz, uz, fmaf(vz, vz, S1.y + l3p));
      const float c01 = fmaf(ux, uy, fmaf(vx, vy, S0.y));
      const float c02 = fmaf(ux, uz, fmaf(vx, vz, S0.z));
      const float c12 = fmaf(uy, uz, fmaf(vy, vz, S1.x));
      const float k00 = fmaf(c11, c22, -c12 * c12), k11 = fmaf(c00, c22, -c02 * c02),
                  k22 = fmaf(c00, c11, -c01 * c01);
      const float k01 = fmaf(c02, c12, -c01 * c22), k02 = fmaf(c01, c12, -c02 * c11),
                  k12 = fmaf(c01, c02, -c00 * c12);
      const float id = rcp_approx(fmaf(c00, k00, fmaf(c01, k01, c02 * k02)));
      const float o00 = k00 * id, o11 = k11 * id, o22 = k22 * id, o01 = k01 * id,
                  o02 = k02 * id, o12 = k12 * id;
      const float w0 = fmaf(o00, bx, fmaf(o01, by, o02 * bz));
      const float w1 = fmaf(o01, bx, fmaf(o11, by, o12 * bz));
      const float w2 = fmaf(o02, bx, fmaf(o12, by, o22 * bz));
      l = fmaf(-bx, w0, fmaf(-by, w1, fmaf(-bz, w2, l)));
      const float p00 = o01 * mz - o02 * my, p01 = o02 * mx - o00 * mz, p02 = o00 * my - o01 * mx;
      const float p10 = o11 * mz - o12 * my, p11 = o12 * mx - o01 * mz, p12 = o01 * my - o11 * mx;
      const float p20 = o12 * mz - o22 * my, p21 = o22 * mx - o02 * mz, p22 = o02 * my - o12 * mx;
      h[0] += o00; h[1] += o01; h[2] += o02;
      h[3] -= p00; h[4] -= p01; h[5] -= p02;
      h[6] += o11; h[7] += o12;
      h[8] -= p10; h[9] -= p11; h[10] -= p12;
      h[11] += o22;
      h[12] -= p20; h[13] -= p21; h[14] -= p22;
      h[15] = fmaf(mz, p10, fmaf(-my, p20, h[15]));
      h[16] = fmaf(mz, p11, fmaf(-my, p21, h[16]));
      h[17] = fmaf(mz, p12, fmaf(-my, p22, h[17]));
      h[18] = fmaf(mx, p21, fmaf(-mz, p01, h[18]));
      h[19] = fmaf(mx, p22, fmaf(-mz, p02, h[19]));
      h[20] = fmaf(my, p02, fmaf(-mx, p12, h[20]));
      bv[0] -= w0; bv[1] -= w1; bv[2] -= w2;
      bv[3] = fmaf(w1, mz, fmaf(-w2, my, bv[3]));
      bv[4] = fmaf(w2, mx, fmaf(-w0, mz, bv[4]));
      bv[5] = fmaf(w0, my, fmaf(-w1, mx, bv[5]));
    }
  }
  float acc = l;
#pragma unroll
  for (int k = 0; k < 21; ++k) acc += h[k];
#pragma unroll
  for (int k = 0; k < 6; ++k) acc += bv[k];
  if (acc == 1234.5f) out[0] = acc;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  float4 h[kPts * 3];
  for (int j = 0; j < kPts; ++j) {
    const float a = 0.01f * j;
    h[3 * j] = make_float4(5.f * cosf(a), 5.f * sinf(a), 0.3f * sinf(3 * a), 1e-3f);
    h[3 * j + 1] = make_float4(0.7f * cosf(a), 0.7f * sinf(a), 0.1f, 0.f);
    h[3 * j + 2] = make_float4(-0.5f * sinf(a), 0.5f * cosf(a), 0.4f, 0.f);
  }
  float4 hc[kPts * 4];
  for (int j = 0; j < kPts; ++j) {
    hc[4 * j] = h[3 * j];
    hc[4 * j + 1] = h[3 * j + 1];
    hc[4 * j + 2] = h[3 * j + 2];
    hc[4 * j + 3] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  float4* d;
  float* out;
  CK(cudaMalloc(&d, sizeof(h)));
  CK(cudaMalloc(&out, 16));
  CK(cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  const int blocks = sms * 4 * 4, reps = 16;  // 4 CTAs/SM resident, 4 waves
  CK(cudaMemcpyToSymbol(c_pts, hc, sizeof(hc)));
  static float hp[1024 * 32];
  for (int i = 0; i < 1024; ++i) {  // rotations about a tilted axis + payloads
    const float th = 1e-3f * i, c = cosf(th), s = sinf(th);
    float* q = hp + 32 * i;
    const float R[9] = {c, -s * 0.8f, s * 0.6f, s, c * 0.8f, -c * 0.6f, 0.f, 0.6f, 0.8f};
    q[0] = R[0]; q[1] = R[1]; q[2] = R[2]; q[3] = 0.3f;
    q[4] = R[3]; q[5] = R[4]; q[6] = R[5]; q[7] = 0.1f;
    q[8] = R[6]; q[9] = R[7]; q[10] = R[8]; q[11] = -0.2f;
    q[12] = 0.5f + th; q[13] = 0.2f; q[14] = 0.1f;
    q[15] = 0.6f; q[16] = 0.7f; q[17] = 0.01f; q[18] = 0.02f; q[19] = 0.8f; q[20] = 0.03f;
    q[21] = 0.6f; q[22] = 0.64f; q[23] = 0.48f; q[24] = 1.0f; q[25] = 1.001f;
  }
  float* dp;
  CK(cudaMalloc(&dp, sizeof(hp)));
  CK(cudaMemcpy(dp, hp, sizeof(hp), cudaMemcpyHostToDevice));
  printf("{\"results\": [");
  const char* names[12] = {"l only (smem)", "l+H+b (smem)", "l+H+b (scan in constant bank)",
                          "v17 body-frame plane l+H+b (constant bank)", "l only (constant bank)",
                          "l+H+b (smem) minB 2", "l+H+b (smem) minB 6", "l+H+b (smem) minB 8",
                          "v18 rotated-frame plane l+H+b (smem)", "v18 (constant bank)",
                          "v19 body-frame general l+H+b (constant bank)",
                          "v19 body-frame general l+H+b (smem)"};
  for (int variant = 0; variant < 12; ++variant) {
    auto run = [&]() {
      if (variant == 0) math_kernel<0, 0><<<blocks, 128>>>(d, reps, out, dp);
      if (variant == 1) math_kernel<1, 0><<<blocks, 128>>>(d, reps, out, dp);
      if (variant == 2) math_kernel<1, 1><<<blocks, 128>>>(d, reps, out, dp);
      if (variant == 3) v17_kernel<<<blocks, 128>>>(reps, out, dp);
      if (variant == 4) math_kernel<0, 1><<<blocks, 128>>>(d, reps, out, dp);
      if (variant == 5) math_kernel<1, 0, 2><<<blocks, 128>>>(d, reps, out, dp);
      if (variant == 6) math_kernel<1, 0, 6><<<blocks, 128>>>(d, reps, out, dp);
      if (variant == 7) math_kernel<1, 0, 8><<<blocks, 128>>>(d, reps, out, dp);
      if (variant == 8) v18_kernel<0><<<blocks, 128>>>(d, reps, out, dp);
      if (variant == 9) v18_kernel<1><<<blocks, 128>>>(d, reps, out, dp);
      if (variant == 10) v19_kernel<1><<<blocks, 128>>>(d, reps, out, dp);
      if (variant == 11) v19_kernel<0><<<blocks, 128>>>(d, reps, out, dp);
    };
    run();
    CK(cudaEventRecord(a));
    run();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, a, b));
    const double warp_points = (double)blocks * 4 * reps * kPts;
    const double smsp_cycles = ms * 1e-3 * 1.965e9 * sms * 4;
    printf("%s{\"variant\": \"%s\", \"ms\": %.3f, \"smsp_cycles_per_warp_point\": %.1f}",
           variant ? ", " : "", names[variant], ms, smsp_cycles / warp_points);
  }
  printf("]}\n");
  return 0;
}
