// se3.cuh — fp64 SE(3) exponential and the right-applied pose update shared by a3 / a4
// (update.cu) and the prediction step (predict.cu).  Right perturbation, twist (rho, phi) (R2).
#pragma once
#include <cuda_runtime.h>

namespace mcs {

__device__ __forceinline__ void se3_exp_d(const double xi[6], double T[12]) {
  const double px = xi[3], py = xi[4], pz = xi[5];
  const double th2 = px * px + py * py + pz * pz;
  const double th = sqrt(th2);
  double A, B, C;
  if (th < 1e-4) {
    A = 1.0 - th2 / 6.0 + th2 * th2 / 120.0;
    B = 0.5 - th2 / 24.0 + th2 * th2 / 720.0;
    C = 1.0 / 6.0 - th2 / 120.0 + th2 * th2 / 5040.0;
  } else {
    double s, c;
    sincos(th, &s, &c);
    A = s / th;
    B = (1.0 - c) / th2;
    C = (th - s) / (th2 * th);
  }
  const double W[9] = {0.0, -pz, py, pz, 0.0, -px, -py, px, 0.0};
  double W2[9];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b)
      W2[3 * a + b] = W[3 * a] * W[b] + W[3 * a + 1] * W[3 + b] + W[3 * a + 2] * W[6 + b];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    double v[3];
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      const double I = (a == b) ? 1.0 : 0.0;
      T[4 * a + b] = I + A * W[3 * a + b] + B * W2[3 * a + b];
      v[b] = I + B * W[3 * a + b] + C * W2[3 * a + b];
    }
    T[4 * a + 3] = v[0] * xi[0] + v[1] * xi[1] + v[2] * xi[2];
  }
}

// T32 <- round_fp32( Newton( T32 * exp(xi) ) )   (Eq.7 / Eq.10, R23, R30)
__device__ __forceinline__ void pose_right_update(float T32[12], const double xi[6]) {
  double E[12], TE[12];
  se3_exp_d(xi, E);
#pragma unroll
  for (int a = 0; a < 3; ++a) {
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      double s = (b == 3) ? (double)T32[4 * a + 3] : 0.0;
#pragma unroll
      for (int c = 0; c < 3; ++c) s += (double)T32[4 * a + c] * E[4 * c + b];
      TE[4 * a + b] = s;
    }
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
      T32[4 * a + b] = (float)(0.5 * s);
    }
    T32[4 * a + 3] = (float)TE[4 * a + 3];
  }
}

}  // namespace mcs
