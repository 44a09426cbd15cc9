// update.cu — a3: combine slots + Gauss-Newton current-pose update (Eqs.2, 5-7; P:114,
// P:125-135), fused with L += l and the first weight reduction (Eq.11);
// a4: keyframe-pose propagation (Eqs.8-10).
//
// a3, one thread per particle, fp64 from the fp32 sweep partials:
//   H_s = B_s^T H~_s B_s, b_s = B_s^T b~_s, B_s = blockdiag(kR_s, kR_s)  (body frame of T_t)
//   l_i = sum_s l_s - kappa sum_s (S - n_s)                    (Eq.2; R8)
//   H = sum_{s in G} H_s, b = sum_{s in G} b_s, g = -2b         (R3, R4)
//   loop_i: lambda = damping_rel tr(H)/6; psi = -(H + lambda I)^-1 b (Cholesky; R1, R11);
//           clamp ||psi|| <= step_clamp; T_t <- T_t exp(psi) (Eq.7) + one Newton
//           re-orthonormalisation step (R30); non-PD -> flag singular, no update.
// a4, one thread per (particle, keyframe): for updated particles and t_o <= k <= latest,
//   r_k = (D_k - D_{t_o}) / (D_now - D_{t_o}) (R14, R15); T_k <- T_k exp(r_k psi) (Eq.10, R16).
#include "mcs_internal.cuh"

#include <algorithm>
#include "reduce.cuh"
#include "se3.cuh"

namespace mcs {

__device__ __forceinline__ int up_idx(int r, int c) {  // r <= c
  return r * 6 - (r * (r - 1)) / 2 + (c - r);
}

struct CombineArgs {
  const float4* items;
  const double* part;    // sweep partials, SoA [kSlotWords][pstride]
  size_t pstride;
  int splits;            // point splits of the sweep (records [splits][kSlotWords][pstride])
  const uint8_t* meta;
  float* pose;
  double* L;
  double* l_out;
  double* psi;
  float* grad;
  float* hess;
  uint8_t* flags;
  double* partials;  // [2][grid]
  Scalars* scal;
  int capN, N, K, nb_max, S, gap, gn_all, eval_mode;
  int do_gn, do_weight;  // update mode: GN step (a3) and/or L += l with the a5 reduction
  double kappa, damping, clamp;
  // eval outputs (device, may be null)
  double* slot_l;
  float* slot_H21;
  float* slot_b6;
  int32_t* slot_n;
  int32_t* slot_kf;
  uint8_t* loop_out;
};

// One thread per particle, the slots in a loop: the better shape when the particles fill the
// GPU (the solve keeps every resident warp busy).
__global__ void __launch_bounds__(128) combine_serial_kernel(CombineArgs a) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  double l = -INFINITY, Lnew = -INFINITY;
  if (i < a.N) {
    const int nb = a.K < a.nb_max ? a.K : a.nb_max;
    const int latest = a.K - 1;
    double H[21], b[6];
#pragma unroll
    for (int k = 0; k < 21; ++k) H[k] = 0.0;
#pragma unroll
    for (int k = 0; k < 6; ++k) b[k] = 0.0;
    double lsum = 0.0;
    long long unmatched = 0;
    for (int s = 0; s < a.nb_max; ++s) {
      const size_t item = (size_t)s * a.capN + i;
      if (s >= nb) {
        if (a.eval_mode) {
          const size_t o = (size_t)i * a.nb_max + s;
          if (a.slot_l) a.slot_l[o] = 0.0;
          if (a.slot_n) a.slot_n[o] = 0;
          if (a.slot_kf) a.slot_kf[o] = -1;
          if (a.slot_H21) for (int k = 0; k < 21; ++k) a.slot_H21[o * 21 + k] = 0.f;
          if (a.slot_b6) for (int k = 0; k < 6; ++k) a.slot_b6[o * 6 + k] = 0.f;
        }
        continue;
      }
      const float4 r0 = a.items[4 * item + 0], r1 = a.items[4 * item + 1],
                   r2 = a.items[4 * item + 2], inf = a.items[4 * item + 3];
      const int kf = __float_as_int(inf.x);
      const double R[9] = {r0.x, r0.y, r0.z, r1.x, r1.y, r1.z, r2.x, r2.y, r2.z};
      // sweep partials, SoA: word k of item at part[k * pstride + item] (coalesced across i)
      // point splits: the same word of every split record, summed in split order (fp64)
      const double* pi = a.part + item;
      const size_t ps = a.pstride;
      auto o = [&](int k) {
        double v = pi[(size_t)k * ps];
        for (int q = 1; q < a.splits; ++q) v += pi[((size_t)q * kSlotWords + k) * ps];
        return v;
      };
      const double ls = o(0);
      const int ns = (int)o(1);
      const bool in_G = a.gn_all ? true : (kf <= latest - a.gap);
      lsum += ls;
      unmatched += a.S - ns;
      if (!a.eval_mode && !a.do_gn) continue;  // weighting-only pass: l is all it needs
      if (!(in_G || a.eval_mode)) continue;
      const size_t so = (size_t)i * a.nb_max + s;
      float* hs_out = (a.eval_mode && a.slot_H21) ? a.slot_H21 + so * 21 : nullptr;
      // H_s = B^T H~ B with B = blockdiag(R, R), block by block on the upper triangle only
      // (blocks (0,0), (0,1), (1,1); block (1,0) lies below the diagonal): T = H~_pq R,
      // H_s,pq = R^T T, accumulated straight into H (slots in G) / written out (eval)
#pragma unroll
      for (int p = 0; p < 2; ++p)
#pragma unroll
        for (int q = p; q < 2; ++q) {
          double Hb[9];
#pragma unroll
          for (int x = 0; x < 3; ++x)
#pragma unroll
            for (int y = 0; y < 3; ++y) {
              const int r = 3 * p + x, c = 3 * q + y;
              Hb[3 * x + y] = o(2 + (r <= c ? up_idx(r, c) : up_idx(c, r)));
            }
          double T[9];
#pragma unroll
          for (int x = 0; x < 3; ++x)
#pragma unroll
            for (int y = 0; y < 3; ++y)
              T[3 * x + y] = Hb[3 * x + 0] * R[0 * 3 + y] + Hb[3 * x + 1] * R[1 * 3 + y] +
                             Hb[3 * x + 2] * R[2 * 3 + y];
#pragma unroll
          for (int x = 0; x < 3; ++x)
#pragma unroll
            for (int y = 0; y < 3; ++y) {
              if (p == q && y < x) continue;
              const double v = R[0 * 3 + x] * T[0 * 3 + y] + R[1 * 3 + x] * T[1 * 3 + y] +
                               R[2 * 3 + x] * T[2 * 3 + y];
              const int u = up_idx(3 * p + x, 3 * q + y);
              if (in_G) H[u] += v;
              if (hs_out) hs_out[u] = (float)v;
            }
        }
      // b_s = B^T b~
#pragma unroll
      for (int p = 0; p < 2; ++p)
#pragma unroll
        for (int x = 0; x < 3; ++x) {
          const double v = R[0 * 3 + x] * o(23 + 3 * p + 0) + R[1 * 3 + x] * o(23 + 3 * p + 1) +
                           R[2 * 3 + x] * o(23 + 3 * p + 2);
          if (in_G) b[3 * p + x] += v;
          if (a.eval_mode && a.slot_b6) a.slot_b6[so * 6 + 3 * p + x] = (float)v;
        }
      if (a.eval_mode) {
        if (a.slot_l) a.slot_l[so] = ls;
        if (a.slot_n) a.slot_n[so] = ns;
        if (a.slot_kf) a.slot_kf[so] = kf;
      }
    }
    l = lsum - a.kappa * (double)unmatched;
    const uint8_t loop = a.meta[i] & 1;
    if (a.eval_mode) {
      if (a.loop_out) a.loop_out[i] = loop;
    } else if (a.do_gn) {
      uint8_t flags = loop;
      double psi[6] = {0, 0, 0, 0, 0, 0};
      // outputs that do not depend on the solve first (frees H's registers for it)
#pragma unroll
      for (int k = 0; k < 6; ++k) a.grad[(size_t)k * a.capN + i] = (float)(-2.0 * b[k]);
#pragma unroll
      for (int k = 0; k < 21; ++k) a.hess[(size_t)k * a.capN + i] = (float)H[k];
      if (loop) {
        // Eq.5 with Levenberg damping (R11): (H + lambda I) psi = -b via Cholesky, in place on
        // the packed lower triangle Lc[r(r+1)/2 + c] (fully unrolled: register-resident); a
        // non-positive pivot marks the system singular, the rest runs on a stand-in value
        const double tr = H[up_idx(0, 0)] + H[up_idx(1, 1)] + H[up_idx(2, 2)] +
                          H[up_idx(3, 3)] + H[up_idx(4, 4)] + H[up_idx(5, 5)];
        const double lam = a.damping * tr / 6.0;
        double Lc[21];
#pragma unroll
        for (int r = 0; r < 6; ++r)
#pragma unroll
          for (int c = 0; c <= r; ++c) Lc[r * (r + 1) / 2 + c] = H[up_idx(c, r)] + (r == c ? lam : 0.0);
        // (inner loops have constant trip counts with index guards so that every loop unrolls
        // and Lc stays in registers)
        bool ok = true;
#pragma unroll
        for (int j = 0; j < 6; ++j) {
          double d = Lc[j * (j + 1) / 2 + j];
#pragma unroll
          for (int k = 0; k < 6; ++k)
            if (k < j) d -= Lc[j * (j + 1) / 2 + k] * Lc[j * (j + 1) / 2 + k];
          ok = ok && (d > 0.0);
          const double ljj = sqrt(d > 0.0 ? d : 1.0);
          Lc[j * (j + 1) / 2 + j] = ljj;
#pragma unroll
          for (int r = 0; r < 6; ++r) {
            if (r <= j) continue;
            double t = Lc[r * (r + 1) / 2 + j];
#pragma unroll
            for (int k = 0; k < 6; ++k)
              if (k < j) t -= Lc[r * (r + 1) / 2 + k] * Lc[j * (j + 1) / 2 + k];
            Lc[r * (r + 1) / 2 + j] = t / ljj;
          }
        }
        if (!ok) {
          flags |= 4;
        } else {
          double z[6];
#pragma unroll
          for (int r = 0; r < 6; ++r) {
            double t = -b[r];
#pragma unroll
            for (int k = 0; k < 6; ++k)
              if (k < r) t -= Lc[r * (r + 1) / 2 + k] * z[k];
            z[r] = t / Lc[r * (r + 1) / 2 + r];
          }
#pragma unroll
          for (int rr = 0; rr < 6; ++rr) {
            const int r = 5 - rr;
            double t = z[r];
#pragma unroll
            for (int k = 0; k < 6; ++k)
              if (k > r) t -= Lc[k * (k + 1) / 2 + r] * psi[k];
            psi[r] = t / Lc[r * (r + 1) / 2 + r];
          }
          double nrm = 0.0;
#pragma unroll
          for (int k = 0; k < 6; ++k) nrm += psi[k] * psi[k];
          nrm = sqrt(nrm);
          if (nrm > a.clamp) {
#pragma unroll
            for (int k = 0; k < 6; ++k) psi[k] *= a.clamp / nrm;
            flags |= 16;
          }
          flags |= 2;
          bool nz = false;
#pragma unroll
          for (int k = 0; k < 6; ++k) nz |= (psi[k] != 0.0);
          if (nz) {
            float T[12];
#pragma unroll
            for (int e = 0; e < 12; ++e) T[e] = a.pose[(size_t)e * a.capN + i];
            pose_right_update(T, psi);
#pragma unroll
            for (int e = 0; e < 12; ++e) a.pose[(size_t)e * a.capN + i] = T[e];
          }
        }
      }
#pragma unroll
      for (int k = 0; k < 6; ++k) a.psi[(size_t)k * a.capN + i] = psi[k];
      a.flags[i] = flags;
    }
    if (!a.eval_mode && a.do_weight) {
      a.l_out[i] = l;
      Lnew = a.L[i] + l;  // Eq.11 in log space (R22)
      a.L[i] = Lnew;
    }
  }
  if (a.eval_mode || !a.do_weight) return;
  // first weight reduction: max L, max l  (a5)
  const double bm = block_reduce(Lnew, MaxOp(), -INFINITY);
  const double bl = block_reduce(l, MaxOp(), -INFINITY);
  if (threadIdx.x == 0) {
    a.partials[blockIdx.x] = bm;
    a.partials[gridDim.x + blockIdx.x] = bl;
  }
  if (last_block(&a.scal->counter[0])) {
    double m = -INFINITY, ls = -INFINITY;
    for (int k = threadIdx.x; k < (int)gridDim.x; k += blockDim.x) {
      m = fmax(m, a.partials[k]);
      ls = fmax(ls, a.partials[gridDim.x + k]);
    }
    m = block_reduce(m, MaxOp(), -INFINITY);
    ls = block_reduce(ls, MaxOp(), -INFINITY);
    if (threadIdx.x == 0) {
      a.scal->m = m;
      a.scal->lstar = ls;
    }
  }
}

// One block per kCombP particles and one thread per (slot, particle), for small shards where
// one thread per particle leaves the GPU mostly idle and a3 is latency-bound: the slot threads
// rotate their slot's H~, b~ back to the body frame (the bulk of a3's fp64 work) in parallel,
// the slot-0 threads then sum the slots in slot order (the same additions as the serial loop,
// so the result is bitwise that of combine_serial_kernel) and run the solve.
constexpr int kCombP = 32;
#ifndef MCS_COMBINE_SLOTS_BELOW
#define MCS_COMBINE_SLOTS_BELOW 40000  // particles per device below which a3 runs per slot
#endif  // (measured: a3 + a4 at 12.5k 0.118 -> 0.069 ms, 25k 0.122 -> 0.112; 50k 0.135 -> 0.156)

__global__ void __launch_bounds__(kCombP * kMaxNb) combine_slots_kernel(CombineArgs a) {
  const int il = threadIdx.x % kCombP, s = threadIdx.x / kCombP;  // particle lane, slot
  const int i = blockIdx.x * kCombP + il;
  __shared__ double sh_hb[kMaxNb][27][kCombP];  // rotated H_s (21) and b_s (6) per slot
  __shared__ double sh_ls[kMaxNb][kCombP];
  __shared__ int sh_ns[kMaxNb][kCombP];
  __shared__ unsigned char sh_g[kMaxNb][kCombP];  // bit0: in G, bit1: H_s / b_s present
  double l = -INFINITY, Lnew = -INFINITY;
  const int nb = a.K < a.nb_max ? a.K : a.nb_max;
  const int latest = a.K - 1;
  // ---- phase 1: slot s of particle i
  if (i < a.N && s < a.nb_max) {
    const size_t item = (size_t)s * a.capN + i;
    unsigned char g = 0;
    double ls = 0.0;
    int ns = 0;
    if (s >= nb) {
      if (a.eval_mode) {
        const size_t o = (size_t)i * a.nb_max + s;
        if (a.slot_l) a.slot_l[o] = 0.0;
        if (a.slot_n) a.slot_n[o] = 0;
        if (a.slot_kf) a.slot_kf[o] = -1;
        if (a.slot_H21) for (int k = 0; k < 21; ++k) a.slot_H21[o * 21 + k] = 0.f;
        if (a.slot_b6) for (int k = 0; k < 6; ++k) a.slot_b6[o * 6 + k] = 0.f;
      }
    } else {
      const float4 r0 = a.items[4 * item + 0], r1 = a.items[4 * item + 1],
                   r2 = a.items[4 * item + 2], inf = a.items[4 * item + 3];
      const int kf = __float_as_int(inf.x);
      const double R[9] = {r0.x, r0.y, r0.z, r1.x, r1.y, r1.z, r2.x, r2.y, r2.z};
      // sweep partials, SoA: word k of item at part[k * pstride + item] (coalesced across i)
      // point splits: the same word of every split record, summed in split order (fp64)
      const double* pi = a.part + item;
      const size_t ps = a.pstride;
      auto o = [&](int k) {
        double v = pi[(size_t)k * ps];
        for (int q = 1; q < a.splits; ++q) v += pi[((size_t)q * kSlotWords + k) * ps];
        return v;
      };
      ls = o(0);
      ns = (int)o(1);
      const bool in_G = a.gn_all ? true : (kf <= latest - a.gap);
      g = in_G ? 1 : 0;
      if ((a.eval_mode || a.do_gn) && (in_G || a.eval_mode)) {
        g |= 2;
        const size_t so = (size_t)i * a.nb_max + s;
        float* hs_out = (a.eval_mode && a.slot_H21) ? a.slot_H21 + so * 21 : nullptr;
        // H_s = B^T H~ B with B = blockdiag(R, R), block by block on the upper triangle only
        // (blocks (0,0), (0,1), (1,1); block (1,0) lies below the diagonal): T = H~_pq R,
        // H_s,pq = R^T T
#pragma unroll
        for (int p = 0; p < 2; ++p)
#pragma unroll
          for (int q = p; q < 2; ++q) {
            double Hb[9];
#pragma unroll
            for (int x = 0; x < 3; ++x)
#pragma unroll
              for (int y = 0; y < 3; ++y) {
                const int r = 3 * p + x, c = 3 * q + y;
                Hb[3 * x + y] = o(2 + (r <= c ? up_idx(r, c) : up_idx(c, r)));
              }
            double T[9];
#pragma unroll
            for (int x = 0; x < 3; ++x)
#pragma unroll
              for (int y = 0; y < 3; ++y)
                T[3 * x + y] = Hb[3 * x + 0] * R[0 * 3 + y] + Hb[3 * x + 1] * R[1 * 3 + y] +
                               Hb[3 * x + 2] * R[2 * 3 + y];
#pragma unroll
            for (int x = 0; x < 3; ++x)
#pragma unroll
              for (int y = 0; y < 3; ++y) {
                if (p == q && y < x) continue;
                const double v = R[0 * 3 + x] * T[0 * 3 + y] + R[1 * 3 + x] * T[1 * 3 + y] +
                                 R[2 * 3 + x] * T[2 * 3 + y];
                const int u = up_idx(3 * p + x, 3 * q + y);
                sh_hb[s][u][il] = v;
                if (hs_out) hs_out[u] = (float)v;
              }
          }
        // b_s = B^T b~
#pragma unroll
        for (int p = 0; p < 2; ++p)
#pragma unroll
          for (int x = 0; x < 3; ++x) {
            const double v = R[0 * 3 + x] * o(23 + 3 * p + 0) + R[1 * 3 + x] * o(23 + 3 * p + 1) +
                             R[2 * 3 + x] * o(23 + 3 * p + 2);
            sh_hb[s][21 + 3 * p + x][il] = v;
            if (a.eval_mode && a.slot_b6) a.slot_b6[so * 6 + 3 * p + x] = (float)v;
          }
      }
      if (a.eval_mode) {
        const size_t so = (size_t)i * a.nb_max + s;
        if (a.slot_l) a.slot_l[so] = ls;
        if (a.slot_n) a.slot_n[so] = ns;
        if (a.slot_kf) a.slot_kf[so] = kf;
      }
    }
    sh_ls[s][il] = ls;
    sh_ns[s][il] = ns;
    sh_g[s][il] = g;
  }
  __syncthreads();
  // ---- phase 2: the slot-0 thread of particle i sums the slots in slot order and solves
  if (s == 0 && i < a.N) {
    double H[21], b[6];
#pragma unroll
    for (int k = 0; k < 21; ++k) H[k] = 0.0;
#pragma unroll
    for (int k = 0; k < 6; ++k) b[k] = 0.0;
    double lsum = 0.0;
    long long unmatched = 0;
    for (int t = 0; t < nb; ++t) {
      lsum += sh_ls[t][il];
      unmatched += a.S - sh_ns[t][il];
      if ((sh_g[t][il] & 3) == 3) {  // in G, rotated
#pragma unroll
        for (int k = 0; k < 21; ++k) H[k] += sh_hb[t][k][il];
#pragma unroll
        for (int k = 0; k < 6; ++k) b[k] += sh_hb[t][21 + k][il];
      }
    }
    l = lsum - a.kappa * (double)unmatched;
    const uint8_t loop = a.meta[i] & 1;
    if (a.eval_mode) {
      if (a.loop_out) a.loop_out[i] = loop;
    } else if (a.do_gn) {
      uint8_t flags = loop;
      double psi[6] = {0, 0, 0, 0, 0, 0};
      // outputs that do not depend on the solve first (frees H's registers for it)
#pragma unroll
      for (int k = 0; k < 6; ++k) a.grad[(size_t)k * a.capN + i] = (float)(-2.0 * b[k]);
#pragma unroll
      for (int k = 0; k < 21; ++k) a.hess[(size_t)k * a.capN + i] = (float)H[k];
      if (loop) {
        // Eq.5 with Levenberg damping (R11): (H + lambda I) psi = -b via Cholesky, in place on
        // the packed lower triangle Lc[r(r+1)/2 + c] (fully unrolled: register-resident); a
        // non-positive pivot marks the system singular, the rest runs on a stand-in value
        const double tr = H[up_idx(0, 0)] + H[up_idx(1, 1)] + H[up_idx(2, 2)] +
                          H[up_idx(3, 3)] + H[up_idx(4, 4)] + H[up_idx(5, 5)];
        const double lam = a.damping * tr / 6.0;
        double Lc[21];
#pragma unroll
        for (int r = 0; r < 6; ++r)
#pragma unroll
          for (int c = 0; c <= r; ++c) Lc[r * (r + 1) / 2 + c] = H[up_idx(c, r)] + (r == c ? lam : 0.0);
        // (inner loops have constant trip counts with index guards so that every loop unrolls
        // and Lc stays in registers)
        bool ok = true;
#pragma unroll
        for (int j = 0; j < 6; ++j) {
          double d = Lc[j * (j + 1) / 2 + j];
#pragma unroll
          for (int k = 0; k < 6; ++k)
            if (k < j) d -= Lc[j * (j + 1) / 2 + k] * Lc[j * (j + 1) / 2 + k];
          ok = ok && (d > 0.0);
          const double ljj = sqrt(d > 0.0 ? d : 1.0);
          Lc[j * (j + 1) / 2 + j] = ljj;
#pragma unroll
          for (int r = 0; r < 6; ++r) {
            if (r <= j) continue;
            double t = Lc[r * (r + 1) / 2 + j];
#pragma unroll
            for (int k = 0; k < 6; ++k)
              if (k < j) t -= Lc[r * (r + 1) / 2 + k] * Lc[j * (j + 1) / 2 + k];
            Lc[r * (r + 1) / 2 + j] = t / ljj;
          }
        }
        if (!ok) {
          flags |= 4;
        } else {
          double z[6];
#pragma unroll
          for (int r = 0; r < 6; ++r) {
            double t = -b[r];
#pragma unroll
            for (int k = 0; k < 6; ++k)
              if (k < r) t -= Lc[r * (r + 1) / 2 + k] * z[k];
            z[r] = t / Lc[r * (r + 1) / 2 + r];
          }
#pragma unroll
          for (int rr = 0; rr < 6; ++rr) {
            const int r = 5 - rr;
            double t = z[r];
#pragma unroll
            for (int k = 0; k < 6; ++k)
              if (k > r) t -= Lc[k * (k + 1) / 2 + r] * psi[k];
            psi[r] = t / Lc[r * (r + 1) / 2 + r];
          }
          double nrm = 0.0;
#pragma unroll
          for (int k = 0; k < 6; ++k) nrm += psi[k] * psi[k];
          nrm = sqrt(nrm);
          if (nrm > a.clamp) {
#pragma unroll
            for (int k = 0; k < 6; ++k) psi[k] *= a.clamp / nrm;
            flags |= 16;
          }
          flags |= 2;
          bool nz = false;
#pragma unroll
          for (int k = 0; k < 6; ++k) nz |= (psi[k] != 0.0);
          if (nz) {
            float T[12];
#pragma unroll
            for (int e = 0; e < 12; ++e) T[e] = a.pose[(size_t)e * a.capN + i];
            pose_right_update(T, psi);
#pragma unroll
            for (int e = 0; e < 12; ++e) a.pose[(size_t)e * a.capN + i] = T[e];
          }
        }
      }
#pragma unroll
      for (int k = 0; k < 6; ++k) a.psi[(size_t)k * a.capN + i] = psi[k];
      a.flags[i] = flags;
    }
    if (!a.eval_mode && a.do_weight) {
      a.l_out[i] = l;
      Lnew = a.L[i] + l;  // Eq.11 in log space (R22)
      a.L[i] = Lnew;
    }
  }
  if (a.eval_mode || !a.do_weight) return;
  // first weight reduction: max L, max l  (a5)
  const double bm = block_reduce(Lnew, MaxOp(), -INFINITY);
  const double bl = block_reduce(l, MaxOp(), -INFINITY);
  if (threadIdx.x == 0) {
    a.partials[blockIdx.x] = bm;
    a.partials[gridDim.x + blockIdx.x] = bl;
  }
  if (last_block(&a.scal->counter[0])) {
    double m = -INFINITY, ls = -INFINITY;
    for (int k = threadIdx.x; k < (int)gridDim.x; k += blockDim.x) {
      m = fmax(m, a.partials[k]);
      ls = fmax(ls, a.partials[gridDim.x + k]);
    }
    m = block_reduce(m, MaxOp(), -INFINITY);
    ls = block_reduce(ls, MaxOp(), -INFINITY);
    if (threadIdx.x == 0) {
      a.scal->m = m;
      a.scal->lstar = ls;
    }
  }
}

void launch_combine(mcs_ctx* c, int S, int mode, double* slot_l, float* slot_H21,
                    float* slot_b6, int32_t* slot_n, int32_t* slot_kf, uint8_t* loop_out) {
  const bool eval_mode = mode == kCombineEval;
  CombineArgs a;
  a.items = c->d_items;
  a.part = c->d_part;
  a.pstride = (size_t)c->cfg.neighbor_count * c->capN;
  a.splits = c->cur_splits;
  a.meta = c->d_meta;
  a.pose = c->d_pose;
  a.L = c->d_L;
  a.l_out = c->d_l;
  a.psi = c->d_psi;
  a.grad = c->d_grad;
  a.hess = c->d_hess;
  a.flags = c->d_flags;
  a.partials = c->d_partials;
  a.scal = c->d_scal;
  a.capN = c->capN;
  a.N = c->N;
  a.K = c->K;
  a.nb_max = c->cfg.neighbor_count;
  a.S = S;
  a.gap = c->cfg.loop_recency_gap;
  a.gn_all = c->cfg.gn_slots == MCS_GN_ALL_SLOTS;
  a.eval_mode = eval_mode ? 1 : 0;
  a.do_gn = (mode == kCombineUpdateWeight || mode == kCombineUpdate) ? 1 : 0;
  a.do_weight = (mode == kCombineUpdateWeight || mode == kCombineWeight) ? 1 : 0;
  a.kappa = c->cfg.unmatched_penalty;
  a.damping = c->cfg.damping_rel;
  a.clamp = c->cfg.step_clamp;
  a.slot_l = slot_l;
  a.slot_H21 = slot_H21;
  a.slot_b6 = slot_b6;
  a.slot_n = slot_n;
  a.slot_kf = slot_kf;
  a.loop_out = loop_out;
  if (c->N >= MCS_COMBINE_SLOTS_BELOW) {
    combine_serial_kernel<<<(c->N + 127) / 128, 128, 0, c->stream>>>(a);
  } else {
    combine_slots_kernel<<<(c->N + kCombP - 1) / kCombP, kCombP * a.nb_max, 0, c->stream>>>(a);
  }
}

// One warp per 32 consecutive particles (grid-stride): each lane decides for its particle
// whether a4 applies (looped and updated; survivor / dead per mode; D_now > D_{t_o}) and how
// many keyframes it moves (t_o .. K-1), a warp scan flattens the (particle, keyframe) pairs of
// the warp, and the lanes take the pairs 32 at a time.  Only the work that exists is spread over
// the lanes: at C2 (one survivor) a4 is a check per particle, not a thread per (particle,
// keyframe) — N K threads cost ~0.1 ms at C3's 200 keyframes even when they all return.
__global__ void __launch_bounds__(256) propagate_kernel(
    float* __restrict__ kfpose, float4* __restrict__ kft, int capK, int K, int N,
    const uint8_t* __restrict__ flags,
    const int32_t* __restrict__ to, const double* __restrict__ psi, int capN,
    const double* __restrict__ D, const Scalars* __restrict__ sc, int mode,
    const double* __restrict__ l, const double* __restrict__ e, double rel_floor,
    double post_floor) {
  if (mode == kPropIfDegenerate && sc->status != (int)MCS_E_DEGENERATE) return;  // usual case
  const int lane = threadIdx.x & 31;
  const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  const double D_now = sc->D_now;
  for (long long base = gw * 32; base < N; base += nw * 32) {
    const long long i = base + lane;
    int cnt = 0, t_o = 0;
    double den = 0.0;
    if (i < N && (flags[i] & 2)) {
      bool act = true;
      if (mode != kPropAll) {  // kPropSurvivors: a dead particle's keyframe poses are its
        // donor's (a6); kPropIfDegenerate: no survivor, a6 kept every state
        const bool dead = particle_dead(l[i], sc->lstar, e[i], sc->S, rel_floor, post_floor);
        act = (mode == kPropSurvivors) ? !dead : dead;
      }
      if (act) {
        t_o = to[i];
        den = D_now - D[t_o];
        if (den > 0.0) cnt = K - t_o;  // keyframes t_o .. K-1; older ones untouched (R15)
      }
    }
    int inc = cnt;  // inclusive scan of the pair counts over the warp
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += v;
    }
    const int total = __shfl_sync(0xffffffffu, inc, 31);
    for (int p0 = 0; p0 < total; p0 += 32) {  // warp-uniform trip count
      const int p = p0 + lane;
      int j = 0;  // owner lane: the first with inc_j > p
#pragma unroll
      for (int step = 16; step > 0; step >>= 1) {
        const int v = __shfl_sync(0xffffffffu, inc, j + step - 1);
        if (v <= p) j += step;
      }
      const int inc_j = __shfl_sync(0xffffffffu, inc, j);
      const int cnt_j = __shfl_sync(0xffffffffu, cnt, j);
      const int to_j = __shfl_sync(0xffffffffu, t_o, j);
      const double den_j = __shfl_sync(0xffffffffu, den, j);
      if (p >= total) continue;
      const int k = to_j + (p - (inc_j - cnt_j));
      const long long ij = base + j;
      const double r = (D[k] - D[to_j]) / den_j;  // Eqs.8-9 (R14)
      if (r == 0.0) continue;                      // k = t_o (and equal path lengths)
      double xi[6];
#pragma unroll
      for (int c = 0; c < 6; ++c) xi[c] = r * psi[(size_t)c * capN + ij];
      MCS_DCHECK(k >= 0 && k < K && K <= capK && ij < N);
      float* Tk = kfpose + ((size_t)ij * capK + k) * 12;
      float T[12];
      const float4* p4 = reinterpret_cast<const float4*>(Tk);
      const float4 v0 = p4[0], v1 = p4[1], v2 = p4[2];
      T[0] = v0.x; T[1] = v0.y; T[2] = v0.z; T[3] = v0.w;
      T[4] = v1.x; T[5] = v1.y; T[6] = v1.z; T[7] = v1.w;
      T[8] = v2.x; T[9] = v2.y; T[10] = v2.z; T[11] = v2.w;
      pose_right_update(T, xi);  // Eq.10
      float4* q4 = reinterpret_cast<float4*>(Tk);
      q4[0] = make_float4(T[0], T[1], T[2], T[3]);
      q4[1] = make_float4(T[4], T[5], T[6], T[7]);
      q4[2] = make_float4(T[8], T[9], T[10], T[11]);
      kft[(size_t)ij * capK + k] = make_float4(T[3], T[7], T[11], 0.f);
    }
  }
}

void launch_propagate(mcs_ctx* c, int mode) {
  if ((long long)c->N * c->K == 0) return;
  const long long warps = (c->N + 31) / 32;
  const int grid = (int)std::min<long long>((warps + 7) / 8, 148LL * 16);
  propagate_kernel<<<grid, 256, 0, c->stream>>>(c->d_kfpose, c->d_kft, c->capK, c->K, c->N,
                                                c->d_flags,
                                                c->d_to, c->d_psi, c->capN, c->d_D, c->d_scal,
                                                mode, c->d_l, c->d_e, c->cfg.loglik_rel_floor,
                                                c->cfg.posterior_floor);
}

// the per-update scalars, by value at launch (outside any captured graph)
__global__ void set_params_kernel(Scalars* sc, double D_now, unsigned int U) {
  sc->D_now = D_now;
  sc->U = U;
}

void launch_set_params(mcs_ctx* c, double D_now, uint32_t U) {
  set_params_kernel<<<1, 1, 0, c->stream>>>(c->d_scal, D_now, U);
}

}  // namespace mcs
