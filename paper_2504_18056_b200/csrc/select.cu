// select.cu — a1: neighbour keyframes, loop flag, relative poses (
// Fig.3).
//
// One thread per particle:
//   d_k = ||t_k^i - t_t^i||^2 with the pinned fp32 order fmaf(dz,dz,fmaf(dy,dy,dx*dx)) (R6, R27)
//   the nb = min(neighbor_count, K) smallest (d, k), ties -> lower id
//   loop_i = exists slot with id <= latest - gap (R5);  t_o = min slot id
//   kT = (T_k^i)^-1 T_t^i per slot, pinned fp32: R = Rk^T Rt, t = Rk^T (t_t - t_k),
//   each entry fmaf(x2,y2, fmaf(x1,y1, x0*y0)) (R27) — the same correspondences as the oracle.
// Writes one 64-byte work item per (particle, slot) for the sweep:
//   float4 rows {R00 R01 R02 tx}{R10 R11 R12 ty}{R20 R21 R22 tz}, int4 {kf, particle, flags, 0}
//   flags bit0: accumulate H~, b~ (slot in G, R4).
#include <cub/cub.cuh>

#include "mcs_internal.cuh"

namespace mcs {

// Lane-coherence sort key of a work item: the keyframe id in the top bits, then
// a 6-D Morton code of where the item's relative pose sends two reference points 16 m out on
// the x and y axes (a typical LiDAR range, which weighs rotation against translation the way
// the scan's own points do; 4 m / 8 m / 24 m / 32 m measured slower), at 1/6 m steps (5 bits
// per coordinate, wrapping every 5.3 m: one radix pass fewer than 6 bits at 1/16 m; 1/8 m
// steps 0.3 % slower once the sparse tables removed the probe chains).  Items that
// are adjacent in this order probe the same cells for the same scan point, so a warp's
// gathers coalesce and its hit/miss branches agree.
#ifndef MCS_MORTON_BITS
#define MCS_MORTON_BITS 5
#endif
#ifndef MCS_MORTON_REF
#define MCS_MORTON_REF 16.0f  // distance of the two reference points (m): a typical LiDAR range
#endif
#ifndef MCS_MORTON_SCALE
#define MCS_MORTON_SCALE 6.0f
#endif
#ifndef MCS_MORTON_PTS
#define MCS_MORTON_PTS 2  // reference points on the x, y (, z) axes
#endif
constexpr int kMortonBitsPerDim = MCS_MORTON_BITS;
#ifndef MCS_SELECT_UNROLL
#define MCS_SELECT_UNROLL 1  // the keyframe-distance loop of select_kernel, unrolled
#endif
constexpr int kSelectUnroll = MCS_SELECT_UNROLL;
#ifndef MCS_SORT_BITS
// the top 32 bits of the (keyframe, Morton) key are sorted: four radix passes instead of five
// (the finest Morton level of 3 of the 6 coordinates stays in input order).  C2 update 5.627 ->
// 5.626 ms, 12.5k particles 0.915 -> 0.907 ms; 24 bits costs the sweep its coherence (C2 5.83)
#define MCS_SORT_BITS 32
#endif
constexpr int kMortonDims = 3 * MCS_MORTON_PTS;
constexpr int kMortonBits = kMortonDims * kMortonBitsPerDim;

__device__ __forceinline__ unsigned long long coherence_key(int kf, const float* rel) {
  const float d = MCS_MORTON_REF;
  float q[kMortonDims];
#pragma unroll
  for (int p = 0; p < MCS_MORTON_PTS; ++p)
#pragma unroll
    for (int a = 0; a < 3; ++a) q[3 * p + a] = d * rel[4 * a + p] + rel[4 * a + 3];
  unsigned int c[kMortonDims];
#pragma unroll
  for (int k = 0; k < kMortonDims; ++k)
    c[k] = (unsigned int)__float2int_rd(q[k] * MCS_MORTON_SCALE) & ((1u << kMortonBitsPerDim) - 1u);
  unsigned long long m = 0ull;
#pragma unroll
  for (int b = kMortonBitsPerDim - 1; b >= 0; --b)
#pragma unroll
    for (int k = 0; k < kMortonDims; ++k) m = (m << 1) | ((c[k] >> b) & 1u);
  return ((unsigned long long)kf << kMortonBits) | m;
}

__global__ void select_kernel(const float* __restrict__ pose, int capN, int N,
                              const float* __restrict__ kfpose,
                              const float4* __restrict__ kft, int capK, int K, int nb_max,
                              int gap, int gn_all, int eval_mode, float4* __restrict__ items,
                              uint8_t* __restrict__ meta, int32_t* __restrict__ t_o_out,
                              unsigned long long* __restrict__ skeys, int32_t* __restrict__ sids,
                              unsigned long long inactive_key) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  float Tt[12];
#pragma unroll
  for (int e = 0; e < 12; ++e) Tt[e] = pose[(size_t)e * capN + i];
  const float* kp = kfpose + (size_t)i * capK * 12;
  const int nb = K < nb_max ? K : nb_max;
  float bd[kMaxNb];
  int bk[kMaxNb];
#pragma unroll
  for (int s = 0; s < kMaxNb; ++s) { bd[s] = 0.f; bk[s] = -1; }
  const float4* tk = kft + (size_t)i * capK;  // the keyframe translations (16 B each)
#pragma unroll kSelectUnroll
  for (int k = 0; k < K; ++k) {
    const float4 t4 = __ldg(tk + k);
    float dx = __fsub_rn(t4.x, Tt[3]);
    float dy = __fsub_rn(t4.y, Tt[7]);
    float dz = __fsub_rn(t4.z, Tt[11]);
    float d = __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
    // insertion into the sorted top-nb list; strict < keeps the lower id on ties
#pragma unroll
    for (int s = 0; s < kMaxNb; ++s) {
      if (s < nb && (bk[s] < 0 || d < bd[s])) {
        for (int u = kMaxNb - 1; u > s; --u) { bd[u] = bd[u - 1]; bk[u] = bk[u - 1]; }
        bd[s] = d;
        bk[s] = k;
        break;
      }
    }
  }
  const int latest = K - 1;
  int loop = 0, t_o = bk[0];
  for (int s = 0; s < nb; ++s) {
    loop |= (bk[s] <= latest - gap);
    t_o = bk[s] < t_o ? bk[s] : t_o;
  }
  meta[i] = (uint8_t)loop;
  t_o_out[i] = t_o;
  for (int s = 0; s < nb_max; ++s) {
    float4* it = items + 4 * ((size_t)s * capN + i);
    const int k = s < nb ? bk[s] : -1;
    MCS_DCHECK(k < K && (s >= nb || k >= 0));
    skeys[(size_t)s * N + i] = inactive_key;
    sids[(size_t)s * N + i] = s * capN + i;
    if (k < 0) {
      it[3] = make_float4(__int_as_float(-1), __int_as_float(i), __int_as_float(0), 0.f);
      continue;
    }
    const float* Tk = kp + 12 * k;
    float Rk[9], d[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
#pragma unroll
      for (int b = 0; b < 3; ++b) Rk[3 * a + b] = Tk[4 * a + b];
      d[a] = __fsub_rn(Tt[4 * a + 3], Tk[4 * a + 3]);
    }
    float rel[12];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
#pragma unroll
      for (int b = 0; b < 3; ++b)
        rel[4 * a + b] = __fmaf_rn(Rk[6 + a], Tt[8 + b],
                                   __fmaf_rn(Rk[3 + a], Tt[4 + b], __fmul_rn(Rk[a], Tt[b])));
      rel[4 * a + 3] =
          __fmaf_rn(Rk[6 + a], d[2], __fmaf_rn(Rk[3 + a], d[1], __fmul_rn(Rk[a], d[0])));
    }
    const int in_G = gn_all ? 1 : (k <= latest - gap);
    const int flags = eval_mode == kSelectEval ? 1 : (eval_mode == kSelectWeight ? 0 : (in_G ? 1 : 0));
    it[0] = make_float4(rel[0], rel[1], rel[2], rel[3]);
    it[1] = make_float4(rel[4], rel[5], rel[6], rel[7]);
    it[2] = make_float4(rel[8], rel[9], rel[10], rel[11]);
    it[3] = make_float4(__int_as_float(k), __int_as_float(i), __int_as_float(flags), 0.f);
    skeys[(size_t)s * N + i] = coherence_key(k, rel);
  }
}

static int sort_end_bit(int capK) {
  int b = 1;
  while ((1 << b) <= capK) ++b;  // room for kf in [0, capK] (capK = inactive)
  return kMortonBits + b;
}

size_t sort_temp_needed(int n, int capK) {
  size_t b = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, b, (unsigned long long*)nullptr,
                                  (unsigned long long*)nullptr, (int32_t*)nullptr,
                                  (int32_t*)nullptr, n, 0, sort_end_bit(capK));
  return b;
}

mcs_status launch_select(mcs_ctx* c, int mode) {
  const int N = c->N;
  const int nb_max = c->cfg.neighbor_count;
  const int end_bit = sort_end_bit(c->capK);
  const unsigned long long inactive = (end_bit >= 64) ? ~0ull : ((1ull << end_bit) - 1ull);
  select_kernel<<<(N + 127) / 128, 128, 0, c->stream>>>(
      c->d_pose, c->capN, N, c->d_kfpose, c->d_kft, c->capK, c->K, nb_max,
      c->cfg.loop_recency_gap,
      c->cfg.gn_slots == MCS_GN_ALL_SLOTS, mode, c->d_items, c->d_meta, c->d_to,
      c->d_skeys, c->d_sids, inactive);
  size_t tb = c->cub_temp_bytes;
  // MCS_SORT_BITS: the number of key bits sorted (the top ones; 0 = all)
  const int begin_bit = (MCS_SORT_BITS > 0 && end_bit > MCS_SORT_BITS) ? end_bit - MCS_SORT_BITS : 0;
  if (cub::DeviceRadixSort::SortPairs(c->d_cub_temp, tb, c->d_skeys, c->d_skeys_out, c->d_sids,
                                      c->d_order, nb_max * N, begin_bit, end_bit, c->stream) !=
      cudaSuccess)
    return MCS_E_CUDA;
  return cudaGetLastError() == cudaSuccess ? MCS_OK : MCS_E_CUDA;
}

}  // namespace mcs
