// dist.cu — host-side plan of the multi-GPU exchange steps of a6.
//
// Particles are sharded into contiguous global index ranges.  After the weights (a5) every rank
// knows its survivor-ladder total Q_g and dead count D_g; an allgather of (Q_g, D_g) lets every
// rank evaluate the GLOBAL systematic-respawn count formula (R18) on its own survivors.  The
// r-th global clone (donors in ascending global index, with multiplicity) goes to the r-th
// global dead slot (ascending global index).  These functions are pure functions of the
// allgathered per-rank totals, so every rank computes the same plan.
#include <stdint.h>

#include "../../include/mcs.h"

namespace {

__int128 ceil_div(__int128 num, __int128 den) {  // den > 0
  __int128 q = num / den;
  if (num > 0 && q * den != num) q += 1;
  return q;
}

// n(c) = #{draws r in [0, D) : (r + U/2^32) Q / D < c}   (R18)
int64_t draws_below(unsigned __int128 c, int64_t D, unsigned __int128 Q, uint32_t U) {
  const __int128 num = (__int128)c * D * ((__int128)1 << 32) - (__int128)U * (__int128)Q;
  const __int128 den = (__int128)Q * ((__int128)1 << 32);
  __int128 v = ceil_div(num, den);
  if (v < 0) v = 0;
  if (v > D) v = D;
  return (int64_t)v;
}

}  // namespace

extern "C" {

mcs_status mcs_plan_ladder(int32_t world, const uint64_t* Q_per_rank, const int64_t* D_per_rank,
                           uint32_t u, uint64_t* q_offset, int64_t* d_offset,
                           int64_t* clones_per_rank, uint64_t* Q_total, int64_t* D_total) {
  if (world < 1 || !Q_per_rank || !D_per_rank) return MCS_E_INVALID_ARG;
  unsigned __int128 Q = 0;
  int64_t D = 0;
  for (int32_t g = 0; g < world; ++g) {
    if (D_per_rank[g] < 0) return MCS_E_INVALID_ARG;
    if (q_offset) q_offset[g] = (uint64_t)Q;
    if (d_offset) d_offset[g] = D;
    Q += Q_per_rank[g];
    D += D_per_rank[g];
  }
  if (Q >> 64) return MCS_E_CAPACITY;  // the exact ladder needs Q < 2^64 (R18)
  if (Q_total) *Q_total = (uint64_t)Q;
  if (D_total) *D_total = D;
  if (clones_per_rank) {
    unsigned __int128 c = 0;
    for (int32_t g = 0; g < world; ++g) {
      const unsigned __int128 c1 = c + Q_per_rank[g];
      clones_per_rank[g] = (D > 0 && Q > 0) ? draws_below(c1, D, Q, u) - draws_below(c, D, Q, u)
                                            : 0;
      c = c1;
    }
  }
  return (D > 0 && Q == 0) ? MCS_E_DEGENERATE : MCS_OK;
}

mcs_status mcs_plan_migration(int32_t world, const int64_t* clones_per_rank,
                              const int64_t* dead_per_rank, int64_t* send_counts) {
  if (world < 1 || !clones_per_rank || !dead_per_rank || !send_counts) return MCS_E_INVALID_ARG;
  int64_t tc = 0, td = 0;
  for (int32_t g = 0; g < world; ++g) {
    if (clones_per_rank[g] < 0 || dead_per_rank[g] < 0) return MCS_E_INVALID_ARG;
    tc += clones_per_rank[g];
    td += dead_per_rank[g];
  }
  if (tc != td) return MCS_E_INVALID_ARG;
  int64_t cs = 0;
  for (int32_t src = 0; src < world; ++src) {
    const int64_t c0 = cs, c1 = cs + clones_per_rank[src];
    int64_t ds = 0;
    for (int32_t dst = 0; dst < world; ++dst) {
      const int64_t d0 = ds, d1 = ds + dead_per_rank[dst];
      const int64_t lo = c0 > d0 ? c0 : d0, hi = c1 < d1 ? c1 : d1;
      send_counts[(size_t)src * world + dst] = hi > lo ? hi - lo : 0;
      ds = d1;
    }
    cs = c1;
  }
  return MCS_OK;
}

}  // extern "C"
