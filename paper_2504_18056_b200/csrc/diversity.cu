// diversity.cu — the neighbour-particle diversity term (flag; reading R35).
//
// The paper cites SVGD / GN-SVGD for "preserving sample diversity through neighbor particle
// information" and defines no term of its own (Eqs.5-10).  R35 takes SVGD's
// kernel-gradient (repulsive) term with an RBF kernel on the current-pose translations:
//   d_i = (2 / (h N)) sum_j (t_i - t_j) exp(-|t_i - t_j|^2 / h)     (all N particles, every rank)
// with t the translations at the start of the update, and after the GN step(s) moves every
// particle's translation by eta d_i in the world frame (rotations, keyframe poses and weights
// untouched).  Off (eta = 0) by default.
//
// Multi-GPU: the term needs every particle's translation — the one neighbour-particle statistic
// the update exchanges: each rank contributes its shard padded to the largest
// shard (an equal-count device allgather, in place), and every rank sums over the global index
// order, so the G-rank result equals the 1-rank result bit for bit.
//
// Kernel: all pairs, N-body style — each CTA stages tiles of 256 translations in shared memory
// and every thread sums its particle's term over them in fp64, j ascending (deterministic).
#include "mcs_internal.cuh"

namespace mcs {

constexpr int kDivT = 256;

// this rank's translations (fp64 of the fp32 poses) into its slot of the gathered array
__global__ void div_snapshot_kernel(const float* __restrict__ pose, int capN, int N,
                                    double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
#pragma unroll
  for (int a = 0; a < 3; ++a) out[3 * (size_t)i + a] = (double)pose[(size_t)(4 * a + 3) * capN + i];
}

// t_all: [world][maxn][3] (rank g's first n_g rows valid); local particle i = global gbase + i
__global__ void __launch_bounds__(kDivT) diversity_kernel(const double* __restrict__ t_all,
                                                          const int* __restrict__ n_rank,
                                                          int world, int maxn, long long n_total,
                                                          int me, int N, float* __restrict__ pose,
                                                          int capN, double eta, double h) {
  __shared__ double st[kDivT][3];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool act = i < N;
  const double* mine = t_all + 3 * ((size_t)me * maxn + (act ? i : 0));
  const double ti0 = mine[0], ti1 = mine[1], ti2 = mine[2];
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  for (int g = 0; g < world; ++g) {
    const int ng = n_rank[g];
    const double* tg = t_all + 3 * (size_t)g * maxn;
    for (int base = 0; base < ng; base += kDivT) {
      const int cnt = min(kDivT, ng - base);
      __syncthreads();
      if (threadIdx.x < cnt) {
        st[threadIdx.x][0] = tg[3 * (size_t)(base + threadIdx.x) + 0];
        st[threadIdx.x][1] = tg[3 * (size_t)(base + threadIdx.x) + 1];
        st[threadIdx.x][2] = tg[3 * (size_t)(base + threadIdx.x) + 2];
      }
      __syncthreads();
      if (act) {
        for (int j = 0; j < cnt; ++j) {
          const double dx = __dsub_rn(ti0, st[j][0]), dy = __dsub_rn(ti1, st[j][1]),
                       dz = __dsub_rn(ti2, st[j][2]);
          const double r2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)),
                                      __dmul_rn(dz, dz));
          const double k = exp(-r2 / h);  // as the definition (R35): no reciprocal
          a0 = __dadd_rn(a0, __dmul_rn(dx, k));
          a1 = __dadd_rn(a1, __dmul_rn(dy, k));
          a2 = __dadd_rn(a2, __dmul_rn(dz, k));
        }
      }
    }
  }
  if (!act) return;
  const double c = 2.0 / (h * (double)n_total);
  const double d[3] = {c * a0, c * a1, c * a2};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    float* tc = pose + (size_t)(4 * a + 3) * capN + i;
    *tc = (float)((double)*tc + eta * d[a]);
  }
}

mcs_status launch_diversity_snapshot(mcs_ctx* c) {
  double* t_all = c->d_tall;
  double* mine = t_all + 3 * (size_t)c->rank * c->div_maxn;
  div_snapshot_kernel<<<(c->N + kDivT - 1) / kDivT, kDivT, 0, c->stream>>>(c->d_pose, c->capN,
                                                                            c->N, mine);
  if (cudaGetLastError() != cudaSuccess) return MCS_E_CUDA;
  if (dist_active(c))  // in place: rank g's block lands at t_all + 3 g maxn
    MCS_TRY(dist_allgather_dev(c, mine, t_all, sizeof(double) * 3 * (size_t)c->div_maxn));
  return MCS_OK;
}

mcs_status launch_diversity_apply(mcs_ctx* c) {
  long long n_total = 0;
  for (long long v : c->n_per_rank) n_total += v;
  diversity_kernel<<<(c->N + kDivT - 1) / kDivT, kDivT, 0, c->stream>>>(
      c->d_tall, c->d_divn, c->world, c->div_maxn, n_total, c->rank, c->N, c->d_pose, c->capN,
      c->cfg.diversity_weight, c->cfg.diversity_bandwidth);
  return cudaGetLastError() == cudaSuccess ? MCS_OK : MCS_E_CUDA;
}

}  // namespace mcs
