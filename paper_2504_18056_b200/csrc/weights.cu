// weights.cu — a5: importance weights (Eq.11) as a max-subtracted log-sum-exp in
// fp64 (R22); a6: dead-particle pruning + respawn (R17-R21); a7: representative
// (P:206).  Single device or one shard of a multi-GPU run.
//
//   m = max L (from a3), e_i = exp(L_i - m), S = sum e (fixed tree), w_i = e_i / S
//   dead_i = (l_i - max l < rel_floor) or (w_i < posterior_floor)            (R17)
//   survivors' rungs q_i = floor(e_i 2^32), dead rungs 0; C = inclusive scan (exact uint64)
//   n(c) = clamp(ceil((c D 2^32 - U Q) / (Q 2^32)), 0, D)  in signed 128-bit  (R18)
//   draw r is made by the survivor j with n(C_{j-1}) <= r < n(C_j) and fills the r-th dead slot
//   clone T_t, every T_k and L (R19, R20); re-normalise; representative = argmax w, ties low.
// Across ranks every quantity above is global: m, l*, S are all-reduced, the ladder offsets and
// totals come from an allgather of (Q_g, D_g), and clones whose dead slot lives on another rank
// travel as packed particle states.
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "mcs_internal.cuh"
#include "reduce.cuh"

namespace mcs {

struct Rung {
  unsigned long long C;
  unsigned int d;
  unsigned int pad;
};
struct RungSum {
  __host__ __device__ Rung operator()(const Rung& a, const Rung& b) const {
    Rung r;
    r.C = a.C + b.C;
    r.d = a.d + b.d;
    r.pad = 0;
    return r;
  }
};

constexpr int kWT = 256;

__global__ void __launch_bounds__(kWT) exp_sum_kernel(const double* __restrict__ L, int N,
                                                      const double* __restrict__ m_ptr,
                                                      double* __restrict__ e,
                                                      double* __restrict__ partials,
                                                      double* __restrict__ S_out,
                                                      unsigned int* counter) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const double m = *m_ptr;
  double v = 0.0;
  if (i < N) {
    v = exp(L[i] - m);
    e[i] = v;
  }
  const double bs = block_reduce(v, SumOp(), 0.0);
  if (threadIdx.x == 0) partials[blockIdx.x] = bs;
  if (last_block(counter)) {
    double s = 0.0;
    for (int k = threadIdx.x; k < (int)gridDim.x; k += blockDim.x) s += partials[k];
    s = block_reduce(s, SumOp(), 0.0);
    if (threadIdx.x == 0) *S_out = s;
  }
}

__global__ void dead_kernel(const double* __restrict__ e, const double* __restrict__ l, int N,
                            const Scalars* __restrict__ sc, double rel_floor, double post_floor,
                            double* __restrict__ w, uint8_t* __restrict__ flags,
                            Rung* __restrict__ rung) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const double wi = e[i] / sc->S;
  w[i] = wi;
  const bool dead = (l[i] - sc->lstar < rel_floor) || (wi < post_floor);
  if (dead) flags[i] |= 8;
  Rung r;
  r.C = dead ? 0ull : (unsigned long long)floor(e[i] * 4294967296.0);
  r.d = dead ? 1u : 0u;
  r.pad = 0;
  rung[i] = r;
}

__global__ void rung_from_inputs_kernel(const double* __restrict__ e,
                                        const uint8_t* __restrict__ dead, int N,
                                        Rung* __restrict__ rung) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  Rung r;
  r.C = dead[i] ? 0ull : (unsigned long long)floor(e[i] * 4294967296.0);
  r.d = dead[i] ? 1u : 0u;
  r.pad = 0;
  rung[i] = r;
}

// local totals; on a single device also the (trivial) global plan
__global__ void totals_kernel(const Rung* __restrict__ scan, int N, int single, Scalars* sc) {
  const Rung last = scan[N - 1];
  sc->Q = last.C;
  sc->D = (long long)last.d;
  if (single) {
    const bool degenerate = last.d > 0 && last.C == 0ull;
    sc->Q_tot = last.C;
    sc->D_tot = (long long)last.d;
    sc->q_off = 0;
    sc->d_off = 0;
    sc->clone_off = 0;
    sc->clones = degenerate ? 0 : (long long)last.d;
    sc->status = degenerate ? (int)MCS_E_DEGENERATE : 0;
  }
}

__device__ __forceinline__ long long draws_below(unsigned long long c, long long D,
                                                 unsigned long long Q, unsigned int U) {
  const __int128 num = (__int128)c * (__int128)D * ((__int128)1 << 32) - (__int128)U * (__int128)Q;
  const __int128 den = (__int128)Q * ((__int128)1 << 32);
  __int128 q = num / den;
  if (num > 0 && q * den != num) q += 1;  // ceil for den > 0
  if (q < 0) q = 0;
  if (q > D) q = D;
  return (long long)q;
}

// n(C_i) on the GLOBAL ladder for every local particle; compacted list of local dead slots
__global__ void ncum_dead_kernel(const Rung* __restrict__ scan, int N,
                                 const Scalars* __restrict__ sc, long long* __restrict__ ncum, int32_t* __restrict__ dead_list,
                                 int32_t* __restrict__ donor_local, int32_t* __restrict__ donor_g) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const Rung s = scan[i];
  const Rung prev = i > 0 ? scan[i - 1] : Rung{0ull, 0u, 0u};
  MCS_DCHECK(s.d >= prev.d && s.d - prev.d <= 1u && s.d <= (unsigned)N);
  if (s.d != prev.d) dead_list[s.d - 1] = i;  // this particle is dead
  donor_local[i] = -1;
  if (donor_g) donor_g[i] = -1;
  if (sc->D_tot == 0 || sc->Q_tot == 0) return;
  ncum[i] = draws_below(sc->q_off + s.C, sc->D_tot, sc->Q_tot, sc->U);
}

// R34 (flag clone_split): a survivor with c draws shares its weight with its clones; it and
// each clone get L - ln(1 + c).  Runs before pack/clone, which copy the adjusted L.
__global__ void split_kernel(const long long* __restrict__ ncum, int N,
                             const Scalars* __restrict__ sc, double* __restrict__ L) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N || sc->D_tot == 0 || sc->Q_tot == 0) return;
  const long long prev =
      i > 0 ? ncum[i - 1] : draws_below(sc->q_off, sc->D_tot, sc->Q_tot, sc->U);
  const long long copies = ncum[i] - prev;
  if (copies > 0) L[i] -= log((double)(1 + copies));
}

// one thread per draw made by this rank's survivors: find the donor (binary search on the
// monotone n(C)), then either record a local clone or queue the donor for a remote rank.
// plan (world > 1): [0..G] dead offsets, [G+1..2G+1] send item offsets, [4(G+1)..] first draw
// sent to each peer.
__global__ void draws_kernel(const long long* __restrict__ ncum, int N,
                             const Scalars* __restrict__ sc, int world, int me, long long gbase,
                             const long long* __restrict__ plan,
                             const int32_t* __restrict__ dead_list,
                             int32_t* __restrict__ donor_local, int32_t* __restrict__ donor_g,
                             int32_t* __restrict__ pack_src) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= sc->clones) return;
  const long long R = sc->clone_off + t;
  int lo = 0, hi = N - 1;  // first j with ncum[j] > R
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (ncum[mid] > R) hi = mid; else lo = mid + 1;
  }
  const int j = lo;
  MCS_DCHECK(j >= 0 && j < N && ncum[j] > R && (j == 0 || ncum[j - 1] <= R));
  int dst = me;
  if (world > 1) {
    const long long* doffs = plan;
    int a = 0, b = world - 1;  // last rank with doffs[rank] <= R
    while (a < b) {
      const int mid = (a + b + 1) >> 1;
      if (doffs[mid] <= R) a = mid; else b = mid - 1;
    }
    dst = a;
  }
  if (dst == me) {
    MCS_DCHECK(R - sc->d_off >= 0 && R - sc->d_off < N);
    const int slot = dead_list[R - sc->d_off];
    MCS_DCHECK(slot >= 0 && slot < N && slot != j);
    donor_local[slot] = j;
    if (donor_g) donor_g[slot] = (int32_t)(gbase + j);
  } else {
    const long long* send_off = plan + (world + 1);
    const long long* sfirst = plan + 4 * (world + 1);
    pack_src[send_off[dst] + (R - sfirst[dst])] = j;
  }
}

// Peer-direct migration (cfg.peer_migration, world > 1): one warp per draw made by this rank's
// survivors.  A clone whose dead slot is local is recorded for clone_kernel; one whose slot is
// on rank p is written straight into p's state (its dead list read over peer memory): pose,
// every keyframe pose, L and the global donor index -- the pack / send / unpack of the
// transport path fused into the kernel that decides the transfer.
__global__ void draws_p2p_kernel(const long long* __restrict__ ncum, int N,
                                 const Scalars* __restrict__ sc, int world, int me,
                                 long long gbase, const long long* __restrict__ plan,
                                 const int32_t* __restrict__ dead_list,
                                 int32_t* __restrict__ donor_local, int32_t* __restrict__ donor_g,
                                 const PeerView* __restrict__ peers, int K,
                                 const float* __restrict__ pose, const float* __restrict__ kfpose,
                                 const double* __restrict__ L, int capN, int capK) {
  const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= sc->clones) return;
  const long long R = sc->clone_off + w;
  int lo = 0, hi = N - 1;  // first j with ncum[j] > R (every lane the same: broadcast loads)
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (ncum[mid] > R) hi = mid; else lo = mid + 1;
  }
  const int j = lo;
  MCS_DCHECK(j >= 0 && j < N && ncum[j] > R && (j == 0 || ncum[j - 1] <= R));
  const long long* doffs = plan;
  int a = 0, b = world - 1;  // destination: last rank with doffs[rank] <= R
  while (a < b) {
    const int mid = (a + b + 1) >> 1;
    if (doffs[mid] <= R) a = mid; else b = mid - 1;
  }
  if (a == me) {
    if (lane == 0) {
      const int slot = dead_list[R - sc->d_off];
      MCS_DCHECK(slot >= 0 && slot < N && slot != j);
      donor_local[slot] = j;
      donor_g[slot] = (int32_t)(gbase + j);
    }
    return;
  }
  const PeerView P = peers[a];
  const int slot = P.dead_list[R - doffs[a]];
  MCS_DCHECK(slot >= 0 && slot < P.capN);
  if (lane < 12) P.pose[(size_t)lane * P.capN + slot] = pose[(size_t)lane * capN + j];
  const float4* src = reinterpret_cast<const float4*>(kfpose + (size_t)j * capK * 12);
  float4* dst = reinterpret_cast<float4*>(P.kfpose + (size_t)slot * P.capK * 12);
  for (int k = lane; k < 3 * K; k += 32) dst[k] = src[k];
  if (lane == 0) {
    P.L[slot] = L[j];
    P.donor_g[slot] = (int32_t)(gbase + j);
  }
  __threadfence_system();  // the stores are visible to the peer before this rank's barrier
}

__global__ void clone_kernel(const int32_t* __restrict__ donor, int N, int K, int capK, int capN,
                             float* __restrict__ pose, float* __restrict__ kfpose,
                             double* __restrict__ L) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int KK = K + 1;
  if (t >= (long long)N * KK) return;
  const int i = (int)(t / KK), k = (int)(t - (long long)i * KK);
  const int d = donor[i];
  if (d < 0) return;
  MCS_DCHECK(d < N && donor[d] < 0);  // a donor is a survivor, never itself overwritten
  if (k == K) {
#pragma unroll
    for (int e = 0; e < 12; ++e) pose[(size_t)e * capN + i] = pose[(size_t)e * capN + d];
    L[i] = L[d];
  } else {
    const float4* src = reinterpret_cast<const float4*>(kfpose + ((size_t)d * capK + k) * 12);
    float4* dst = reinterpret_cast<float4*>(kfpose + ((size_t)i * capK + k) * 12);
    dst[0] = src[0];
    dst[1] = src[1];
    dst[2] = src[2];
  }
}

// packed particle state: [pose 12][K keyframe poses x 12][L (2 words)][global donor (2 words)]
__host__ __device__ inline int state_floats(int K) { return 12 + 12 * K + 4; }

__global__ void pack_kernel(const int32_t* __restrict__ pack_src, long long n_items, int K,
                            int capK, int capN, long long gbase, const float* __restrict__ pose,
                            const float* __restrict__ kfpose, const double* __restrict__ L,
                            float* __restrict__ out) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int KK = K + 1;
  if (t >= n_items * KK) return;
  const long long it = t / KK;
  const int k = (int)(t - it * KK);
  const int j = pack_src[it];
  MCS_DCHECK(j >= 0 && j < capN);
  float* o = out + it * state_floats(K);
  if (k == K) {
    for (int e = 0; e < 12; ++e) o[e] = pose[(size_t)e * capN + j];
    double* od = reinterpret_cast<double*>(o + 12 + 12 * K);
    od[0] = L[j];
    long long* og = reinterpret_cast<long long*>(o + 12 + 12 * K + 2);
    og[0] = gbase + j;
  } else {
    const float* src = kfpose + ((size_t)j * capK + k) * 12;
    for (int e = 0; e < 12; ++e) o[12 + 12 * k + e] = src[e];
  }
}

// plan: [2(G+1)..3(G+1)) recv item offsets, [3(G+1)..4(G+1)) first local dead index per source
__global__ void unpack_kernel(const float* __restrict__ in, long long n_items, int K, int capK,
                              int capN, int world, const long long* __restrict__ plan,
                              const int32_t* __restrict__ dead_list, float* __restrict__ pose,
                              float* __restrict__ kfpose, double* __restrict__ L,
                              int32_t* __restrict__ donor_g) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int KK = K + 1;
  if (t >= n_items * KK) return;
  const long long it = t / KK;
  const int k = (int)(t - it * KK);
  const long long* roff = plan + 2 * (world + 1);
  const long long* kstart = plan + 3 * (world + 1);
  int a = 0, b = world - 1;  // source rank: last with roff[src] <= it
  while (a < b) {
    const int mid = (a + b + 1) >> 1;
    if (roff[mid] <= it) a = mid; else b = mid - 1;
  }
  MCS_DCHECK(kstart[a] + (it - roff[a]) >= 0 && kstart[a] + (it - roff[a]) < capN);
  const int slot = dead_list[kstart[a] + (it - roff[a])];
  MCS_DCHECK(slot >= 0 && slot < capN);
  const float* s = in + it * state_floats(K);
  if (k == K) {
    for (int e = 0; e < 12; ++e) pose[(size_t)e * capN + slot] = s[e];
    L[slot] = reinterpret_cast<const double*>(s + 12 + 12 * K)[0];
    donor_g[slot] = (int32_t)reinterpret_cast<const long long*>(s + 12 + 12 * K + 2)[0];
  } else {
    float* dst = kfpose + ((size_t)slot * capK + k) * 12;
    for (int e = 0; e < 12; ++e) dst[e] = s[12 + 12 * k + e];
  }
}

__global__ void __launch_bounds__(kWT) max_kernel(const double* __restrict__ L, int N,
                                                  double* __restrict__ partials,
                                                  double* __restrict__ out,
                                                  unsigned int* counter) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const double v = i < N ? L[i] : -INFINITY;
  const double bm = block_reduce(v, MaxOp(), -INFINITY);
  if (threadIdx.x == 0) partials[blockIdx.x] = bm;
  if (last_block(counter)) {
    double m = -INFINITY;
    for (int k = threadIdx.x; k < (int)gridDim.x; k += blockDim.x) m = fmax(m, partials[k]);
    m = block_reduce(m, MaxOp(), -INFINITY);
    if (threadIdx.x == 0) *out = m;
  }
}

// argmax with ties -> lowest index, on (value, index) pairs
__device__ __forceinline__ void better(double& w, int& i, double w2, int i2) {
  if (w2 > w || (w2 == w && i2 < i)) { w = w2; i = i2; }
}

__device__ void block_argmax(double& w, int& idx) {
  __shared__ double sw[32];
  __shared__ int si[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double w2 = __shfl_xor_sync(0xffffffffu, w, o);
    const int i2 = __shfl_xor_sync(0xffffffffu, idx, o);
    better(w, idx, w2, i2);
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) { sw[wid] = w; si[wid] = idx; }
  __syncthreads();
  const int nw = blockDim.x >> 5;
  w = lane < nw ? sw[lane] : -INFINITY;
  idx = lane < nw ? si[lane] : 0x7fffffff;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double w2 = __shfl_xor_sync(0xffffffffu, w, o);
    const int i2 = __shfl_xor_sync(0xffffffffu, idx, o);
    better(w, idx, w2, i2);
  }
}

__global__ void __launch_bounds__(kWT) weight_argmax_kernel(const double* __restrict__ e, int N,
                                                            const double* __restrict__ S_ptr,
                                                            double* __restrict__ w,
                                                            double* __restrict__ pw,
                                                            int32_t* __restrict__ pi,
                                                            Scalars* sc, long long gbase,
                                                            unsigned int* counter) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  double wi = -INFINITY;
  int idx = 0x7fffffff;
  if (i < N) {
    wi = e[i] / *S_ptr;
    w[i] = wi;
    idx = i;
  }
  block_argmax(wi, idx);
  if (threadIdx.x == 0) { pw[blockIdx.x] = wi; pi[blockIdx.x] = idx; }
  if (last_block(counter)) {
    double bw = -INFINITY;
    int bi = 0x7fffffff;
    for (int k = threadIdx.x; k < (int)gridDim.x; k += blockDim.x) better(bw, bi, pw[k], pi[k]);
    block_argmax(bw, bi);
    if (threadIdx.x == 0) {
      sc->rep = gbase + bi;
      sc->wbest = bw;
    }
  }
}

size_t cub_temp_needed(int n) {
  size_t b = 0;
  cub::DeviceScan::InclusiveScan(nullptr, b, (Rung*)nullptr, (Rung*)nullptr, RungSum(), n);
  return b;
}


// Global respawn plan for world > 1: allgather (Q_g, D_g), plan on the host, upload.
static mcs_status plan_global(mcs_ctx* c, uint32_t U, long long* n_send_items,
                              long long* n_recv_items, std::vector<size_t>& sb,
                              std::vector<size_t>& so, std::vector<size_t>& rb,
                              std::vector<size_t>& ro) {
  const int G = c->world, me = c->rank;
  long long mine[2];
  MCS_CUDA(cudaMemcpyAsync(mine, &c->d_scal->Q, 16, cudaMemcpyDeviceToHost, c->stream));
  MCS_CUDA(cudaStreamSynchronize(c->stream));
  std::vector<long long> all(2 * G);
  MCS_TRY(dist_allgather_host(c, mine, all.data(), 16));
  std::vector<uint64_t> Q(G);
  std::vector<int64_t> D(G), qoff(G), clones(G), send((size_t)G * G);
  std::vector<uint64_t> qo(G);
  for (int g = 0; g < G; ++g) {
    Q[g] = (uint64_t)all[2 * g];
    D[g] = all[2 * g + 1];
  }
  uint64_t Qt = 0;
  int64_t Dt = 0;
  std::vector<int64_t> doff(G);
  const mcs_status st = mcs_plan_ladder(G, Q.data(), D.data(), U, qo.data(), doff.data(),
                                        clones.data(), &Qt, &Dt);
  if (st != MCS_OK && st != MCS_E_DEGENERATE) return st;
  if (st == MCS_E_DEGENERATE)
    for (auto& x : clones) x = 0;
  if (st == MCS_OK || st == MCS_E_DEGENERATE) {
    if (st == MCS_OK) MCS_TRY(mcs_plan_migration(G, clones.data(), D.data(), send.data()));
  }
  std::vector<long long> coff(G + 1, 0), doffs(G + 1, 0);
  for (int g = 0; g < G; ++g) {
    coff[g + 1] = coff[g] + clones[g];
    doffs[g + 1] = doffs[g] + D[g];
  }
  // plan table: [0] dead offsets, [1] send item offsets, [2] recv item offsets,
  //             [3] first local dead index per source, [4] first draw sent per destination
  std::vector<long long> plan(5 * (G + 1), 0);
  for (int g = 0; g <= G; ++g) plan[g] = doffs[g];
  long long s = 0, r = 0;
  sb.assign(G, 0);
  rb.assign(G, 0);
  so.assign(G + 1, 0);
  ro.assign(G + 1, 0);
  const size_t SB = sizeof(float) * 12 * (1 + c->K) + 16;
  for (int p = 0; p < G; ++p) {
    plan[(G + 1) + p] = s;
    plan[2 * (G + 1) + p] = r;
    const long long ns = (p == me || st != MCS_OK) ? 0 : send[(size_t)me * G + p];
    const long long nr = (p == me || st != MCS_OK) ? 0 : send[(size_t)p * G + me];
    plan[3 * (G + 1) + p] = std::max(coff[p], doffs[me]) - doffs[me];
    plan[4 * (G + 1) + p] = std::max(coff[me], doffs[p]);
    sb[p] = (size_t)ns * SB;
    rb[p] = (size_t)nr * SB;
    so[p] = (size_t)s * SB;
    ro[p] = (size_t)r * SB;
    s += ns;
    r += nr;
  }
  plan[(G + 1) + G] = s;
  plan[2 * (G + 1) + G] = r;
  so[G] = (size_t)s * SB;
  ro[G] = (size_t)r * SB;
  *n_send_items = s;
  *n_recv_items = r;
  // scalars Q_tot .. clones are contiguous in Scalars
  const long long host_sc[6] = {(long long)Qt, (long long)Dt, (long long)qo[me], (long long)doff[me],
                                coff[me], st == MCS_OK ? (long long)clones[me] : 0};
  MCS_CUDA(cudaMemcpyAsync(&c->d_scal->Q_tot, host_sc, sizeof(host_sc), cudaMemcpyHostToDevice,
                           c->stream));
  const int status = st == MCS_E_DEGENERATE ? (int)MCS_E_DEGENERATE : 0;
  MCS_CUDA(cudaMemcpyAsync(&c->d_scal->status, &status, sizeof(int), cudaMemcpyHostToDevice,
                           c->stream));
  MCS_CUDA(cudaMemcpyAsync(c->d_plan, plan.data(), sizeof(long long) * plan.size(),
                           cudaMemcpyHostToDevice, c->stream));
  MCS_CUDA(cudaStreamSynchronize(c->stream));  // host arrays above go out of scope
  return MCS_OK;
}

static mcs_status ensure_xfer(mcs_ctx* c, long long items) {
  if ((size_t)items <= c->xfer_cap_items) return MCS_OK;
  mem_free(c, c->d_send);
  mem_free(c, c->d_recv);
  mem_free(c, c->d_pack_src);
  c->d_send = c->d_recv = nullptr;
  c->d_pack_src = nullptr;
  const size_t cap = (size_t)items + (items >> 2) + 1024;
  const size_t bytes = cap * (sizeof(float) * 12 * (1 + c->capK) + 16);
  if (mem_alloc(c, (void**)&c->d_send, bytes) != cudaSuccess ||
      mem_alloc(c, (void**)&c->d_recv, bytes) != cudaSuccess ||
      mem_alloc(c, (void**)&c->d_pack_src, sizeof(int32_t) * cap) != cudaSuccess)
    return MCS_E_OUT_OF_MEMORY;
  c->xfer_cap_items = cap;
  return MCS_OK;
}

mcs_status launch_weights_resample(mcs_ctx* c, uint32_t U) {
  cudaStream_t st = c->stream;
  const int N = c->N;
  const int g = (N + kWT - 1) / kWT;
  const bool single = !dist_active(c);
  Scalars* sc = c->d_scal;
  double* p0 = c->d_partials;
  // a5: m and l* (reduced locally by a3) are global maxima across ranks
  MCS_TRY(dist_allreduce_f64(c, &sc->m, 2, 1));
  exp_sum_kernel<<<g, kWT, 0, st>>>(c->d_L, N, &sc->m, c->d_e, p0, &sc->S, &sc->counter[1]);
  MCS_TRY(dist_allreduce_f64(c, &sc->S, 1, 0));
  // a6: dead set and the survivor ladder
  Rung* rung = reinterpret_cast<Rung*>(c->d_ladder);
  Rung* scan = reinterpret_cast<Rung*>(c->d_ladder_scan);
  dead_kernel<<<g, kWT, 0, st>>>(c->d_e, c->d_l, N, sc, c->cfg.loglik_rel_floor,
                                 c->cfg.posterior_floor, c->d_w, c->d_flags, rung);
  size_t tb = c->cub_temp_bytes;
  MCS_CUDA(cub::DeviceScan::InclusiveScan(c->d_cub_temp, tb, rung, scan, RungSum(), N, st));
  totals_kernel<<<1, 1, 0, st>>>(scan, N, single ? 1 : 0, sc);
  long long n_send = 0, n_recv = 0, n_draws_bound = N;
  std::vector<size_t> sb, so, rb, ro;
  if (!single) MCS_TRY(dist_peer_setup(c));  // once per context (collective)
  const bool p2p = !single && c->p2p == 1;
  if (!single) {
    MCS_TRY(plan_global(c, U, &n_send, &n_recv, sb, so, rb, ro));
    long long h_clones = 0;
    MCS_CUDA(cudaMemcpy(&h_clones, &sc->clones, sizeof(long long), cudaMemcpyDeviceToHost));
    n_draws_bound = h_clones;
    if (!p2p) MCS_TRY(ensure_xfer(c, std::max(n_send, n_recv)));
  }
  ncum_dead_kernel<<<g, kWT, 0, st>>>(scan, N, sc, c->d_ncum, c->d_dead_list, c->d_donor,
                                      c->d_donor_g);
  if (c->cfg.clone_split) split_kernel<<<g, kWT, 0, st>>>(c->d_ncum, N, sc, c->d_L);
  if (p2p) {
    // every rank's dead list is complete before any rank writes into it
    MCS_TRY(dist_barrier(c));
    if (n_draws_bound > 0)
      draws_p2p_kernel<<<(int)((n_draws_bound * 32 + 255) / 256), 256, 0, st>>>(
          c->d_ncum, N, sc, c->world, c->rank, c->gbase, c->d_plan, c->d_dead_list, c->d_donor,
          c->d_donor_g, c->d_peers, c->K, c->d_pose, c->d_kfpose, c->d_L, c->capN, c->capK);
  } else if (n_draws_bound > 0) {
    draws_kernel<<<(int)((n_draws_bound + kWT - 1) / kWT), kWT, 0, st>>>(
        c->d_ncum, N, sc, c->world, c->rank, c->gbase, c->d_plan, c->d_dead_list, c->d_donor,
        c->d_donor_g, c->d_pack_src);
  }
  if (!p2p && !single && n_send > 0) {
    const long long tot = n_send * (c->K + 1);
    pack_kernel<<<(int)((tot + 255) / 256), 256, 0, st>>>(c->d_pack_src, n_send, c->K, c->capK,
                                                          c->capN, c->gbase, c->d_pose,
                                                          c->d_kfpose, c->d_L, c->d_send);
  }
  const long long tot = (long long)N * (c->K + 1);
  clone_kernel<<<(int)((tot + 255) / 256), 256, 0, st>>>(c->d_donor, N, c->K, c->capK, c->capN,
                                                         c->d_pose, c->d_kfpose, c->d_L);
  if (p2p) {
    MCS_TRY(dist_barrier(c));  // every rank's incoming clones have landed
  } else if (!single) {
    MCS_TRY(dist_alltoallv(c, c->d_send, sb.data(), so.data(), c->d_recv, rb.data(), ro.data()));
    if (n_recv > 0) {
      const long long tr = n_recv * (c->K + 1);
      unpack_kernel<<<(int)((tr + 255) / 256), 256, 0, st>>>(
          c->d_recv, n_recv, c->K, c->capK, c->capN, c->world, c->d_plan, c->d_dead_list,
          c->d_pose, c->d_kfpose, c->d_L, c->d_donor_g);
    }
  }
  // re-normalise on the new L (global max and sum), then a7
  max_kernel<<<g, kWT, 0, st>>>(c->d_L, N, p0, &sc->m2, &sc->counter[2]);
  MCS_TRY(dist_allreduce_f64(c, &sc->m2, 1, 1));
  exp_sum_kernel<<<g, kWT, 0, st>>>(c->d_L, N, &sc->m2, c->d_e, p0, &sc->S2, &sc->counter[3]);
  MCS_TRY(dist_allreduce_f64(c, &sc->S2, 1, 0));
  weight_argmax_kernel<<<g, kWT, 0, st>>>(c->d_e, N, &sc->S2, c->d_w, p0, c->d_ipartials, sc,
                                          c->gbase, &sc->counter[4]);
  if (!single) {  // representative: best (w, global index) over ranks, ties -> lowest index
    double mine[2];
    MCS_CUDA(cudaMemcpyAsync(&mine[0], &sc->wbest, 8, cudaMemcpyDeviceToHost, st));
    MCS_CUDA(cudaMemcpyAsync(&mine[1], &sc->rep, 8, cudaMemcpyDeviceToHost, st));
    MCS_CUDA(cudaStreamSynchronize(st));
    std::vector<double> all(2 * c->world);
    MCS_TRY(dist_allgather_host(c, mine, all.data(), 16));
    double bw = -INFINITY;
    long long bi = 0x7fffffffffffffffLL;
    for (int r = 0; r < c->world; ++r) {
      long long ri;
      memcpy(&ri, &all[2 * r + 1], 8);
      if (all[2 * r] > bw || (all[2 * r] == bw && ri < bi)) { bw = all[2 * r]; bi = ri; }
    }
    MCS_CUDA(cudaMemcpyAsync(&sc->rep, &bi, 8, cudaMemcpyHostToDevice, st));
    MCS_CUDA(cudaMemcpyAsync(&sc->wbest, &bw, 8, cudaMemcpyHostToDevice, st));
    MCS_CUDA(cudaStreamSynchronize(st));
  }
  return cudaGetLastError() == cudaSuccess ? MCS_OK : MCS_E_CUDA;
}

mcs_status launch_resample_only(mcs_ctx* c, const double* d_e, const uint8_t* d_dead, int n,
                                uint32_t U, int32_t* d_donor) {
  cudaStream_t st = c->stream;
  Rung* rung = reinterpret_cast<Rung*>(c->d_ladder);
  Rung* scan = reinterpret_cast<Rung*>(c->d_ladder_scan);
  const int g = (n + kWT - 1) / kWT;
  launch_set_params(c, 0.0, U);
  rung_from_inputs_kernel<<<g, kWT, 0, st>>>(d_e, d_dead, n, rung);
  size_t tb = c->cub_temp_bytes;
  MCS_CUDA(cub::DeviceScan::InclusiveScan(c->d_cub_temp, tb, rung, scan, RungSum(), n, st));
  totals_kernel<<<1, 1, 0, st>>>(scan, n, 1, c->d_scal);
  ncum_dead_kernel<<<g, kWT, 0, st>>>(scan, n, c->d_scal, c->d_ncum, c->d_dead_list, d_donor,
                                      nullptr);
  draws_kernel<<<g, kWT, 0, st>>>(c->d_ncum, n, c->d_scal, 1, 0, 0, nullptr, c->d_dead_list,
                                  d_donor, nullptr, nullptr);
  return cudaGetLastError() == cudaSuccess ? MCS_OK : MCS_E_CUDA;
}

}  // namespace mcs
