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
//
// Four launches on one device, all stream-ordered and graph-capturable:
//   exp_sum_kernel     e, S (block sums + last-block finisher)
//   ladder_kernel      dead set, rungs, the hand-written single-pass inclusive scan of
//                      {uint64 rung, uint32 dead} (decoupled look-back over 1,024-particle
//                      tiles), the ascending dead list, local totals (and the one-device plan),
//                      the survivors' max of L for the re-normalisation
//   draws_kernel       one thread per draw: its donor by binary search on the ladder with the
//                      exact 128-bit test (r 2^32 + U) Q < C_j D 2^32; then the warp copies the
//                      32 donors' states (T_t, every T_k, L) into their dead slots — locally, or
//                      straight into a peer rank's state over peer memory
//   renorm_kernel      e' = exp(L - m'), S' and the argmax (ties -> lowest index); w = e' / S'
//                      is formed where it is read (outputs, mcs_get_particles)
// Across ranks every quantity above is global: m, l* and S are all-reduced; the ladder
// offsets and totals and the survivors' max m' come from one device allgather of
// {Q_g, D_g, m'_g} and a one-thread plan kernel; S' and the representative from one device
// allgather of {S'_g, best e'_g, index} (S' summed in rank order).  Five collectives with
// peer-direct migration (the fifth is the barrier after the draws).  With NCCL and peer access
// no step waits on the host; the host-transport and pack/send/recv fallbacks do.
#include <algorithm>
#include <vector>

#include "mcs_internal.cuh"
#include "reduce.cuh"

namespace mcs {

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

// ---------------------------------------------------------------- the ladder (a6 steps 1-4)
constexpr int kLT = 256, kLI = 4, kTile = kLT * kLI;  // 1,024 particles per scan tile

// decoupled look-back tile state: flag = (epoch << 2) | 1 (aggregate published) or 2 (inclusive
// prefix published too).  The two values live in separate fields, each written once before its
// flag: a reader that saw "aggregate" must not pick up an inclusive value written after it
// read the flag.
struct TileSt {
  unsigned long long aC;  // tile aggregate
  unsigned int aD;
  unsigned int flag;
  unsigned long long iC;  // inclusive prefix through this tile
  unsigned int iD;
  unsigned int pad;
};
static_assert(sizeof(TileSt) == 32, "tile state is one 32-byte record");

struct LadderArgs {
  const double* e;          // [N] e_i (update) or the caller's e (mcs_resample)
  const double* l;          // [N] l_i (update)
  const uint8_t* dead_in;   // [N] caller's dead mask (mcs_resample) or nullptr
  const double* L;          // [N] cumulative log-likelihood (survivors' max), or nullptr
  int N;
  Scalars* sc;
  double rel_floor, post_floor;
  uint8_t* flags;           // bit3 dead (update) or nullptr
  unsigned long long* C;    // [N] inclusive ladder (local)
  int32_t* dead_list;       // [N] local dead slots, ascending
  int32_t* donor;           // [N] reset to -1
  int32_t* donor_g;         // [N] reset to -1, or nullptr
  TileSt* tiles;            // [ceil(N / kTile)] (32 B each, d_ladder)
  double* partials;         // [ceil(N / kTile)] survivors' max of L per tile
  int single;               // one device: also write the (trivial) global plan
};

__device__ __forceinline__ void st_tile(TileSt* t, unsigned long long C, unsigned int d,
                                        unsigned int flag) {
  volatile TileSt* v = t;
  if ((flag & 3u) == 2u) {
    v->iC = C;
    v->iD = d;
  } else {
    v->aC = C;
    v->aD = d;
  }
  __threadfence();  // value before flag
  v->flag = flag;
}

__global__ void __launch_bounds__(kLT) ladder_kernel(LadderArgs a) {
  __shared__ int s_tile;
  __shared__ unsigned int s_epoch;
  __shared__ unsigned long long s_wc[kLT / 32];
  __shared__ unsigned int s_wd[kLT / 32];
  __shared__ unsigned long long s_pc;
  __shared__ unsigned int s_pd;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) {
    s_tile = (int)atomicAdd(&a.sc->tile_ctr, 1u);  // tiles in start order: look-back progresses
    s_epoch = a.sc->epoch & 0x3FFFFFFFu;
  }
  __syncthreads();
  const int tile = s_tile;
  const unsigned int ep = s_epoch;
  const int ntiles = (a.N + kTile - 1) / kTile;
  const int base = tile * kTile + tid * kLI;  // this thread's kLI consecutive particles
  const double S = a.sc->S, lstar = a.sc->lstar;
  unsigned long long q[kLI];
  unsigned int dk[kLI];
  double lmax = -INFINITY;
#pragma unroll
  for (int k = 0; k < kLI; ++k) {
    const int i = base + k;
    q[k] = 0ull;
    dk[k] = 0u;
    if (i >= a.N) continue;
    const double ei = a.e[i];
    bool dead;
    if (a.dead_in) {
      dead = a.dead_in[i] != 0;
    } else {
      dead = particle_dead(a.l[i], lstar, ei, S, a.rel_floor, a.post_floor);  // P:190, R17
      if (dead) a.flags[i] |= 8;
    }
    if (!dead) q[k] = (unsigned long long)floor(ei * 4294967296.0);  // rung (R18)
    dk[k] = dead ? 1u : 0u;
    if (!dead && a.L) lmax = fmax(lmax, a.L[i]);
    a.donor[i] = -1;
    if (a.donor_g) a.donor_g[i] = -1;
  }
  // thread-local inclusive prefixes, then the block's exclusive scan of the thread totals
  unsigned long long tc = 0ull;
  unsigned int td = 0u;
#pragma unroll
  for (int k = 0; k < kLI; ++k) {
    tc += q[k];
    td += dk[k];
  }
  unsigned long long ic = tc;
  unsigned int id = td;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long c2 = __shfl_up_sync(0xffffffffu, ic, o);
    const unsigned int d2 = __shfl_up_sync(0xffffffffu, id, o);
    if (lane >= o) {
      ic += c2;
      id += d2;
    }
  }
  if (lane == 31) {
    s_wc[wid] = ic;
    s_wd[wid] = id;
  }
  __syncthreads();
  unsigned long long wc = 0ull, AC = 0ull;
  unsigned int wd = 0u, AD = 0u;
#pragma unroll
  for (int w = 0; w < kLT / 32; ++w) {
    if (w < wid) {
      wc += s_wc[w];
      wd += s_wd[w];
    }
    AC += s_wc[w];
    AD += s_wd[w];
  }
  const unsigned long long bc = wc + ic - tc;  // exclusive prefix of this thread in the tile
  const unsigned int bd = wd + id - td;
  // publish the aggregate at once, then look back for the exclusive prefix of the tile
  if (wid == 0) {
    unsigned long long pc = 0ull;
    unsigned int pd = 0u;
    if (tile == 0) {
      if (lane == 0) st_tile(&a.tiles[0], AC, AD, (ep << 2) | 2u);
    } else {
      if (lane == 0) st_tile(&a.tiles[tile], AC, AD, (ep << 2) | 1u);
      int pos = tile - 1;
      while (true) {
        const int idx = pos - lane;  // lane 0: the nearest predecessor
        unsigned long long c = 0ull;
        unsigned int d = 0u, stt = 2u;  // before tile 0: an inclusive zero
        if (idx >= 0) {
          volatile TileSt* t = a.tiles + idx;
          unsigned int f;
          do {
            f = t->flag;
          } while ((f >> 2) != ep || (f & 3u) == 0u);
          __threadfence();
          stt = f & 3u;
          c = stt == 2u ? t->iC : t->aC;
          d = stt == 2u ? t->iD : t->aD;
        }
        const unsigned int incl = __ballot_sync(0xffffffffu, stt == 2u);
        const int stop = incl ? __ffs(incl) - 1 : 31;
        unsigned long long vc = lane <= stop ? c : 0ull;
        unsigned int vd = lane <= stop ? d : 0u;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          vc += __shfl_xor_sync(0xffffffffu, vc, o);
          vd += __shfl_xor_sync(0xffffffffu, vd, o);
        }
        pc += vc;
        pd += vd;
        if (incl) break;
        pos -= 32;
      }
      if (lane == 0) st_tile(&a.tiles[tile], pc + AC, pd + AD, (ep << 2) | 2u);
    }
    if (lane == 0) {
      s_pc = pc;
      s_pd = pd;
    }
  }
  __syncthreads();
  unsigned long long C = s_pc + bc;
  unsigned int D = s_pd + bd;
#pragma unroll
  for (int k = 0; k < kLI; ++k) {
    const int i = base + k;
    if (i >= a.N) break;
    if (dk[k]) a.dead_list[D] = i;  // the D-th dead slot (ascending)
    C += q[k];
    D += dk[k];
    a.C[i] = C;
    if (i == a.N - 1) {  // local totals; one device: the global plan is the local one
      Scalars* sc = a.sc;
      sc->Q = C;
      sc->D = (long long)D;
      if (a.single) {
        const bool degenerate = D > 0u && C == 0ull;
        sc->Q_tot = C;
        sc->D_tot = (long long)D;
        sc->q_off = 0ull;
        sc->d_off = 0;
        sc->clone_off = 0;
        sc->clones = degenerate ? 0 : (long long)D;
        sc->status = degenerate ? (int)MCS_E_DEGENERATE : 0;
      }
    }
  }
  // the survivors' max of L: the shift of the re-normalisation (clones copy survivors' L)
  lmax = block_reduce(lmax, MaxOp(), -INFINITY);
  if (tid == 0) a.partials[tile] = lmax;
  if (last_block(&a.sc->counter[2])) {
    double m = -INFINITY;
    for (int k = tid; k < ntiles; k += kLT) m = fmax(m, a.partials[k]);
    m = block_reduce(m, MaxOp(), -INFINITY);
    if (tid == 0) {
      a.sc->m2 = m;
      a.sc->tile_ctr = 0u;  // every block has drawn its tile
      a.sc->epoch = a.sc->epoch + 1u;
    }
  }
}

// ---------------------------------------------------------------- the global plan (world > 1)
// n(c) = #{draws r in [0, D) : (r + U/2^32) Q / D < c}   (R18)
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

// One thread: every rank's (Q_g, D_g) -> this rank's ladder offset, dead offset, first draw and
// draw count, the global totals, and the dead-slot offsets of every rank (plan[0..G]).  The same
// arithmetic as the host mcs_plan_ladder (dist.cu), which the CPU tests pin.
__global__ void plan_kernel(const long long* __restrict__ QD, int G, int me, Scalars* sc,
                            long long* __restrict__ plan) {
  unsigned __int128 Q = 0;
  long long D = 0, qo = 0, dof = 0;
  double m2 = -INFINITY;
  for (int g = 0; g < G; ++g) {
    if (g == me) {
      qo = (long long)Q;
      dof = D;
    }
    plan[g] = D;
    Q += (unsigned long long)QD[4 * g];
    D += QD[4 * g + 1];
    double mg;
    memcpy(&mg, &QD[4 * g + 2], 8);
    m2 = fmax(m2, mg);  // the global survivors' max of L (-inf where a rank has none)
  }
  sc->m2 = m2;
  plan[G] = D;
  const bool over = (Q >> 64) != 0;  // the exact ladder needs Q < 2^64 (R18)
  const unsigned long long Qt = (unsigned long long)Q;
  const bool degenerate = D > 0 && Qt == 0ull;
  sc->Q_tot = Qt;
  sc->D_tot = D;
  sc->q_off = (unsigned long long)qo;
  sc->d_off = dof;
  long long c0 = 0, c1 = 0;
  if (!over && !degenerate && D > 0) {
    c0 = draws_below((unsigned long long)qo, D, Qt, sc->U);
    c1 = draws_below((unsigned long long)qo + sc->Q, D, Qt, sc->U);
  }
  sc->clone_off = c0;
  sc->clones = c1 - c0;
  sc->status = over ? (int)MCS_E_CAPACITY : degenerate ? (int)MCS_E_DEGENERATE : 0;
}

// ---------------------------------------------------------------- draws + clones (a6 step 5)
struct DrawArgs {
  const unsigned long long* C;  // [N] local inclusive ladder
  int N;
  const Scalars* sc;
  int world, me;
  long long gbase;
  const long long* plan;        // [0..G] dead-slot offsets (world > 1)
  const int32_t* dead_list;     // local dead slots, ascending
  int32_t* donor;               // [N] local donor index or -1
  int32_t* donor_g;             // [N] global donor index or -1 (nullptr: donors only)
  int copy;                     // 1: clone states; 0: donors only (mcs_resample)
  int split;                    // R34: clones (and donors, in renorm) get L - ln(1 + copies)
  const PeerView* peers;        // world > 1 with peer-direct migration, else nullptr
  int32_t* pack_src;            // world > 1 without peer access: local donors to pack
  int K, capK, capN;
  float* pose;
  float* kfpose;
  float4* kft;
  double* L;
};

__global__ void __launch_bounds__(kWT) draws_kernel(DrawArgs a) {
  const Scalars* sc = a.sc;
  const long long clones = sc->clones;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  const unsigned long long Qt = sc->Q_tot, qoff = sc->q_off;
  const unsigned __int128 Dt2 = (unsigned __int128)(unsigned long long)sc->D_tot << 32;
  for (long long t0 = (long long)blockIdx.x * blockDim.x; t0 < clones; t0 += stride) {
    const long long t = t0 + threadIdx.x;
    const bool valid = t < clones;
    int j = 0, dst = a.me, slot = -1;
    if (valid) {
      const long long R = sc->clone_off + t;
      // donor: the first j with (R 2^32 + U) Q < (q_off + C_j) D 2^32  (n(C_j) > R, R18)
      const unsigned __int128 lhs = ((unsigned __int128)((unsigned long long)R << 32 | 0ull) +
                                     sc->U) * Qt;
      int lo = 0, hi = a.N - 1;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (lhs < (unsigned __int128)(qoff + a.C[mid]) * Dt2) hi = mid; else lo = mid + 1;
      }
      j = lo;
      MCS_DCHECK(lhs < (unsigned __int128)(qoff + a.C[j]) * Dt2);
      if (a.world > 1) {  // destination rank: the last with plan[g] <= R
        int x = 0, y = a.world - 1;
        while (x < y) {
          const int mid = (x + y + 1) >> 1;
          if (a.plan[mid] <= R) x = mid; else y = mid - 1;
        }
        dst = x;
      }
      if (dst == a.me) {
        slot = a.dead_list[R - sc->d_off];
        MCS_DCHECK(slot >= 0 && slot < a.N && slot != j);
        a.donor[slot] = j;
        if (a.donor_g) a.donor_g[slot] = (int32_t)(a.gbase + j);
      } else if (a.peers) {
        slot = a.peers[dst].dead_list[R - a.plan[dst]];
      } else {
        // pack path: plan[G+1 + p] send offsets, plan[4(G+1) + p] first draw sent to p
        const long long* send_off = a.plan + (a.world + 1);
        const long long* sfirst = a.plan + 4 * (a.world + 1);
        a.pack_src[send_off[dst] + (R - sfirst[dst])] = j;
      }
    }
    if (!a.copy) continue;
    // the warp copies its lanes' clones one after another: T_t (SoA), every T_k (contiguous
    // 48-B records), L — locally, or into the destination rank's state over peer memory
    unsigned int todo = __ballot_sync(0xffffffffu, valid && (dst == a.me || a.peers));
    bool remote_any = false;
    while (todo) {
      const int src = __ffs(todo) - 1;
      todo &= todo - 1;
      const int jj = __shfl_sync(0xffffffffu, j, src);
      const int dd = __shfl_sync(0xffffffffu, dst, src);
      const int ss = __shfl_sync(0xffffffffu, slot, src);
      float* dpose = a.pose;
      float* dkf = a.kfpose;
      float4* dkt = a.kft;
      double* dL = a.L;
      int dcapN = a.capN, dcapK = a.capK;
      if (dd != a.me) {
        const PeerView& P = a.peers[dd];
        dpose = P.pose;
        dkf = P.kfpose;
        dkt = P.kft;
        dL = P.L;
        dcapN = P.capN;
        dcapK = P.capK;
        remote_any = true;
      }
      MCS_DCHECK(ss >= 0 && ss < dcapN);
      if (lane < 12) dpose[(size_t)lane * dcapN + ss] = a.pose[(size_t)lane * a.capN + jj];
      const float4* s4 = reinterpret_cast<const float4*>(a.kfpose + (size_t)jj * a.capK * 12);
      float4* d4 = reinterpret_cast<float4*>(dkf + (size_t)ss * dcapK * 12);
      // keyframe poses: 3K float4, four loads in flight per lane (C3: 9.6 KB per clone)
      const int n4 = 3 * a.K;
      int k = lane;
      for (; k + 96 < n4; k += 128) {
        const float4 x0 = __ldg(s4 + k), x1 = __ldg(s4 + k + 32), x2 = __ldg(s4 + k + 64),
                     x3 = __ldg(s4 + k + 96);
        d4[k] = x0;
        d4[k + 32] = x1;
        d4[k + 64] = x2;
        d4[k + 96] = x3;
      }
      for (; k < n4; k += 32) d4[k] = __ldg(s4 + k);
      const float4* st4 = a.kft + (size_t)jj * a.capK;  // the translation plane, K float4
      float4* dt4 = dkt + (size_t)ss * dcapK;
      for (k = lane; k < a.K; k += 32) dt4[k] = __ldg(st4 + k);
      if (lane == 0) {
        double Lc = a.L[jj];
        if (a.split) {  // R34: the donor's draw count from its own rungs
          const long long c = draws_below(qoff + a.C[jj], sc->D_tot, Qt, sc->U) -
                              draws_below(qoff + (jj > 0 ? a.C[jj - 1] : 0ull), sc->D_tot, Qt,
                                          sc->U);
          Lc -= log((double)(1 + c));
        }
        dL[ss] = Lc;
        if (dd != a.me) a.peers[dd].donor_g[ss] = (int32_t)(a.gbase + jj);
      }
    }
    if (__any_sync(0xffffffffu, remote_any)) __threadfence_system();  // before the barrier
  }
}

// ---------------------------------------------------------------- re-normalisation + a7
// argmax with ties -> lowest index, on (value, index) pairs
__device__ __forceinline__ void better(double& w, long long& i, double w2, long long i2) {
  if (w2 > w || (w2 == w && i2 < i)) { w = w2; i = i2; }
}

__device__ void block_argmax(double& w, long long& idx) {
  __shared__ double sw[32];
  __shared__ long long si[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double w2 = __shfl_xor_sync(0xffffffffu, w, o);
    const long long i2 = __shfl_xor_sync(0xffffffffu, idx, o);
    better(w, idx, w2, i2);
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) { sw[wid] = w; si[wid] = idx; }
  __syncthreads();
  const int nw = blockDim.x >> 5;
  w = lane < nw ? sw[lane] : -INFINITY;
  idx = lane < nw ? si[lane] : 0x7fffffffffffffffLL;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double w2 = __shfl_xor_sync(0xffffffffu, w, o);
    const long long i2 = __shfl_xor_sync(0xffffffffu, idx, o);
    better(w, idx, w2, i2);
  }
}

// e'_i = exp(L_i - m') with m' the global survivors' max of L (the old max m when every
// particle is dead: respawn skipped, L unchanged); S' = sum e' and the argmax of e' (ties ->
// lowest global index).  R34: a donor's own L drops by ln(1 + its draw count) first.
__global__ void __launch_bounds__(kWT) renorm_kernel(double* __restrict__ L, int N, Scalars* sc,
                                                     const uint8_t* __restrict__ flags,
                                                     const unsigned long long* __restrict__ C,
                                                     int split, long long gbase, int single,
                                                     double* __restrict__ e,
                                                     double* __restrict__ partials,
                                                     double* __restrict__ pw,
                                                     long long* __restrict__ pi) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const double m2 = sc->m2;
  const double shift = m2 > -INFINITY ? m2 : sc->m;
  double v = 0.0, best = -INFINITY;
  long long bi = 0x7fffffffffffffffLL;
  if (i < N) {
    double Li = L[i];
    if (split && !(flags[i] & 8) && sc->status == 0 && sc->D_tot > 0) {
      const unsigned long long qo = sc->q_off;
      const long long c = draws_below(qo + C[i], sc->D_tot, sc->Q_tot, sc->U) -
                          draws_below(qo + (i > 0 ? C[i - 1] : 0ull), sc->D_tot, sc->Q_tot, sc->U);
      if (c > 0) {
        Li -= log((double)(1 + c));
        L[i] = Li;
      }
    }
    v = exp(Li - shift);
    e[i] = v;
    best = v;
    bi = gbase + i;
  }
  const double bs = block_reduce(v, SumOp(), 0.0);
  block_argmax(best, bi);
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = bs;
    pw[blockIdx.x] = best;
    pi[blockIdx.x] = bi;
  }
  if (last_block(&sc->counter[3])) {
    double s = 0.0, bw = -INFINITY;
    long long bk = 0x7fffffffffffffffLL;
    for (int k = threadIdx.x; k < (int)gridDim.x; k += blockDim.x) {
      s += partials[k];
      better(bw, bk, pw[k], pi[k]);
    }
    s = block_reduce(s, SumOp(), 0.0);
    block_argmax(bw, bk);
    if (threadIdx.x == 0) {
      sc->S2 = s;
      sc->rep = bk;
      sc->wbest = single ? bw / s : bw;  // world > 1: e' of the local best, normalised in pick
    }
  }
}

// world > 1: every rank's {S'_g, e'_best, global index, -}: S' = sum over ranks in rank order
// (the same on every rank, whatever NCCL's reduction order), the representative = the best
// (e', index) pair, ties -> lowest index
__global__ void pick_kernel(const double* __restrict__ all, int G, Scalars* sc) {
  double bw = -INFINITY, S2 = 0.0;
  long long bi = 0x7fffffffffffffffLL;
  for (int g = 0; g < G; ++g) {
    long long ig;
    memcpy(&ig, &all[4 * g + 2], 8);
    S2 += all[4 * g];
    better(bw, bi, all[4 * g + 1], ig);
  }
  sc->S2 = S2;
  sc->rep = bi;
  sc->wbest = bw / S2;
}

// {Q_g, D_g, m'_g, -} for the allgather that feeds plan_kernel (one collective for the ladder
// totals and the survivors' max of L)
__global__ void qd_kernel(const Scalars* sc, long long* out) {
  out[0] = (long long)sc->Q;
  out[1] = sc->D;
  memcpy(&out[2], &sc->m2, 8);
  out[3] = 0;
}

__global__ void best_kernel(const Scalars* sc, double* out) {  // {S'_g, e'_best, index, -}
  out[0] = sc->S2;
  out[1] = sc->wbest;
  memcpy(&out[2], &sc->rep, 8);
  out[3] = 0.0;
}

// ---------------------------------------------------------------- transport fallback (pack)
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
                              float* __restrict__ kfpose, float4* __restrict__ kft,
                              double* __restrict__ L, int32_t* __restrict__ donor_g) {
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
    kft[(size_t)slot * capK + k] =
        make_float4(s[12 + 12 * k + 3], s[12 + 12 * k + 7], s[12 + 12 * k + 11], 0.f);
  }
}

// R34 on the pack path: a clone's L is packed before the donor-side adjustment, so the donor
// rank applies ln(1 + c) to the packed copies here (the p2p / local path does it in draws)
__global__ void split_packed_kernel(float* __restrict__ buf, const int32_t* __restrict__ pack_src,
                                    long long n_items, int K,
                                    const unsigned long long* __restrict__ C,
                                    const Scalars* __restrict__ sc) {
  const long long it = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (it >= n_items) return;
  const int j = pack_src[it];
  const unsigned long long qo = sc->q_off;
  const long long c = draws_below(qo + C[j], sc->D_tot, sc->Q_tot, sc->U) -
                      draws_below(qo + (j > 0 ? C[j - 1] : 0ull), sc->D_tot, sc->Q_tot, sc->U);
  double* od = reinterpret_cast<double*>(buf + it * state_floats(K) + 12 + 12 * K);
  od[0] -= log((double)(1 + c));
}

// Host-planned migration for world > 1 without peer access (the pack / send / recv fallback):
// the plan scalars come back to the host once, which derives the per-peer transfer counts.
static mcs_status plan_transfers(mcs_ctx* c, long long* n_send_items, long long* n_recv_items,
                                 std::vector<size_t>& sb, std::vector<size_t>& so,
                                 std::vector<size_t>& rb, std::vector<size_t>& ro) {
  const int G = c->world, me = c->rank;
  const long long* dQD = reinterpret_cast<const long long*>(c->d_xg);
  std::vector<long long> QD(4 * G);
  Scalars hs;
  MCS_CUDA(cudaMemcpyAsync(QD.data(), dQD, sizeof(long long) * 4 * G, cudaMemcpyDeviceToHost,
                           c->stream));
  MCS_CUDA(cudaMemcpyAsync(&hs, c->d_scal, sizeof(Scalars), cudaMemcpyDeviceToHost, c->stream));
  MCS_CUDA(cudaStreamSynchronize(c->stream));
  std::vector<uint64_t> Q(G);
  std::vector<int64_t> D(G), doff(G), clones(G), send((size_t)G * G, 0);
  std::vector<uint64_t> qo(G);
  for (int g = 0; g < G; ++g) {
    Q[g] = (uint64_t)QD[4 * g];
    D[g] = QD[4 * g + 1];
  }
  uint64_t Qt = 0;
  int64_t Dt = 0;
  const mcs_status st = mcs_plan_ladder(G, Q.data(), D.data(), hs.U, qo.data(), doff.data(),
                                        clones.data(), &Qt, &Dt);
  if (st != MCS_OK && st != MCS_E_DEGENERATE) return st;
  if (st == MCS_OK) MCS_TRY(mcs_plan_migration(G, clones.data(), D.data(), send.data()));
  std::vector<long long> coff(G + 1, 0), doffs(G + 1, 0);
  for (int g = 0; g < G; ++g) {
    coff[g + 1] = coff[g] + (st == MCS_OK ? clones[g] : 0);
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
  const size_t SB = sizeof(float) * state_floats(c->K);
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
  MCS_CUDA(cudaMemcpyAsync(c->d_plan, plan.data(), sizeof(long long) * plan.size(),
                           cudaMemcpyHostToDevice, c->stream));
  MCS_CUDA(cudaStreamSynchronize(c->stream));  // the host plan goes out of scope
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
  const size_t bytes = cap * (sizeof(float) * state_floats(c->capK));
  if (mem_alloc(c, (void**)&c->d_send, bytes) != cudaSuccess ||
      mem_alloc(c, (void**)&c->d_recv, bytes) != cudaSuccess ||
      mem_alloc(c, (void**)&c->d_pack_src, sizeof(int32_t) * cap) != cudaSuccess)
    return MCS_E_OUT_OF_MEMORY;
  c->xfer_cap_items = cap;
  return MCS_OK;
}

static int draw_grid(const mcs_ctx* c) {  // grid-stride: enough warps for a few draws each
  const int n = c->N > 0 ? c->N : 1;
  return std::max(1, std::min((n + kWT - 1) / kWT, 148 * 8));
}

static void ladder_args(mcs_ctx* c, LadderArgs& a, int N) {
  a.N = N;
  a.sc = c->d_scal;
  a.C = reinterpret_cast<unsigned long long*>(c->d_ladder_scan);
  a.dead_list = c->d_dead_list;
  a.tiles = reinterpret_cast<TileSt*>(c->d_ladder);
  a.partials = c->d_partials;
}

bool weights_device_resident(const mcs_ctx* c) {
  return !dist_active(c) || (c->nccl_comm && c->p2p == 1);
}

// fork_a4: a4 runs on the side stream for the survivors only, from the moment the dead set is
// decided (after the S allreduce) and concurrently with the ladder; the draws (and, across
// ranks, the allgather that lets other ranks write into this rank's dead slots) wait for it
mcs_status launch_weights_resample(mcs_ctx* c, uint32_t U, bool fork_a4) {
  (void)U;  // the uniform reaches the kernels through d_scal (set_params), graph-replay safe
  cudaStream_t st = c->stream;
  const int N = c->N;
  const int g = (N + kWT - 1) / kWT;
  const bool single = !dist_active(c);
  Scalars* sc = c->d_scal;
  // a5: m and l* (reduced locally by a3) are global maxima across ranks
  MCS_TRY(dist_allreduce_f64(c, &sc->m, 2, 1));
  exp_sum_kernel<<<g, kWT, 0, st>>>(c->d_L, N, &sc->m, c->d_e, c->d_partials, &sc->S,
                                    &sc->counter[1]);
  MCS_TRY(dist_allreduce_f64(c, &sc->S, 1, 0));
  cudaEvent_t join = nullptr;
  if (fork_a4) {  // a4 for the survivors, beside the ladder
    MCS_CUDA(cudaEventRecord(c->fork_ev, st));
    MCS_CUDA(cudaStreamWaitEvent(c->side, c->fork_ev, 0));
    c->stream = c->side;
    launch_propagate(c, kPropSurvivors);
    c->stream = st;
    MCS_CUDA(cudaEventRecord(c->join_ev, c->side));
    join = c->join_ev;
  }
  // a6: dead set, ladder scan, dead list, local totals
  if (!single) MCS_TRY(dist_peer_setup(c));  // once per context (collective)
  LadderArgs la{};
  ladder_args(c, la, N);
  la.e = c->d_e;
  la.l = c->d_l;
  la.L = c->d_L;
  la.rel_floor = c->cfg.loglik_rel_floor;
  la.post_floor = c->cfg.posterior_floor;
  la.flags = c->d_flags;
  la.donor = c->d_donor;
  la.donor_g = c->d_donor_g;
  la.single = single ? 1 : 0;
  ladder_kernel<<<(N + kTile - 1) / kTile, kLT, 0, st>>>(la);
  if (join) MCS_CUDA(cudaStreamWaitEvent(st, join, 0));  // a4 done: keyframe poses final
  const bool p2p = !single && c->p2p == 1;
  long long n_send = 0, n_recv = 0;
  std::vector<size_t> sb, so, rb, ro;
  if (!single) {
    // every rank's (Q_g, D_g) on the device, then the plan; the allgather also orders every
    // rank's ladder kernel (its dead list) before any rank's draws read it over peer memory
    long long* dQD = reinterpret_cast<long long*>(c->d_xg);
    qd_kernel<<<1, 1, 0, st>>>(sc, dQD + 4 * c->world);
    MCS_TRY(dist_allgather_dev(c, dQD + 4 * c->world, dQD, 32));
    plan_kernel<<<1, 1, 0, st>>>(dQD, c->world, c->rank, sc, c->d_plan);
    if (!p2p) {
      MCS_TRY(plan_transfers(c, &n_send, &n_recv, sb, so, rb, ro));
      MCS_TRY(ensure_xfer(c, std::max(n_send, n_recv)));
    }
  }
  // no survivor anywhere (sc->status, final here): the respawn is skipped and every state kept,
  // so the particles the survivor-only a4 skipped are propagated after all
  if (fork_a4) launch_propagate(c, kPropIfDegenerate);
  DrawArgs da{};
  da.C = la.C;
  da.N = N;
  da.sc = sc;
  da.world = c->world;
  da.me = c->rank;
  da.gbase = c->gbase;
  da.plan = c->d_plan;
  da.dead_list = c->d_dead_list;
  da.donor = c->d_donor;
  da.donor_g = c->d_donor_g;
  da.copy = 1;
  da.split = c->cfg.clone_split ? 1 : 0;
  da.peers = p2p ? c->d_peers : nullptr;
  da.pack_src = c->d_pack_src;
  da.K = c->K;
  da.capK = c->capK;
  da.capN = c->capN;
  da.pose = c->d_pose;
  da.kfpose = c->d_kfpose;
  da.kft = c->d_kft;
  da.L = c->d_L;
  draws_kernel<<<draw_grid(c), kWT, 0, st>>>(da);
  if (p2p) {
    MCS_TRY(dist_barrier(c));  // every rank's incoming clones have landed
  } else if (!single) {
    if (n_send > 0) {
      const long long tot = n_send * (c->K + 1);
      pack_kernel<<<(int)((tot + 255) / 256), 256, 0, st>>>(c->d_pack_src, n_send, c->K, c->capK,
                                                            c->capN, c->gbase, c->d_pose,
                                                            c->d_kfpose, c->d_L, c->d_send);
      if (c->cfg.clone_split)
        split_packed_kernel<<<(int)((n_send + 255) / 256), 256, 0, st>>>(
            c->d_send, c->d_pack_src, n_send, c->K, la.C, sc);
    }
    MCS_TRY(dist_alltoallv(c, c->d_send, sb.data(), so.data(), c->d_recv, rb.data(), ro.data()));
    if (n_recv > 0) {
      const long long tr = n_recv * (c->K + 1);
      unpack_kernel<<<(int)((tr + 255) / 256), 256, 0, st>>>(
          c->d_recv, n_recv, c->K, c->capK, c->capN, c->world, c->d_plan, c->d_dead_list,
          c->d_pose, c->d_kfpose, c->d_kft, c->d_L, c->d_donor_g);
    }
  }
  // re-normalise on the new L (global shift and sum), then a7
  renorm_kernel<<<g, kWT, 0, st>>>(c->d_L, N, sc, c->d_flags, la.C, da.split, c->gbase,
                                   single ? 1 : 0, c->d_e, c->d_partials,
                                   c->d_partials + g, reinterpret_cast<long long*>(c->d_ipartials));
  if (!single) {  // one allgather: every rank's S'_g and best (e', index)
    double* dB = reinterpret_cast<double*>(c->d_xg) + 4 * (c->world + 1);
    best_kernel<<<1, 1, 0, st>>>(sc, dB + 4 * c->world);
    MCS_TRY(dist_allgather_dev(c, dB + 4 * c->world, dB, 32));
    pick_kernel<<<1, 1, 0, st>>>(dB, c->world, sc);
  }
  return cudaGetLastError() == cudaSuccess ? MCS_OK : MCS_E_CUDA;
}

mcs_status launch_resample_only(mcs_ctx* c, const double* d_e, const uint8_t* d_dead, int n,
                                uint32_t U, int32_t* d_donor) {
  cudaStream_t st = c->stream;
  launch_set_params(c, 0.0, U);
  LadderArgs la{};
  ladder_args(c, la, n);
  la.e = d_e;
  la.dead_in = d_dead;
  la.donor = d_donor;
  la.single = 1;
  ladder_kernel<<<(n + kTile - 1) / kTile, kLT, 0, st>>>(la);
  DrawArgs da{};
  da.C = la.C;
  da.N = n;
  da.sc = c->d_scal;
  da.world = 1;
  da.dead_list = c->d_dead_list;
  da.donor = d_donor;
  draws_kernel<<<std::max(1, std::min((n + kWT - 1) / kWT, 148 * 8)), kWT, 0, st>>>(da);
  return cudaGetLastError() == cudaSuccess ? MCS_OK : MCS_E_CUDA;
}

// w_i = e'_i / S' (weights are formed where they are read)
__global__ void weights_out_kernel(const double* __restrict__ e, int N, const Scalars* sc,
                                   double* __restrict__ w) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < N) w[i] = e[i] / sc->S2;
}

void launch_weights_out(mcs_ctx* c, double* d_w) {
  weights_out_kernel<<<(c->N + kWT - 1) / kWT, kWT, 0, c->stream>>>(c->d_e, c->N, c->d_scal, d_w);
}

}  // namespace mcs
