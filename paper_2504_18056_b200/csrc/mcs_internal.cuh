// mcs_internal.cuh — internal types of libmcs (B200 / sm_100a).  Not part of the ABI.
//
// HBM layout:
//   current poses T_t      : SoA fp32 [12][Ncap]            (coalesced per element)
//   keyframe poses T_k^i   : fp32 [Ncap][Kcap][12]          (a particle's map is contiguous:
//                                                            clone = one memcpy)
//   cumulative log-lik L   : fp64 [Ncap]                    (R22)
//   keyframe hash tables   : per keyframe, 64-B slots float4 [cap + 1][4] (key in the first
//                            word, then mu', Sigma'; slot cap = always-empty sentinel)
//   work items (a1 -> a2)  : float4 [3*Ncap][4]  = (kR|kt rows, {kf, particle, flags, 0})
//   sweep partials (a2->a3): fp64 SoA [32][3*Ncap] = {l, n, H~21, b~6, pad} per item
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/mcs.h"

namespace mcs {

// Device-side invariant checks: compiled in with -DMCS_DEVICE_CHECKS (the checked build that
// tests/test_gpu_checked.py runs), nothing otherwise.  A failed check prints and traps, so the
// call returns MCS_E_CUDA.
#ifdef MCS_DEVICE_CHECKS
#define MCS_DCHECK(cond)                                                                      \
  do {                                                                                        \
    if (!(cond)) {                                                                            \
      printf("MCS_DCHECK %s:%d: %s\n", __FILE__, __LINE__, #cond);                           \
      __trap();                                                                               \
    }                                                                                         \
  } while (0)
#else
#define MCS_DCHECK(cond) \
  do {                   \
  } while (0)
#endif

// status plumbing of the host-side launch sequences
#define MCS_TRY(x)               \
  do {                           \
    const mcs_status _s = (x);   \
    if (_s != MCS_OK) return _s; \
  } while (0)
#define MCS_CUDA(x)                            \
  do {                                         \
    if ((x) != cudaSuccess) return MCS_E_CUDA; \
  } while (0)

constexpr int kCellMin = -1048576;               // 21-bit signed cell coordinates (R27)
constexpr int kCellMax = 1048575;
constexpr int kSlotWords = 32;                    // sweep partial record per (particle, slot), fp64
constexpr int kMaxNb = MCS_MAX_NEIGHBORS;

// Per-keyframe open-addressing table in the keyframe's own cell grid.  Keys are 32-bit
// bbox-local cell coordinates (dx << 21 | dy << 10 | dz), so a query outside the keyframe's
// occupied bounding box is a miss without a probe, and a probe is one 64-byte slot:
//   float4 {key, mu'x, mu'y, mu'z}  {S'yy, S'zz, S'xy, S'xz}  {S'xx, S'yz, count, 0}  {0,0,0,0}
// (the key shares the first 16 bytes with the mean, so the first-probe payload loads are
// issued together with the key; the (y, z) pairs (mu'y, mu'z), (S'yy, S'zz), (S'xy, S'xz) land
// in aligned register pairs, the operands of the sweep's packed FFMA2 math).  Load factor <= 1/4
// (down to 1/64 within a 64 MiB table, kf_store.cu).
constexpr unsigned int kEmptyKey32 = 0xFFFFFFFFu;  // dx = 2047 never occurs (ex <= 2046)
constexpr unsigned int kNoKey32 = 0xFFFFFFFEu;     // query key of an out-of-bbox point (dx = 2047)
// keyframe bbox extents (cells): one below the 11/11/10-bit fields, so that a query cell clamped
// to the extents (sweep.cu, MCS_SWEEP_CLAMP) stays a key no slot holds, below the markers
constexpr int kMaxEx = 2046, kMaxEy = 2047, kMaxEz = 1023;
constexpr unsigned int kHashMul32 = 0x9E3779B1u;

struct KfMeta {                 // one per keyframe (device array, read through L1)
  const float4* slots;          // [cap + 1][4]; slot cap is an always-empty sentinel
  int ox, oy, oz;               // bbox origin (cell coordinates)
  unsigned int ex, ey, ez;      // bbox extents (cells)
  unsigned int shift;           // 32 - log2(cap)
  unsigned int mask;            // cap - 1
};

__host__ __device__ inline unsigned long long pack_cell(int x, int y, int z) {
  return ((unsigned long long)(x & 0x1FFFFF) << 42) | ((unsigned long long)(y & 0x1FFFFF) << 21) |
         (unsigned long long)(z & 0x1FFFFF);
}

__host__ __device__ inline unsigned int local_key(unsigned int dx, unsigned int dy,
                                                  unsigned int dz) {
  return (dx << 21) | (dy << 10) | dz;
}
// the same key for in-range fields (dx < 2^11, dy < 2^11, dz < 2^10), as two shift-adds (LEA)
__host__ __device__ inline unsigned int local_key_lea(unsigned int dx, unsigned int dy,
                                                      unsigned int dz) {
  return (((dx << 11) + dy) << 10) + dz;
}

__host__ __device__ inline unsigned int slot_hash(unsigned int key, unsigned int shift) {
  return (key * kHashMul32) >> shift;
}

struct KfHost {
  float4* slots = nullptr;
  int32_t cap = 0, n_cells = 0, n_points = 0;
  KfMeta meta{};
};

struct PeerView;                // dist.cu: a rank's state as another rank writes it

struct Scalars {                // device-side reduction results of one update
  double m;                     // max_i L_i (after L += l)            } exchanged together
  double lstar;                 // max_i l_i                           } (allreduce MAX)
  double S;                     // sum_i exp(L_i - m)                    (allreduce SUM)
  double m2;                    // after respawn                         (allreduce MAX)
  double S2;                    //                                       (allreduce SUM)
  unsigned long long Q;         // local survivor ladder total
  long long D;                  // local dead count
  unsigned long long Q_tot;     // global ladder total
  long long D_tot;              // global dead count
  unsigned long long q_off;     // ladder offset of this rank
  long long d_off;              // dead-slot offset of this rank
  long long clone_off;          // first global draw made by this rank's survivors
  long long clones;             // number of draws made by this rank's survivors
  double wbest;                 // best local weight, then global
  long long rep;                // representative (global index)
  int32_t status;               // 0 ok, MCS_E_DEGENERATE
  unsigned int counter[8];      // last-block counters (reset by the last block)
  double D_now;                 // per-update parameters, written by set_params_kernel before
  unsigned int U;               // the update body (so a captured CUDA graph can be replayed)
  unsigned int tile_ctr;        // ladder scan: next tile to hand out (reset by the last block)
  unsigned int epoch;           // ladder scan: launch epoch tagging the look-back tile flags
};

}  // namespace mcs

struct mcs_ctx {
  mcs_config cfg{};
  int dev = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  mcs_allocator alloc{};      // user device-memory hook (alloc.alloc == nullptr: CUDA's own)
  std::string err;
  mcs_status sticky = MCS_OK;
  bool profiling = false;
  float phase_ms[5] = {0, 0, 0, 0, 0};
  cudaEvent_t ev[6] = {};
  // a4 runs on a side stream concurrently with a5 / the ladder (fork after a3, join before the
  // first step that reads keyframe poses of other particles: the draws' clones)
  cudaStream_t side = nullptr;
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr;

  // keyframe store (a0)
  int K = 0;
  std::vector<mcs::KfHost> kf;
  std::vector<double> D;        // shared cumulative odometry path length per keyframe (R14)
  mcs::KfMeta* d_kf_meta = nullptr;
  double* d_D = nullptr;

  // particle state
  int N = 0;                    // local particles
  float* d_pose = nullptr;      // [12][Ncap]
  float* d_kfpose = nullptr;    // [Ncap][Kcap][12]
  // the keyframe translations again, {t_x, t_y, t_z, 0} per (particle, keyframe) [Ncap][Kcap]:
  // a1's nearest-keyframe search reads 16 B per keyframe instead of the 48-B pose.  Every
  // writer of d_kfpose writes it too (insertion, set_particles, a4, clones, unpack, restore)
  float4* d_kft = nullptr;
  double* d_L = nullptr;        // [Ncap]
  void* d_snapshot = nullptr;   // mcs_snapshot buffer
  size_t snapshot_bytes = 0;

  // per-update scratch
  float* d_scan_raw = nullptr;  // [Scap][9]
  float4* d_scan = nullptr;     // [Scap][3], then d_scan_plane, then one float4 for d_scan_np
  float4* d_scan_plane = nullptr;  // [Scap][2] plane-form layout (R36)
  int* d_scan_np = nullptr;     // number of scan points not in plane form (prepare_scan)
  bool scan_prepared = false;   // a scan went through prepare_scan (mcs_scan_nonplanar)
  float4* d_items = nullptr;    // [nb*Ncap][4]
  int32_t* d_order = nullptr;   // [nb*Ncap] sweep order (item ids, coherence-sorted)
  unsigned long long* d_skeys = nullptr;      // [nb*Ncap] coherence keys (a1)
  unsigned long long* d_skeys_out = nullptr;  // [nb*Ncap]
  int32_t* d_sids = nullptr;                  // [nb*Ncap] item ids before sorting
  double* d_part = nullptr;     // [nb*Ncap][32] fp64 {l, n, H~21, b~6, pad}
  uint8_t* d_meta = nullptr;    // [Ncap] bit0 loop
  int32_t* d_to = nullptr;      // [Ncap] oldest neighbour keyframe t_o
  double* d_l = nullptr;        // [Ncap] l_i
  double* d_psi = nullptr;      // [6][Ncap] fp64 psi
  float* d_grad = nullptr;      // [6][Ncap]
  float* d_hess = nullptr;      // [21][Ncap]
  uint8_t* d_flags = nullptr;   // [Ncap]
  double* d_e = nullptr;        // [Ncap] e_i, then e'_i after the respawn: w_i = e'_i / S'
  char* d_xg = nullptr;         // [8][world+1] x 8 B: device allgathers {Q_g, D_g, m'_g, -},
                                // {S'_g, e'_g, rep_g, -},
                                // then 12 doubles: the all-reduced pose of mcs_get_global_pose
  void* d_ladder = nullptr;     // 32-B look-back tile states of the ladder scan, one per 1,024
                                // particles (zeroed at create)
  void* d_ladder_scan = nullptr;  // [Ncap] u64 inclusive survivor ladder C_i
  int32_t* d_donor = nullptr;   // [Ncap]
  double* d_partials = nullptr; // [4][max_blocks]
  int32_t* d_ipartials = nullptr;
  mcs::Scalars* d_scal = nullptr;
  mcs::Scalars* h_scal = nullptr;  // pinned
  char* d_stage = nullptr;      // output staging for synchronous calls
  size_t stage_bytes = 0;
  int* d_bad = nullptr;         // validation counter
  void* d_cub_temp = nullptr;
  size_t cub_temp_bytes = 0;
  int32_t capN = 0, capK = 0, capS = 0, nbcap = 0;
  // sweep point splits (cfg.point_splits): splits the partial buffer holds, splits in use by
  // the current update (set by launch_sweep, read by combine)
  int part_splits = 1;
  int cur_splits = 1;

  // multi-rank (world > 1): particle shards with global index = gbase + local index
  int world = 1, rank = 0;
  long long gbase = 0;
  std::vector<long long> n_per_rank;
  const mcs_transport* tr = nullptr;  // host transport, or
  void* nccl_comm = nullptr;          // NCCL communicator (dlopen'ed libnccl)
  int32_t* d_dead_list = nullptr;     // [Ncap] local dead slots, ascending
  int32_t* d_donor_g = nullptr;       // [Ncap] global donor index or -1
  long long* d_plan = nullptr;        // [5][world+1] d_offs, send_off, recv_off, kstart, sfirst
  int32_t* d_pack_src = nullptr;      // [xfer_cap_items] local donors to pack, send order
  float* d_send = nullptr;            // packed particle states to send / received
  float* d_recv = nullptr;
  size_t xfer_cap_items = 0;
  void* h_stage = nullptr;            // pinned host staging for the host transport
  size_t h_stage_bytes = 0;
  char* d_ag = nullptr;               // device scratch of the NCCL host allgather / barrier
  size_t d_ag_bytes = 0;
  // peer-direct migration (cfg.peer_migration): 0 not set up yet, 1 on, -1 off
  int p2p = 0;
  // CUDA graph of the single-rank update body (run_update), replayed while its key holds
  cudaGraphExec_t gexec = nullptr;
  long long gkey[5] = {-1, -1, -1, -1, -1};  // n_pts, N, K, diversity gather rows, profiling
  bool graph_off = false;                // capture failed once: eager from then on
  // neighbour-particle diversity term (R35, cfg.diversity_weight != 0): every rank's
  // translations at the start of the update, padded to the largest shard
  double* d_tall = nullptr;            // [world][div_maxn][3]
  int* d_divn = nullptr;               // [world] shard sizes
  int div_maxn = 0;
  mcs::PeerView* d_peers = nullptr;    // [world] device views of every rank's state
  std::vector<void*> ipc_opened;       // CUDA IPC mappings of other processes' buffers
};

namespace mcs {

// ---- launchers (all stream-ordered on ctx->stream) ----
// a0: build keyframe k's table from device mean3/cov6 (n points).  Returns cudaError;
// *bad_cell = number of points outside the 21-bit range, *bad_extent = 1 if the occupied
// bounding box exceeds 2047 x 2048 x 1024 cells.
cudaError_t kf_build(mcs_ctx* c, const float* d_mean3, const float* d_cov6, int n, KfHost& out,
                     int* bad_cell, int* bad_extent);
// raw [S][3] + [S][6] -> the sweep's float4 x3 layout {mu, lambda3} {u, 0} {v, 0} (spectral
// form Sigma = lambda3 I + u u^T + v v^T, fp64 Jacobi), and the plane-form layout {mu, lambda3}
// {x, 0} (Sigma = lambda3 I + [x]x^T [x]x, R36) in out_plane; *nonplanar = number of points
// that are not plane-form
cudaError_t launch_prepare_scan(const float* mean3, const float* cov6, int S, float4* out,
                                float4* out_plane, int* nonplanar, cudaStream_t st);
// a1; mode: kSelectUpdate (H~, b~ for slots in G), kSelectEval (all slots), kSelectWeight (none)
enum { kSelectUpdate = 0, kSelectEval = 1, kSelectWeight = 2 };
mcs_status launch_select(mcs_ctx* c, int mode);  // MCS_E_CUDA if a launch (or the sort) fails
// a2
void launch_sweep(mcs_ctx* c, int S);
// point splits the sweep would use for n local particles (cfg.point_splits, or auto)
int sweep_splits_for(const mcs_ctx* c, int n);

// device memory through the allocator hook (include/mcs.h): persistent buffers (context
// lifetime) and stream-ordered temporaries
cudaError_t mem_alloc(mcs_ctx* c, void** p, size_t bytes);
void mem_free(mcs_ctx* c, void* p);
cudaError_t mem_alloc_async(mcs_ctx* c, void** p, size_t bytes, cudaStream_t st);
void mem_free_async(mcs_ctx* c, void* p, cudaStream_t st);
// a3; modes: per-slot eval outputs; GN update and/or L += l with the first a5 reduction
enum { kCombineEval = 0, kCombineUpdateWeight = 1, kCombineUpdate = 2, kCombineWeight = 3 };
void launch_combine(mcs_ctx* c, int S, int mode, double* slot_l, float* slot_H21,
                    float* slot_b6, int32_t* slot_n, int32_t* slot_kf, uint8_t* loop_out);
// a4
// a4 over every loop particle (kPropAll); over the survivors of this update's a6 only
// (kPropSurvivors: a dead particle's keyframe poses are replaced by its donor's clone); or, after
// a6 found no survivor at all (respawn skipped, sc->status = MCS_E_DEGENERATE), over the rest
// (kPropIfDegenerate, a no-op otherwise).  D_now from d_scal (launch_set_params)
enum { kPropAll = 0, kPropSurvivors = 1, kPropIfDegenerate = 2 };
void launch_propagate(mcs_ctx* c, int mode = kPropAll);
// a6's dead test (R17) — the ladder and the survivor-only a4 take the same decision
__device__ __forceinline__ bool particle_dead(double l_i, double lstar, double e_i, double S,
                                              double rel_floor, double post_floor) {
  return (l_i - lstar < rel_floor) || (e_i / S < post_floor);
}
// writes D_now and U into d_scal (a tiny kernel: by value, outside any captured graph)
void launch_set_params(mcs_ctx* c, double D_now, uint32_t U);
// a5-a7 (+ the exchange steps when world > 1); degenerate status in d_scal
// fork_a4: run a4 (survivors only) on c->side once the dead set is decided (after the S
// allreduce), concurrently with the ladder, joined before the draws
mcs_status launch_weights_resample(mcs_ctx* c, uint32_t U, bool fork_a4 = false);
// isolated respawn on caller arrays (single device)
mcs_status launch_resample_only(mcs_ctx* c, const double* d_e, const uint8_t* d_dead, int n,
                                uint32_t U, int32_t* d_donor);
// true when a5-a7 need no host round trip (one device, or NCCL with peer-direct migration):
// the update body can then be captured into a CUDA graph
bool weights_device_resident(const mcs_ctx* c);
// w = e' / S' into d_w (N doubles)
void launch_weights_out(mcs_ctx* c, double* d_w);

// A rank's particle state as another rank writes it (peer-direct migration).
struct PeerView {
  float* pose;         // SoA [12][capN]
  float* kfpose;       // [capN][capK][12]
  float4* kft;         // [capN][capK] keyframe translations
  double* L;           // [capN]
  int32_t* dead_list;  // [capN] local dead slots, ascending
  int32_t* donor_g;    // [capN] global donor index
  int capN, capK;
};

// ---- multi-rank exchange (dist.cu); world == 1 => no-ops returning MCS_OK ----
mcs_status dist_init(mcs_ctx* c, std::string& err);
bool dist_active(const mcs_ctx* c);  // exchange path in use (world > 1, or a transport/NCCL)
// collective: returns once every rank's stream has reached this point (NCCL: stream-ordered)
mcs_status dist_barrier(mcs_ctx* c);
// collective: exchange state views (raw pointers in one process, CUDA IPC across processes);
// sets c->p2p to 1 when every rank can write every other rank's state, else -1
mcs_status dist_peer_setup(mcs_ctx* c);
void dist_destroy(mcs_ctx* c);
// in place on device doubles; op 0 = sum, 1 = max (stream-ordered; host transport syncs)
mcs_status dist_allreduce_f64(mcs_ctx* c, double* d_buf, int n, int op);
// device buffers gathered on the device (NCCL: stream-ordered; host transport: staged, syncs)
mcs_status dist_allgather_dev(mcs_ctx* c, const void* d_send, void* d_recv, size_t bytes);
// host values gathered to host (small, synchronous)
mcs_status dist_allgather_host(mcs_ctx* c, const void* send, void* recv, size_t bytes);
// device buffers; byte counts per peer on the host
mcs_status dist_alltoallv(mcs_ctx* c, const float* d_send, const size_t* send_bytes,
                          const size_t* send_off, float* d_recv, const size_t* recv_bytes,
                          const size_t* recv_off);
size_t sort_temp_needed(int n, int capK);
// NEXT rows (predict.cu): Eq.1 prediction; keyframe-insertion overlap
// R35: snapshot this rank's translations (+ the device allgather over ranks) / apply eta d_i
mcs_status launch_diversity_snapshot(mcs_ctx* c);
mcs_status launch_diversity_apply(mcs_ctx* c);
mcs_status launch_predict(mcs_ctx* c, double* d_buf, int* d_bad, unsigned long long seed,
                          unsigned long long frame, double vsig);
mcs_status launch_overlap(mcs_ctx* c, const float* d_mean3, int S, const float* d_rel, int kf,
                          unsigned long long* d_count, unsigned long long* h_count);

}  // namespace mcs
