/*
 * mcs.h — C-ABI of the B200-native hot path of gradient-guided 6-DoF Monte Carlo
 * SLAM (arXiv 2504.18056).  Product library: libmcs.so (sm_100a CUDA).
 *
 * What it computes (PAPER.md line numbers "P:n"; readings "Rn" in DESIGN.md §3):
 *   per particle i and each of its neighbour keyframes k:
 *     kT = (T_k^i)^-1 T_t^i                                      (Eq.4)
 *     log p = -sum_j e_j^T Omega_j e_j,  e_j = mu'_j - kT mu_j,
 *             Omega_j = (Sigma'_j + kR Sigma_j kR^T)^-1          (Eqs.2-4)
 *     H = sum J^T Omega J, b = sum J^T Omega e, J = de/d(kT)     (Eq.6)
 *   then, for loop particles: psi = -(H + lambda I)^-1 b (Eq.5; R1, R11),
 *   T_t <- T_t exp(psi) (Eq.7), keyframe propagation
 *   T_k <- T_k exp(r_k psi), r_k = d(t_k, t_o)/d(t, t_o)         (Eqs.8-10; R14-R16),
 *   importance weights L_i += log p, w = softmax(L)              (Eq.11; R22),
 *   dead-particle pruning + respawn from the survivors' weights  (R17, R18),
 *   representative = argmax w.
 *
 * Conventions
 *   Pose12  : row-major 3x4 [R|t], fp32; p[4a+b] = R[a][b], p[4a+3] = t[a] (P:91 implies fp32).
 *   Cov6    : (xx, xy, xz, yy, yz, zz), fp32, symmetric positive definite.
 *   Twist6  : (rho, phi), translation first, right perturbation T exp(xi) (R2).
 *   Hess21  : upper triangle of a symmetric 6x6, row-major: (0,0),(0,1)..(0,5),(1,1)..(5,5).
 *   Keyframe clouds are Gaussians in the keyframe's own sensor frame.
 *
 * Ownership: the caller owns every buffer passed in.  Data the library keeps
 *   (keyframe clouds, particles) is copied into context-owned device memory.
 *   Synchronous calls accept HOST or DEVICE pointers (unified addressing) and keep
 *   no pointer after returning.  *_async calls take DEVICE pointers only and borrow
 *   them until the given stream reaches the work.
 * Errors: every call returns mcs_status; mcs_last_error() gives the message.
 *   Argument errors are detected before any state change.  CUDA/NCCL errors are
 *   sticky: the context then returns MCS_E_CUDA / MCS_E_NCCL until destroyed.
 *   MCS_E_DEGENERATE (every particle dead): weights were updated, respawn
 *   was skipped; the caller must re-initialise the particles.
 * Threading: a context is not thread-safe; distinct contexts are independent.
 */
#ifndef MCS_H
#define MCS_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define MCS_API __attribute__((visibility("default")))
#else
#define MCS_API
#endif

#define MCS_ABI_VERSION 1
#define MCS_MAX_NEIGHBORS 4

typedef struct mcs_ctx mcs_ctx; /* opaque; owns all device state */

typedef enum {
  MCS_OK = 0,
  MCS_E_INVALID_ARG = 1,  /* null / size / non-finite / non-SPD input            */
  MCS_E_OUT_OF_MEMORY = 2,
  MCS_E_CUDA = 3,         /* sticky                                             */
  MCS_E_NCCL = 4,         /* sticky                                             */
  MCS_E_CAPACITY = 5,     /* exceeds a capacity fixed at mcs_create             */
  MCS_E_STATE = 6,        /* call order, e.g. update before any keyframe        */
  MCS_E_DEGENERATE = 7    /* every particle dead                        */
} mcs_status;

typedef enum { MCS_GN_OLD_SLOTS = 0, /* Fig.3: gradient w.r.t. non-recent keyframes (R4) */
               MCS_GN_ALL_SLOTS = 1  /* every neighbour slot                      */
} mcs_gn_slots;

/* Correspondence search ("voxel-based corresponding point search"; R7, R33). */
typedef enum { MCS_CORR_CELL = 0, /* the single voxel containing q (one probe)                  */
               MCS_CORR_NN27 = 1  /* nearest cell representative within nn_radius among the 27
                                     voxels around q: exact NN for nn_radius <= r (pinned fp32
                                     squared distance, ties -> lower (oz, oy, ox) index)       */
} mcs_corr_mode;

/* Collective transport for world_size > 1 when NCCL is not used (e.g. torch.distributed gloo or
 * the in-process transport below).  Buffers are HOST memory; every rank calls the same sequence
 * of operations.  allreduce: in place over n values (dtype 0 = f64, 1 = i64; op 0 = sum,
 * 1 = max), reduced in rank order.  allgather: `bytes` from every rank into recv[world][bytes].
 * alltoallv: send[p] (send_bytes[p]) goes to rank p, recv[p] (recv_bytes[p]) comes from rank p.
 * Each returns 0 on success. */
typedef struct mcs_transport {
  void* user;
  int (*allreduce)(void* user, int32_t rank, void* buf, int32_t n, int32_t dtype, int32_t op);
  int (*allgather)(void* user, int32_t rank, const void* send, void* recv, size_t bytes);
  int (*alltoallv)(void* user, int32_t rank, const void* const* send, const size_t* send_bytes,
                   void* const* recv, const size_t* recv_bytes);
} mcs_transport;

/* Device-memory hook (e.g. PyTorch's caching allocator).  Every device buffer of a context is
 * taken from alloc(bytes, stream, user) and returned through free(ptr, stream, user), with the
 * context's stream at the time of the call (persistent buffers: the stream current at create).
 * alloc returns NULL on failure (-> MCS_E_OUT_OF_MEMORY) and must return 256-byte aligned
 * memory, like cudaMalloc (the sweep reads table slots with 32-byte vector loads); a misaligned
 * block is handed back through free and the call fails (MCS_E_INVALID_ARG from mcs_create,
 * MCS_E_CUDA with cudaErrorMisalignedAddress in mcs_last_error later).  Both must be
 * thread-compatible with the caller; the struct is copied at mcs_create. */
typedef struct mcs_allocator {
  void* (*alloc)(size_t bytes, void* cuda_stream, void* user);
  void  (*free)(void* ptr, void* cuda_stream, void* user);
  void* user;
} mcs_allocator;

typedef struct mcs_config {
  uint32_t abi_version;          /* MCS_ABI_VERSION                                         */
  int32_t  capacity_particles;   /* particles on this device (its shard when world_size>1)  */
  int32_t  capacity_keyframes;   /* K_max: per-particle keyframe pose storage is N x K_max  */
  int32_t  capacity_scan_points; /* S_max                                                   */
  int32_t  neighbor_count;       /* 1..MCS_MAX_NEIGHBORS; 3                          */
  int32_t  loop_recency_gap;     /* slot old iff kf id <= latest - gap (R5); 10             */
  float    voxel_resolution;     /* r in metres; a power of two (R27); 0.5 indoor          */
  int32_t  gn_slots;             /* mcs_gn_slots                                            */
  double   damping_rel;          /* lambda = damping_rel * tr(H) / 6 (R11); 1e-6            */
  double   step_clamp;           /* ||psi||_2 <= step_clamp (R11); 1.0                      */
  double   unmatched_penalty;    /* kappa per unmatched (point, slot) (R8); 0               */
  double   loglik_rel_floor;     /* dead if l_i - max_j l_j < this (R17); ln 1e-16   */
  double   posterior_floor;      /* dead if w_i < this; 1e-8                        */
  int32_t  device;               /* CUDA ordinal                                            */
  int32_t  rank, world_size;     /* particle shards (one process per GPU)                   */
  const void* nccl_unique_id;    /* 128-byte ncclUniqueId when world_size > 1, else NULL    */
  const mcs_transport* transport; /* host transport when world_size > 1 without NCCL        */
  int32_t  gn_iterations;        /* GN steps per update, each a full a1-a4 pass (R12); 1        */
  int32_t  weight_after_update;  /* 0: weight with the pre-update l (R13); 1: re-evaluate l   */
  int32_t  corr_mode;            /* mcs_corr_mode: MCS_CORR_CELL (R7, default) or NN27 (R33)  */
  float    nn_radius;            /* NN27 candidate radius in metres, 0 < nn_radius <= r (R33) */
  int32_t  clone_split;          /* 0: a clone copies its donor's L (R19); 1: the donor and its
                                    c clones each get L - ln(1 + c) (R34)                    */
  const mcs_allocator* allocator; /* NULL: cudaMalloc / cudaMallocAsync on the context stream */
  int32_t  peer_migration;       /* world_size > 1: 1 (default) = respawned particles that land
                                    on another rank are written straight into that rank's state
                                    by the draws kernel over peer memory (NVLink; CUDA IPC across
                                    processes) when every rank's state is reachable, else (and
                                    with 0) packed and exchanged by NCCL send/recv or the
                                    transport's alltoallv                                     */
  int32_t  point_splits;         /* scan-point ranges per work item in the sweep, 1..16; 0 (default)
                                    = auto: more splits when the particles alone cannot fill the
                                    GPU (results differ only in fp rounding; bitwise equality of
                                    runs holds for a fixed value)                               */
  int32_t  graph_replay;         /* 1 (default): a single-rank update body is captured once into
                                    a CUDA graph and replayed while the scan size, particle and
                                    keyframe counts stay the same; 0: launched kernel by kernel */
  int32_t  kf_table_mib;         /* per-keyframe hash-table budget (MiB): the table's power-of-two
                                    capacity is >= 4 x the occupied cells and is doubled up to 64 x
                                    the cells while it stays within this budget (a sparse table:
                                    first probes almost never walk a linear-probing chain; C2: 32
                                    MiB per keyframe); 64 (default); 0 = minimum capacity (load up
                                    to 1/4, least memory).  Results do not depend on it.        */
  double   diversity_weight;     /* eta (m^2) of the neighbour-particle diversity term (R35): after
                                    the GN step(s) every translation moves by eta d_i in the world
                                    frame, d_i = (2 / (h N)) sum_j (t_i - t_j) exp(-|t_i - t_j|^2
                                    / h) over all N particles (every rank) at the translations the
                                    update started from (SVGD's repulsive term; the paper cites it,
                                    P:32, and defines none); 0 (default) = off           */
  double   diversity_bandwidth;  /* h (m^2) of that RBF kernel, > 0; 1.0 (default)              */
} mcs_config;

/* sizeof(mcs_config) of this build: bindings check their mirror of the struct against it. */
MCS_API size_t mcs_config_size(void);

/* Fills *cfg with the defaults above (capacities 0: caller sets them). */
MCS_API void mcs_config_default(mcs_config* cfg);

MCS_API mcs_status  mcs_create(const mcs_config* cfg, mcs_ctx** out);
MCS_API mcs_status  mcs_destroy(mcs_ctx* ctx);
/* ctx == NULL: the calling thread's last mcs_create error. */
MCS_API const char* mcs_last_error(const mcs_ctx* ctx);
/* Stream every call of this context is ordered on (cudaStream_t; NULL = library-owned). */
MCS_API mcs_status  mcs_set_stream(mcs_ctx* ctx, void* cuda_stream);

/* Register keyframe k = K (returned in *out_kf_id): n Gaussians (mean3[n][3], cov6[n][6])
 * in the keyframe's own sensor frame, and D_k, the cumulative odometry path length at the
 * keyframe (Eq.9 reading R14).  Builds the keyframe's voxel hash once (off the update
 * clock).  Every particle's new keyframe pose is its current pose: T_k^i := T_t^i (R24).
 * MCS_E_INVALID_ARG if a point's cell lies outside the 21-bit range, if the occupied cells'
 * bounding box is wider than 2046 x 2047 x 1023 cells (the 32-bit bbox-local table keys: at
 * r = 0.5 m that is 1023 x 1023.5 x 511.5 m), or if n < 1. */
MCS_API mcs_status mcs_add_keyframe(mcs_ctx* ctx, const float* mean3, const float* cov6, int32_t n,
                            double path_length, int32_t* out_kf_id);

/* Set the local particle set: pose12[n][12] current poses; kf_pose12[n][K][12] (K = current
 * keyframe count) or NULL (every T_k^i := T_t^i); cum_loglik[n] (fp64 L_i, Eq.11) or NULL (0). */
MCS_API mcs_status mcs_set_particles(mcs_ctx* ctx, int32_t n_local, const float* pose12,
                             const float* kf_pose12, const double* cum_loglik);
/* Read back (any pointer may be NULL): pose12[n][12], kf_pose12[n][K][12], L[n], w[n]. */
MCS_API mcs_status mcs_get_particles(mcs_ctx* ctx, float* pose12, float* kf_pose12, double* cum_loglik,
                             double* weight);
MCS_API mcs_status mcs_get_sizes(const mcs_ctx* ctx, int32_t* n_local, int32_t* n_keyframes);
/* One local particle's current pose (row-major 3x4 [R|t] into pose12[12], host or device), e.g.
 * the representative's without reading back the whole set.  MCS_E_INVALID_ARG if
 * index is outside [0, n_local). */
MCS_API mcs_status mcs_get_pose(mcs_ctx* ctx, int32_t index, float* pose12);
/* Collective over the ranks of a multi-GPU job (every rank calls it with the same index): the
 * current pose of the particle with GLOBAL index global_index (e.g. mcs_update_out's
 * representative) on every rank — the owning rank's pose reaches the others through one fp64
 * all-reduce of 12 values.  On one device it equals mcs_get_pose.  MCS_E_INVALID_ARG if the
 * index is outside [0, N_total). */
MCS_API mcs_status mcs_get_global_pose(mcs_ctx* ctx, int64_t global_index, float* pose12);

/* Outputs of one update; every pointer optional (NULL = not produced).  Per-particle rows are
 * indexed by LOCAL particle index.  loglik = l_i over ALL neighbour slots (Eq.2) minus the kappa
 * term; grad6 = dl/d(delta) = -2 sum_{s in G} b_s (0 for non-loop particles under
 * MCS_GN_OLD_SLOTS); hess21 = undamped H over G; psi6 = applied update (0 if none);
 * weight = w_i after respawn; donor = -1 or the GLOBAL index cloned into slot i;
 * flags: bit0 loop, bit1 updated, bit2 singular, bit3 dead before respawn, bit4 clamped;
 * representative = GLOBAL argmax w (ties -> lowest); n_dead = global dead count.
 * Global index = sum of the local particle counts of lower ranks + local index. */
typedef struct {
  double*  loglik;
  float*   grad6;
  float*   hess21;
  float*   psi6;
  double*  weight;
  int32_t* donor;
  uint8_t* flags;
  int32_t* representative;
  int64_t* n_dead;
} mcs_update_out;

/* One full filter update with one scan (mean3[n_pts][3], cov6[n_pts][6] in the current
 * sensor frame): a1 neighbours/relative poses, a2 likelihood+gradient sweep, a3 GN update,
 * a4 keyframe propagation, a5 weights, a6 pruning/respawn, a7 representative.
 * D_now = current cumulative odometry path length (R14); resample_u = the respawn uniform
 * u0 = resample_u / 2^32 (R18).  Synchronous; host or device pointers.
 * MCS_E_INVALID_ARG (before any state change) for a null or non-finite scan, a non-SPD scan
 * covariance, n_pts < 1, or D_now below the newest keyframe's path length (the cumulative path
 * length never decreases, R14).
 * Precision (fp32 sweep, fp64 combine/solve): loglik within 1e-4 relative of the exact value
 * for scans of >= 64 points; below that a single point's fp32 transform rounding (~1e-6 m at
 * 10-20 m against centimetre residuals, ~1e-4 of e) is not averaged out and the bound is 2e-3.
 * grad6 within 1e-3 (vector norm), poses within 1e-5 rad / 1e-5 m after one step. */
MCS_API mcs_status mcs_update(mcs_ctx* ctx, const float* scan_mean3, const float* scan_cov6,
                      int32_t n_pts, double D_now, uint32_t resample_u,
                      const mcs_update_out* out);
/* Same, stream-ordered on cuda_stream (NULL = context stream); DEVICE pointers only; the
 * scan is not validated (caller guarantees finite SPD covariances).  On one device, and across
 * ranks joined by NCCL with peer-direct migration, no step waits on the host: the call can be
 * captured into the caller's CUDA graph (a host transport or the pack/send/recv fallback
 * synchronises). */
MCS_API mcs_status mcs_update_async(mcs_ctx* ctx, const float* d_scan_mean3, const float* d_scan_cov6,
                            int32_t n_pts, double D_now, uint32_t resample_u,
                            const mcs_update_out* d_out, void* cuda_stream);

/* Isolated likelihood + gradient evaluation (a1 + a2 + per-slot combine), no state change.
 * Per (particle, slot) s < neighbor_count, row-major [n][neighbor_count]: slot_loglik (fp64
 * value of the fp32 sum), slot_H21 (body frame of T_t), slot_b6 (sum J^T Omega e), slot_n
 * (matched points), slot_kf (keyframe id, -1 if K < slot+1); loop[n] (bit0). */
MCS_API mcs_status mcs_eval(mcs_ctx* ctx, const float* scan_mean3, const float* scan_cov6,
                    int32_t n_pts, double* slot_loglik, float* slot_H21, float* slot_b6,
                    int32_t* slot_n, int32_t* slot_kf, uint8_t* loop);

/* Isolated respawn (a6) on given inputs, no state change: e[n] (fp64 exp(L - max L)),
 * dead[n] (0 = survivor, nonzero = dead), uniform u -> donor[n] (-1 or donor index).
 * Domain: every e_i finite in [0, 1] (e = exp(L - max L)); otherwise MCS_E_INVALID_ARG.  Within
 * it the result is bit-exact with the oracle's integer-ladder systematic resampler (R18) for
 * any e, including survivors whose rung floor(e 2^32) is 0 (they never donate);
 * MCS_E_DEGENERATE when some particle is dead and every rung is 0.  Single-device. */
MCS_API mcs_status mcs_resample(mcs_ctx* ctx, const double* e, const uint8_t* dead, int32_t n,
                        uint32_t u, int32_t* donor_out);

/* Device-side checkpoint of the particle state (poses, keyframe poses, L): mcs_snapshot copies
 * it into a context-owned buffer, mcs_restore copies it back.  Stream-ordered. */
MCS_API mcs_status mcs_snapshot(mcs_ctx* ctx);
MCS_API mcs_status mcs_restore(mcs_ctx* ctx);

/* Multi-GPU respawn plan (host functions; pure functions of allgathered per-rank totals).
 * mcs_plan_ladder: from every rank's survivor-ladder total Q_g (sum of floor(e_i 2^32) over its
 * survivors, R18) and dead count D_g, in rank order: each rank's ladder and dead offsets, the
 * number of clones its survivors make under the GLOBAL systematic count formula with uniform u,
 * and the totals.  MCS_E_DEGENERATE if D > 0 and Q = 0.  Output pointers may be NULL.
 * mcs_plan_migration: send_counts[src * world + dst] = clones made on rank src that land in dead
 * slots of rank dst (the r-th global clone fills the r-th global dead slot, both ascending). */
MCS_API mcs_status mcs_plan_ladder(int32_t world, const uint64_t* Q_per_rank,
                                   const int64_t* D_per_rank, uint32_t u, uint64_t* q_offset,
                                   int64_t* d_offset, int64_t* clones_per_rank, uint64_t* Q_total,
                                   int64_t* D_total);
MCS_API mcs_status mcs_plan_migration(int32_t world, const int64_t* clones_per_rank,
                                      const int64_t* dead_per_rank, int64_t* send_counts);

/* Prediction step (Eq.1): for every local particle i (global index g),
 *   T_t^i = T_{t-1}^i dT exp(delta_i),  delta_i = chol(cov) z,  z ~ N(0, I)
 * with z from Philox4x32-10 keyed by seed, counter (block, g, frame), and fp64 Box-Muller
 * (R31).  dT12: odometry relative motion (pose12, host or device); cov36: 6x6 row-major SPD
 * covariance of the twist (rho, phi) or all zeros.  vertical_sigma > 0 adds the elevator
 * heuristic's world-frame vertical random walk t_z += vertical_sigma z_6.
 * MCS_E_INVALID_ARG if cov is neither SPD nor zero. */
MCS_API mcs_status mcs_predict(mcs_ctx* ctx, const float* dT12, const double* cov36,
                               uint64_t seed, uint64_t frame, double vertical_sigma);

/* Keyframe-insertion test: the fraction of scan points (mean3[n_pts][3]) whose
 * cell, after the transform rel12 (T_kf^-1 T_now from odometry), is occupied in keyframe kf's
 * voxel map (same pinned key path as the likelihood, R27).  Insert a keyframe when it falls
 * below 0.7. */
MCS_API mcs_status mcs_overlap(mcs_ctx* ctx, const float* scan_mean3, int32_t n_pts,
                               const float* rel12, int32_t kf, double* out_rate);

/* NCCL unique id (128 bytes) for mcs_config.nccl_unique_id; rank 0 creates it and the caller
 * broadcasts it (e.g. through torch.distributed).  MCS_E_NCCL if libnccl.so.2 is unavailable. */
MCS_API mcs_status mcs_nccl_unique_id(void* out128);

/* In-process transport joining `world` contexts of one process (one thread per rank); for tests
 * of the multi-rank path on a single device.  Reductions run in rank order. */
MCS_API mcs_transport* mcs_inproc_transport_create(int32_t world);
MCS_API void mcs_inproc_transport_destroy(mcs_transport* t);

/* Per-particle state bytes with K keyframes: 48 (T_t) + 48 K (T_k) + 8 (L). */
MCS_API size_t mcs_state_bytes_per_particle(int32_t n_keyframes);

/* Cumulative device time of the last update's phases, milliseconds (CUDA events):
 * [0] a1 select, [1] a2 sweep, [2] a3+a4 update, [3] a5-a7 weights/respawn, [4] total.
 * Only filled when profiling is enabled with mcs_set_profiling(ctx, 1). */
MCS_API mcs_status mcs_set_profiling(mcs_ctx* ctx, int32_t enable);
MCS_API mcs_status mcs_get_phase_ms(const mcs_ctx* ctx, float* ms5);
/* Migration path of a multi-rank context after its first respawn: 1 peer-direct (the draws
 * kernel writes clones into other ranks' memory), -1 packed + NCCL / transport exchange,
 * 0 not decided yet (no respawn so far, or world_size 1 without an exchange path). */
MCS_API int32_t mcs_peer_migration_state(const mcs_ctx* ctx);
/* 1 if the library holds a captured CUDA graph of the update body (mcs_config.graph_replay and
 * a device-resident exchange path: one device, or NCCL with peer-direct migration), else 0. */
MCS_API int32_t mcs_graph_state(const mcs_ctx* ctx);
/* Scan form of the last scan prepared by mcs_update / mcs_update_async / mcs_eval (R36,
 * DESIGN.md §3): *n_out = the number of its points whose covariance is NOT plane-form (the two
 * largest eigenvalues of the fp32 covariance differ by more than 2^-21 of the largest).  0
 * selects the sweep's plane-form instantiation (one rotated vector per point, Sigma =
 * lambda3 I + [x]x^T [x]x); any other value the general one (Sigma = lambda3 I + u u^T + v v^T).
 * Both compute C = Sigma' + R Sigma R^T of Eq.4 up to rounding.  Synchronises the
 * context's stream (after mcs_update_async on another stream, synchronise that stream first);
 * MCS_E_STATE before any scan was prepared, MCS_E_INVALID_ARG if n_out is NULL. */
MCS_API mcs_status mcs_scan_nonplanar(mcs_ctx* ctx, int32_t* n_out);

#ifdef __cplusplus
}
#endif
#endif /* MCS_H */
