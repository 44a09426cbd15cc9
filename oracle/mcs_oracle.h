/*
 * mcs_oracle.h — TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * Plain, slow CPU oracle for the hot path of arXiv 2504.18056 (gradient-guided
 * 6-DoF Monte Carlo SLAM): per-particle GICP log-likelihood + SE(3) gradient
 * against a shared keyframe map, Gauss-Newton current-pose update, keyframe
 * propagation, importance weights, dead-particle pruning / respawn.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
 * --impl reference) may load this library.  It shares no code, header, table or
 * helper with paper_2504_18056_b200/ (the CUDA product path), and neither
 * includes the other.
 *
 * Citations: P:n = line n of the paper's PAPER.md; S:n = line n of SPEC.md;
 * Rn = reading n in DESIGN.md §3 (the paper is silent/garbled there).
 * Arithmetic is fp64 except the pinned fp32 correspondence-key path (R27).
 *
 * Pose format everywhere: row-major 3x4 [R|t]; p[4*a+b] = R[a][b], p[4*a+3] = t[a].
 * Twist order: (rho, phi) — translation first (R2).
 * Covariance format cov6: (xx, xy, xz, yy, yz, zz).
 *
 * Pins (tests/test_oracle_pins.py, test_oracle_rules.py, test_oracle_next.py,
 * test_oracle_diversity.py; golden hand cases in tests/golden/): every function
 * here is pinned by closed forms, hand cases, invariants or brute force — the
 * G-slot combine (R4), the unmatched penalty (R8), the posterior floor
 * and pre/post-update weighting (R13) by hand cases since round 2.  What no pin
 * can fix are the readings themselves: the absolute likelihood
 * scale on synthetic scenes (the paper prints no worked example), the
 * pruning-threshold semantics (R17), Eq.10's frame convention (R16) and the
 * diversity term as a whole (R35) are interpretations of the paper, implemented
 * and pinned as stated.
 */
#ifndef MCS_ORACLE_H
#define MCS_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int32_t neighbor_count;      /* 3                                    */
  int32_t loop_recency_gap;    /* 10 (R5): slot "old" iff kf <= latest - gap   */
  float   voxel_resolution;    /* r, power of two (R27)                        */
  int32_t gn_slots;            /* 0: old slots only (Fig.3, R4); 1: all slots  */
  double  damping_rel;         /* lambda = damping_rel * tr(H)/6 (R11)         */
  double  step_clamp;          /* ||psi|| <= step_clamp (R11)                  */
  double  unmatched_penalty;   /* kappa (R8), 0 default                        */
  double  loglik_rel_floor;    /* ln(1e-16) (R17)                       */
  double  posterior_floor;     /* 1e-8                                 */
  int32_t gn_iterations;       /* GN steps per update (R12), 1 default         */
  int32_t weight_after_update; /* 0: weight with the pre-update l (R13); 1: re-evaluate */
  int32_t corr_mode;           /* 0: CELL, the containing voxel (R7); 1: NN27 (R33)       */
  float   nn_radius;           /* NN27 candidate radius, 0 < nn_radius <= r (R33)        */
  int32_t clone_split;         /* 0: a clone copies the donor's L (R19); 1: split (R34)  */
  double  diversity_weight;    /* eta (m^2) of the neighbour-particle term (R35); 0: off  */
  double  diversity_bandwidth; /* h (m^2) of its RBF kernel (R35)                        */
} orc_config;

/* ---- SE(3) (right-applied exp) ---- */
void orc_se3_exp(const double xi[6], double T[12]);
int  orc_se3_log(const double T[12], double xi[6]);          /* 0 ok, 1 near pi */
void orc_compose(const double A[12], const double B[12], double AB[12]);

/* ---- keyframe voxel map (aggregation S:112) ---- */
typedef struct orc_map orc_map;
orc_map* orc_map_build(const float* mean3, const float* cov6, int32_t n, float r);
void     orc_map_free(orc_map* m);
int32_t  orc_map_size(const orc_map* m);
/* the k-th cell of the sorted cell list (the index orc_pair_linearize's corr[] reports) */
int32_t  orc_map_cell(const orc_map* m, int32_t k, double mean[3], double cov6[6]);
/* returns member count (0 = empty cell); writes fp64 mean-of-means / mean-of-covs */
int32_t  orc_map_lookup(const orc_map* m, int32_t cx, int32_t cy, int32_t cz,
                        double mean[3], double cov6[6]);
/* correspondence rule the map answers with (orc_particles / orc_update set it from the
 * config): mode 0 CELL (R7), 1 NN27 with radius nn_radius (R33) */
void     orc_map_set_corr(orc_map* m, int32_t mode, float nn_radius);
/* the correspondence of an already transformed fp32 point q under the map's rule: index into
 * the sorted cell list, or -1 (unmatched) */
int32_t  orc_map_correspond(const orc_map* m, const float q[3]);
/* pinned fp32 cell of a point: returns 0 if out of the 21-bit range (R27) */
int      orc_cell_of(float qx, float qy, float qz, float inv_r, int32_t cell[3]);

/* ---- relative pose kT = (T_k)^-1 T_t (Eq.4): pinned fp32 copy + fp64 copy ---- */
void orc_relpose(const float Tk[12], const float Tt[12], float rel32[12], double rel64[12]);

/* ---- Eqs.3-4 + Eq.6 for one (particle, keyframe) pair ----
 * l = -sum_j e_j^T Omega_j e_j over matched points; H = sum J^T Omega J; b = sum J^T Omega e,
 * J = de/d(delta) under right perturbation of kT (R1-R3).  Optional per-point outputs:
 * corr[j] = index of the matched cell in the map's sorted cell list or -1. */
int orc_pair_linearize(const orc_map* m, const float* mean3, const float* cov6, int32_t S,
                       const float rel32[12], const double rel64[12],
                       double* l, double H[36], double b[6], int32_t* n, int32_t* corr);
/* l for FIXED correspondences and FIXED Omega (GN convention, R3): the function
 * whose derivative H/b linearise.  corr from orc_pair_linearize, Omega36 per point
 * (row-major 3x3 per point, 9 doubles) as evaluated at the linearisation point. */
double orc_pair_loglik_frozen(const orc_map* m, const float* mean3, int32_t S,
                              const double rel64[12], const int32_t* corr,
                              const double* omega9);
/* per-point Omega at rel64 for matched points (for the frozen-FD pin). */
void orc_pair_omegas(const orc_map* m, const float* cov6, int32_t S, const double rel64[12],
                     const int32_t* corr, double* omega9);

/* ---- Eq.5 with damping and clamp (R1, R11) ----
 * psi = -(H + lambda I)^-1 b.  returns 0 ok, 1 singular (not PD).  *clamped set. */
int orc_gn_step(const double H[36], const double b[6], double damping_rel, double step_clamp,
                double psi[6], int32_t* clamped);

/* ---- Eqs.8-9: propagation ratios r_k for k = t_o..latest (R14, R15) ---- */
int orc_propagation_ratio(const double* D, int32_t K, int32_t t_o, double D_now, double* r);

/* ---- per-particle steps 2-7 (neighbours, relpose, likelihood, combine, GN, propagation) ----
 * Runs on the particles listed in idx[0..n_idx) (NULL = all N), in place on pose12 / kf_pose12.
 * Outputs indexed by list position p (0..n_idx).  kf_stride = keyframe capacity per particle
 * (>= K).  slot_* outputs sized n_idx * neighbor_count (slot_H: 36 per slot, body frame). */
typedef struct {
  double*  loglik;     /* [n_idx]          */
  double*  grad6;      /* [n_idx][6]       */
  double*  hess36;     /* [n_idx][36]      */
  double*  psi6;       /* [n_idx][6]       */
  uint8_t* flags;      /* [n_idx] bit0 loop, bit1 updated, bit2 singular, bit4 clamped */
  double*  slot_l;     /* [n_idx][nb] optional */
  double*  slot_H36;   /* [n_idx][nb][36]  */
  double*  slot_b6;    /* [n_idx][nb][6]   */
  int32_t* slot_n;     /* [n_idx][nb]      */
  int32_t* slot_kf;    /* [n_idx][nb]      */
} orc_particle_out;

int orc_particles(const orc_config* cfg,
                  int32_t K, orc_map* const* maps, const double* D, double D_now,
                  int32_t N, float* pose12, float* kf_pose12, int32_t kf_stride,
                  const float* scan_mean3, const float* scan_cov6, int32_t S,
                  const int32_t* idx, int32_t n_idx, int32_t apply_update,
                  orc_particle_out* out);

/* ---- Eq.11 in log space (R22): L += l (if l != NULL); m = max L;
 * e = exp(L - m); S = sum e (ascending index order); w = e / S. ---- */
void orc_weights(int32_t N, double* L, const double* l, double* e, double* w,
                 double* m_out, double* S_out);

/* ---- dead set (R17): dead_i = (l_i - max l < rel_floor) or (w_i < post_floor) ---- */
int64_t orc_dead(int32_t N, const double* l, const double* w, double rel_floor,
                 double post_floor, uint8_t* dead);

/* ---- respawn by exact systematic resampling on the integer ladder (R18) ----
 * donor[i] = -1 for survivors, else the survivor cloned into dead slot i.
 * returns 0 ok, 1 degenerate (no survivor). */
int orc_resample(int32_t N, const double* e, const uint8_t* dead, uint32_t U, int32_t* donor);

/* ---- representative: argmax w, ties -> lowest index ---- */
int32_t orc_representative(int32_t N, const double* w);

/* ---- the whole update, steps 2-11 (SURVEY 8(c) algorithm; P:85 order) ----
 * returns 0 ok, 1 degenerate. */
typedef struct {
  double*  loglik; double* grad6; double* hess36; double* psi6;
  double*  weight; int32_t* donor; uint8_t* flags;
  int32_t* representative; int64_t* n_dead;
} orc_update_out;

/* R35: SVGD's repulsive (diversity) term over the particles' translations t[N][3] (P:32,
 * P:41, P:78 cite it; the paper defines none): d_i = (2 / (h N)) sum_j (t_i - t_j)
 * exp(-|t_i - t_j|^2 / h), i.e. d_i = -grad_{t_i} (1/N) sum_j k(t_i, t_j), k the RBF kernel. */
void orc_diversity(int32_t N, const double* t, double h, double* d);
int orc_update(const orc_config* cfg,
               int32_t K, orc_map* const* maps, const double* D, double D_now,
               int32_t N, float* pose12, float* kf_pose12, int32_t kf_stride, double* L,
               const float* scan_mean3, const float* scan_cov6, int32_t S, uint32_t U,
               orc_update_out* out);

/* ---- Philox4x32-10 (counter-based generator; Salmon et al., SC'11) ---- */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);

/* ---- prediction (Eq.1; R31): for particle i (global index gbase + i)
 * T_t^i = T_{t-1}^i dT exp(delta_i), delta_i = chol(cov) z, z ~ N(0, I) from Philox keyed by
 * seed with counter (block, gbase + i, frame) and fp64 Box-Muller; vertical_sigma > 0 adds the
 * elevator heuristic's world-frame vertical random walk t_z += vertical_sigma * z_6.
 * cov36 row-major 6x6 SPD, or all zero (deterministic prediction).  returns 0, or 1 if cov is
 * neither. ---- */
int orc_predict(int32_t N, float* pose12, const float dT12[12], const double cov36[36],
                uint64_t seed, uint64_t frame, int64_t gbase, double vertical_sigma);
/* the 8 standard normals of particle gi (exposed for the statistical pins) */
void orc_normals8(uint64_t seed, uint64_t frame, int64_t gi, double z[8]);

/* ---- keyframe-insertion overlap: fraction of scan points whose pinned fp32 cell
 * under rel32 is occupied in the map ---- */
double orc_overlap(const orc_map* m, const float* mean3, int32_t S, const float rel32[12]);

int orc_num_threads(void);
void orc_set_num_threads(int n);  /* OpenMP threads of the particle loops (timing only) */

#ifdef __cplusplus
}
#endif
#endif
