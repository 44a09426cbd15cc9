/* c_api_demo.c — the boundary (include/mcs.h) used from plain C99: no Python, no PyTorch.
 *
 * One keyframe (a room of three walls and a floor, r = 0.5 m), N particles scattered around
 * the true pose (identity), one mcs_update with the keyframe's own cloud as the scan, so the
 * Gauss-Newton step of every loop particle points back towards the identity (Eqs.5-7).
 * Every particle's keyframe pose is the identity (the keyframe was taken at the origin), and
 * the keyframe is old (loop_recency_gap = 0), so every particle loops.
 *
 *   gcc -std=c99 -O2 -Iinclude examples/c_api_demo.c -Lpaper_2504_18056_b200 -lmcs \
 *       -Wl,-rpath,$PWD/paper_2504_18056_b200 -lm -o c_api_demo
 *   ./c_api_demo [N [S [out.bin]]]
 *
 * Prints one JSON line.  With out.bin it also writes the inputs and outputs (layout below) so
 * tests/test_gpu_c_api.py can check them against the oracle.  Exit code = the mcs_status of
 * the first failing call (0 on success); the library's message goes to stderr.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "mcs.h"

static uint64_t rng_state = 0x9E3779B97F4A7C15ull;
static double urand(void) { /* splitmix64 -> [0, 1) */
  uint64_t z = (rng_state += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return (double)(z >> 11) * (1.0 / 9007199254740992.0);
}

/* S surface points of a room: walls x = 7.75, y = 7.75, y = -7.75 (heights 0.5-3 m) and the
 * floor z = 0.25 (|x|, |y| < 7.5), each surface in the middle of a voxel layer (r = 0.5 m) and
 * no two surfaces sharing a voxel, so a particle off by less than r / 2 along a surface normal
 * still finds that surface's cells; each point's covariance is thin along the normal (GICP
 * plane-like Gaussians) */
static void make_cloud(int S, float* mean3, float* cov6) {
  for (int j = 0; j < S; ++j) {
    const int face = j % 4;
    const double a = 15.0 * urand() - 7.5, h = 0.5 + 2.5 * urand();
    double p[3], n[3] = {0, 0, 0};
    if (face == 0) { p[0] = 7.75;  p[1] = a;     p[2] = h;    n[0] = 1; }
    if (face == 1) { p[0] = a;     p[1] = 7.75;  p[2] = h;    n[1] = 1; }
    if (face == 2) { p[0] = a;     p[1] = -7.75; p[2] = h;    n[1] = 1; }
    if (face == 3) { p[0] = a;     p[1] = 15.0 * urand() - 7.5; p[2] = 0.25; n[2] = 1; }
    const double sn = 0.01 * 0.01, st = 0.1 * 0.1; /* normal / tangential variances */
    double C[3][3];
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) C[r][c] = (r == c ? st : 0.0) + (sn - st) * n[r] * n[c];
    for (int r = 0; r < 3; ++r) mean3[3 * j + r] = (float)p[r];
    cov6[6 * j + 0] = (float)C[0][0]; cov6[6 * j + 1] = (float)C[0][1];
    cov6[6 * j + 2] = (float)C[0][2]; cov6[6 * j + 3] = (float)C[1][1];
    cov6[6 * j + 4] = (float)C[1][2]; cov6[6 * j + 5] = (float)C[2][2];
  }
}

#define CHECK(call)                                                                 \
  do {                                                                              \
    const mcs_status st_ = (call);                                                  \
    if (st_ != MCS_OK) {                                                            \
      fprintf(stderr, "%s failed (%d): %s\n", #call, (int)st_, mcs_last_error(ctx)); \
      printf("{\"status\": %d, \"call\": \"%s\"}\n", (int)st_, #call);              \
      if (ctx) mcs_destroy(ctx);                                                    \
      return (int)st_;                                                              \
    }                                                                               \
  } while (0)

int main(int argc, char** argv) {
  const int N = argc > 1 ? atoi(argv[1]) : 1000;
  const int S = argc > 2 ? atoi(argv[2]) : 512;
  const char* out_path = argc > 3 ? argv[3] : NULL;
  mcs_ctx* ctx = NULL;
  if (N < 1 || S < 1) return (int)MCS_E_INVALID_ARG;
  float* mean3 = malloc(sizeof(float) * 3 * S);
  float* cov6 = malloc(sizeof(float) * 6 * S);
  float* pose_in = malloc(sizeof(float) * 12 * N);
  float* kf_pose = malloc(sizeof(float) * 12 * N);
  float* pose_out = malloc(sizeof(float) * 12 * N);
  double* loglik = malloc(sizeof(double) * N);
  double* weight = malloc(sizeof(double) * N);
  float* psi = malloc(sizeof(float) * 6 * N);
  int32_t* donor = malloc(sizeof(int32_t) * N);
  uint8_t* flags = malloc(N);
  int32_t rep = -1;
  int64_t n_dead = -1;
  if (!mean3 || !cov6 || !pose_in || !kf_pose || !pose_out || !loglik || !weight || !psi ||
      !donor || !flags)
    return (int)MCS_E_OUT_OF_MEMORY;
  make_cloud(S, mean3, cov6);
  /* particles: yaw in +-0.03 rad, translation in +-0.15 m (x, y), +-0.05 m (z): less than
   * r / 2 off every surface */
  for (int i = 0; i < N; ++i) {
    const double yaw = 0.06 * urand() - 0.03, c = cos(yaw), s = sin(yaw);
    const float T[12] = {(float)c, (float)-s, 0.f, (float)(0.3 * urand() - 0.15),
                         (float)s, (float)c,  0.f, (float)(0.3 * urand() - 0.15),
                         0.f,      0.f,       1.f, (float)(0.1 * urand() - 0.05)};
    const float I[12] = {1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0};
    for (int e = 0; e < 12; ++e) {
      pose_in[12 * i + e] = T[e];
      kf_pose[12 * i + e] = I[e];
    }
  }

  mcs_config cfg;
  mcs_config_default(&cfg);
  cfg.capacity_particles = N;
  cfg.capacity_keyframes = 1;
  cfg.capacity_scan_points = S;
  cfg.voxel_resolution = 0.5f;
  cfg.loop_recency_gap = 0; /* the one keyframe is old: every particle loops */
  CHECK(mcs_create(&cfg, &ctx));
  int32_t kf = -1;
  CHECK(mcs_add_keyframe(ctx, mean3, cov6, S, 0.0, &kf));
  CHECK(mcs_set_particles(ctx, N, pose_in, kf_pose, NULL));
  mcs_update_out out = {0};
  out.loglik = loglik;
  out.psi6 = psi;
  out.weight = weight;
  out.donor = donor;
  out.flags = flags;
  out.representative = &rep;
  out.n_dead = &n_dead;
  const double D_now = 1.0;
  const uint32_t U = 0x5EED1234u;
  CHECK(mcs_update(ctx, mean3, cov6, S, D_now, U, &out));
  CHECK(mcs_get_particles(ctx, pose_out, NULL, NULL, NULL));
  CHECK(mcs_destroy(ctx));
  ctx = NULL;

  double sw = 0.0, t_in = 0.0, t_out = 0.0;
  int updated = 0;
  for (int i = 0; i < N; ++i) {
    sw += weight[i];
    updated += (flags[i] >> 1) & 1;
    if (donor[i] < 0) { /* survivors: summed translation error before / after the GN step */
      t_in += sqrt(pose_in[12 * i + 3] * pose_in[12 * i + 3] +
                   pose_in[12 * i + 7] * pose_in[12 * i + 7] +
                   pose_in[12 * i + 11] * pose_in[12 * i + 11]);
      t_out += sqrt(pose_out[12 * i + 3] * pose_out[12 * i + 3] +
                    pose_out[12 * i + 7] * pose_out[12 * i + 7] +
                    pose_out[12 * i + 11] * pose_out[12 * i + 11]);
    }
  }
  printf("{\"status\": 0, \"N\": %d, \"S\": %d, \"updated\": %d, \"n_dead\": %lld, "
         "\"representative\": %d, \"sum_w\": %.15f, \"survivor_t_err_in\": %.6g, "
         "\"survivor_t_err_out\": %.6g}\n",
         N, S, updated, (long long)n_dead, rep, sw, t_in, t_out);

  if (out_path) {
    /* layout: int32 N, S; f32 mean3[S][3], cov6[S][6], pose_in[N][12]; f64 D_now; u32 U;
     * f64 loglik[N]; f32 psi6[N][6]; f64 weight[N]; i32 donor[N]; u8 flags[N]; i32 rep;
     * i64 n_dead; f32 pose_out[N][12] */
    FILE* f = fopen(out_path, "wb");
    if (!f) return 1;
    const int32_t hdr[2] = {N, S};
    fwrite(hdr, sizeof(int32_t), 2, f);
    fwrite(mean3, sizeof(float), 3 * (size_t)S, f);
    fwrite(cov6, sizeof(float), 6 * (size_t)S, f);
    fwrite(pose_in, sizeof(float), 12 * (size_t)N, f);
    fwrite(&D_now, sizeof(double), 1, f);
    fwrite(&U, sizeof(uint32_t), 1, f);
    fwrite(loglik, sizeof(double), (size_t)N, f);
    fwrite(psi, sizeof(float), 6 * (size_t)N, f);
    fwrite(weight, sizeof(double), (size_t)N, f);
    fwrite(donor, sizeof(int32_t), (size_t)N, f);
    fwrite(flags, 1, (size_t)N, f);
    fwrite(&rep, sizeof(int32_t), 1, f);
    fwrite(&n_dead, sizeof(int64_t), 1, f);
    fwrite(pose_out, sizeof(float), 12 * (size_t)N, f);
    fclose(f);
  }
  free(mean3); free(cov6); free(pose_in); free(kf_pose); free(pose_out);
  free(loglik); free(weight); free(psi); free(donor); free(flags);
  return 0;
}
