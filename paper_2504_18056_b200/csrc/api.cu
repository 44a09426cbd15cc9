// api.cu — the C-ABI of libmcs (include/mcs.h): validation, lifecycle, state, orchestration of
// the hot path a1..a7 on the context stream.  No compute happens on the host: every step of
// the path runs in the kernels of select.cu, sweep.cu, update.cu, weights.cu, kf_store.cu.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "mcs_internal.cuh"

using namespace mcs;

static thread_local std::string g_create_error;

#define FAIL(ctx, code, ...)                                   \
  do {                                                         \
    char _b[512];                                              \
    snprintf(_b, sizeof(_b), __VA_ARGS__);                     \
    (ctx)->err = _b;                                           \
    return (code);                                             \
  } while (0)

#define CUDA_TRY(ctx, x)                                                               \
  do {                                                                                 \
    cudaError_t _e = (x);                                                              \
    if (_e != cudaSuccess) {                                                           \
      (ctx)->sticky = MCS_E_CUDA;                                                      \
      char _b[512];                                                                    \
      snprintf(_b, sizeof(_b), "CUDA error %s at %s:%d: %s", cudaGetErrorName(_e),     \
               __FILE__, __LINE__, cudaGetErrorString(_e));                            \
      (ctx)->err = _b;                                                                 \
      return MCS_E_CUDA;                                                               \
    }                                                                                  \
  } while (0)

#define CHECK_CTX(ctx)                                  \
  do {                                                  \
    if (!(ctx)) return MCS_E_INVALID_ARG;               \
    if ((ctx)->sticky != MCS_OK) return (ctx)->sticky;  \
  } while (0)

// ------------------------------------------------------------------ small device kernels
__global__ void fill_kf_from_current_kernel(const float* __restrict__ pose, int capN, int N,
                                            float* __restrict__ kfpose, float4* __restrict__ kft,
                                            int capK, int k0, int k1) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int nk = k1 - k0;
  if (t >= (long long)N * nk) return;
  const int i = (int)(t / nk), k = k0 + (int)(t - (long long)i * nk);
  float* dst = kfpose + ((size_t)i * capK + k) * 12;
#pragma unroll
  for (int e = 0; e < 12; ++e) dst[e] = pose[(size_t)e * capN + i];
  kft[(size_t)i * capK + k] = make_float4(dst[3], dst[7], dst[11], 0.f);
}

// the translation plane of keyframes [0, K) from the poses (after a bulk pose copy)
__global__ void kft_from_kfpose_kernel(const float* __restrict__ kfpose, int capK, int N, int K,
                                       float4* __restrict__ kft) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)N * K) return;
  const int i = (int)(t / K), k = (int)(t - (long long)i * K);
  const float* T = kfpose + ((size_t)i * capK + k) * 12;
  kft[(size_t)i * capK + k] = make_float4(T[3], T[7], T[11], 0.f);
}

__global__ void aos_to_soa_kernel(const float* __restrict__ aos, int N, int capN,
                                  float* __restrict__ soa) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
#pragma unroll
  for (int e = 0; e < 12; ++e) soa[(size_t)e * capN + i] = aos[(size_t)i * 12 + e];
}

__global__ void soa_to_aos_kernel(const float* __restrict__ soa, int N, int capN,
                                  float* __restrict__ aos) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
#pragma unroll
  for (int e = 0; e < 12; ++e) aos[(size_t)i * 12 + e] = soa[(size_t)e * capN + i];
}

// counts non-finite values and rotation blocks that are not orthonormal (|R^T R - I| > 1e-3)
__global__ void validate_poses_kernel(const float* __restrict__ p, long long n_poses,
                                      int* __restrict__ bad) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_poses) return;
  const float* T = p + t * 12;
  bool ok = true;
  for (int e = 0; e < 12; ++e) ok = ok && isfinite(T[e]);
  if (ok) {
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        float s = 0.f;
        for (int c = 0; c < 3; ++c) s += T[4 * c + a] * T[4 * c + b];
        ok = ok && fabsf(s - (a == b ? 1.f : 0.f)) < 1e-3f;
      }
  }
  if (!ok) atomicAdd(bad, 1);
}

// non-finite means or non-SPD covariances (Sylvester on fp64)
__global__ void validate_gauss_kernel(const float* __restrict__ mean3,
                                      const float* __restrict__ cov6, int n,
                                      int* __restrict__ bad) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  bool ok = isfinite(mean3[3 * j]) && isfinite(mean3[3 * j + 1]) && isfinite(mean3[3 * j + 2]);
  const float* c = cov6 + 6 * j;
  for (int k = 0; k < 6; ++k) ok = ok && isfinite(c[k]);
  if (ok) {
    const double xx = c[0], xy = c[1], xz = c[2], yy = c[3], yz = c[4], zz = c[5];
    const double m2 = xx * yy - xy * xy;
    const double m3 = xx * (yy * zz - yz * yz) - xy * (xy * zz - yz * xz) + xz * (xy * yz - yy * xz);
    ok = xx > 0.0 && m2 > 0.0 && m3 > 0.0;
  }
  if (!ok) atomicAdd(bad, 1);
}

__global__ void pose_column_kernel(const float* __restrict__ pose, int capN, int i,
                                   double* __restrict__ out) {
  const int k = threadIdx.x;
  if (k < 12) out[k] = i >= 0 ? (double)pose[(size_t)k * capN + i] : 0.0;
}

__global__ void validate_unit_kernel(const double* __restrict__ e, int n, int* bad) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && !(e[i] >= 0.0 && e[i] <= 1.0)) atomicAdd(bad, 1);  // NaN fails both
}

__global__ void fill_double_kernel(double* __restrict__ p, int n, double v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

struct OutPtrs {
  double* loglik;
  float* grad6;
  float* hess21;
  float* psi6;
  double* weight;
  int32_t* donor;
  uint8_t* flags;
  int32_t* rep;
  int64_t* n_dead;
};

__global__ void gather_outputs_kernel(OutPtrs o, int N, int capN, const double* __restrict__ l,
                                      const float* __restrict__ grad,
                                      const float* __restrict__ hess,
                                      const double* __restrict__ psi,
                                      const double* __restrict__ e,
                                      const int32_t* __restrict__ donor,
                                      const uint8_t* __restrict__ flags, const Scalars* sc) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0) {
    if (o.rep) *o.rep = (int32_t)sc->rep;
    if (o.n_dead) *o.n_dead = sc->D_tot;
  }
  if (i >= N) return;
  if (o.loglik) o.loglik[i] = l[i];
  if (o.grad6)
    for (int k = 0; k < 6; ++k) o.grad6[(size_t)i * 6 + k] = grad[(size_t)k * capN + i];
  if (o.hess21)
    for (int k = 0; k < 21; ++k) o.hess21[(size_t)i * 21 + k] = hess[(size_t)k * capN + i];
  if (o.psi6)
    for (int k = 0; k < 6; ++k) o.psi6[(size_t)i * 6 + k] = (float)psi[(size_t)k * capN + i];
  if (o.weight) o.weight[i] = e[i] / sc->S2;  // w = e' / S' (weights.cu)
  if (o.donor) o.donor[i] = donor[i];
  if (o.flags) o.flags[i] = flags[i];
}

// ------------------------------------------------------------------ helpers
namespace mcs {
// a user allocator's block must be 256-byte aligned like cudaMalloc's (vector loads of table
// slots); a misaligned one is returned and reported as cudaErrorMisalignedAddress, which the
// callers turn into MCS_E_INVALID_ARG
static cudaError_t user_block(mcs_ctx* c, void** p, cudaStream_t st) {
  if (!*p) return cudaErrorMemoryAllocation;
  if (reinterpret_cast<uintptr_t>(*p) % 256 != 0) {
    c->alloc.free(*p, (void*)st, c->alloc.user);
    *p = nullptr;
    return cudaErrorMisalignedAddress;
  }
  return cudaSuccess;
}
cudaError_t mem_alloc(mcs_ctx* c, void** p, size_t bytes) {
  if (!bytes) bytes = 1;
  if (c->alloc.alloc) {
    *p = c->alloc.alloc(bytes, (void*)c->stream, c->alloc.user);
    return user_block(c, p, c->stream);
  }
  return cudaMalloc(p, bytes);
}
void mem_free(mcs_ctx* c, void* p) {
  if (!p) return;
  if (c->alloc.alloc) c->alloc.free(p, (void*)c->stream, c->alloc.user);
  else cudaFree(p);
}
cudaError_t mem_alloc_async(mcs_ctx* c, void** p, size_t bytes, cudaStream_t st) {
  if (!bytes) bytes = 1;
  if (c->alloc.alloc) {
    *p = c->alloc.alloc(bytes, (void*)st, c->alloc.user);
    return user_block(c, p, st);
  }
  return cudaMallocAsync(p, bytes, st);
}
void mem_free_async(mcs_ctx* c, void* p, cudaStream_t st) {
  if (!p) return;
  if (c->alloc.alloc) c->alloc.free(p, (void*)st, c->alloc.user);
  else cudaFreeAsync(p, st);
}
}  // namespace mcs

template <typename T>
static cudaError_t dalloc(mcs_ctx* c, T** p, size_t count) {
  return mem_alloc(c, (void**)p, sizeof(T) * (count ? count : 1));
}

static bool is_pow2_float(float r) {
  if (!(r > 0.f) || !std::isfinite(r)) return false;
  int ex;
  float m = std::frexp(r, &ex);
  return m == 0.5f;
}

static void free_all(mcs_ctx* c) {
  for (auto& k : c->kf) mem_free_async(c, k.slots, c->stream);
  void* ptrs[] = {c->d_kf_meta, c->d_D,       c->d_pose,     c->d_kfpose,   c->d_kft, c->d_L,
                  c->d_snapshot, c->d_scan_raw, c->d_scan,    c->d_items,    c->d_order,
                  c->d_part,    c->d_meta,    c->d_to,       c->d_l,        c->d_psi,
                  c->d_grad,    c->d_hess,    c->d_flags,    c->d_e,        c->d_xg,
                  c->d_ladder,  c->d_ladder_scan, c->d_donor,    c->d_partials,
                  c->d_ipartials, c->d_scal,  c->d_cub_temp, c->d_skeys, c->d_skeys_out,
                  c->d_sids,    c->d_stage,   c->d_bad,      c->d_dead_list, c->d_donor_g,
                  c->d_plan,    c->d_pack_src, c->d_send,    c->d_recv,     c->d_tall,
                  c->d_divn};
  for (void* p : ptrs) mem_free(c, p);
  if (c->h_scal) cudaFreeHost(c->h_scal);
  if (c->h_stage) cudaFreeHost(c->h_stage);
  if (c->gexec) cudaGraphExecDestroy(c->gexec);
  c->gexec = nullptr;
  dist_destroy(c);
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  if (c->fork_ev) cudaEventDestroy(c->fork_ev);
  if (c->join_ev) cudaEventDestroy(c->join_ev);
  if (c->side) cudaStreamDestroy(c->side);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
}

// output staging layout of the synchronous mcs_update (per-particle rows, 256-B aligned)
struct StageLayout {
  size_t l, g, h, p, w, d, f, total;
  explicit StageLayout(size_t N) {
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 255) & ~size_t(255); return o; };
    l = take(8 * N); g = take(24 * N); h = take(84 * N); p = take(24 * N);
    w = take(8 * N); d = take(4 * N); f = take(N);
    total = off;
  }
};

// copy n bytes from a host-or-device pointer into device memory, stream-ordered
static cudaError_t to_device(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, st);
}

// ------------------------------------------------------------------ ABI
extern "C" {

size_t mcs_config_size(void) { return sizeof(mcs_config); }

void mcs_config_default(mcs_config* cfg) {
  if (!cfg) return;
  memset(cfg, 0, sizeof(*cfg));
  cfg->abi_version = MCS_ABI_VERSION;
  cfg->neighbor_count = 3;
  cfg->loop_recency_gap = 10;
  cfg->voxel_resolution = 0.5f;
  cfg->gn_slots = MCS_GN_OLD_SLOTS;
  cfg->damping_rel = 1e-6;
  cfg->step_clamp = 1.0;
  cfg->unmatched_penalty = 0.0;
  cfg->loglik_rel_floor = std::log(1e-16);
  cfg->posterior_floor = 1e-8;
  cfg->device = 0;
  cfg->gn_iterations = 1;
  cfg->weight_after_update = 0;
  cfg->corr_mode = MCS_CORR_CELL;
  cfg->nn_radius = 0.0f;
  cfg->clone_split = 0;
  cfg->peer_migration = 1;
  cfg->graph_replay = 1;
  cfg->kf_table_mib = 64;
  cfg->diversity_weight = 0.0;
  cfg->diversity_bandwidth = 1.0;
  cfg->point_splits = 0;
  cfg->rank = 0;
  cfg->world_size = 1;
  cfg->nccl_unique_id = nullptr;
}

size_t mcs_state_bytes_per_particle(int32_t n_keyframes) {
  return 48u + 48u * (size_t)(n_keyframes < 0 ? 0 : n_keyframes) + 8u;
}

const char* mcs_last_error(const mcs_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_create_error.c_str();
}

mcs_status mcs_create(const mcs_config* cfg, mcs_ctx** out) {
  g_create_error.clear();
  if (!cfg || !out) { g_create_error = "null argument"; return MCS_E_INVALID_ARG; }
  *out = nullptr;
  if (cfg->abi_version != MCS_ABI_VERSION) {
    g_create_error = "abi_version mismatch";
    return MCS_E_INVALID_ARG;
  }
  if (cfg->capacity_particles < 1 || cfg->capacity_keyframes < 1 ||
      cfg->capacity_scan_points < 1) {
    g_create_error = "capacities must be >= 1";
    return MCS_E_INVALID_ARG;
  }
  if (cfg->neighbor_count < 1 || cfg->neighbor_count > MCS_MAX_NEIGHBORS) {
    g_create_error = "neighbor_count must be in [1, MCS_MAX_NEIGHBORS]";
    return MCS_E_INVALID_ARG;
  }
  if (!is_pow2_float(cfg->voxel_resolution)) {
    g_create_error = "voxel_resolution must be a positive power of two (DESIGN.md R27)";
    return MCS_E_INVALID_ARG;
  }
  if (cfg->loop_recency_gap < 0 || (cfg->gn_slots != 0 && cfg->gn_slots != 1) ||
      !(cfg->damping_rel >= 0) || !(cfg->step_clamp > 0) || !(cfg->unmatched_penalty >= 0) ||
      std::isnan(cfg->loglik_rel_floor) || std::isnan(cfg->posterior_floor)) {
    g_create_error = "invalid numeric configuration";
    return MCS_E_INVALID_ARG;
  }
  if (!std::isfinite(cfg->diversity_weight) ||
      (cfg->diversity_weight != 0.0 &&
       !(cfg->diversity_bandwidth > 0.0 && std::isfinite(cfg->diversity_bandwidth)))) {
    g_create_error = "diversity_weight must be finite, diversity_bandwidth > 0 and finite (R35)";
    return MCS_E_INVALID_ARG;
  }
  if (cfg->gn_iterations < 1 || cfg->gn_iterations > 64 ||
      (cfg->weight_after_update != 0 && cfg->weight_after_update != 1)) {
    g_create_error = "gn_iterations must be in [1, 64], weight_after_update 0 or 1";
    return MCS_E_INVALID_ARG;
  }
  if ((cfg->corr_mode != MCS_CORR_CELL && cfg->corr_mode != MCS_CORR_NN27) ||
      (cfg->corr_mode == MCS_CORR_NN27 &&
       !(cfg->nn_radius > 0.0f && cfg->nn_radius <= cfg->voxel_resolution)) ||
      (cfg->clone_split != 0 && cfg->clone_split != 1) ||
      (cfg->peer_migration != 0 && cfg->peer_migration != 1) ||
      (cfg->graph_replay != 0 && cfg->graph_replay != 1) ||
      cfg->point_splits < 0 || cfg->point_splits > 16 || cfg->kf_table_mib < 0 ||
      cfg->kf_table_mib > 65536) {
    g_create_error = "corr_mode must be CELL or NN27 (with 0 < nn_radius <= voxel_resolution), "
                     "clone_split, peer_migration and graph_replay 0 or 1; point_splits 0..16; "
                     "kf_table_mib 0..65536";
    return MCS_E_INVALID_ARG;
  }
  if (cfg->world_size < 1 || cfg->rank < 0 || cfg->rank >= cfg->world_size) {
    g_create_error = "need 0 <= rank < world_size";
    return MCS_E_INVALID_ARG;
  }
  if (cfg->world_size > 1 && !cfg->transport && !cfg->nccl_unique_id) {
    g_create_error = "world_size > 1 needs nccl_unique_id or a transport";
    return MCS_E_INVALID_ARG;
  }
  if ((long long)cfg->capacity_particles * cfg->neighbor_count > 0x7fffffffLL) {
    g_create_error = "capacity_particles * neighbor_count exceeds 2^31";
    return MCS_E_CAPACITY;
  }
  if (cfg->capacity_particles > (1 << 21)) {  // exact ladder: N * 2^32 < 2^53 (R18)
    g_create_error = "capacity_particles > 2^21 per device (integer-ladder bound, R18)";
    return MCS_E_CAPACITY;
  }
  if (cfg->allocator && (!cfg->allocator->alloc || !cfg->allocator->free)) {
    g_create_error = "allocator needs both alloc and free";
    return MCS_E_INVALID_ARG;
  }
  mcs_ctx* c = new mcs_ctx();
  c->cfg = *cfg;
  if (cfg->allocator) c->alloc = *cfg->allocator;
  c->cfg.allocator = nullptr;  // copied above; the caller's struct need not outlive the call
  c->dev = cfg->device;
  c->capN = cfg->capacity_particles;
  c->capK = cfg->capacity_keyframes;
  c->capS = cfg->capacity_scan_points;
  c->nbcap = cfg->neighbor_count;
  cudaError_t e = cudaSetDevice(c->dev);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
  c->own_stream = (e == cudaSuccess);
  const size_t N = c->capN, K = c->capK, S = c->capS, nb = c->nbcap;
  const size_t maxb = (N + 31) / 32 + 64;  // block partials: combine runs 32 particles per block
  if (e == cudaSuccess) e = dalloc(c, &c->d_kf_meta, K);
  if (e == cudaSuccess) e = dalloc(c, &c->d_D, K);
  if (e == cudaSuccess) e = dalloc(c, &c->d_pose, 12 * N);
  if (e == cudaSuccess) e = dalloc(c, &c->d_kfpose, N * K * 12);
  if (e == cudaSuccess) e = dalloc(c, &c->d_kft, N * K);
  if (e == cudaSuccess) e = dalloc(c, &c->d_L, N);
  if (e == cudaSuccess) e = dalloc(c, &c->d_scan_raw, 9 * S);
  if (e == cudaSuccess) e = dalloc(c, &c->d_scan, 5 * S + 1);
  if (e == cudaSuccess) {
    c->d_scan_plane = c->d_scan + 3 * S;
    c->d_scan_np = reinterpret_cast<int*>(c->d_scan + 5 * S);
  }
  if (e == cudaSuccess) e = dalloc(c, &c->d_items, 4 * nb * N);
  if (e == cudaSuccess) e = dalloc(c, &c->d_order, nb * N);
  if (e == cudaSuccess) e = dalloc(c, &c->d_skeys, nb * N);
  if (e == cudaSuccess) e = dalloc(c, &c->d_skeys_out, nb * N);
  if (e == cudaSuccess) e = dalloc(c, &c->d_sids, nb * N);
  if (e == cudaSuccess) e = dalloc(c, &c->d_bad, 1);
  if (e == cudaSuccess) e = dalloc(c, &c->d_dead_list, N);
  if (e == cudaSuccess) e = dalloc(c, &c->d_donor_g, N);
  if (e == cudaSuccess) e = dalloc(c, &c->d_plan, 5 * (size_t)(cfg->world_size + 1));
  if (e == cudaSuccess) {
    c->stage_bytes = StageLayout(N).total;
    e = dalloc(c, &c->d_stage, c->stage_bytes);
  }
  if (e == cudaSuccess) {  // keep stream-ordered allocations mapped between calls
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, c->dev) == cudaSuccess) {
      uint64_t thr = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    // Reserve the keyframe tables' share of the pool now (capacity_keyframes tables at the
    // per-keyframe budget, at most 16 GiB): the pool keeps the block mapped after the free, so
    // a later insertion (a0) takes its table without growing the pool (page mapping: ms).
    if (!c->alloc.alloc && K > 0) {
      const size_t tab = (size_t)std::max(cfg->kf_table_mib, 1) << 20;
      const size_t want = std::min((size_t)K * (tab + 4096), (size_t)16 << 30);
      void* p = nullptr;
      if (cudaMallocAsync(&p, want, c->stream) == cudaSuccess) {
        cudaFreeAsync(p, c->stream);
      } else {
        cudaGetLastError();  // not enough memory to reserve: insertions grow the pool instead
      }
    }
  }
  c->part_splits = cfg->point_splits > 0 ? cfg->point_splits : 1;
  if (e == cudaSuccess) e = dalloc(c, &c->d_part, (size_t)kSlotWords * nb * N * c->part_splits);
  if (e == cudaSuccess) e = dalloc(c, &c->d_meta, N);
  if (e == cudaSuccess) e = dalloc(c, &c->d_to, N);
  if (e == cudaSuccess) e = dalloc(c, &c->d_l, N);
  if (e == cudaSuccess) e = dalloc(c, &c->d_psi, 6 * N);
  if (e == cudaSuccess) e = dalloc(c, &c->d_grad, 6 * N);
  if (e == cudaSuccess) e = dalloc(c, &c->d_hess, 21 * N);
  if (e == cudaSuccess) e = dalloc(c, &c->d_flags, N);
  if (e == cudaSuccess) e = dalloc(c, &c->d_e, N);
  if (e == cudaSuccess) e = dalloc(c, &c->d_xg, 64 * (size_t)(cfg->world_size + 1) + 96);
  // look-back tile states of the ladder scan: 32 B per 1,024-particle tile
  const size_t ladder_bytes = 32 * ((N + 1023) / 1024 + 1);
  // look-back tile flags carry a launch epoch; zero memory matches no published tile
  if (e == cudaSuccess) e = mem_alloc(c, &c->d_ladder, ladder_bytes);
  if (e == cudaSuccess) e = cudaMemset(c->d_ladder, 0, ladder_bytes);
  if (e == cudaSuccess) e = mem_alloc(c, &c->d_ladder_scan, 8 * N);
  if (e == cudaSuccess) e = dalloc(c, &c->d_donor, N);
  if (e == cudaSuccess) e = dalloc(c, &c->d_partials, 2 * maxb);
  if (e == cudaSuccess) e = dalloc(c, &c->d_ipartials, 2 * maxb);
  if (e == cudaSuccess) e = dalloc(c, &c->d_scal, 1);
  if (e == cudaSuccess) e = cudaMemset(c->d_scal, 0, sizeof(Scalars));
  if (e == cudaSuccess) e = cudaMallocHost((void**)&c->h_scal, sizeof(Scalars));
  if (e == cudaSuccess) {
    c->cub_temp_bytes = sort_temp_needed((int)(nb * N), (int)K);
    e = mem_alloc(c, &c->d_cub_temp, c->cub_temp_bytes);
  }
  for (int k = 0; k < 6 && e == cudaSuccess; ++k) e = cudaEventCreate(&c->ev[k]);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->fork_ev, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->join_ev, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e == cudaSuccess) {
    std::string derr;
    const mcs_status ds = dist_init(c, derr);
    if (ds != MCS_OK) {
      g_create_error = derr;
      free_all(c);
      delete c;
      return ds;
    }
  }
  if (e != cudaSuccess) {
    g_create_error = std::string("CUDA: ") + cudaGetErrorString(e);
    free_all(c);
    delete c;
    if (e == cudaErrorMisalignedAddress)
      g_create_error = "the allocator hook returned memory that is not 256-byte aligned";
    return e == cudaErrorMemoryAllocation ? MCS_E_OUT_OF_MEMORY
           : e == cudaErrorMisalignedAddress ? MCS_E_INVALID_ARG : MCS_E_CUDA;
  }
  *out = c;
  return MCS_OK;
}

mcs_status mcs_destroy(mcs_ctx* ctx) {
  if (!ctx) return MCS_E_INVALID_ARG;
  cudaSetDevice(ctx->dev);
  cudaStreamSynchronize(ctx->stream);
  free_all(ctx);
  delete ctx;
  return MCS_OK;
}

mcs_status mcs_set_stream(mcs_ctx* ctx, void* cuda_stream) {
  CHECK_CTX(ctx);
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
  if (cuda_stream) {
    ctx->stream = (cudaStream_t)cuda_stream;
    ctx->own_stream = false;
  } else {
    CUDA_TRY(ctx, cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    ctx->own_stream = true;
  }
  return MCS_OK;
}

mcs_status mcs_get_sizes(const mcs_ctx* ctx, int32_t* n_local, int32_t* n_keyframes) {
  if (!ctx) return MCS_E_INVALID_ARG;
  if (n_local) *n_local = ctx->N;
  if (n_keyframes) *n_keyframes = ctx->K;
  return MCS_OK;
}

mcs_status mcs_add_keyframe(mcs_ctx* ctx, const float* mean3, const float* cov6, int32_t n,
                            double path_length, int32_t* out_kf_id) {
  CHECK_CTX(ctx);
  if (!mean3 || !cov6 || n < 1) FAIL(ctx, MCS_E_INVALID_ARG, "mcs_add_keyframe: null or n < 1");
  if (!std::isfinite(path_length)) FAIL(ctx, MCS_E_INVALID_ARG, "path_length not finite");
  if (ctx->K >= ctx->capK) FAIL(ctx, MCS_E_CAPACITY, "capacity_keyframes (%d) reached", ctx->capK);
  if (ctx->K > 0 && path_length < ctx->D.back())
    FAIL(ctx, MCS_E_INVALID_ARG, "path_length must be non-decreasing (cumulative, R14)");
  cudaStream_t st = ctx->stream;
  float *dm = nullptr, *dc = nullptr;
  int* bad = nullptr;
  CUDA_TRY(ctx, mem_alloc_async(ctx, (void**)&dm, sizeof(float) * 3 * n, st));
  CUDA_TRY(ctx, mem_alloc_async(ctx, (void**)&dc, sizeof(float) * 6 * n, st));
  CUDA_TRY(ctx, mem_alloc_async(ctx, (void**)&bad, sizeof(int), st));
  CUDA_TRY(ctx, cudaMemsetAsync(bad, 0, sizeof(int), st));
  CUDA_TRY(ctx, to_device(dm, mean3, sizeof(float) * 3 * n, st));
  CUDA_TRY(ctx, to_device(dc, cov6, sizeof(float) * 6 * n, st));
  validate_gauss_kernel<<<(n + 255) / 256, 256, 0, st>>>(dm, dc, n, bad);
  int h_bad = 0;
  CUDA_TRY(ctx, cudaMemcpyAsync(&h_bad, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(ctx, cudaStreamSynchronize(st));
  if (h_bad) {
    mem_free_async(ctx, dm, st); mem_free_async(ctx, dc, st); mem_free_async(ctx, bad, st);
    FAIL(ctx, MCS_E_INVALID_ARG, "%d keyframe points non-finite or covariance not SPD", h_bad);
  }
  KfHost kh;
  int bad_cell = 0, bad_extent = 0;
  cudaError_t e = kf_build(ctx, dm, dc, n, kh, &bad_cell, &bad_extent);
  mem_free_async(ctx, dm, st);
  mem_free_async(ctx, dc, st);
  mem_free_async(ctx, bad, st);
  CUDA_TRY(ctx, e);
  if (bad_cell)
    FAIL(ctx, MCS_E_INVALID_ARG, "%d keyframe points outside the 21-bit cell range", bad_cell);
  if (bad_extent) {
    if (kh.slots) mem_free_async(ctx, kh.slots, st);
    FAIL(ctx, MCS_E_INVALID_ARG,
         "keyframe occupied extent exceeds 2047 x 2048 x 1024 cells at r = %g m",
         (double)ctx->cfg.voxel_resolution);
  }
  const int k = ctx->K;
  const KfMeta m = kh.meta;
  CUDA_TRY(ctx, cudaMemcpyAsync(ctx->d_kf_meta + k, &m, sizeof(m), cudaMemcpyHostToDevice, st));
  CUDA_TRY(ctx, cudaMemcpyAsync(ctx->d_D + k, &path_length, sizeof(double), cudaMemcpyHostToDevice,
                                st));
  // lockstep extension: T_k^i := T_t^i (R24)
  if (ctx->N > 0) {
    fill_kf_from_current_kernel<<<(ctx->N + 255) / 256, 256, 0, st>>>(
        ctx->d_pose, ctx->capN, ctx->N, ctx->d_kfpose, ctx->d_kft, ctx->capK, k, k + 1);
    CUDA_TRY(ctx, cudaGetLastError());
  }
  CUDA_TRY(ctx, cudaStreamSynchronize(st));
  ctx->kf.push_back(kh);
  ctx->D.push_back(path_length);
  ctx->K = k + 1;
  if (out_kf_id) *out_kf_id = k;
  return MCS_OK;
}

mcs_status mcs_set_particles(mcs_ctx* ctx, int32_t n, const float* pose12,
                             const float* kf_pose12, const double* cum_loglik) {
  CHECK_CTX(ctx);
  if (!pose12 || n < 1) FAIL(ctx, MCS_E_INVALID_ARG, "mcs_set_particles: null pose12 or n < 1");
  if (n > ctx->capN) FAIL(ctx, MCS_E_CAPACITY, "n (%d) > capacity_particles (%d)", n, ctx->capN);
  cudaStream_t st = ctx->stream;
  const int K = ctx->K;
  float *tp = nullptr, *tk = nullptr;
  double* tl = nullptr;
  int* bad = nullptr;
  CUDA_TRY(ctx, mem_alloc_async(ctx, (void**)&tp, sizeof(float) * 12 * n, st));
  CUDA_TRY(ctx, mem_alloc_async(ctx, (void**)&bad, sizeof(int), st));
  CUDA_TRY(ctx, cudaMemsetAsync(bad, 0, sizeof(int), st));
  CUDA_TRY(ctx, to_device(tp, pose12, sizeof(float) * 12 * n, st));
  validate_poses_kernel<<<(n + 255) / 256, 256, 0, st>>>(tp, n, bad);
  if (kf_pose12 && K > 0) {
    const long long np = (long long)n * K;
    CUDA_TRY(ctx, mem_alloc_async(ctx, (void**)&tk, sizeof(float) * 12 * np, st));
    CUDA_TRY(ctx, to_device(tk, kf_pose12, sizeof(float) * 12 * np, st));
    validate_poses_kernel<<<(int)((np + 255) / 256), 256, 0, st>>>(tk, np, bad);
  }
  if (cum_loglik) {
    CUDA_TRY(ctx, mem_alloc_async(ctx, (void**)&tl, sizeof(double) * n, st));
    CUDA_TRY(ctx, to_device(tl, cum_loglik, sizeof(double) * n, st));
  }
  int h_bad = 0;
  CUDA_TRY(ctx, cudaMemcpyAsync(&h_bad, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(ctx, cudaStreamSynchronize(st));
  bool lbad = false;
  if (cum_loglik && !h_bad) {
    std::vector<double> hl(n);
    CUDA_TRY(ctx, cudaMemcpy(hl.data(), tl, sizeof(double) * n, cudaMemcpyDeviceToHost));
    for (double v : hl) lbad |= !std::isfinite(v);
  }
  if (h_bad || lbad) {
    mem_free_async(ctx, tp, st);
    if (tk) mem_free_async(ctx, tk, st);
    if (tl) mem_free_async(ctx, tl, st);
    mem_free_async(ctx, bad, st);
    FAIL(ctx, MCS_E_INVALID_ARG, "non-finite or non-orthonormal pose / non-finite L (%d)", h_bad);
  }
  // commit
  aos_to_soa_kernel<<<(n + 255) / 256, 256, 0, st>>>(tp, n, ctx->capN, ctx->d_pose);
  if (K > 0) {
    if (tk) {
      CUDA_TRY(ctx, cudaMemcpy2DAsync(ctx->d_kfpose, sizeof(float) * 12 * ctx->capK, tk,
                                      sizeof(float) * 12 * K, sizeof(float) * 12 * K, n,
                                      cudaMemcpyDeviceToDevice, st));
      const long long tot = (long long)n * K;
      kft_from_kfpose_kernel<<<(int)((tot + 255) / 256), 256, 0, st>>>(ctx->d_kfpose, ctx->capK,
                                                                         n, K, ctx->d_kft);
    } else {
      const long long tot = (long long)n * K;
      fill_kf_from_current_kernel<<<(int)((tot + 255) / 256), 256, 0, st>>>(
          ctx->d_pose, ctx->capN, n, ctx->d_kfpose, ctx->d_kft, ctx->capK, 0, K);
    }
  }
  if (tl) {
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->d_L, tl, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  } else {
    CUDA_TRY(ctx, cudaMemsetAsync(ctx->d_L, 0, sizeof(double) * n, st));
  }
  fill_double_kernel<<<(n + 255) / 256, 256, 0, st>>>(ctx->d_e, n, 1.0);  // w = 1 / N_total
  CUDA_TRY(ctx, cudaGetLastError());
  mem_free_async(ctx, tp, st);
  if (tk) mem_free_async(ctx, tk, st);
  if (tl) mem_free_async(ctx, tl, st);
  mem_free_async(ctx, bad, st);
  CUDA_TRY(ctx, cudaStreamSynchronize(st));
  ctx->N = n;
  {  // sweep partials for the point splits this particle count will use (outside any capture)
    const int P = sweep_splits_for(ctx, n);
    if (P > ctx->part_splits) {
      double* np = nullptr;
      CUDA_TRY(ctx, mem_alloc(ctx, (void**)&np,
                              sizeof(double) * kSlotWords * ctx->nbcap * ctx->capN * P));
      mem_free(ctx, ctx->d_part);
      ctx->d_part = np;
      ctx->part_splits = P;
    }
  }
  // global index base of this shard (collective over ranks)
  ctx->n_per_rank.assign(ctx->world, 0);
  const long long mine = n;
  const mcs_status ds = dist_allgather_host(ctx, &mine, ctx->n_per_rank.data(), sizeof(long long));
  if (ds != MCS_OK) {
    ctx->sticky = ds;
    FAIL(ctx, ds, "allgather of the shard sizes failed");
  }
  ctx->gbase = 0;
  for (int g = 0; g < ctx->rank; ++g) ctx->gbase += ctx->n_per_rank[g];
  if (ctx->cfg.diversity_weight != 0.0) {  // R35: every rank's translations, padded
    long long mx = 0;
    for (long long v : ctx->n_per_rank) mx = v > mx ? v : mx;
    if ((int)mx > ctx->div_maxn) {
      mem_free(ctx, ctx->d_tall);
      ctx->d_tall = nullptr;
      ctx->div_maxn = 0;
      CUDA_TRY(ctx, mem_alloc(ctx, (void**)&ctx->d_tall,
                              sizeof(double) * 3 * (size_t)mx * ctx->world));
      if (!ctx->d_divn) CUDA_TRY(ctx, mem_alloc(ctx, (void**)&ctx->d_divn, sizeof(int) * ctx->world));
    }
    ctx->div_maxn = (int)mx;
    std::vector<int> nr(ctx->world);
    for (int g = 0; g < ctx->world; ++g) nr[g] = (int)ctx->n_per_rank[g];
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->d_divn, nr.data(), sizeof(int) * ctx->world,
                                  cudaMemcpyHostToDevice, st));
    CUDA_TRY(ctx, cudaStreamSynchronize(st));
  }
  double n_total = 0.0;  // uniform initial weights over the particles of every rank
  for (int g = 0; g < ctx->world; ++g) n_total += (double)ctx->n_per_rank[g];
  CUDA_TRY(ctx, cudaMemcpyAsync(&ctx->d_scal->S2, &n_total, sizeof(double),
                                cudaMemcpyHostToDevice, st));
  CUDA_TRY(ctx, cudaStreamSynchronize(st));
  return MCS_OK;
}

mcs_status mcs_get_particles(mcs_ctx* ctx, float* pose12, float* kf_pose12, double* cum_loglik,
                             double* weight) {
  CHECK_CTX(ctx);
  cudaStream_t st = ctx->stream;
  const int n = ctx->N, K = ctx->K;
  if (n == 0) return MCS_OK;
  if (pose12) {
    float* tp = nullptr;
    CUDA_TRY(ctx, mem_alloc_async(ctx, (void**)&tp, sizeof(float) * 12 * n, st));
    soa_to_aos_kernel<<<(n + 255) / 256, 256, 0, st>>>(ctx->d_pose, n, ctx->capN, tp);
    CUDA_TRY(ctx, cudaMemcpyAsync(pose12, tp, sizeof(float) * 12 * n, cudaMemcpyDefault, st));
    mem_free_async(ctx, tp, st);
  }
  if (kf_pose12 && K > 0)
    CUDA_TRY(ctx, cudaMemcpy2DAsync(kf_pose12, sizeof(float) * 12 * K, ctx->d_kfpose,
                                    sizeof(float) * 12 * ctx->capK, sizeof(float) * 12 * K, n,
                                    cudaMemcpyDefault, st));
  if (cum_loglik)
    CUDA_TRY(ctx, cudaMemcpyAsync(cum_loglik, ctx->d_L, sizeof(double) * n, cudaMemcpyDefault, st));
  if (weight) {
    double* tw = nullptr;
    CUDA_TRY(ctx, mem_alloc_async(ctx, (void**)&tw, sizeof(double) * n, st));
    launch_weights_out(ctx, tw);
    CUDA_TRY(ctx, cudaMemcpyAsync(weight, tw, sizeof(double) * n, cudaMemcpyDefault, st));
    mem_free_async(ctx, tw, st);
  }
  CUDA_TRY(ctx, cudaStreamSynchronize(st));
  return MCS_OK;
}

mcs_status mcs_get_pose(mcs_ctx* ctx, int32_t index, float* pose12) {
  CHECK_CTX(ctx);
  if (!pose12 || index < 0 || index >= ctx->N)
    FAIL(ctx, MCS_E_INVALID_ARG, "mcs_get_pose: index %d outside [0, %d)", index, ctx->N);
  // SoA column: 12 strided floats in one 2-D copy
  CUDA_TRY(ctx, cudaMemcpy2DAsync(pose12, sizeof(float), ctx->d_pose + index,
                                  sizeof(float) * ctx->capN, sizeof(float), 12, cudaMemcpyDefault,
                                  ctx->stream));
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return MCS_OK;
}

mcs_status mcs_get_global_pose(mcs_ctx* ctx, int64_t global_index, float* pose12) {
  CHECK_CTX(ctx);
  long long n_total = 0;
  for (long long v : ctx->n_per_rank) n_total += v;
  if (!pose12 || global_index < 0 || global_index >= n_total)
    FAIL(ctx, MCS_E_INVALID_ARG, "mcs_get_global_pose: index %lld outside [0, %lld)",
         (long long)global_index, n_total);
  cudaStream_t st = ctx->stream;
  double* d = reinterpret_cast<double*>(ctx->d_xg) + 8 * (ctx->world + 1);  // 12 doubles
  const long long li = global_index - ctx->gbase;
  const int owner = li >= 0 && li < ctx->N;
  pose_column_kernel<<<1, 12, 0, st>>>(ctx->d_pose, ctx->capN, owner ? (int)li : -1, d);
  const mcs_status s = dist_allreduce_f64(ctx, d, 12, 0);  // exactly one rank is nonzero
  if (s != MCS_OK) FAIL(ctx, s, "mcs_get_global_pose: all-reduce failed");
  double h[12];
  CUDA_TRY(ctx, cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(ctx, cudaStreamSynchronize(st));
  float f[12];
  for (int k = 0; k < 12; ++k) f[k] = (float)h[k];  // fp32 values: exact round trip
  CUDA_TRY(ctx, cudaMemcpy(pose12, f, sizeof(f), cudaMemcpyDefault));
  return MCS_OK;
}

// validate a scan already in device memory (d_scan_raw layout: mean3 then cov6)
static mcs_status validate_scan(mcs_ctx* ctx, int n_pts) {
  cudaStream_t st = ctx->stream;
  CUDA_TRY(ctx, cudaMemsetAsync(ctx->d_bad, 0, sizeof(int), st));
  validate_gauss_kernel<<<(n_pts + 255) / 256, 256, 0, st>>>(
      ctx->d_scan_raw, ctx->d_scan_raw + 3 * (size_t)ctx->capS, n_pts, ctx->d_bad);
  CUDA_TRY(ctx, cudaMemcpyAsync(&ctx->h_scal->status, ctx->d_bad, sizeof(int),
                                cudaMemcpyDeviceToHost, st));
  CUDA_TRY(ctx, cudaStreamSynchronize(st));
  const int h_bad = ctx->h_scal->status;
  if (h_bad) FAIL(ctx, MCS_E_INVALID_ARG, "%d scan points non-finite or covariance not SPD", h_bad);
  return MCS_OK;
}

static mcs_status check_update_args(mcs_ctx* ctx, const void* m, const void* c, int n_pts,
                                    double D_now) {
  if (ctx->K < 1) FAIL(ctx, MCS_E_STATE, "no keyframe registered");
  if (ctx->N < 1) FAIL(ctx, MCS_E_STATE, "no particles set");
  if (!m || !c) FAIL(ctx, MCS_E_INVALID_ARG, "null scan");
  if (n_pts < 1) FAIL(ctx, MCS_E_INVALID_ARG, "n_pts < 1");
  if (n_pts > ctx->capS) FAIL(ctx, MCS_E_CAPACITY, "n_pts > capacity_scan_points");
  if (!std::isfinite(D_now)) FAIL(ctx, MCS_E_INVALID_ARG, "D_now not finite");
  if (!ctx->D.empty() && D_now < ctx->D.back())  // cumulative path length never decreases (R14)
    FAIL(ctx, MCS_E_INVALID_ARG, "D_now (%g) < the newest keyframe's path length (%g)", D_now,
         ctx->D.back());
  return MCS_OK;
}

// phase events; inside a stream capture they become event-record nodes of the graph (the
// External flag), so each replay records them and the phases of a replayed update are timed
static void record(mcs_ctx* ctx, int k) {
  if (!ctx->profiling) return;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(ctx->stream, &cap);
  if (cap == cudaStreamCaptureStatusActive)
    cudaEventRecordWithFlags(ctx->ev[k], ctx->stream, cudaEventRecordExternal);
  else
    cudaEventRecord(ctx->ev[k], ctx->stream);
}

// the hot path a1..a7, stream-ordered; scan already prepared in d_scan
static mcs_status run_update_body(mcs_ctx* ctx, int n_pts, uint32_t U) {
  const int iters = ctx->cfg.gn_iterations > 0 ? ctx->cfg.gn_iterations : 1;
  const bool post = ctx->cfg.weight_after_update != 0;
  const bool div = ctx->cfg.diversity_weight != 0.0;
  record(ctx, 0);
  if (div) MCS_TRY(launch_diversity_snapshot(ctx));  // R35: translations at the start
  // the default path (one GN step, pre-update weighting, no R35) runs a4 inside a5-a7, on a
  // side stream beside the ladder and for the survivors only: nothing before the draws reads
  // keyframe poses, and a dead particle's are replaced by its donor's
  const bool fork = iters == 1 && !post && !div;
  for (int it = 0; it < iters; ++it) {  // R12: each iteration is a full a1-a4 pass
    MCS_TRY(launch_select(ctx, kSelectUpdate));                         // a1
    if (it == 0) record(ctx, 1);
    launch_sweep(ctx, n_pts);                                           // a2
    if (it == 0) record(ctx, 2);
    launch_combine(ctx, n_pts, (it == 0 && !post) ? kCombineUpdateWeight : kCombineUpdate,
                   nullptr, nullptr, nullptr, nullptr, nullptr, nullptr);  // a3 (+ L += l)
    if (!fork) launch_propagate(ctx);                                   // a4
  }
  if (div) MCS_TRY(launch_diversity_apply(ctx));  // R35: t_i += eta d_i after the GN step(s)
  if (post) {  // R13 variant: weight with l re-evaluated at the updated poses
    MCS_TRY(launch_select(ctx, kSelectWeight));
    launch_sweep(ctx, n_pts);
    launch_combine(ctx, n_pts, kCombineWeight, nullptr, nullptr, nullptr, nullptr, nullptr,
                   nullptr);
  }
  record(ctx, 3);
  const mcs_status s = launch_weights_resample(ctx, U, fork);           // (a4,) a5-a7
  record(ctx, 4);
  return s;
}

// The update body (a1-a7) of a single-rank context is captured once into a CUDA graph and
// replayed while its shape holds (scan size, particle and keyframe counts); the per-update
// scalars D_now and U reach it through d_scal (launch_set_params, outside the graph).
// Multi-rank updates (host-side exchange steps), profiled updates (phase events) and calls
// made inside the caller's own stream capture run the body directly.
static mcs_status run_update(mcs_ctx* ctx, int n_pts, double D_now, uint32_t U) {
  launch_set_params(ctx, D_now, U);
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(ctx->stream, &cap);
  // multi-rank: the peer views are exchanged (collectively, with host steps) before any capture
  if (dist_active(ctx) && ctx->p2p == 0) {
    const mcs_status ps = dist_peer_setup(ctx);
    if (ps != MCS_OK) return ps;
  }
  // (with profiling on, the phase events are recorded inside the graph: timed replays)
  const bool graph = ctx->cfg.graph_replay && !ctx->graph_off &&
                     weights_device_resident(ctx) && cap == cudaStreamCaptureStatusNone;
  if (!graph) return run_update_body(ctx, n_pts, U);
  const long long key[5] = {n_pts, ctx->N, ctx->K, ctx->div_maxn,  // R35's gather shape
                            ctx->profiling ? 1 : 0};                // phase events inside
  if (!ctx->gexec || memcmp(key, ctx->gkey, sizeof(key)) != 0) {
    if (ctx->gexec) cudaGraphExecDestroy(ctx->gexec);
    ctx->gexec = nullptr;
    cudaGraph_t g = nullptr;
    if (cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
      cudaGetLastError();
      ctx->graph_off = true;
      return run_update_body(ctx, n_pts, U);
    }
    const mcs_status s = run_update_body(ctx, n_pts, U);
    const cudaError_t ec = cudaStreamEndCapture(ctx->stream, &g);
    cudaError_t ei = cudaErrorUnknown;
    if (s == MCS_OK && ec == cudaSuccess && g) ei = cudaGraphInstantiate(&ctx->gexec, g, 0);
    if (g) cudaGraphDestroy(g);
    if (ei != cudaSuccess) {  // not capturable here: eager from now on
      ctx->gexec = nullptr;
      cudaGetLastError();
      ctx->graph_off = true;
      return run_update_body(ctx, n_pts, U);
    }
    memcpy(ctx->gkey, key, sizeof(key));
  }
  return cudaGraphLaunch(ctx->gexec, ctx->stream) == cudaSuccess ? MCS_OK : MCS_E_CUDA;
}

mcs_status mcs_update(mcs_ctx* ctx, const float* scan_mean3, const float* scan_cov6,
                      int32_t n_pts, double D_now, uint32_t resample_u,
                      const mcs_update_out* out) {
  CHECK_CTX(ctx);
  mcs_status s = check_update_args(ctx, scan_mean3, scan_cov6, n_pts, D_now);
  if (s != MCS_OK) return s;
  cudaStream_t st = ctx->stream;
  float* raw_m = ctx->d_scan_raw;
  float* raw_c = ctx->d_scan_raw + 3 * (size_t)ctx->capS;
  CUDA_TRY(ctx, to_device(raw_m, scan_mean3, sizeof(float) * 3 * n_pts, st));
  CUDA_TRY(ctx, to_device(raw_c, scan_cov6, sizeof(float) * 6 * n_pts, st));
  s = validate_scan(ctx, n_pts);
  if (s != MCS_OK) return s;
  CUDA_TRY(ctx, launch_prepare_scan(raw_m, raw_c, n_pts, ctx->d_scan, ctx->d_scan_plane,
                                    ctx->d_scan_np, st));
  ctx->scan_prepared = true;
  s = run_update(ctx, n_pts, D_now, resample_u);
  if (s != MCS_OK) {
    ctx->sticky = s;
    FAIL(ctx, s, "update failed in the weights/exchange phase (%d)", (int)s);
  }
  CUDA_TRY(ctx, cudaGetLastError());
  const int N = ctx->N;
  if (out) {
    // gather per-particle rows into a device staging area, then one copy per output
    OutPtrs o{};
    const StageLayout lay(N);
    char* stage = ctx->d_stage;
    if (out->loglik) o.loglik = (double*)(stage + lay.l);
    if (out->grad6) o.grad6 = (float*)(stage + lay.g);
    if (out->hess21) o.hess21 = (float*)(stage + lay.h);
    if (out->psi6) o.psi6 = (float*)(stage + lay.p);
    if (out->weight) o.weight = (double*)(stage + lay.w);
    if (out->donor) o.donor = (int32_t*)(stage + lay.d);
    if (out->flags) o.flags = (uint8_t*)(stage + lay.f);
    gather_outputs_kernel<<<(N + 255) / 256, 256, 0, st>>>(
        o, N, ctx->capN, ctx->d_l, ctx->d_grad, ctx->d_hess, ctx->d_psi, ctx->d_e, ctx->d_donor_g,
        ctx->d_flags, ctx->d_scal);
    if (out->loglik) CUDA_TRY(ctx, cudaMemcpyAsync(out->loglik, o.loglik, 8 * N, cudaMemcpyDefault, st));
    if (out->grad6) CUDA_TRY(ctx, cudaMemcpyAsync(out->grad6, o.grad6, 24 * N, cudaMemcpyDefault, st));
    if (out->hess21) CUDA_TRY(ctx, cudaMemcpyAsync(out->hess21, o.hess21, 84 * N, cudaMemcpyDefault, st));
    if (out->psi6) CUDA_TRY(ctx, cudaMemcpyAsync(out->psi6, o.psi6, 24 * N, cudaMemcpyDefault, st));
    if (out->weight) CUDA_TRY(ctx, cudaMemcpyAsync(out->weight, o.weight, 8 * N, cudaMemcpyDefault, st));
    if (out->donor) CUDA_TRY(ctx, cudaMemcpyAsync(out->donor, o.donor, 4 * N, cudaMemcpyDefault, st));
    if (out->flags) CUDA_TRY(ctx, cudaMemcpyAsync(out->flags, o.flags, N, cudaMemcpyDefault, st));
  }
  CUDA_TRY(ctx, cudaMemcpyAsync(ctx->h_scal, ctx->d_scal, sizeof(Scalars), cudaMemcpyDeviceToHost,
                                st));
  CUDA_TRY(ctx, cudaStreamSynchronize(st));
  if (out && out->representative) *out->representative = (int32_t)ctx->h_scal->rep;
  if (out && out->n_dead) *out->n_dead = ctx->h_scal->D_tot;
  if (ctx->h_scal->status == MCS_E_DEGENERATE)
    FAIL(ctx, MCS_E_DEGENERATE, "every particle dead (S:381); respawn skipped");
  return MCS_OK;
}

mcs_status mcs_update_async(mcs_ctx* ctx, const float* d_scan_mean3, const float* d_scan_cov6,
                            int32_t n_pts, double D_now, uint32_t resample_u,
                            const mcs_update_out* d_out, void* cuda_stream) {
  CHECK_CTX(ctx);
  mcs_status s = check_update_args(ctx, d_scan_mean3, d_scan_cov6, n_pts, D_now);
  if (s != MCS_OK) return s;
  cudaStream_t saved = ctx->stream;
  if (cuda_stream) ctx->stream = (cudaStream_t)cuda_stream;
  const cudaError_t pe = launch_prepare_scan(d_scan_mean3, d_scan_cov6, n_pts, ctx->d_scan,
                                             ctx->d_scan_plane, ctx->d_scan_np, ctx->stream);
  if (pe != cudaSuccess) ctx->stream = saved;  // (CUDA_TRY returns)
  CUDA_TRY(ctx, pe);
  ctx->scan_prepared = true;
  s = run_update(ctx, n_pts, D_now, resample_u);
  if (s != MCS_OK) {
    ctx->stream = saved;
    ctx->sticky = s;
    FAIL(ctx, s, "update failed in the weights/exchange phase (%d)", (int)s);
  }
  if (d_out) {
    OutPtrs o{d_out->loglik, d_out->grad6,  d_out->hess21,         d_out->psi6,  d_out->weight,
              d_out->donor,  d_out->flags,  d_out->representative, d_out->n_dead};
    gather_outputs_kernel<<<(ctx->N + 255) / 256, 256, 0, ctx->stream>>>(
        o, ctx->N, ctx->capN, ctx->d_l, ctx->d_grad, ctx->d_hess, ctx->d_psi, ctx->d_e,
        ctx->d_donor_g, ctx->d_flags, ctx->d_scal);
  }
  cudaError_t e = cudaGetLastError();
  ctx->stream = saved;
  CUDA_TRY(ctx, e);
  return MCS_OK;
}

mcs_status mcs_eval(mcs_ctx* ctx, const float* scan_mean3, const float* scan_cov6, int32_t n_pts,
                    double* slot_loglik, float* slot_H21, float* slot_b6, int32_t* slot_n,
                    int32_t* slot_kf, uint8_t* loop) {
  CHECK_CTX(ctx);
  mcs_status s = check_update_args(ctx, scan_mean3, scan_cov6, n_pts,
                                   ctx->D.empty() ? 0.0 : ctx->D.back());  // no D_now in eval
  if (s != MCS_OK) return s;
  cudaStream_t st = ctx->stream;
  float* raw_m = ctx->d_scan_raw;
  float* raw_c = ctx->d_scan_raw + 3 * (size_t)ctx->capS;
  CUDA_TRY(ctx, to_device(raw_m, scan_mean3, sizeof(float) * 3 * n_pts, st));
  CUDA_TRY(ctx, to_device(raw_c, scan_cov6, sizeof(float) * 6 * n_pts, st));
  s = validate_scan(ctx, n_pts);
  if (s != MCS_OK) return s;
  CUDA_TRY(ctx, launch_prepare_scan(raw_m, raw_c, n_pts, ctx->d_scan, ctx->d_scan_plane,
                                    ctx->d_scan_np, st));
  ctx->scan_prepared = true;
  const size_t NS = (size_t)ctx->N * ctx->cfg.neighbor_count;
  double* dl = nullptr;
  float *dH = nullptr, *db = nullptr;
  int32_t *dn = nullptr, *dk = nullptr;
  uint8_t* dloop = nullptr;
  CUDA_TRY(ctx, mem_alloc_async(ctx, (void**)&dl, 8 * NS, st));
  CUDA_TRY(ctx, mem_alloc_async(ctx, (void**)&dH, 84 * NS, st));
  CUDA_TRY(ctx, mem_alloc_async(ctx, (void**)&db, 24 * NS, st));
  CUDA_TRY(ctx, mem_alloc_async(ctx, (void**)&dn, 4 * NS, st));
  CUDA_TRY(ctx, mem_alloc_async(ctx, (void**)&dk, 4 * NS, st));
  CUDA_TRY(ctx, mem_alloc_async(ctx, (void**)&dloop, ctx->N, st));
  if (launch_select(ctx, kSelectEval) != MCS_OK) CUDA_TRY(ctx, cudaErrorLaunchFailure);
  launch_sweep(ctx, n_pts);
  launch_combine(ctx, n_pts, kCombineEval, dl, dH, db, dn, dk, dloop);
  CUDA_TRY(ctx, cudaGetLastError());
  if (slot_loglik) CUDA_TRY(ctx, cudaMemcpyAsync(slot_loglik, dl, 8 * NS, cudaMemcpyDefault, st));
  if (slot_H21) CUDA_TRY(ctx, cudaMemcpyAsync(slot_H21, dH, 84 * NS, cudaMemcpyDefault, st));
  if (slot_b6) CUDA_TRY(ctx, cudaMemcpyAsync(slot_b6, db, 24 * NS, cudaMemcpyDefault, st));
  if (slot_n) CUDA_TRY(ctx, cudaMemcpyAsync(slot_n, dn, 4 * NS, cudaMemcpyDefault, st));
  if (slot_kf) CUDA_TRY(ctx, cudaMemcpyAsync(slot_kf, dk, 4 * NS, cudaMemcpyDefault, st));
  if (loop) CUDA_TRY(ctx, cudaMemcpyAsync(loop, dloop, ctx->N, cudaMemcpyDefault, st));
  mem_free_async(ctx, dl, st); mem_free_async(ctx, dH, st); mem_free_async(ctx, db, st);
  mem_free_async(ctx, dn, st); mem_free_async(ctx, dk, st); mem_free_async(ctx, dloop, st);
  CUDA_TRY(ctx, cudaStreamSynchronize(st));
  return MCS_OK;
}

mcs_status mcs_resample(mcs_ctx* ctx, const double* e, const uint8_t* dead, int32_t n, uint32_t u,
                        int32_t* donor_out) {
  CHECK_CTX(ctx);
  if (!e || !dead || !donor_out || n < 1) FAIL(ctx, MCS_E_INVALID_ARG, "mcs_resample: bad args");
  if (n > ctx->capN) FAIL(ctx, MCS_E_CAPACITY, "n > capacity_particles");
  cudaStream_t st = ctx->stream;
  uint8_t* dd = nullptr;
  double* de = nullptr;
  CUDA_TRY(ctx, mem_alloc_async(ctx, (void**)&dd, n, st));
  CUDA_TRY(ctx, mem_alloc_async(ctx, (void**)&de, 8 * (size_t)n, st));
  CUDA_TRY(ctx, to_device(dd, dead, n, st));
  CUDA_TRY(ctx, to_device(de, e, 8 * (size_t)n, st));
  // domain of the exact ladder (R18): 0 <= e_i <= 1 (e = exp(L - max L)), so every rung
  // floor(e 2^32) and the N-term prefix sums are exact uint64
  CUDA_TRY(ctx, cudaMemsetAsync(ctx->d_bad, 0, sizeof(int), st));
  validate_unit_kernel<<<(n + 255) / 256, 256, 0, st>>>(de, n, ctx->d_bad);
  CUDA_TRY(ctx, cudaMemcpyAsync(&ctx->h_scal->status, ctx->d_bad, sizeof(int),
                                cudaMemcpyDeviceToHost, st));
  CUDA_TRY(ctx, cudaStreamSynchronize(st));
  if (ctx->h_scal->status) {
    const int nb = ctx->h_scal->status;
    mem_free_async(ctx, dd, st);
    mem_free_async(ctx, de, st);
    FAIL(ctx, MCS_E_INVALID_ARG, "mcs_resample: %d values of e outside [0, 1] or not finite", nb);
  }
  int32_t* ddon = nullptr;
  CUDA_TRY(ctx, mem_alloc_async(ctx, (void**)&ddon, 4 * (size_t)n, st));
  if (launch_resample_only(ctx, de, dd, n, u, ddon) != MCS_OK) CUDA_TRY(ctx, cudaGetLastError());
  CUDA_TRY(ctx, cudaGetLastError());
  CUDA_TRY(ctx, cudaMemcpyAsync(donor_out, ddon, 4 * (size_t)n, cudaMemcpyDefault, st));
  CUDA_TRY(ctx, cudaMemcpyAsync(ctx->h_scal, ctx->d_scal, sizeof(Scalars), cudaMemcpyDeviceToHost,
                                st));
  mem_free_async(ctx, dd, st); mem_free_async(ctx, de, st); mem_free_async(ctx, ddon, st);
  CUDA_TRY(ctx, cudaStreamSynchronize(st));
  if (ctx->h_scal->status == MCS_E_DEGENERATE)
    FAIL(ctx, MCS_E_DEGENERATE, "every particle dead (S:381)");
  return MCS_OK;
}

mcs_status mcs_predict(mcs_ctx* ctx, const float* dT12, const double* cov36, uint64_t seed,
                       uint64_t frame, double vertical_sigma) {
  CHECK_CTX(ctx);
  if (!dT12 || !cov36) FAIL(ctx, MCS_E_INVALID_ARG, "mcs_predict: null dT or covariance");
  if (!std::isfinite(vertical_sigma) || vertical_sigma < 0)
    FAIL(ctx, MCS_E_INVALID_ARG, "vertical_sigma must be finite and >= 0");
  float hdT[12];
  double hbuf[48];
  CUDA_TRY(ctx, cudaMemcpy(hdT, dT12, sizeof(hdT), cudaMemcpyDefault));
  CUDA_TRY(ctx, cudaMemcpy(hbuf + 12, cov36, sizeof(double) * 36, cudaMemcpyDefault));
  for (int k = 0; k < 12; ++k) {
    if (!std::isfinite(hdT[k])) FAIL(ctx, MCS_E_INVALID_ARG, "dT not finite");
    hbuf[k] = (double)hdT[k];
  }
  for (int a = 0; a < 6; ++a)
    for (int b = 0; b < 6; ++b)
      if (!std::isfinite(hbuf[12 + 6 * a + b]) || hbuf[12 + 6 * a + b] != hbuf[12 + 6 * b + a])
        FAIL(ctx, MCS_E_INVALID_ARG, "covariance not finite/symmetric");
  cudaStream_t st = ctx->stream;
  double* d = nullptr;
  CUDA_TRY(ctx, mem_alloc_async(ctx, (void**)&d, sizeof(double) * 84, st));
  CUDA_TRY(ctx, cudaMemcpyAsync(d, hbuf, sizeof(double) * 48, cudaMemcpyHostToDevice, st));
  CUDA_TRY(ctx, cudaMemsetAsync(ctx->d_bad, 0, sizeof(int), st));
  const mcs_status s = launch_predict(ctx, d, ctx->d_bad, seed, frame, vertical_sigma);
  mem_free_async(ctx, d, st);
  CUDA_TRY(ctx, cudaStreamSynchronize(st));
  if (s == MCS_E_INVALID_ARG) FAIL(ctx, s, "covariance neither SPD nor zero");
  if (s != MCS_OK) CUDA_TRY(ctx, cudaGetLastError());
  return s;
}

mcs_status mcs_overlap(mcs_ctx* ctx, const float* scan_mean3, int32_t n_pts, const float* rel12,
                       int32_t kf, double* out_rate) {
  CHECK_CTX(ctx);
  if (!scan_mean3 || !rel12 || !out_rate || n_pts < 1)
    FAIL(ctx, MCS_E_INVALID_ARG, "mcs_overlap: bad arguments");
  if (kf < 0 || kf >= ctx->K) FAIL(ctx, MCS_E_INVALID_ARG, "mcs_overlap: no keyframe %d", kf);
  cudaStream_t st = ctx->stream;
  char* d = nullptr;
  const size_t bm = (sizeof(float) * 3 * (size_t)n_pts + 255) & ~(size_t)255;  // keep alignment
  CUDA_TRY(ctx, mem_alloc_async(ctx, (void**)&d, bm + 64 + 8, st));
  CUDA_TRY(ctx, to_device(d, scan_mean3, sizeof(float) * 3 * (size_t)n_pts, st));
  CUDA_TRY(ctx, to_device(d + bm, rel12, 48, st));
  unsigned long long cnt = 0;
  const mcs_status s = launch_overlap(ctx, (const float*)d, n_pts, (const float*)(d + bm), kf,
                                      (unsigned long long*)(d + bm + 64), &cnt);
  mem_free_async(ctx, d, st);
  if (s != MCS_OK) CUDA_TRY(ctx, cudaGetLastError());
  *out_rate = (double)cnt / (double)n_pts;
  return s;
}

mcs_status mcs_snapshot(mcs_ctx* ctx) {
  CHECK_CTX(ctx);
  const size_t bp = sizeof(float) * 12 * ctx->capN, bk = sizeof(float) * 12 * ctx->capN * ctx->capK,
               bt = sizeof(float4) * ctx->capN * ctx->capK, bl = sizeof(double) * ctx->capN;
  if (!ctx->d_snapshot) {
    CUDA_TRY(ctx, mem_alloc(ctx, &ctx->d_snapshot, bp + bk + bt + bl));
    ctx->snapshot_bytes = bp + bk + bt + bl;
  }
  char* s = (char*)ctx->d_snapshot;
  cudaStream_t st = ctx->stream;
  CUDA_TRY(ctx, cudaMemcpyAsync(s, ctx->d_pose, bp, cudaMemcpyDeviceToDevice, st));
  CUDA_TRY(ctx, cudaMemcpyAsync(s + bp, ctx->d_kfpose, bk, cudaMemcpyDeviceToDevice, st));
  CUDA_TRY(ctx, cudaMemcpyAsync(s + bp + bk, ctx->d_kft, bt, cudaMemcpyDeviceToDevice, st));
  CUDA_TRY(ctx, cudaMemcpyAsync(s + bp + bk + bt, ctx->d_L, bl, cudaMemcpyDeviceToDevice, st));
  return MCS_OK;
}

mcs_status mcs_restore(mcs_ctx* ctx) {
  CHECK_CTX(ctx);
  if (!ctx->d_snapshot) FAIL(ctx, MCS_E_STATE, "no snapshot");
  const size_t bp = sizeof(float) * 12 * ctx->capN, bk = sizeof(float) * 12 * ctx->capN * ctx->capK,
               bt = sizeof(float4) * ctx->capN * ctx->capK, bl = sizeof(double) * ctx->capN;
  char* s = (char*)ctx->d_snapshot;
  cudaStream_t st = ctx->stream;
  CUDA_TRY(ctx, cudaMemcpyAsync(ctx->d_pose, s, bp, cudaMemcpyDeviceToDevice, st));
  CUDA_TRY(ctx, cudaMemcpyAsync(ctx->d_kfpose, s + bp, bk, cudaMemcpyDeviceToDevice, st));
  CUDA_TRY(ctx, cudaMemcpyAsync(ctx->d_kft, s + bp + bk, bt, cudaMemcpyDeviceToDevice, st));
  CUDA_TRY(ctx, cudaMemcpyAsync(ctx->d_L, s + bp + bk + bt, bl, cudaMemcpyDeviceToDevice, st));
  return MCS_OK;
}

mcs_status mcs_set_profiling(mcs_ctx* ctx, int32_t enable) {
  CHECK_CTX(ctx);
  ctx->profiling = enable != 0;
  return MCS_OK;
}

int32_t mcs_peer_migration_state(const mcs_ctx* ctx) { return ctx ? ctx->p2p : 0; }
int32_t mcs_graph_state(const mcs_ctx* ctx) { return ctx && ctx->gexec ? 1 : 0; }

mcs_status mcs_scan_nonplanar(mcs_ctx* ctx, int32_t* n_out) {
  CHECK_CTX(ctx);
  if (!n_out) FAIL(ctx, MCS_E_INVALID_ARG, "n_out is NULL");
  if (!ctx->scan_prepared) FAIL(ctx, MCS_E_STATE, "no scan prepared yet");
  int v = 0;
  CUDA_TRY(ctx, cudaMemcpyAsync(&v, ctx->d_scan_np, sizeof(int), cudaMemcpyDeviceToHost,
                                ctx->stream));
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  *n_out = v;
  return MCS_OK;
}

mcs_status mcs_get_phase_ms(const mcs_ctx* ctx, float* ms5) {
  if (!ctx || !ms5) return MCS_E_INVALID_ARG;
  if (!ctx->profiling) {
    for (int k = 0; k < 5; ++k) ms5[k] = 0.f;
    return MCS_OK;
  }
  // events of the last update (sync or async) on the context stream
  if (cudaEventSynchronize(ctx->ev[4]) != cudaSuccess) return MCS_E_CUDA;
  for (int k = 0; k < 4; ++k) cudaEventElapsedTime(&ms5[k], ctx->ev[k], ctx->ev[k + 1]);
  cudaEventElapsedTime(&ms5[4], ctx->ev[0], ctx->ev[4]);
  return MCS_OK;
}

}  // extern "C"
