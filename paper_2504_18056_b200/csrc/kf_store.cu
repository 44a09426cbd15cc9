// kf_store.cu — a0: keyframe store + per-keyframe spatial hash, built once per keyframe
// (P:88-91 shared keyframe clouds, Fig.2; P:112 voxel-based correspondence search).
//
// For keyframe k's Gaussians (mu', Sigma') in its own sensor frame: cell = floorf(mu' * (1/r))
// per axis (pinned fp32, R27), one aggregate per occupied cell — mean of means and mean of
// covariances accumulated in fp64 in input order (stable radix sort), stored
// fp32 — inserted into an open-addressing table keyed by bbox-local 32-bit cell coordinates
// (power-of-two capacity, load <= 1/4 and down to 1/64 when the table fits 64 MiB,
// multiplicative hash, linear probing, 64-byte slots;
// see mcs_internal.cuh).  One table serves every particle because it lives in the keyframe
// frame.
#include <cub/cub.cuh>

#include "mcs_internal.cuh"

// Table capacity: the smallest power of two >= 4 x the occupied cells (load <= 1/4), then
// doubled up to MCS_HASH_SLOTS_PER_CELL x the cells while the table stays within the
// context's budget (mcs_config.kf_table_mib, 64 MiB by default).  A sparse table costs HBM
// (64 B per slot; C2: 32 MiB per keyframe) and buys first probes that almost never meet
// another key: at load 1/4, about a quarter of the probes for empty cells (36 % of the
// sweep's probes at C2) and a sixth of those for occupied cells continue down a dependent
// linear-probing chain; at 1/64 the C2 sweep runs 7.5 % faster and NN27 12 %.
#ifndef MCS_HASH_SLOTS_PER_CELL
#define MCS_HASH_SLOTS_PER_CELL 64
#endif

namespace mcs {

__global__ void cell_keys_kernel(const float* __restrict__ mean3, int n, float inv_r,
                                 unsigned long long* __restrict__ keys, int* __restrict__ idx,
                                 int* __restrict__ bbox, int* __restrict__ bad) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int c[3];
  bool ok = true;
  for (int a = 0; a < 3; ++a) {
    float f = floorf(__fmul_rn(mean3[3 * i + a], inv_r));
    ok = ok && (f >= (float)kCellMin && f <= (float)kCellMax);
    c[a] = ok ? (int)f : 0;
  }
  if (!ok) {
    atomicAdd(bad, 1);
  } else {
    for (int a = 0; a < 3; ++a) {
      atomicMin(&bbox[a], c[a]);
      atomicMax(&bbox[3 + a], c[a]);
    }
  }
  keys[i] = pack_cell(c[0], c[1], c[2]);
  idx[i] = i;
}

__global__ void heads_kernel(const unsigned long long* __restrict__ keys, int n,
                             int* __restrict__ head) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  head[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

__global__ void aggregate_insert_kernel(const unsigned long long* __restrict__ skeys,
                                        const int* __restrict__ sidx, const int* __restrict__ head,
                                        int n, const float* __restrict__ mean3,
                                        const float* __restrict__ cov6, float inv_r, KfMeta m,
                                        float4* __restrict__ slots) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || !head[i]) return;
  const unsigned long long key = skeys[i];
  double mu[3] = {0, 0, 0}, s[6] = {0, 0, 0, 0, 0, 0};
  int cnt = 0;
  for (int j = i; j < n && skeys[j] == key; ++j) {  // members in input order (stable sort)
    int p = sidx[j];
    for (int a = 0; a < 3; ++a) mu[a] += (double)mean3[3 * p + a];
    for (int a = 0; a < 6; ++a) s[a] += (double)cov6[6 * p + a];
    ++cnt;
  }
  for (int a = 0; a < 3; ++a) mu[a] /= (double)cnt;
  for (int a = 0; a < 6; ++a) s[a] /= (double)cnt;
  // the cell of this group (recomputed from its first member, identical by construction)
  const int p0 = sidx[i];
  int c[3];
  for (int a = 0; a < 3; ++a) c[a] = (int)floorf(__fmul_rn(mean3[3 * p0 + a], inv_r));
  const unsigned int lk =
      local_key((unsigned)(c[0] - m.ox), (unsigned)(c[1] - m.oy), (unsigned)(c[2] - m.oz));
  unsigned int h = slot_hash(lk, m.shift);
  unsigned int* kw;
  while (true) {
    kw = reinterpret_cast<unsigned int*>(&slots[4 * h].x);
    unsigned int prev = atomicCAS(kw, kEmptyKey32, lk);
    if (prev == kEmptyKey32) break;
    h = (h + 1) & m.mask;
    MCS_DCHECK(h != (slot_hash(lk, m.shift) & m.mask));  // table never full (load <= 1/4)
  }
  // layout (mcs_internal.cuh): the (y, z) pairs sit in aligned register pairs for the sweep's
  // packed FFMA2 math; s[] = (xx, xy, xz, yy, yz, zz)
  slots[4 * h + 0] = make_float4(__uint_as_float(lk), (float)mu[0], (float)mu[1], (float)mu[2]);
  slots[4 * h + 1] = make_float4((float)s[3], (float)s[5], (float)s[1], (float)s[2]);
  slots[4 * h + 2] = make_float4((float)s[0], (float)s[4], __int_as_float(cnt), 0.f);
}

__global__ void init_slots_kernel(float4* __restrict__ slots, int cap) {
  int h = blockIdx.x * blockDim.x + threadIdx.x;
  if (h >= cap) return;
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  slots[4 * h + 0] = make_float4(__uint_as_float(kEmptyKey32), 0.f, 0.f, 0.f);
  slots[4 * h + 1] = z;
  slots[4 * h + 2] = z;
  slots[4 * h + 3] = z;
}

cudaError_t kf_build(mcs_ctx* c, const float* d_mean3, const float* d_cov6, int n, KfHost& out,
                     int* bad_cell, int* bad_extent) {
  cudaStream_t st = c->stream;
  float inv_r = 1.0f / c->cfg.voxel_resolution;
  unsigned long long *keys = nullptr, *skeys = nullptr;
  int *idx = nullptr, *sidx = nullptr, *head = nullptr, *cid = nullptr, *bad = nullptr;
  int* bbox = nullptr;
  void* temp = nullptr;
  size_t tb1 = 0, tb2 = 0;
  int h_bbox[6];
  const int bbox_init[6] = {0x7fffffff, 0x7fffffff, 0x7fffffff, (int)0x80000000, (int)0x80000000,
                            (int)0x80000000};
  cudaError_t e = cudaSuccess;
  *bad_cell = 0;
  *bad_extent = 0;
#define CK(x)                           \
  do {                                  \
    e = (x);                            \
    if (e != cudaSuccess) goto cleanup; \
  } while (0)
  CK(mem_alloc_async(c, (void**)&keys, sizeof(unsigned long long) * n, st));
  CK(mem_alloc_async(c, (void**)&skeys, sizeof(unsigned long long) * n, st));
  CK(mem_alloc_async(c, (void**)&idx, sizeof(int) * n, st));
  CK(mem_alloc_async(c, (void**)&sidx, sizeof(int) * n, st));
  CK(mem_alloc_async(c, (void**)&head, sizeof(int) * n, st));
  CK(mem_alloc_async(c, (void**)&cid, sizeof(int) * n, st));
  CK(mem_alloc_async(c, (void**)&bad, sizeof(int), st));
  CK(mem_alloc_async(c, (void**)&bbox, sizeof(int) * 6, st));
  CK(cudaMemsetAsync(bad, 0, sizeof(int), st));
  CK(cudaMemcpyAsync(bbox, bbox_init, sizeof(bbox_init), cudaMemcpyHostToDevice, st));
  {
    int g = (n + 255) / 256;
    cell_keys_kernel<<<g, 256, 0, st>>>(d_mean3, n, inv_r, keys, idx, bbox, bad);
    CK(cudaGetLastError());
    cub::DeviceRadixSort::SortPairs(nullptr, tb1, keys, skeys, idx, sidx, n, 0, 63, st);
    cub::DeviceScan::ExclusiveSum(nullptr, tb2, head, cid, n, st);
    size_t tb = tb1 > tb2 ? tb1 : tb2;
    CK(mem_alloc_async(c, (void**)&temp, tb, st));
    CK(cub::DeviceRadixSort::SortPairs(temp, tb, keys, skeys, idx, sidx, n, 0, 63, st));
    heads_kernel<<<g, 256, 0, st>>>(skeys, n, head);
    CK(cudaGetLastError());
    CK(cub::DeviceScan::ExclusiveSum(temp, tb, head, cid, n, st));
    int last_cid = 0, last_head = 0, h_bad = 0;
    CK(cudaMemcpyAsync(&last_cid, cid + n - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&last_head, head + n - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&h_bad, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(h_bbox, bbox, sizeof(h_bbox), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    *bad_cell = h_bad;
    if (h_bad) goto cleanup;
    KfMeta m;
    m.ox = h_bbox[0];
    m.oy = h_bbox[1];
    m.oz = h_bbox[2];
    m.ex = (unsigned)(h_bbox[3] - h_bbox[0] + 1);
    m.ey = (unsigned)(h_bbox[4] - h_bbox[1] + 1);
    m.ez = (unsigned)(h_bbox[5] - h_bbox[2] + 1);
    if (m.ex > (unsigned)kMaxEx || m.ey > (unsigned)kMaxEy || m.ez > (unsigned)kMaxEz) {
      *bad_extent = 1;
      goto cleanup;
    }
    int n_cells = last_cid + last_head;
    int cap = 64, lg = 6;
    while (cap < 4 * n_cells) { cap <<= 1; ++lg; }
    while ((long long)cap < (long long)MCS_HASH_SLOTS_PER_CELL * n_cells &&
           2ll * cap * 64 <= ((long long)c->cfg.kf_table_mib << 20) && lg < 30) {
      cap <<= 1;
      ++lg;
    }
    m.shift = (unsigned)(32 - lg);
    m.mask = (unsigned)(cap - 1);
    out.cap = cap;
    out.n_cells = n_cells;
    out.n_points = n;
    // cap probe slots + one always-empty sentinel slot (index cap) that out-of-bbox queries read
    // stream-ordered from the pool the context keeps mapped (a sparse table is tens of MiB: a
    // plain cudaMalloc of that size synchronises the device and maps pages on every insertion)
    CK(mem_alloc_async(c, (void**)&out.slots, sizeof(float4) * 4 * (size_t)(cap + 1), st));
    m.slots = out.slots;
    out.meta = m;
    init_slots_kernel<<<(cap + 1 + 255) / 256, 256, 0, st>>>(out.slots, cap + 1);
    aggregate_insert_kernel<<<g, 256, 0, st>>>(skeys, sidx, head, n, d_mean3, d_cov6, inv_r, m,
                                               out.slots);
    CK(cudaGetLastError());
  }
cleanup:
  mem_free_async(c, keys, st);
  mem_free_async(c, skeys, st);
  mem_free_async(c, idx, st);
  mem_free_async(c, sidx, st);
  mem_free_async(c, head, st);
  mem_free_async(c, cid, st);
  mem_free_async(c, bad, st);
  mem_free_async(c, bbox, st);
  if (temp) mem_free_async(c, temp, st);
#undef CK
  return e;
}

}  // namespace mcs
