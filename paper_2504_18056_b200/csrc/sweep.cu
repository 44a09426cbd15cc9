// sweep.cu — a2 ★: the fused transform -> hash lookup -> residual -> reduce sweep
// (Eqs.2-4; Eq.6).
//
// One thread per (particle, neighbour slot) work item; items are sorted by a pose-coherence
// key in a1, and the whole CTA walks the scan in lock-step, so every lane of a warp reads the
// SAME scan point from shared memory (a broadcast) and lanes with similar poses probe the same
// table slots (coalesced gathers).  Per point j:
//   q = kT mu_j            pinned fp32 key path (R27) -> cell = floor(q / r) -> bbox-local key
//   unmatched -> skip (R8)
//   e = mu' - q            C = Sigma' + R Sigma_j R^T      Omega = C^-1 (adjugate / det)
//   l -= e^T Omega e       n += 1
//   H~ += K^T Omega K,  b~ += K^T Omega e,   K = [-I, [m]x],  m = R mu_j = q - t
// K is the Jacobian in the rotated frame: J = de/d(delta) = [-R, R[mu]x] = K blockdiag(R, R)
// (R2), so the per-slot rotation back to the body frame happens once in a3, not per point.
// Table probes (key + 40 B of payload from one 64-byte slot) are issued in batches of two
// points, two points ahead of the math, so the L2 gather latency hides behind it; the (y, z)
// halves of the 3-vector / 3x3 math run as packed FFMA2.  R Sigma_j R^T uses the per-scan
// spectral form of Sigma_j (prepare_scan_kernel below); a scan whose points are all plane-form
// (GICP's plane regularisation, R36) runs the kPlane instantiation, one rotated vector per
// point.  A query cell outside the keyframe's bbox is clamped to the bbox extents (a key no slot
// holds).  Accumulation is two-level (fp32 within a stage of 256 / 448 points, fp64 across
// stages) in a fixed order: bitwise reproducible.  DESIGN.md §5.
#include <algorithm>
#include <atomic>
#include <type_traits>

#include "mcs_internal.cuh"

namespace mcs {

#ifndef MCS_SWEEP_THREADS
#define MCS_SWEEP_THREADS 128
#endif
#ifndef MCS_SWEEP_CHUNK
#define MCS_SWEEP_CHUNK 256
#endif
#ifndef MCS_SWEEP_AHEAD
#define MCS_SWEEP_AHEAD 4   // 4: probes issued in batches of two, two points ahead; 1: one ahead
#endif
#ifndef MCS_SWEEP_TMA
#define MCS_SWEEP_TMA 0  // 1: scan stages double-buffered by TMA bulk copies + mbarriers
#endif
#ifndef MCS_SWEEP_CONVERGENT
#define MCS_SWEEP_CONVERGENT 1  // 1: threads without an item run the stage loop (always missing)
#endif
#ifndef MCS_SWEEP_PACKED_H
#define MCS_SWEEP_PACKED_H 2  // 1: the H~ path's rows 1-2 as packed column pairs; 2: all of
                              // P, phi-phi and b~_phi as pairs (signs folded, undone at flush)
#endif
#ifndef MCS_SWEEP_CLAMP
#define MCS_SWEEP_CLAMP 1  // 1: out-of-bbox cells clamped to the extents instead of the sentinel
                           // (C2 sweep 5.546 -> 5.490 ms: two fewer ALU instructions per point)
#endif
#ifndef MCS_SWEEP_LEA_KEY
#define MCS_SWEEP_LEA_KEY 1  // 1: the clamped key as two shift-adds (LEA; C2 sweep -0.5 %)
#endif
#ifndef MCS_SWEEP_TMEM_ACC
#define MCS_SWEEP_TMEM_ACC 0  // 1: the fp64 stage totals in tensor memory (tcgen05.ld/st, 64
                              // columns per CTA) instead of 28 KB of shared memory: parity green,
                              // C2 sweep 5.409 -> 5.442 ms (the larger L1 does not pay for the
                              // per-stage TMEM round trips)
#endif
#ifndef MCS_SWEEP_GACC
#define MCS_SWEEP_GACC 0  // 1: fp64 stage totals in the (SoA) partial records, not shared memory
#endif
#ifndef MCS_SWEEP_STATIC_SMEM  // static shared arrays when they fit in 48 KB (default build)
#if MCS_SWEEP_TMA || MCS_SWEEP_GACC || (MCS_SWEEP_CHUNK + 2) * 48 + 224 * MCS_SWEEP_THREADS > 49152 || \
    (MCS_SWEEP_CHUNK_PLANE + 2) * 32 + 232 * MCS_SWEEP_THREADS > 49152
#define MCS_SWEEP_STATIC_SMEM 0
#else
#define MCS_SWEEP_STATIC_SMEM 1
#endif
#endif
#ifndef MCS_SWEEP_MINBLOCKS
#define MCS_SWEEP_MINBLOCKS 4
#endif
#ifndef MCS_NN27_MINBLOCKS
#define MCS_NN27_MINBLOCKS 4
#endif
#ifndef MCS_NN27_BATCH
#define MCS_NN27_BATCH 9  // NN27: cells whose first-probe loads are issued together (1, 3, 9, 27)
#endif
constexpr int kSweepThreads = MCS_SWEEP_THREADS;
#ifndef MCS_SWEEP_REDUCE
#define MCS_SWEEP_REDUCE 1  // 1: reduce_splits_kernel sums the point splits; 0: a3 reads them all
#endif
#ifndef MCS_SWEEP_CARVEOUT
#define MCS_SWEEP_CARVEOUT -1  // shared-memory carveout hint (percent) for the plane sweep; -1 default
#endif
#ifndef MCS_SWEEP_TRIM_SPLITS
#define MCS_SWEEP_TRIM_SPLITS 1  // 1: as many point splits as the plane-form stages fill
#endif
#ifndef MCS_SWEEP_CHUNK_PLANE
// stage points of the plane-form instantiation (32 B each).  C2 sweep by stage size (ms): 256
// 5.48, 384 5.45, 416 5.42, 448 5.40, 456 5.47, 480 5.46, 512 5.43 (3 splits of 4/4/2 stages
// at 448 beat 3/3/3 at 456); with the split count trimmed to the stages (12.5k particles:
// 10 stages over 5 splits, not 8 with 3 empty) 448 is also the best for the strong-scaling
// shards (12.5k 0.915, 25k 1.617, 50k 2.959 ms per update vs 0.932 / 1.647 / 2.980 at 256)
#define MCS_SWEEP_CHUNK_PLANE 448
#endif
constexpr int kChunkGeneral = MCS_SWEEP_CHUNK;      // scan points per shared-memory stage (48 B)
constexpr int kChunkPlane = MCS_SWEEP_CHUNK_PLANE;  // the same for plane-form points (32 B)

struct Probe {
  float4 s0, s1, s2;   // slot payload at the first probe position (speculatively loaded)
  float qx;            // pinned fp32 transform of the point: x, and (y, z) as one register pair
  float2 qyz;
  unsigned int key;    // bbox-local key; kNoKey32 = outside the keyframe bbox
  unsigned int h;      // slot index of the first probe
};

__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// packed-pair helpers: one FFMA2/FMUL2/FADD2 does the (y, z) halves of two scalar ops; each
// lane is the same IEEE fp32 operation as the scalar form (so the R27 key path stays pinned)
__device__ __forceinline__ float2 bc(float a) { return make_float2(a, a); }
__device__ __forceinline__ float2 sw(float2 a) { return make_float2(a.y, a.x); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 neg2(float2 a) { return make_float2(-a.x, -a.y); }

#ifndef MCS_SWEEP_LDG256
#define MCS_SWEEP_LDG256 1  // 1: the slot's first sector (key, mu', 4 of Sigma') as one 256-bit load
#endif
// the 40 used bytes of a 64-byte slot: sector 0 {key, mu'} {S'yy, S'zz, S'xy, S'xz} and the
// first 8 bytes of sector 1 {S'xx, S'yz}.  sm_100 loads a whole 32-byte sector per lane in one
// instruction (LDG.256): one request and its L1 wavefronts instead of two
__device__ __forceinline__ void ld_slot(const float4* sl, float4& s0, float4& s1, float4& s2) {
#if MCS_SWEEP_LDG256
  asm volatile("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=f"(s0.x), "=f"(s0.y), "=f"(s0.z), "=f"(s0.w), "=f"(s1.x), "=f"(s1.y),
                 "=f"(s1.z), "=f"(s1.w)
               : "l"(sl));
#else
  asm volatile("ld.global.nc.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(s0.x), "=f"(s0.y), "=f"(s0.z), "=f"(s0.w) : "l"(sl));
  asm volatile("ld.global.nc.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(s1.x), "=f"(s1.y), "=f"(s1.z), "=f"(s1.w) : "l"(sl + 1));
#endif
  asm volatile("ld.global.nc.v2.f32 {%0, %1}, [%2];" : "=f"(s2.x), "=f"(s2.y) : "l"(sl + 2));
  s2.z = 0.f;
  s2.w = 0.f;
}

// shared-memory load through a 32-bit shared-window address (kept in one register; a generic
// pointer would make ptxas re-derive the window base from %cgactaid at every use)
__device__ __forceinline__ float4 lds4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}

// ---- TMEM (tcgen05) for the fp64 stage totals (MCS_SWEEP_TMEM_ACC): each thread owns one TMEM
// lane (its warp's quarter of the 128 lanes), 64 columns = 28 doubles as (lo, hi) word pairs
__device__ __forceinline__ void tm_st8(uint32_t ta, const uint32_t (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};"
               ::"r"(ta), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]),
               "r"(v[6]), "r"(v[7])
               : "memory");
}
__device__ __forceinline__ void tm_ld8(uint32_t ta, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                 "=r"(v[6]), "=r"(v[7])
               : "r"(ta)
               : "memory");
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// ---- TMA bulk-copy staging (MCS_SWEEP_TMA): mbarrier + cp.async.bulk wrappers ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void bulk_stage(void* dst, const void* src, uint32_t bytes,
                                           uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// floor(x) as the bits of x + 1.5*2^23 rounded toward -inf: exact for |x| < 2^22, and every
// other finite x maps far outside any keyframe bbox after the offset.
constexpr float kMagic = 12582912.0f;

// kCorr: MCS_CORR_CELL (one probe of the containing voxel, R7) or MCS_CORR_NN27 (R33)
// kPlane: the instantiation for scans whose points are all plane-form (R36); both CELL
// instantiations are launched and the one that does not match the scan's flag (written by
// prepare_scan_kernel) returns at once (two instantiations, not a branch per stage: with both
// stage loops in one kernel ptxas spills the probe buffers)
template <int kCorr, bool kPlane>
__global__ void __launch_bounds__(kSweepThreads, kCorr == MCS_CORR_NN27 ? MCS_NN27_MINBLOCKS
                                                                       : MCS_SWEEP_MINBLOCKS)
    sweep_kernel(const float4* __restrict__ items, const int32_t* __restrict__ order,
                 int n_items, const float4* __restrict__ scan, int S,
                 const KfMeta* __restrict__ kmeta, float inv_r, float nn_r2,
                 double* __restrict__ part, size_t pstride, const int* __restrict__ nonplanar) {
  static_assert(!kPlane || kCorr == MCS_CORR_CELL, "NN27 has one (general) instantiation");
  if (kCorr == MCS_CORR_CELL && ((*nonplanar == 0) != kPlane)) return;
  using PlaneTag = std::integral_constant<bool, kPlane>;
  // dynamic shared memory: [(kChunk + 2) * 3] float4 scan stage, then [28][threads] fp64 totals
  constexpr int kW = kPlane ? 2 : 3;          // float4 words per scan point in the stage
  constexpr int kChunk = kPlane ? kChunkPlane : kChunkGeneral;
  constexpr int kStage = (kChunk + 2) * kW;  // float4 per stage buffer (2 spare points)
  constexpr int kBufs = MCS_SWEEP_TMA ? 2 : 1;
#if MCS_SWEEP_STATIC_SMEM
  // static shared memory: link-time addresses, nothing to rematerialise per point
  __shared__ float4 smem_dyn[kBufs * kStage];
#if !MCS_SWEEP_TMEM_ACC
  __shared__ double s_acc_st[28][kSweepThreads];
  double(*s_acc)[kSweepThreads] = s_acc_st;
#endif
#else
  extern __shared__ float4 smem_dyn[];
  // two-level accumulation: fp32 registers within a stage, fp64 totals per thread in shared
  // memory across stages (the fp32 running sums over a whole 4,096-point scan lose ~1e-5
  // relative, which an ill-conditioned H turns into >1e-5 m of pose error)
  double(*s_acc)[kSweepThreads] =
      reinterpret_cast<double(*)[kSweepThreads]>(smem_dyn + kBufs * kStage);
#endif
  float4* s_pt = smem_dyn;  // the current stage (MCS_SWEEP_TMA: one of two buffers)
  uint32_t s_pt_u32 = (uint32_t)__cvta_generic_to_shared(smem_dyn);  // same, shared window
  // a point is named by its shared-window address (48 B per point): a loop-carried register
  // that ptxas cannot rematerialise from %cgactaid at every use, as it does for a stage-constant
  // base plus an index
  constexpr uint32_t kPt = 16u * kW;
  auto pt = [&](uint32_t j, int w) { return lds4(j + 16u * w); };  // word w of point j
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int item = t < n_items ? order[t] : -1;
  // point splits (gridDim.y): this CTA's run of whole stages, and its own partial records
  const int stages_all = (S + kChunk - 1) / kChunk;
  const int st_per = (stages_all + gridDim.y - 1) / gridDim.y;
  const int st_lo = min((int)blockIdx.y * st_per, stages_all);
  const int st_hi = min(st_lo + st_per, stages_all);
  part += (size_t)blockIdx.y * kSlotWords * pstride;
  // this item's partial record, SoA: word k at part[k * pstride + item] (coalesced per warp)
  auto rec = [&](int k) -> double& { return part[(size_t)k * pstride + item]; };
  float4 r0 = make_float4(0, 0, 0, 0), r1 = r0, r2 = r0, inf = r0;
  if (item >= 0) {
    r0 = items[4 * (size_t)item + 0];
    r1 = items[4 * (size_t)item + 1];
    r2 = items[4 * (size_t)item + 2];
    inf = items[4 * (size_t)item + 3];
  }
  const int kf = item >= 0 ? __float_as_int(inf.x) : -1;
  MCS_DCHECK(t >= n_items || (item >= 0 && kf < 4096));
  const bool active = kf >= 0;
  const bool hb = active && (__float_as_int(inf.z) & 1);
  KfMeta m;
#if MCS_SWEEP_CONVERGENT
  // a thread without an item runs the stage loop with the others, on keyframe 0's table with an
  // empty bbox: every point probes one fixed slot (the sentinel, or with MCS_SWEEP_CLAMP the
  // clamped cell (0, 0, 0)), and the record is never written.  The loop then stays warp-convergent, and ptxas keeps its bound in
  // a uniform register instead of a spilled one
  m = kmeta[active ? kf : 0];
  if (!active) m.ex = m.ey = m.ez = 0;
#else
  if (active) {
    m = kmeta[kf];
  } else {
    m.slots = nullptr;
    m.ox = m.oy = m.oz = 0;
    m.ex = m.ey = m.ez = 0;
    m.shift = 31;
    m.mask = 0;
  }
#endif
  const unsigned int offx = (unsigned)__float_as_int(kMagic) + (unsigned)m.ox;
  const unsigned int offy = (unsigned)__float_as_int(kMagic) + (unsigned)m.oy;
  const unsigned int offz = (unsigned)__float_as_int(kMagic) + (unsigned)m.oz;
  // row 0 of kT as scalars, rows 1 and 2 as (y, z) column pairs
  const float R00 = r0.x, R01 = r0.y, R02 = r0.z, tx = r0.w;
  const float2 Ryz0 = make_float2(r1.x, r2.x), Ryz1 = make_float2(r1.y, r2.y);
  const float2 Ryz2 = make_float2(r1.z, r2.z), tyz = make_float2(r1.w, r2.w);
  const float2 ntyz = neg2(tyz);

  // transform, cell and key of point j (pinned, R27) and its first probe slot
  auto locate = [&](uint32_t j) {
    Probe p;
    const float4 A = pt(j, 0);
    // q = kR mu + kt with the pinned chain fma(R2, z, fma(R1, y, fma(R0, x, t))) per lane (R27)
    p.qx = __fmaf_rn(R02, A.z, __fmaf_rn(R01, A.y, __fmaf_rn(R00, A.x, tx)));
    p.qyz = fma2(Ryz2, bc(A.z), fma2(Ryz1, bc(A.y), fma2(Ryz0, bc(A.x), tyz)));
    // floor(q / r) -> bbox-local cell coordinates.  q * (1/r) is exact (r a power of two,
    // R27), so one fma rounded toward -inf equals the separate multiply and add
    const unsigned int dx = (unsigned)__float_as_int(__fmaf_rd(p.qx, inv_r, kMagic)) - offx;
    const float2 fyz = __ffma2_rd(p.qyz, bc(inv_r), bc(kMagic));
    const unsigned int dy = (unsigned)__float_as_int(fyz.x) - offy;
    const unsigned int dz = (unsigned)__float_as_int(fyz.y) - offz;
#if MCS_SWEEP_CLAMP
    // outside the keyframe's bbox: the cell clamped to the extents has a coordinate equal to
    // its extent, so no slot holds its key (every stored cell lies inside, and extents of at
    // most 2046 x 2047 x 1023 keep it below the empty / no-key markers); it probes an
    // ordinary, almost always empty, slot
#if MCS_SWEEP_LEA_KEY
    const unsigned int lk = local_key_lea(min(dx, m.ex), min(dy, m.ey), min(dz, m.ez));
#else
    const unsigned int lk = local_key(min(dx, m.ex), min(dy, m.ey), min(dz, m.ez));
#endif
    p.key = lk;
    p.h = slot_hash(lk, m.shift);
#else
    // outside the keyframe's bbox: a key no slot holds, probing the always-empty sentinel slot
    const bool in = (dx < m.ex) & (dy < m.ey) & (dz < m.ez);
    const unsigned int lk = local_key(dx, dy, dz);
    p.key = in ? lk : kNoKey32;
    p.h = in ? slot_hash(lk, m.shift) : m.mask + 1;  // the hash is < cap already
#endif
    MCS_DCHECK(!active || p.h <= m.mask + 1);
    return p;
  };
  // the (unconditional) first-probe loads; volatile: the compiler may not sink them towards
  // their use (that would undo the look-ahead)
  auto load = [&](Probe& p) {
    if (MCS_SWEEP_CONVERGENT || active) ld_slot(m.slots + 4 * (size_t)p.h, p.s0, p.s1, p.s2);
  };
  auto issue = [&](uint32_t j) {
    Probe p = locate(j);
    load(p);
    return p;
  };
  // issue whose loads are predicated on a key already loaded (never 0xFFFFFFFD: dx = 2047):
  // ptxas must then drain the earlier probe loads before it issues these (all probe loads
  // share one scoreboard, so a later wait would also drain the new ones)
  auto issue_after = [&](uint32_t j, unsigned int kdep) {
    Probe p = locate(j);
    if ((MCS_SWEEP_CONVERGENT || active) & (kdep != 0xFFFFFFFDu)) ld_slot(m.slots + 4 * (size_t)p.h, p.s0, p.s1, p.s2);
    return p;
  };

  float l = 0.f;
  int n = 0;
  float h[21];
  float bv[6];
#pragma unroll
  for (int k = 0; k < 21; ++k) h[k] = 0.f;
#pragma unroll
  for (int k = 0; k < 6; ++k) bv[k] = 0.f;
#if MCS_SWEEP_PACKED_H
  // pair accumulators (their h[]/bv[] words stay 0 until flush): H(0,1..2), H(1,1..2), b(1..2)
  float2 hp01 = bc(0.f), hp11 = bc(0.f), bp12 = bc(0.f);
#endif
#if MCS_SWEEP_PACKED_H >= 2
  // ((1,3), (2,3)), and with the second lane negated: ((0,4), (0,5)) ((1,4), (1,5))
  // ((2,4), (2,5)) ((3,4), (3,5)) ((4,4), (4,5)) (b4, b5)
  float2 hy = bc(0.f), hx0 = bc(0.f), hx1 = bc(0.f), hx2 = bc(0.f), hf34 = bc(0.f),
         hf45 = bc(0.f), bp45 = bc(0.f);
#elif MCS_SWEEP_PACKED_H
  // the rho-phi rows 1-2 column by column: ((1,3),(2,3)) ((1,4),(2,4)) ((1,5),(2,5))
  float2 hq0 = bc(0.f), hq1 = bc(0.f), hq2 = bc(0.f);
#endif

  // continue linear probing (rare): loads into fresh registers q.s*, waited on inside this
  // path, so the common path never inherits a pending scoreboard from it
  auto probe_on = [&](Probe& q) -> bool {
    unsigned int hh = slot_hash(q.key, m.shift) & m.mask;  // (recomputed: rare path)
    while (true) {
      hh = (hh + 1) & m.mask;
      MCS_DCHECK(hh != (slot_hash(q.key, m.shift) & m.mask));  // table never full (load <= 1/4)
      const float4* sl = m.slots + 4 * (size_t)hh;
      const float4 t0 = __ldg(sl);
      const unsigned int kk = __float_as_uint(t0.x);
      if (kk == q.key) {
        q.s0 = t0;
        q.s1 = __ldg(sl + 1);
        q.s2 = __ldg(sl + 2);
        return true;
      }
      if (kk == kEmptyKey32) return false;
    }
  };

  // Eqs.3-4 and Eq.6 for one matched (item, point); the (y, z) halves of the 3-vectors and of
  // the symmetric 3x3 matrices travel as register pairs (packed FFMA2/FMUL2/FADD2)
  // general scan point: Sigma_j = lam3 I + u u^T + v v^T (words {mu, lam3} {u, 0} {v, 0});
  // plane-form point (kPlane, R36): Sigma_j = lam3 I + |n|^2 I - n n^T = lam3 I + [n]x^T [n]x
  // (words {mu, lam3} {n, 0}), whose diagonal is a sum of squares, as in the general form
  auto accumulate = [&](auto plane_tag, uint32_t j, const Probe& p) {
    constexpr bool kPl = decltype(plane_tag)::value;
    const float4 A = pt(j, 0);  // {mu, lam3}
    const float4 U = pt(j, 1);  // {u, 0}, or {n, 0}
    // payload {key, mu'} {S'yy, S'zz, S'xy, S'xz} {S'xx, S'yz}
    const float4 P0 = p.s0, P1 = p.s1, P2 = p.s2;
    // e = mu' - kT mu   (Eq.4);  m = R mu = q - t
    const float ex = P0.y - p.qx;
    const float2 eyz = fma2(p.qyz, bc(-1.f), make_float2(P0.z, P0.w));
    const float mx = p.qx - tx;
    const float2 myz = add2(p.qyz, ntyz);
    const float my = myz.x, mz = myz.y;
    // C = Sigma' + R Sigma R^T  (Eq.4):  Sigma' + lam3 I + (Ru)(Ru)^T + (Rv)(Rv)^T, or with
    // x = R n:  Sigma' + lam3 I + [x]x^T [x]x,  diagonal (x1^2 + x2^2, x0^2 + x2^2, x0^2 + x1^2)
    const float ux = fmaf(R02, U.z, fmaf(R01, U.y, R00 * U.x));
    const float2 uyz = fma2(Ryz2, bc(U.z), fma2(Ryz1, bc(U.y), mul2(Ryz0, bc(U.x))));
    float c00, c12;
    float2 c1122, c0102;
    if constexpr (kPl) {
      c00 = fmaf(uyz.x, uyz.x, fmaf(uyz.y, uyz.y, P2.x + A.w));
      c1122 = fma2(bc(ux), bc(ux), fma2(sw(uyz), sw(uyz), add2(make_float2(P1.x, P1.y), bc(A.w))));
      c0102 = fma2(bc(-ux), uyz, make_float2(P1.z, P1.w));
      c12 = fmaf(-uyz.x, uyz.y, P2.y);
    } else {
      const float4 V = pt(j, 2);  // {v, 0}
      const float vx = fmaf(R02, V.z, fmaf(R01, V.y, R00 * V.x));
      const float2 vyz = fma2(Ryz2, bc(V.z), fma2(Ryz1, bc(V.y), mul2(Ryz0, bc(V.x))));
      c00 = fmaf(ux, ux, fmaf(vx, vx, P2.x + A.w));
      c1122 = fma2(uyz, uyz, fma2(vyz, vyz, add2(make_float2(P1.x, P1.y), bc(A.w))));
      c0102 = fma2(bc(ux), uyz, fma2(bc(vx), vyz, make_float2(P1.z, P1.w)));
      c12 = fmaf(uyz.x, uyz.y, fmaf(vyz.x, vyz.y, P2.y));
    }
    // Omega = C^-1 = adj(C) / det(C):  (k11, k22) = c00 (c22, c11) - (c02, c01)^2,
    // (k01, k02) = c12 (c02, c01) - (c01 c22, c02 c11)
    const float k00 = fmaf(c1122.x, c1122.y, -c12 * c12);
    const float2 c0201 = sw(c0102);
    const float2 k1122 = fma2(bc(c00), sw(c1122), mul2(c0201, neg2(c0201)));
    const float2 k0102 = fma2(bc(c12), c0201, mul2(c0102, neg2(sw(c1122))));
    const float k12 = fmaf(c0102.x, c0102.y, -c00 * c12);
    const float id = rcp_approx(fmaf(c00, k00, fmaf(c0102.x, k0102.x, c0102.y * k0102.y)));
#if MCS_SWEEP_PACKED_H
    // Omega as o00 and the pairs C = (o01, o02), A = (o11, o12), B = (o12, o22): rows 1-2 of
    // Omega [m]x then come out column by column as pairs (o12 is formed twice, one FMUL, so
    // that A and B need no register moves)
    const float o00 = k00 * id;
    const float2 oC = mul2(k0102, bc(id));
    const float2 oA = make_float2(k1122.x * id, k12 * id);
    // (o12 formed again by an opaque multiply — the same product, in a second register, so
    // that the compiler does not merge it with A's and move registers to build the pairs)
    float o12b;
    asm("mul.rn.f32 %0, %1, %2;" : "=f"(o12b) : "f"(k12), "f"(id));
    const float2 oB = make_float2(o12b, k1122.y * id);
    const float ey = eyz.x, ez = eyz.y;
    // w = Omega e: w0 = o00 ex + o01 ey + o02 ez; (w1, w2) = ex C + ey A + ez B;  l -= e^T w
    const float w0 = fmaf(o00, ex, fmaf(oC.x, ey, oC.y * ez));
    const float2 w12 = fma2(bc(ex), oC, fma2(bc(ey), oA, mul2(bc(ez), oB)));
    const float w1 = w12.x, w2 = w12.y;
    l = fmaf(-ex, w0, fmaf(-ey, w1, fmaf(-ez, w2, l)));
    ++n;
#if MCS_SWEEP_PACKED_H >= 2
    if (hb) {
      // H~ = K^T Omega K = [[Omega, -Omega M], [-M^T Omega, M^T Omega M]], M = [m]x; P = Omega M
      // as X_r = (P_r1, -P_r2) = mx (Omega_r2, Omega_r1) - Omega_r0 (mz, my)  (r = 0, 1, 2),
      // Y = (P10, P20) = mz A - my B and the scalar P00
      const float2 mzy = sw(myz);
      const float o01 = oC.x, o02 = oC.y;
      const float2 X0 = fma2(bc(mx), sw(oC), mul2(bc(-o00), mzy));
      const float2 X1 = fma2(bc(mx), sw(oA), mul2(bc(-o01), mzy));
      const float2 X2 = fma2(bc(mx), sw(oB), mul2(bc(-o02), mzy));
      const float2 Y = fma2(bc(-my), oB, mul2(bc(mz), oA));
      const float p00 = o01 * mz - o02 * my;
      h[0] += o00;
      hp01 = add2(hp01, oC);
      hp11 = add2(hp11, oA);
      h[11] += oB.y;
      h[3] -= p00;
      hx0 = add2(hx0, neg2(X0));
      hx1 = add2(hx1, neg2(X1));
      hx2 = add2(hx2, neg2(X2));
      hy = add2(hy, neg2(Y));
      // M^T Omega M = -M P:  (3,3) = mz P10 - my P20;  ((3,4), -(3,5)) = mz X1 - my X2;
      // ((4,4), -(4,5)) = mx X2 - mz X0;  (5,5) = my P02 - mx P12
      h[15] = fmaf(mz, Y.x, fmaf(-my, Y.y, h[15]));
      hf34 = fma2(bc(mz), X1, fma2(bc(-my), X2, hf34));
      hf45 = fma2(bc(mx), X2, fma2(bc(-mz), X0, hf45));
      h[20] = fmaf(mx, X1.y, fmaf(-my, X0.y, h[20]));
      // b~ = K^T Omega e = [-w ; w x m]:  b3 = w1 mz - w2 my;  (b4, -b5) = mx (w2, w1) - w0 (mz, my)
      bv[0] -= w0;
      bp12 = add2(bp12, neg2(w12));
      bv[3] = fmaf(w1, mz, fmaf(-w2, my, bv[3]));
      bp45 = fma2(bc(mx), sw(w12), fma2(bc(-w0), mzy, bp45));
    }
#else
    if (hb) {
      // H~ = K^T Omega K = [[Omega, -Omega M], [-M^T Omega, M^T Omega M]], M = [m]x; P = Omega M
      // row 0 scalar; rows 1-2 per column k: (P1k, P2k)
      const float o01 = oC.x, o02 = oC.y;
      const float p00 = o01 * mz - o02 * my, p01 = o02 * mx - o00 * mz, p02 = o00 * my - o01 * mx;
      const float2 pc0 = fma2(oB, bc(-my), mul2(oA, bc(mz)));  // (P10, P20)
      const float2 pc1 = fma2(oC, bc(-mz), mul2(oB, bc(mx)));  // (P11, P21)
      const float2 pc2 = fma2(oA, bc(-mx), mul2(oC, bc(my)));  // (P12, P22)
      h[0] += o00;
      hp01 = add2(hp01, oC);
      hp11 = add2(hp11, oA);
      h[11] += oB.y;
      h[3] -= p00; h[4] -= p01; h[5] -= p02;
      hq0 = add2(hq0, neg2(pc0));
      hq1 = add2(hq1, neg2(pc1));
      hq2 = add2(hq2, neg2(pc2));
      // M^T Omega M = -M P
      h[15] = fmaf(mz, pc0.x, fmaf(-my, pc0.y, h[15]));  // (3,3)
      h[16] = fmaf(mz, pc1.x, fmaf(-my, pc1.y, h[16]));  // (3,4)
      h[17] = fmaf(mz, pc2.x, fmaf(-my, pc2.y, h[17]));  // (3,5)
      h[18] = fmaf(mx, pc1.y, fmaf(-mz, p01, h[18]));    // (4,4)
      h[19] = fmaf(mx, pc2.y, fmaf(-mz, p02, h[19]));    // (4,5)
      h[20] = fmaf(my, p02, fmaf(-mx, pc2.x, h[20]));    // (5,5)
      // b~ = K^T Omega e = [-w ; w x m]
      bv[0] -= w0;
      bp12 = add2(bp12, neg2(w12));
      bv[3] = fmaf(w1, mz, fmaf(-w2, my, bv[3]));
      bv[4] = fmaf(w2, mx, fmaf(-w0, mz, bv[4]));
      bv[5] = fmaf(w0, my, fmaf(-w1, mx, bv[5]));
    }
#endif
#else
    const float o00 = k00 * id, o12 = k12 * id;
    const float2 o1122 = mul2(k1122, bc(id)), o0102 = mul2(k0102, bc(id));
    const float o01 = o0102.x, o02 = o0102.y, o11 = o1122.x, o22 = o1122.y;
    const float ey = eyz.x, ez = eyz.y;
    // w = Omega e: w0 = o00 ex + o01 ey + o02 ez; (w1, w2) = ex (o01, o02) + (o11 ey, o22 ez)
    // + o12 (ez, ey);  l -= e^T Omega e  (Eq.3)
    const float w0 = fmaf(o00, ex, fmaf(o01, ey, o02 * ez));
    const float2 w12 = fma2(bc(ex), o0102, fma2(o1122, eyz, mul2(bc(o12), sw(eyz))));
    const float w1 = w12.x, w2 = w12.y;
    l = fmaf(-ex, w0, fmaf(-ey, w1, fmaf(-ez, w2, l)));
    ++n;
    if (hb) {
      // H~ = K^T Omega K = [[Omega, -Omega M], [-M^T Omega, M^T Omega M]], M = [m]x; P = Omega M
      const float p00 = o01 * mz - o02 * my, p01 = o02 * mx - o00 * mz, p02 = o00 * my - o01 * mx;
      const float p10 = o11 * mz - o12 * my, p11 = o12 * mx - o01 * mz, p12 = o01 * my - o11 * mx;
      const float p20 = o12 * mz - o22 * my, p21 = o22 * mx - o02 * mz, p22 = o02 * my - o12 * mx;
      h[0] += o00; h[1] += o01; h[2] += o02;
      h[3] -= p00; h[4] -= p01; h[5] -= p02;
      h[6] += o11; h[7] += o12;
      h[8] -= p10; h[9] -= p11; h[10] -= p12;
      h[11] += o22;
      h[12] -= p20; h[13] -= p21; h[14] -= p22;
      // M^T Omega M = -M P
      h[15] = fmaf(mz, p10, fmaf(-my, p20, h[15]));  // (3,3)
      h[16] = fmaf(mz, p11, fmaf(-my, p21, h[16]));  // (3,4)
      h[17] = fmaf(mz, p12, fmaf(-my, p22, h[17]));  // (3,5)
      h[18] = fmaf(mx, p21, fmaf(-mz, p01, h[18]));  // (4,4)
      h[19] = fmaf(mx, p22, fmaf(-mz, p02, h[19]));  // (4,5)
      h[20] = fmaf(my, p02, fmaf(-mx, p12, h[20]));  // (5,5)
      // b~ = K^T Omega e = [-w ; w x m]
      bv[0] -= w0; bv[1] -= w1; bv[2] -= w2;
      bv[3] = fmaf(w1, mz, fmaf(-w2, my, bv[3]));
      bv[4] = fmaf(w2, mx, fmaf(-w0, mz, bv[4]));
      bv[5] = fmaf(w0, my, fmaf(-w1, mx, bv[5]));
    }
#endif
  };

  // first probe: hit -> accumulate; empty slot (or the sentinel) -> miss; else keep probing
  auto act = [&](auto tg, uint32_t j, const Probe& p, unsigned int k0) {
    if (k0 == p.key) {
      accumulate(tg, j, p);
    } else if (k0 != kEmptyKey32) {
      Probe q;
      q.qx = p.qx; q.qyz = p.qyz; q.key = p.key;
      if (probe_on(q)) accumulate(tg, j, q);
    }
  };
  auto consume = [&](auto tg, uint32_t j, const Probe& p) {
    act(tg, j, p, __float_as_uint(p.s0.x));
  };

  // NN27 (R33): the nearest cell representative within nn_radius among the 27 voxels around
  // q's voxel, d = mu'32 - q32, d2 = fma(dz, dz, fma(dy, dy, dx * dx)) (pinned fp32), ties ->
  // lower (oz, oy, ox) index.
  // Per cell (ox, oy, oz) the key and hash follow from the centre's by one add each: with the
  // key taken as the modular sum kc = (bx << 21) + (by << 10) + bz, the key of an in-bbox
  // neighbour is kc + (ox << 21) + (oy << 10) + oz (mod 2^32, equal to local_key's OR form
  // there), and its hash product (kc + off) * M = kc * M + off * M; the bbox test is the AND
  // of three per-axis flags computed once per point.
  const float nn_r2_up = __int_as_float(__float_as_int(nn_r2) + 1);  // next float above nn_r2
  auto nn27_point = [&](uint32_t j) {
    Probe p = locate(j);
    const unsigned int bx = (unsigned)__float_as_int(__fmaf_rd(p.qx, inv_r, kMagic)) - offx;
    const float2 fyz = __ffma2_rd(p.qyz, bc(inv_r), bc(kMagic));
    const unsigned int by = (unsigned)__float_as_int(fyz.x) - offy;
    const unsigned int bz = (unsigned)__float_as_int(fyz.y) - offz;
    const unsigned int kc = (bx << 21) + (by << 10) + bz;
    const unsigned int hc = kc * kHashMul32;
    bool fx[3], fy[3], fz[3];
#pragma unroll
    for (int o = 0; o < 3; ++o) {
      fx[o] = bx + (unsigned)(o - 1) < m.ex;
      fy[o] = by + (unsigned)(o - 1) < m.ey;
      fz[o] = bz + (unsigned)(o - 1) < m.ez;
    }
    int best = -1;
    // d2 <= nn_r2 and strictly below the best so far (ties keep the lower enumeration index;
    // cells are visited in (oz, oy, ox) order) is one compare against a running bound that
    // starts just above nn_r2
    float best_d2 = nn_r2_up;
    auto consider = [&](unsigned int h, const float4 t0) {  // t0 = {key, mu'} of slot h
      const float dx = __fsub_rn(t0.y, p.qx);
      const float dy = __fsub_rn(t0.z, p.qyz.x);
      const float dz = __fsub_rn(t0.w, p.qyz.y);
      const float d2 = __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
      if (d2 < best_d2) {
        best = (int)h;
        best_d2 = d2;
      }
    };
    // the first-probe loads (key + mu', 16 B) of kB cells at a time issue together, then are
    // consumed in (oz, oy, ox) order
    constexpr int kB = MCS_NN27_BATCH;
    static_assert(27 % kB == 0, "MCS_NN27_BATCH: 1, 3, 9 or 27");
#pragma unroll
    for (int c0 = 0; c0 < 27; c0 += kB) {
      unsigned int key[kB], h[kB];
      float4 t[kB];
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        const int c = c0 + u;
        const int ox = c % 3 - 1, oy = (c / 3) % 3 - 1, oz = c / 9 - 1;
        const unsigned int off = (unsigned)(ox * (1 << 21) + oy * (1 << 10) + oz);
        const bool in = fx[ox + 1] & fy[oy + 1] & fz[oz + 1];
        key[u] = in ? kc + off : kNoKey32;
        h[u] = in ? (hc + off * kHashMul32) >> m.shift : m.mask + 1;  // sentinel: always empty
        MCS_DCHECK(!in || (key[u] == local_key(bx + ox, by + oy, bz + oz) &&
                           h[u] == slot_hash(key[u], m.shift)));
        t[u] = __ldg(m.slots + 4 * (size_t)h[u]);
      }
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        const unsigned int k0 = __float_as_uint(t[u].x);
        if (k0 == key[u]) {
          consider(h[u], t[u]);
        } else if (k0 != kEmptyKey32) {  // rare: continue linear probing
          unsigned int hh = h[u];
          while (true) {
            hh = (hh + 1) & m.mask;
            const float4 tt = __ldg(m.slots + 4 * (size_t)hh);
            const unsigned int kk = __float_as_uint(tt.x);
            if (kk == key[u]) {
              consider(hh, tt);
              break;
            }
            if (kk == kEmptyKey32) break;
          }
        }
      }
    }
    if (best >= 0) {
      const float4* sl = m.slots + 4 * (size_t)best;
      p.s0 = __ldg(sl);
      p.s1 = __ldg(sl + 1);
      p.s2 = __ldg(sl + 2);
      accumulate(std::false_type{}, j, p);
    }
  };



  // fp64 totals across stages: [0] l, [1..21] H~, [22..27] b~ (shared memory, or with
  // MCS_SWEEP_GACC the record words 0, 2..22, 23..28 themselves)
#if MCS_SWEEP_TMEM_ACC
  static_assert(MCS_SWEEP_STATIC_SMEM && MCS_SWEEP_CONVERGENT && !MCS_SWEEP_TMA &&
                    !MCS_SWEEP_GACC && kSweepThreads == 128,
                "TMEM totals: four convergent warps, one TMEM lane quarter each");
  __shared__ uint32_t s_tmem;
  if (threadIdx.x < 32) {  // warp 0 allocates 64 columns for the CTA
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&s_tmem))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = s_tmem + ((threadIdx.x & ~31u) << 16);  // this warp's lanes, column 0
  {
    const uint32_t z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int c = 0; c < 7; ++c) tm_st8(tm + 8 * c, z);
    tm_wait_st();
  }
#else
  auto tot = [&](int k) -> double& {
#if MCS_SWEEP_GACC
    return rec(k == 0 ? 0 : k + 1);
#else
    return s_acc[k][threadIdx.x];
#endif
  };
#if MCS_SWEEP_GACC
  if (active)
#endif
#pragma unroll
    for (int k = 0; k < 28; ++k) tot(k) = 0.0;
#endif
  auto flush = [&]() {
#if MCS_SWEEP_TMEM_ACC
    float d0 = l;
#else
    tot(0) += (double)l;
#endif
    l = 0.f;
#if MCS_SWEEP_PACKED_H
    h[1] = hp01.x; h[2] = hp01.y; h[6] = hp11.x; h[7] = hp11.y; bv[1] = bp12.x; bv[2] = bp12.y;
    hp01 = hp11 = bp12 = bc(0.f);
#endif
#if MCS_SWEEP_PACKED_H >= 2
    h[8] = hy.x; h[12] = hy.y;
    h[4] = hx0.x; h[5] = -hx0.y; h[9] = hx1.x; h[10] = -hx1.y; h[13] = hx2.x; h[14] = -hx2.y;
    h[16] = hf34.x; h[17] = -hf34.y; h[18] = hf45.x; h[19] = -hf45.y;
    bv[4] = bp45.x; bv[5] = -bp45.y;
    hy = hx0 = hx1 = hx2 = hf34 = hf45 = bp45 = bc(0.f);
#elif MCS_SWEEP_PACKED_H
    h[8] = hq0.x; h[12] = hq0.y; h[9] = hq1.x; h[13] = hq1.y; h[10] = hq2.x; h[14] = hq2.y;
    hq0 = hq1 = hq2 = bc(0.f);
#endif
#if MCS_SWEEP_TMEM_ACC
    // totals k = 4c .. 4c + 3 (l, H~21, b~6 in that order) in chunk c: load, add, store
#pragma unroll
    for (int c = 0; c < 7; ++c) {
      uint32_t w[8];
      tm_ld8(tm + 8 * c, w);
      tm_wait_ld();
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int k = 4 * c + u;
        const float dk = k == 0 ? d0 : (k <= 21 ? h[k - 1] : bv[k - 22]);
        const double t = __hiloint2double((int)w[2 * u + 1], (int)w[2 * u]) + (double)dk;
        w[2 * u] = (uint32_t)__double2loint(t);
        w[2 * u + 1] = (uint32_t)__double2hiint(t);
      }
      tm_st8(tm + 8 * c, w);
    }
    tm_wait_st();
#pragma unroll
    for (int k = 0; k < 21; ++k) h[k] = 0.f;
#pragma unroll
    for (int k = 0; k < 6; ++k) bv[k] = 0.f;
#else
#pragma unroll
    for (int k = 0; k < 21; ++k) {
      tot(1 + k) += (double)h[k];
      h[k] = 0.f;
    }
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      tot(22 + k) += (double)bv[k];
      bv[k] = 0.f;
    }
#endif
  };

  // the math of one stage of cnt points in s_pt (active threads)
  auto stage = [&](auto tg, const int cnt) {
    const uint32_t e = s_pt_u32 + kPt * (uint32_t)cnt;  // one past the last point
    if (kCorr == MCS_CORR_NN27) {
      for (uint32_t j = s_pt_u32; j < e; j += kPt) nn27_point(j);
      return;
    }
    // Probe buffers in rotation, no register copies between iterations.  Every probe load
    // shares one scoreboard, so any wait drains all loads issued so far: the loop therefore
    // drains batch n (its key words), issues batch n+1 (two points, predicated on those keys so
    // the issue cannot be hoisted above the drain), then does the math of batch n while batch
    // n+1 is in flight.  s_pt has two spare points, so the look-ahead issues past the stage end
    // need no guard (their stale key probes a real slot or the sentinel, and is never consumed)
#if MCS_SWEEP_AHEAD == 4
    Probe pa = issue(s_pt_u32), pb = issue(s_pt_u32 + kPt), pc, pd;
    uint32_t j = s_pt_u32;
    for (; j + 3 * kPt < e; j += 4 * kPt) {
      const unsigned int ka = __float_as_uint(pa.s0.x), kb = __float_as_uint(pb.s0.x);
      pc = issue_after(j + 2 * kPt, ka);
      pd = issue_after(j + 3 * kPt, kb);
      act(tg, j, pa, ka);
      act(tg, j + kPt, pb, kb);
      const unsigned int kc = __float_as_uint(pc.s0.x), kd = __float_as_uint(pd.s0.x);
      pa = issue_after(j + 4 * kPt, kc);
      pb = issue_after(j + 5 * kPt, kd);
      act(tg, j + 2 * kPt, pc, kc);
      act(tg, j + 3 * kPt, pd, kd);
    }
    if (j < e) consume(tg, j, pa);
    if (j + kPt < e) consume(tg, j + kPt, pb);
    if (j + 2 * kPt < e) {
      pc = issue(j + 2 * kPt);
      consume(tg, j + 2 * kPt, pc);
    }
#else
    Probe pa = issue(s_pt_u32), pb;
    uint32_t j = s_pt_u32;
    for (; j + kPt < e; j += 2 * kPt) {
      pb = issue(j + kPt);
      consume(tg, j, pa);
      pa = issue(j + 2 * kPt);
      consume(tg, j + kPt, pb);
    }
    if (j < e) consume(tg, j, pa);
#endif
  };

#if MCS_SWEEP_TMA
  // Scan stages double-buffered in shared memory by TMA bulk copies (cp.async.bulk, one thread
  // issues, an mbarrier counts the bytes).  No CTA-wide barrier per stage: the last warp to
  // finish stage k (a shared-memory counter) refills that buffer with stage k + 2, so fast
  // warps run up to a stage ahead of slow ones.
  uint64_t* full = reinterpret_cast<uint64_t*>(&s_acc[28][0]);  // [2] mbarriers
  int* done = reinterpret_cast<int*>(full + 2);                   // [2] warps done with stage
  const int n_stages = st_hi - st_lo;  // stages k of this CTA: st_lo + k
  constexpr int kWarps = kSweepThreads / 32;
  auto refill = [&](int k) {  // one thread: stage st_lo + k into buffer k & 1
    const int base = (st_lo + k) * kChunk;
    const int cnt = min(kChunk, S - base);
    bulk_stage(smem_dyn + (k & 1) * kStage, scan + kW * (size_t)base, kPt * cnt, &full[k & 1]);
  };
  if (threadIdx.x < 4 * kW)
    smem_dyn[(threadIdx.x / (2 * kW)) * kStage + kW * kChunk + threadIdx.x % (2 * kW)] =
        make_float4(0.f, 0.f, 0.f, 0.f);
  if (threadIdx.x == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    done[0] = done[1] = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    refill(0);
    if (n_stages > 1) refill(1);
  }
  for (int k = 0; k < n_stages; ++k) {
    s_pt = smem_dyn + (k & 1) * kStage;
    s_pt_u32 = (uint32_t)__cvta_generic_to_shared(s_pt);
    mbar_wait(&full[k & 1], (k >> 1) & 1);
    if (active) {
      stage(PlaneTag{}, min(kChunk, S - (st_lo + k) * kChunk));
      flush();
    }
    __syncwarp();
    if ((threadIdx.x & 31) == 0) {
      __threadfence_block();  // this warp's reads of the buffer precede the count
      if (atomicAdd(&done[k & 1], 1) == kWarps - 1) {
        done[k & 1] = 0;
        if (k + 2 < n_stages) {
          __threadfence_block();
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          refill(k + 2);
        }
      }
    }
  }
#else
  if (threadIdx.x < 2 * kW) s_pt[kW * kChunk + threadIdx.x] = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int base = st_lo * kChunk; base < st_hi * kChunk; base += kChunk) {
    const int cnt = min(kChunk, S - base);
    __syncthreads();
    for (int k = threadIdx.x; k < cnt * kW; k += kSweepThreads) s_pt[k] = scan[kW * base + k];
    __syncthreads();
    if (!MCS_SWEEP_CONVERGENT && !active) continue;
    stage(PlaneTag{}, cnt);
    flush();
  }
#endif
#if MCS_SWEEP_TMEM_ACC
#pragma unroll
  for (int c = 0; c < 7; ++c) {  // (every thread: the TMEM loads are warp-collective)
    uint32_t w[8];
    tm_ld8(tm + 8 * c, w);
    tm_wait_ld();
    if (active) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int k = 4 * c + u;  // total k -> record word (k == 0 ? 0 : k + 1)
        rec(k == 0 ? 0 : k + 1) = __hiloint2double((int)w[2 * u + 1], (int)w[2 * u]);
      }
    }
  }
  if (active) rec(1) = (double)n;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(s_tmem) : "memory");
  }
#else
  if (active) {
    rec(1) = (double)n;
#if !MCS_SWEEP_GACC
    rec(0) = tot(0);
#pragma unroll
    for (int k = 0; k < 21; ++k) rec(2 + k) = tot(1 + k);
#pragma unroll
    for (int k = 0; k < 6; ++k) rec(23 + k) = tot(22 + k);
#endif
  }
#endif
}

// Point splits (gridDim.y = P > 1 in the sweep): split 0's record of every item becomes the sum
// of the P records in split order (the same additions a3 made before), one thread per (word,
// item), so a3 reads one record per item whatever P (a3 reading P records per particle was
// latency-bound: +0.09 ms at P = 3 for C2, more than the splits saved).
__global__ void reduce_splits_kernel(double* __restrict__ part, size_t pstride, int nb, int N,
                                     int capN, int P) {
  const long long n_items = (long long)nb * N;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 29LL * n_items) return;
  const int k = (int)(t / n_items);
  const long long rem = t - (long long)k * n_items;
  const int s = (int)(rem / N), i = (int)(rem - (long long)s * N);  // item s * capN + i
  double* r = part + (size_t)k * pstride + (size_t)s * capN + i;
  double v = r[0];
#pragma unroll
  for (int q = 1; q < P; ++q) v += r[(size_t)q * kSlotWords * pstride];
  r[0] = v;
}

// Scan preparation (once per update): Sigma_j = lambda3 I + u u^T + v v^T with u, v the two
// leading eigenvectors scaled by sqrt(lambda_k - lambda3) — the spectral decomposition,
// exact up to rounding for any symmetric Sigma (fp64 cyclic Jacobi, then rounded).  The sweep
// then forms R Sigma R^T as lambda3 I + (Ru)(Ru)^T + (Rv)(Rv)^T (33 FP32 ops instead of 45).
// Plane-form points also get {mu, lambda3} {x, 0} in out_plane (R36 below), and *nonplanar
// counts the points that are not plane-form: 0 selects the plane instantiation of the sweep.
__global__ void prepare_scan_kernel(const float* __restrict__ mean3,
                                    const float* __restrict__ cov6, int S,
                                    float4* __restrict__ out, float4* __restrict__ out_plane,
                                    int* __restrict__ nonplanar) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= S) return;
  const float* c = cov6 + 6 * j;
  double a[3][3] = {{c[0], c[1], c[2]}, {c[1], c[3], c[4]}, {c[2], c[4], c[5]}};
  double v[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  for (int sweep = 0; sweep < 12; ++sweep) {
    const double off = a[0][1] * a[0][1] + a[0][2] * a[0][2] + a[1][2] * a[1][2];
    const double dg = a[0][0] * a[0][0] + a[1][1] * a[1][1] + a[2][2] * a[2][2];
    if (off <= 1e-36 * dg) break;
    for (int pq = 0; pq < 3; ++pq) {
      const int p = pq == 2 ? 1 : 0, q = pq == 0 ? 1 : 2;
      if (a[p][q] == 0.0) continue;
      const double theta = (a[q][q] - a[p][p]) / (2.0 * a[p][q]);
      const double tt = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
      const double cs = 1.0 / sqrt(tt * tt + 1.0), sn = tt * cs;
      for (int k = 0; k < 3; ++k) {  // A <- J^T A J
        const double akp = a[k][p], akq = a[k][q];
        a[k][p] = cs * akp - sn * akq;
        a[k][q] = sn * akp + cs * akq;
      }
      for (int k = 0; k < 3; ++k) {
        const double apk = a[p][k], aqk = a[q][k];
        a[p][k] = cs * apk - sn * aqk;
        a[q][k] = sn * apk + cs * aqk;
      }
      for (int k = 0; k < 3; ++k) {  // V <- V J
        const double vkp = v[k][p], vkq = v[k][q];
        v[k][p] = cs * vkp - sn * vkq;
        v[k][q] = sn * vkp + cs * vkq;
      }
    }
  }
  // order eigenvalues: l0 >= l1 >= l2
  int i0 = 0, i1 = 1, i2 = 2;
  double lam[3] = {a[0][0], a[1][1], a[2][2]};
  if (lam[i0] < lam[i1]) { int t = i0; i0 = i1; i1 = t; }
  if (lam[i1] < lam[i2]) { int t = i1; i1 = i2; i2 = t; }
  if (lam[i0] < lam[i1]) { int t = i0; i0 = i1; i1 = t; }
  const double l3 = lam[i2];
  const double su = sqrt(fmax(lam[i0] - l3, 0.0)), sv = sqrt(fmax(lam[i1] - l3, 0.0));
  const float* m = mean3 + 3 * j;
  out[3 * j + 0] = make_float4(m[0], m[1], m[2], (float)l3);
  out[3 * j + 1] = make_float4((float)(su * v[0][i0]), (float)(su * v[1][i0]),
                               (float)(su * v[2][i0]), 0.f);
  out[3 * j + 2] = make_float4((float)(sv * v[0][i1]), (float)(sv * v[1][i1]),
                               (float)(sv * v[2][i1]), 0.f);
  // plane form (R36): GICP's plane-regularised covariances (eigenvalues (1, 1, eps), R9) have
  // l0 = l1 up to the rounding of their fp32 entries.  A split within 4 ulps of l0 is merged:
  // Sigma = l3 I + a (I - n n^T) = l3 I + [x]x^T [x]x with a = (l0 + l1) / 2 - l3 and
  // x = sqrt(a) n, n the eigenvector of l3 — one vector for the sweep to rotate instead of two
  const bool plane = lam[i0] - lam[i1] <= 0x1p-21 * fabs(lam[i0]);
  const double sa = sqrt(fmax(0.5 * (lam[i0] + lam[i1]) - l3, 0.0));
  out_plane[2 * j + 0] = make_float4(m[0], m[1], m[2], (float)l3);
  out_plane[2 * j + 1] = make_float4((float)(sa * v[0][i2]), (float)(sa * v[1][i2]),
                                     (float)(sa * v[2][i2]), 0.f);
  if (!plane) atomicAdd(nonplanar, 1);
}

cudaError_t launch_prepare_scan(const float* mean3, const float* cov6, int S, float4* out,
                                float4* out_plane, int* nonplanar, cudaStream_t st) {
  const cudaError_t e = cudaMemsetAsync(nonplanar, 0, sizeof(int), st);
  if (e != cudaSuccess) return e;
  prepare_scan_kernel<<<(S + 127) / 128, 128, 0, st>>>(mean3, cov6, S, out, out_plane,
                                                       nonplanar);
  return cudaGetLastError();
}

#ifndef MCS_SPLIT_MIDRANGE
#define MCS_SPLIT_MIDRANGE 1
#endif
#ifndef MCS_SPLIT_TARGET_CTAS
// auto point splits aim for ~7,000 CTAs (~12 waves of 148 x 4): more, shorter CTAs balance the
// uneven per-item hit rates (C2 sweep: 1 split 6.27 ms, 2 6.19, 3 6.13, 4 6.17; with a3's
// extra partial reads the update is fastest at 3); at most 8 splits (small shards)
#define MCS_SPLIT_TARGET_CTAS 7000
#endif

int sweep_splits_for(const mcs_ctx* c, int n) {
  if (c->cfg.point_splits > 0) return c->cfg.point_splits;
  const long long ctas = ((long long)c->cfg.neighbor_count * n + kSweepThreads - 1) / kSweepThreads;
  long long p = (MCS_SPLIT_TARGET_CTAS + ctas - 1) / (ctas > 0 ? ctas : 1);
#if MCS_SPLIT_MIDRANGE
  // 500-7,000 item CTAs (25k-300k particles at 3 slots): three splits (4/4/2 of the ten
  // 448-point stages at S = 4,096) measured best — 25k 1.591 vs 1.616 ms with five, 50k 2.930
  // vs 2.954 with five, 100k (already 3) 5.63; 12.5k (293 CTAs) keeps five, 1M (23k CTAs) one
  if (ctas >= 500 && ctas < MCS_SPLIT_TARGET_CTAS && p > 3) p = 3;
#endif
  return (int)(p < 1 ? 1 : (p > 8 ? 8 : p));
}

void launch_sweep(mcs_ctx* c, int S) {
  const int n_items = c->cfg.neighbor_count * c->N;
  const int stages = (S + kChunkGeneral - 1) / kChunkGeneral;  // (an instantiation with fewer
  // stages than splits leaves the surplus splits' records zero)
  int P = sweep_splits_for(c, c->N);
  P = P > c->part_splits ? c->part_splits : P;
  P = P > stages ? stages : P;
#if MCS_SWEEP_TRIM_SPLITS
  {  // no split without a stage in the plane-form instantiation: P = ceil(stages / per split)
    const int sp = (S + kChunkPlane - 1) / kChunkPlane, per = (sp + P - 1) / P;
    P = (sp + per - 1) / per;
  }
#endif
#if MCS_SWEEP_REDUCE
  c->cur_splits = 1;  // reduce_splits_kernel sums the point splits into split 0's records
#else
  c->cur_splits = P;  // a3 sums the P records of every item itself
#endif
  const dim3 grid((n_items + kSweepThreads - 1) / kSweepThreads, P);
  const float inv_r = 1.0f / c->cfg.voxel_resolution;
  static_assert(!(MCS_SWEEP_TMA && MCS_SWEEP_GACC), "the TMA mbarriers follow s_acc");
  constexpr size_t smem = MCS_SWEEP_STATIC_SMEM ? 0 :
                          sizeof(float4) * (std::max(3 * (kChunkGeneral + 2),
                                                     2 * (kChunkPlane + 2))) *
                              (MCS_SWEEP_TMA ? 2 : 1) +
                          (MCS_SWEEP_GACC ? 0 : sizeof(double) * 28 * kSweepThreads) +
                          (MCS_SWEEP_TMA ? 32 : 0);
  const size_t pstride = (size_t)c->cfg.neighbor_count * c->capN;
  // opt in beyond 48 KB once per device (both instantiations); atomic flags: contexts may be
  // driven from several host threads (repeating the idempotent call is harmless)
  static std::atomic<bool> attr_set[128];
  if (c->dev < 0 || c->dev >= 128 || !attr_set[c->dev].load(std::memory_order_acquire)) {
    cudaFuncSetAttribute(sweep_kernel<MCS_CORR_CELL, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(sweep_kernel<MCS_CORR_CELL, false>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(sweep_kernel<MCS_CORR_NN27, false>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
#if MCS_SWEEP_CARVEOUT >= 0
    cudaFuncSetAttribute(sweep_kernel<MCS_CORR_CELL, true>,
                         cudaFuncAttributePreferredSharedMemoryCarveout, MCS_SWEEP_CARVEOUT);
#endif
    if (c->dev >= 0 && c->dev < 128) attr_set[c->dev].store(true, std::memory_order_release);
  }
  if (c->cfg.corr_mode == MCS_CORR_NN27) {
    const float nn_r2 = c->cfg.nn_radius * c->cfg.nn_radius;
    sweep_kernel<MCS_CORR_NN27, false><<<grid, kSweepThreads, smem, c->stream>>>(
        c->d_items, c->d_order, n_items, c->d_scan, S, c->d_kf_meta, inv_r, nn_r2, c->d_part,
        pstride, c->d_scan_np);
  } else {
    // the plane-form instantiation first: it is the one that runs on GICP scans (R36)
    sweep_kernel<MCS_CORR_CELL, true><<<grid, kSweepThreads, smem, c->stream>>>(
        c->d_items, c->d_order, n_items, c->d_scan_plane, S, c->d_kf_meta, inv_r, 0.f, c->d_part,
        pstride, c->d_scan_np);
    sweep_kernel<MCS_CORR_CELL, false><<<grid, kSweepThreads, smem, c->stream>>>(
        c->d_items, c->d_order, n_items, c->d_scan, S, c->d_kf_meta, inv_r, 0.f, c->d_part,
        pstride, c->d_scan_np);
  }
  if (P > 1 && MCS_SWEEP_REDUCE) {
    const long long tot = 29LL * n_items;
    reduce_splits_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, c->stream>>>(
        c->d_part, pstride, c->cfg.neighbor_count, c->N, c->capN, P);
  }
}

}  // namespace mcs
