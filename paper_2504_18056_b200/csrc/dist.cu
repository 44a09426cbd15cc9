// dist.cu — host-side plan of the multi-GPU exchange steps of a6.
//
// Particles are sharded into contiguous global index ranges.  After the weights (a5) every rank
// knows its survivor-ladder total Q_g and dead count D_g; an allgather of (Q_g, D_g) lets every
// rank evaluate the GLOBAL systematic-respawn count formula (R18) on its own survivors.  The
// r-th global clone (donors in ascending global index, with multiplicity) goes to the r-th
// global dead slot (ascending global index).  These functions are pure functions of the
// allgathered per-rank totals, so every rank computes the same plan.
#include <stdint.h>

#include "../../include/mcs.h"

namespace {

__int128 ceil_div(__int128 num, __int128 den) {  // den > 0
  __int128 q = num / den;
  if (num > 0 && q * den != num) q += 1;
  return q;
}

// n(c) = #{draws r in [0, D) : (r + U/2^32) Q / D < c}   (R18)
int64_t draws_below(unsigned __int128 c, int64_t D, unsigned __int128 Q, uint32_t U) {
  const __int128 num = (__int128)c * D * ((__int128)1 << 32) - (__int128)U * (__int128)Q;
  const __int128 den = (__int128)Q * ((__int128)1 << 32);
  __int128 v = ceil_div(num, den);
  if (v < 0) v = 0;
  if (v > D) v = D;
  return (int64_t)v;
}

}  // namespace

extern "C" {

mcs_status mcs_plan_ladder(int32_t world, const uint64_t* Q_per_rank, const int64_t* D_per_rank,
                           uint32_t u, uint64_t* q_offset, int64_t* d_offset,
                           int64_t* clones_per_rank, uint64_t* Q_total, int64_t* D_total) {
  if (world < 1 || !Q_per_rank || !D_per_rank) return MCS_E_INVALID_ARG;
  unsigned __int128 Q = 0;
  int64_t D = 0;
  for (int32_t g = 0; g < world; ++g) {
    if (D_per_rank[g] < 0) return MCS_E_INVALID_ARG;
    if (q_offset) q_offset[g] = (uint64_t)Q;
    if (d_offset) d_offset[g] = D;
    Q += Q_per_rank[g];
    D += D_per_rank[g];
  }
  if (Q >> 64) return MCS_E_CAPACITY;  // the exact ladder needs Q < 2^64 (R18)
  if (Q_total) *Q_total = (uint64_t)Q;
  if (D_total) *D_total = D;
  if (clones_per_rank) {
    unsigned __int128 c = 0;
    for (int32_t g = 0; g < world; ++g) {
      const unsigned __int128 c1 = c + Q_per_rank[g];
      clones_per_rank[g] = (D > 0 && Q > 0) ? draws_below(c1, D, Q, u) - draws_below(c, D, Q, u)
                                            : 0;
      c = c1;
    }
  }
  return (D > 0 && Q == 0) ? MCS_E_DEGENERATE : MCS_OK;
}

mcs_status mcs_plan_migration(int32_t world, const int64_t* clones_per_rank,
                              const int64_t* dead_per_rank, int64_t* send_counts) {
  if (world < 1 || !clones_per_rank || !dead_per_rank || !send_counts) return MCS_E_INVALID_ARG;
  int64_t tc = 0, td = 0;
  for (int32_t g = 0; g < world; ++g) {
    if (clones_per_rank[g] < 0 || dead_per_rank[g] < 0) return MCS_E_INVALID_ARG;
    tc += clones_per_rank[g];
    td += dead_per_rank[g];
  }
  if (tc != td) return MCS_E_INVALID_ARG;
  int64_t cs = 0;
  for (int32_t src = 0; src < world; ++src) {
    const int64_t c0 = cs, c1 = cs + clones_per_rank[src];
    int64_t ds = 0;
    for (int32_t dst = 0; dst < world; ++dst) {
      const int64_t d0 = ds, d1 = ds + dead_per_rank[dst];
      const int64_t lo = c0 > d0 ? c0 : d0, hi = c1 < d1 ? c1 : d1;
      send_counts[(size_t)src * world + dst] = hi > lo ? hi - lo : 0;
      ds = d1;
    }
    cs = c1;
  }
  return MCS_OK;
}

}  // extern "C"

// ======================================================================================
// Exchange layer: NCCL (dlopen'ed libnccl.so.2, collectives on the context stream) or a host
// transport (mcs_transport callbacks; small device buffers staged through pinned memory).
// ======================================================================================
#include <dlfcn.h>
#include <string.h>
#include <unistd.h>

#include <chrono>
#include <condition_variable>
#include <mutex>
#include <string>
#include <vector>

#include "mcs_internal.cuh"

namespace {

// minimal NCCL ABI (nccl.h 2.x), resolved at run time
typedef struct { char internal[128]; } NcclId;
typedef void* NcclComm;
enum { kNcclInt8 = 0, kNcclUint8 = 1, kNcclFloat64 = 8 };
enum { kNcclSum = 0, kNcclMax = 2 };
struct NcclApi {
  void* h = nullptr;
  int (*GetUniqueId)(NcclId*) = nullptr;
  int (*CommInitRank)(NcclComm*, int, NcclId, int) = nullptr;
  int (*CommDestroy)(NcclComm) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, NcclComm, cudaStream_t) = nullptr;
  int (*AllGather)(const void*, void*, size_t, int, NcclComm, cudaStream_t) = nullptr;
  int (*Send)(const void*, size_t, int, int, NcclComm, cudaStream_t) = nullptr;
  int (*Recv)(void*, size_t, int, int, NcclComm, cudaStream_t) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
};

// resolved once per process (a function-local static: thread-safe initialisation, so contexts
// created concurrently from several threads see one fully filled table)
static NcclApi load_nccl() {
  NcclApi api;
  {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return api;
    api.h = h;
#define SYM(f, n) api.f = reinterpret_cast<decltype(api.f)>(dlsym(h, n))
    SYM(GetUniqueId, "ncclGetUniqueId");
    SYM(CommInitRank, "ncclCommInitRank");
    SYM(CommDestroy, "ncclCommDestroy");
    SYM(AllReduce, "ncclAllReduce");
    SYM(AllGather, "ncclAllGather");
    SYM(Send, "ncclSend");
    SYM(Recv, "ncclRecv");
    SYM(GroupStart, "ncclGroupStart");
    SYM(GroupEnd, "ncclGroupEnd");
    SYM(GetErrorString, "ncclGetErrorString");
#undef SYM
    if (!api.GetUniqueId || !api.CommInitRank || !api.AllReduce || !api.AllGather || !api.Send ||
        !api.Recv || !api.GroupStart || !api.GroupEnd)
      api.h = nullptr;
  }
  return api;
}

NcclApi* nccl() {
  static NcclApi api = load_nccl();
  return api.h ? &api : nullptr;
}

// ---------------------------------------------------------------- in-process transport
struct Inproc {
  int world;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long long gen = 0;
  std::vector<const void*> in;        // per-rank input pointers of the current operation
  std::vector<const size_t*> in_sizes;
  mcs_transport t;

  bool barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const long long g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return true;
    }
    return cv.wait_for(lk, std::chrono::seconds(300), [&] { return gen != g; });
  }
};

int ip_allreduce(void* user, int32_t rank, void* buf, int32_t n, int32_t dtype, int32_t op) {
  Inproc* P = static_cast<Inproc*>(user);
  const size_t esz = 8;
  std::vector<char> mine((char*)buf, (char*)buf + esz * n);
  P->in[rank] = mine.data();
  if (!P->barrier()) return 1;
  for (int32_t k = 0; k < n; ++k) {  // rank order: deterministic
    if (dtype == 0) {
      double acc = reinterpret_cast<const double*>(P->in[0])[k];
      for (int g = 1; g < P->world; ++g) {
        const double v = reinterpret_cast<const double*>(P->in[g])[k];
        acc = op == 0 ? acc + v : (v > acc ? v : acc);
      }
      reinterpret_cast<double*>(buf)[k] = acc;
    } else {
      long long acc = reinterpret_cast<const long long*>(P->in[0])[k];
      for (int g = 1; g < P->world; ++g) {
        const long long v = reinterpret_cast<const long long*>(P->in[g])[k];
        acc = op == 0 ? acc + v : (v > acc ? v : acc);
      }
      reinterpret_cast<long long*>(buf)[k] = acc;
    }
  }
  return P->barrier() ? 0 : 1;
}

int ip_allgather(void* user, int32_t rank, const void* send, void* recv, size_t bytes) {
  Inproc* P = static_cast<Inproc*>(user);
  P->in[rank] = send;
  if (!P->barrier()) return 1;
  for (int g = 0; g < P->world; ++g) memcpy((char*)recv + g * bytes, P->in[g], bytes);
  return P->barrier() ? 0 : 1;
}

int ip_alltoallv(void* user, int32_t rank, const void* const* send, const size_t* send_bytes,
                 void* const* recv, const size_t* recv_bytes) {
  Inproc* P = static_cast<Inproc*>(user);
  P->in[rank] = send;
  P->in_sizes[rank] = send_bytes;
  if (!P->barrier()) return 1;
  for (int g = 0; g < P->world; ++g) {
    const void* const* theirs = reinterpret_cast<const void* const*>(P->in[g]);
    const size_t nb = P->in_sizes[g][rank];
    if (nb != recv_bytes[g]) return 2;
    if (nb) memcpy(recv[g], theirs[rank], nb);
  }
  return P->barrier() ? 0 : 1;
}

}  // namespace

extern "C" {

mcs_status mcs_nccl_unique_id(void* out128) {
  NcclApi* a = nccl();
  if (!a || !out128) return MCS_E_NCCL;
  NcclId id;
  if (a->GetUniqueId(&id) != 0) return MCS_E_NCCL;
  memcpy(out128, &id, sizeof(id));
  return MCS_OK;
}

mcs_transport* mcs_inproc_transport_create(int32_t world) {
  if (world < 1) return nullptr;
  Inproc* P = new Inproc();
  P->world = world;
  P->in.assign(world, nullptr);
  P->in_sizes.assign(world, nullptr);
  P->t.user = P;
  P->t.allreduce = ip_allreduce;
  P->t.allgather = ip_allgather;
  P->t.alltoallv = ip_alltoallv;
  return &P->t;
}

void mcs_inproc_transport_destroy(mcs_transport* t) {
  if (t) delete static_cast<Inproc*>(t->user);
}

}  // extern "C"

namespace mcs {

mcs_status dist_init(mcs_ctx* c, std::string& err) {
  c->world = c->cfg.world_size;
  c->rank = c->cfg.rank;
  // world_size 1 with a transport or an NCCL id still runs the exchange path (tests of it)
  if (c->world == 1 && !c->cfg.transport && !c->cfg.nccl_unique_id) return MCS_OK;
  if (c->cfg.transport) {
    c->tr = c->cfg.transport;
    return MCS_OK;
  }
  NcclApi* a = nccl();
  if (!a) {
    err = "world_size > 1 needs libnccl.so.2 (dlopen failed) or a host transport";
    return MCS_E_NCCL;
  }
  NcclId id;
  memcpy(&id, c->cfg.nccl_unique_id, sizeof(id));
  NcclComm comm = nullptr;
  const int r = a->CommInitRank(&comm, c->world, id, c->rank);
  if (r != 0) {
    err = std::string("ncclCommInitRank: ") + (a->GetErrorString ? a->GetErrorString(r) : "?");
    return MCS_E_NCCL;
  }
  c->nccl_comm = comm;
  return MCS_OK;
}

void dist_destroy(mcs_ctx* c) {
  for (void* p : c->ipc_opened) cudaIpcCloseMemHandle(p);
  c->ipc_opened.clear();
  if (c->d_peers) cudaFree(c->d_peers);
  c->d_peers = nullptr;
  if (c->d_ag) mem_free(c, c->d_ag);
  c->d_ag = nullptr;
  c->d_ag_bytes = 0;
  if (c->nccl_comm) {
    NcclApi* a = nccl();
    if (a && a->CommDestroy) a->CommDestroy(c->nccl_comm);
    c->nccl_comm = nullptr;
  }
}

static mcs_status stage(mcs_ctx* c, size_t bytes) {
  if (c->h_stage_bytes >= bytes) return MCS_OK;
  if (c->h_stage) cudaFreeHost(c->h_stage);
  c->h_stage = nullptr;
  c->h_stage_bytes = 0;
  if (cudaMallocHost(&c->h_stage, bytes) != cudaSuccess) return MCS_E_OUT_OF_MEMORY;
  c->h_stage_bytes = bytes;
  return MCS_OK;
}

bool dist_active(const mcs_ctx* c) { return c->world > 1 || c->tr || c->nccl_comm; }

mcs_status dist_allreduce_f64(mcs_ctx* c, double* d_buf, int n, int op) {
  if (!dist_active(c)) return MCS_OK;
  if (c->nccl_comm) {
    NcclApi* a = nccl();
    return a->AllReduce(d_buf, d_buf, n, kNcclFloat64, op ? kNcclMax : kNcclSum, c->nccl_comm,
                        c->stream) == 0 ? MCS_OK : MCS_E_NCCL;
  }
  if (stage(c, 8 * n) != MCS_OK) return MCS_E_OUT_OF_MEMORY;
  if (cudaMemcpyAsync(c->h_stage, d_buf, 8 * n, cudaMemcpyDeviceToHost, c->stream) != cudaSuccess ||
      cudaStreamSynchronize(c->stream) != cudaSuccess)
    return MCS_E_CUDA;
  if (c->tr->allreduce(c->tr->user, c->rank, c->h_stage, n, 0, op)) return MCS_E_NCCL;
  if (cudaMemcpyAsync(d_buf, c->h_stage, 8 * n, cudaMemcpyHostToDevice, c->stream) != cudaSuccess ||
      cudaStreamSynchronize(c->stream) != cudaSuccess)
    return MCS_E_CUDA;
  return MCS_OK;
}

mcs_status dist_allgather_host(mcs_ctx* c, const void* send, void* recv, size_t bytes) {
  if (!dist_active(c)) {
    memcpy(recv, send, bytes);
    return MCS_OK;
  }
  if (c->nccl_comm) {
    NcclApi* a = nccl();
    const size_t need = bytes * (c->world + 1);
    if (c->d_ag_bytes < need) {  // persistent scratch: no allocation on the per-update path
      mem_free(c, c->d_ag);
      c->d_ag = nullptr;
      c->d_ag_bytes = 0;
      if (mem_alloc(c, (void**)&c->d_ag, need) != cudaSuccess) return MCS_E_OUT_OF_MEMORY;
      c->d_ag_bytes = need;
    }
    char* d = c->d_ag;
    mcs_status st = MCS_OK;
    if (cudaMemcpyAsync(d, send, bytes, cudaMemcpyHostToDevice, c->stream) != cudaSuccess)
      st = MCS_E_CUDA;
    if (st == MCS_OK &&
        a->AllGather(d, d + bytes, bytes, kNcclUint8, c->nccl_comm, c->stream) != 0)
      st = MCS_E_NCCL;
    if (st == MCS_OK && (cudaMemcpyAsync(recv, d + bytes, bytes * c->world, cudaMemcpyDeviceToHost,
                                         c->stream) != cudaSuccess ||
                         cudaStreamSynchronize(c->stream) != cudaSuccess))
      st = MCS_E_CUDA;
    return st;
  }
  return c->tr->allgather(c->tr->user, c->rank, send, recv, bytes) ? MCS_E_NCCL : MCS_OK;
}

mcs_status dist_allgather_dev(mcs_ctx* c, const void* d_send, void* d_recv, size_t bytes) {
  if (!dist_active(c)) {
    return cudaMemcpyAsync(d_recv, d_send, bytes, cudaMemcpyDeviceToDevice, c->stream) ==
                   cudaSuccess ? MCS_OK : MCS_E_CUDA;
  }
  if (c->nccl_comm) {
    NcclApi* a = nccl();
    return a->AllGather(d_send, d_recv, bytes, kNcclUint8, c->nccl_comm, c->stream) == 0
               ? MCS_OK : MCS_E_NCCL;
  }
  const size_t tot = bytes * (c->world + 1);
  if (stage(c, tot) != MCS_OK) return MCS_E_OUT_OF_MEMORY;
  char* h = (char*)c->h_stage;
  if (cudaMemcpyAsync(h, d_send, bytes, cudaMemcpyDeviceToHost, c->stream) != cudaSuccess ||
      cudaStreamSynchronize(c->stream) != cudaSuccess)
    return MCS_E_CUDA;
  if (c->tr->allgather(c->tr->user, c->rank, h, h + bytes, bytes)) return MCS_E_NCCL;
  if (cudaMemcpyAsync(d_recv, h + bytes, bytes * c->world, cudaMemcpyHostToDevice, c->stream) !=
          cudaSuccess ||
      cudaStreamSynchronize(c->stream) != cudaSuccess)
    return MCS_E_CUDA;
  return MCS_OK;
}

mcs_status dist_barrier(mcs_ctx* c) {
  if (!dist_active(c)) return MCS_OK;
  if (c->nccl_comm) {  // a 1-element allreduce: later work on this stream waits for every rank
    if (c->d_ag_bytes < 8) {
      mem_free(c, c->d_ag);
      c->d_ag = nullptr;
      c->d_ag_bytes = 0;
      if (mem_alloc(c, (void**)&c->d_ag, 64) != cudaSuccess) return MCS_E_OUT_OF_MEMORY;
      c->d_ag_bytes = 64;
    }
    NcclApi* a = nccl();
    return a->AllReduce(c->d_ag, c->d_ag, 1, kNcclFloat64, kNcclMax, c->nccl_comm, c->stream) == 0
               ? MCS_OK : MCS_E_NCCL;
  }
  if (cudaStreamSynchronize(c->stream) != cudaSuccess) return MCS_E_CUDA;
  double z = 0.0;
  return c->tr->allreduce(c->tr->user, c->rank, &z, 1, 0, 1) ? MCS_E_NCCL : MCS_OK;
}

namespace {
struct PeerInfo {  // what a rank publishes about its state buffers
  int32_t pid, dev, capN, capK, ipc_ok, pad;
  uint64_t ptr[6];                 // pose, kfpose, L, dead_list, donor_g, kft
  cudaIpcMemHandle_t handle[6];
};
}  // namespace

mcs_status dist_peer_setup(mcs_ctx* c) {
  if (c->p2p != 0) return MCS_OK;
  c->p2p = -1;
  if (!dist_active(c) || !c->cfg.peer_migration) return MCS_OK;
  const int G = c->world;
  PeerInfo me;
  memset(&me, 0, sizeof(me));
  me.pid = (int32_t)getpid();
  me.dev = c->dev;
  me.capN = c->capN;
  me.capK = c->capK;
  void* mine[6] = {c->d_pose, c->d_kfpose, c->d_L, c->d_dead_list, c->d_donor_g, c->d_kft};
  // CUDA IPC needs whole cudaMalloc allocations: not available under a user allocator
  me.ipc_ok = c->alloc.alloc ? 0 : 1;
  for (int k = 0; k < 6; ++k) {
    me.ptr[k] = (uint64_t)(uintptr_t)mine[k];
    if (me.ipc_ok && cudaIpcGetMemHandle(&me.handle[k], mine[k]) != cudaSuccess) me.ipc_ok = 0;
  }
  cudaGetLastError();
  std::vector<PeerInfo> all(G);
  MCS_TRY(dist_allgather_host(c, &me, all.data(), sizeof(PeerInfo)));
  std::vector<PeerView> views(G);
  int32_t ok = 1;
  std::vector<void*> opened;
  for (int p = 0; p < G && ok; ++p) {
    const PeerInfo& q = all[p];
    void* ptr[6];
    if (q.pid == me.pid) {  // same process: raw pointers (peer access if another device)
      for (int k = 0; k < 6; ++k) ptr[k] = (void*)(uintptr_t)q.ptr[k];
      if (q.dev != c->dev) {
        int can = 0;
        if (cudaDeviceCanAccessPeer(&can, c->dev, q.dev) != cudaSuccess || !can) {
          ok = 0;
          break;
        }
        const cudaError_t e = cudaDeviceEnablePeerAccess(q.dev, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) ok = 0;
        cudaGetLastError();
      }
    } else {
      if (!q.ipc_ok) {
        ok = 0;
        break;
      }
      for (int k = 0; k < 6 && ok; ++k) {
        if (cudaIpcOpenMemHandle(&ptr[k], q.handle[k], cudaIpcMemLazyEnablePeerAccess) !=
            cudaSuccess) {
          ok = 0;
          cudaGetLastError();
        } else {
          opened.push_back(ptr[k]);
        }
      }
    }
    if (!ok) break;
    views[p] = PeerView{(float*)ptr[0], (float*)ptr[1], (float4*)ptr[5], (double*)ptr[2],
                        (int32_t*)ptr[3], (int32_t*)ptr[4], q.capN, q.capK};
  }
  // every rank must agree (one failed open anywhere -> all use the transport path)
  std::vector<int32_t> oks(G);
  MCS_TRY(dist_allgather_host(c, &ok, oks.data(), sizeof(int32_t)));
  for (int p = 0; p < G; ++p) ok &= oks[p];
  if (!ok) {
    for (void* p : opened) cudaIpcCloseMemHandle(p);
    return MCS_OK;
  }
  c->ipc_opened = opened;
  if (cudaMalloc(&c->d_peers, sizeof(PeerView) * G) != cudaSuccess) return MCS_E_OUT_OF_MEMORY;
  if (cudaMemcpy(c->d_peers, views.data(), sizeof(PeerView) * G, cudaMemcpyHostToDevice) !=
      cudaSuccess)
    return MCS_E_CUDA;
  c->p2p = 1;
  return MCS_OK;
}

mcs_status dist_alltoallv(mcs_ctx* c, const float* d_send, const size_t* send_bytes,
                          const size_t* send_off, float* d_recv, const size_t* recv_bytes,
                          const size_t* recv_off) {
  if (!dist_active(c)) return MCS_OK;
  const int G = c->world;
  if (c->nccl_comm) {
    NcclApi* a = nccl();
    if (a->GroupStart() != 0) return MCS_E_NCCL;
    bool ok = true;  // the group is always closed, even after a failed enqueue
    for (int p = 0; p < G && ok; ++p) {
      if (p == c->rank) continue;
      if (send_bytes[p] &&
          a->Send((const char*)d_send + send_off[p], send_bytes[p], kNcclUint8, p, c->nccl_comm,
                  c->stream) != 0)
        ok = false;
      if (ok && recv_bytes[p] &&
          a->Recv((char*)d_recv + recv_off[p], recv_bytes[p], kNcclUint8, p, c->nccl_comm,
                  c->stream) != 0)
        ok = false;
    }
    const bool closed = a->GroupEnd() == 0;
    return (ok && closed) ? MCS_OK : MCS_E_NCCL;
  }
  size_t ts = send_off[G], tr = recv_off[G];
  if (stage(c, ts + tr + 16) != MCS_OK) return MCS_E_OUT_OF_MEMORY;
  char* hs = (char*)c->h_stage;
  char* hr = hs + ts;
  if ((ts && cudaMemcpyAsync(hs, d_send, ts, cudaMemcpyDeviceToHost, c->stream) != cudaSuccess) ||
      cudaStreamSynchronize(c->stream) != cudaSuccess)
    return MCS_E_CUDA;
  std::vector<const void*> sp(G);
  std::vector<void*> rp(G);
  for (int p = 0; p < G; ++p) {
    sp[p] = hs + send_off[p];
    rp[p] = hr + recv_off[p];
  }
  if (c->tr->alltoallv(c->tr->user, c->rank, sp.data(), send_bytes, rp.data(), recv_bytes))
    return MCS_E_NCCL;
  if ((tr && cudaMemcpyAsync(d_recv, hr, tr, cudaMemcpyHostToDevice, c->stream) != cudaSuccess) ||
      cudaStreamSynchronize(c->stream) != cudaSuccess)
    return MCS_E_CUDA;
  return MCS_OK;
}

}  // namespace mcs
