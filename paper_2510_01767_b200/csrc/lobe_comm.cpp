// lobe_comm.cpp -- multi-rank exchange and communicators.
// See lobe_comm.h for the choreography; this file holds its one
// implementation, the three XOps memory spaces and the NCCL loader.
//
// NCCL is resolved at run time (dlopen / dlsym; nccl.h supplies only the
// types): a process that already loaded libnccl.so.2 (torch does) shares that
// copy, otherwise the system library is loaded on the first NCCL scene. A
// library without NCCL still loads and runs every world = 1 or host-comm path.
#include "lobe_comm.h"

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <tuple>
#include <vector>

#include "lobe_internal.h"

namespace lobe {

// ============================================================================
// the choreography (written once; memory space and transport come from XOps)
// ============================================================================
namespace {
struct Scratch {  // RAII over XOps::alloc
  XOps& x;
  std::vector<void*> ps;
  explicit Scratch(XOps& o) : x(o) {}
  ~Scratch() {
    for (void* p : ps) x.release(p);
  }
  template <class T>
  lobe_status get(T** p, size_t count, bool zero = false) {
    void* q = nullptr;
    lobe_status st = x.alloc(&q, std::max<size_t>(count, 1) * sizeof(T));
    if (st != LOBE_OK) return st;
    ps.push_back(q);
    *p = static_cast<T*>(q);
    if (zero) return x.zero(q, std::max<size_t>(count, 1) * sizeof(T));
    return LOBE_OK;
  }
};
#define XT(expr)                            \
  do {                                      \
    const lobe_status st_ = (expr);         \
    if (st_ != LOBE_OK) return st_;         \
  } while (0)
}  // namespace

lobe_status xchg_block_loads(XOps& x, int rank, int world, int B, size_t words, const uint32_t* partial,
                             uint64_t* counts, uint32_t* own, uint32_t* g_vis_host, uint64_t* counts_host) {
  const int W = world, r = rank;
  std::vector<int> nb(W), b0(W);
  int P = 0;
  for (int j = 0; j < W; ++j) {
    b0[j] = (int)shard_begin(B, j, W);
    nb[j] = (int)shard_begin(B, j + 1, W) - b0[j];
    P = std::max(P, nb[j]);
  }
  const size_t wb = words * sizeof(uint32_t);
  Scratch S(x);
  // 1. reduce-scatter by owned blocks: partial masks of rank j's blocks go to j
  uint32_t* recv = nullptr;
  XT(S.get(&recv, (size_t)W * nb[r] * words));
  std::vector<size_t> sb(W), so(W), rb(W), ro(W);
  for (int j = 0; j < W; ++j) {
    sb[j] = (size_t)nb[j] * wb;
    so[j] = (size_t)b0[j] * wb;
    rb[j] = (size_t)nb[r] * wb;
    ro[j] = (size_t)j * nb[r] * wb;
  }
  XT(x.all_to_all_v(partial, sb.data(), so.data(), recv, rb.data(), ro.data()));
  // 2. OR of the W partials of the own blocks + popcount
  uint32_t *gv = nullptr, *gv_all = nullptr;
  XT(S.get(&gv, (size_t)P, true));
  if (nb[r] > 0) XT(x.or_combine(recv, W, nb[r], words, own, gv));
  // 3. G_vis of every block, |C^(b)| and I_b
  XT(S.get(&gv_all, (size_t)W * P));
  XT(x.all_gather(gv, gv_all, (size_t)P * sizeof(uint32_t)));
  XT(x.all_reduce_u64(counts, 2 * (size_t)B));
  std::vector<uint32_t> h((size_t)W * P);
  XT(x.to_host(h.data(), gv_all, h.size() * sizeof(uint32_t)));
  for (int j = 0; j < W; ++j)
    for (int k = 0; k < nb[j]; ++k) g_vis_host[b0[j] + k] = h[(size_t)j * P + k];
  XT(x.to_host(counts_host, counts, 2 * (size_t)B * sizeof(uint64_t)));
  return LOBE_OK;
}

lobe_status xchg_all_masks(XOps& x, int rank, int world, int B, size_t words, const uint32_t* own, uint32_t* all) {
  const int W = world, r = rank;
  std::vector<int> nb(W), b0(W);
  int P = 0;
  for (int j = 0; j < W; ++j) {
    b0[j] = (int)shard_begin(B, j, W);
    nb[j] = (int)shard_begin(B, j + 1, W) - b0[j];
    P = std::max(P, nb[j]);
  }
  if (P == 0) return LOBE_OK;
  const size_t wb = words * sizeof(uint32_t);
  Scratch S(x);
  uint32_t *send = nullptr, *recv = nullptr;
  XT(S.get(&send, (size_t)P * words, true));  // own blocks, padded to the largest share
  if (nb[r] > 0) XT(x.copy(send, own, (size_t)nb[r] * wb));
  XT(S.get(&recv, (size_t)W * P * words));
  XT(x.all_gather(send, recv, (size_t)P * wb));
  for (int j = 0; j < W; ++j)
    if (nb[j] > 0) XT(x.copy(all + (size_t)b0[j] * words, recv + (size_t)j * P * words, (size_t)nb[j] * wb));
  return LOBE_OK;
}

lobe_status xchg_gather_cameras(XOps& x, int rank, int world, int64_t N, size_t elem, const void* local, void* out) {
  const int W = world, r = rank;
  int64_t P = 0;
  for (int j = 0; j < W; ++j) P = std::max(P, shard_begin(N, j + 1, W) - shard_begin(N, j, W));
  if (P == 0) return LOBE_OK;
  const int64_t n_r = shard_begin(N, r + 1, W) - shard_begin(N, r, W);
  Scratch S(x);
  uint8_t *send = nullptr, *recv = nullptr;
  XT(S.get(&send, (size_t)P * elem, true));
  if (n_r > 0) XT(x.copy(send, local, (size_t)n_r * elem));
  XT(S.get(&recv, (size_t)W * P * elem));
  XT(x.all_gather(send, recv, (size_t)P * elem));
  uint8_t* o = static_cast<uint8_t*>(out);
  for (int j = 0; j < W; ++j) {
    const int64_t c0 = shard_begin(N, j, W), n_j = shard_begin(N, j + 1, W) - c0;
    if (n_j > 0) XT(x.copy(o + (size_t)c0 * elem, recv + (size_t)j * P * elem, (size_t)n_j * elem));
  }
  return LOBE_OK;
}

// ============================================================================
// NCCL (run-time loaded)
// ============================================================================
namespace {
struct NcclApi {
  void* handle = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  std::string why;
};

NcclApi* nccl_api() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* env = std::getenv("LOBE_NCCL_LIB");
    void* h = nullptr;
    // prefer a copy the process already has (torch's), then the loader's search path
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      if (!h) h = dlopen(name, RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
    }
    if (!h && env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.why = std::string("cannot load libnccl.so.2: ") + (dlerror() ? dlerror() : "?");
      return;
    }
    api.handle = h;
#define LOBE_SYM(field, name)                                                 \
  api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name));          \
  if (!api.field) {                                                           \
    api.why = std::string("libnccl lacks ") + name;                           \
    api.handle = nullptr;                                                     \
    return;                                                                   \
  }
    LOBE_SYM(GetUniqueId, "ncclGetUniqueId");
    LOBE_SYM(CommInitRank, "ncclCommInitRank");
    LOBE_SYM(CommDestroy, "ncclCommDestroy");
    LOBE_SYM(AllGather, "ncclAllGather");
    LOBE_SYM(AllReduce, "ncclAllReduce");
    LOBE_SYM(Send, "ncclSend");
    LOBE_SYM(Recv, "ncclRecv");
    LOBE_SYM(GroupStart, "ncclGroupStart");
    LOBE_SYM(GroupEnd, "ncclGroupEnd");
    LOBE_SYM(GetErrorString, "ncclGetErrorString");
#undef LOBE_SYM
  });
  return api.handle ? &api : nullptr;
}

std::string nccl_msg(const char* what, ncclResult_t r) {
  NcclApi* a = nccl_api();
  return std::string(what) + ": " + (a ? a->GetErrorString(r) : "nccl unavailable");
}
}  // namespace

struct Comm {
  int kind = 0;  // 1 NCCL, 2 host callbacks
  int rank = 0, world = 1, device = 0;
  ncclComm_t nccl = nullptr;
  lobe_host_comm host{};
};

namespace {
std::mutex g_comm_mu;
// NCCL communicators live for the process (creation is collective and costs
// ~0.1 s; every scene of a run with the same unique id reuses one)
std::map<std::tuple<std::string, int, int, int>, std::unique_ptr<Comm>> g_nccl_comms;
}  // namespace

lobe_status comm_acquire(const lobe_options& o, Comm** out, std::string* err) {
  *out = nullptr;
  if (o.nccl_unique_id && o.host_comm) {
    *err = "give either nccl_unique_id or host_comm";
    return LOBE_E_INVALID_CONFIG;
  }
  if (o.host_comm) {
    const lobe_host_comm& h = *o.host_comm;
    if (!h.all_gather || !h.all_reduce_u64 || !h.all_to_all_v) {
      *err = "host_comm: every callback must be set";
      return LOBE_E_INVALID_CONFIG;
    }
    Comm* c = new Comm();
    c->kind = 2;
    c->rank = o.rank;
    c->world = o.world;
    c->device = o.device;
    c->host = h;
    *out = c;  // owned by the scene
    return LOBE_OK;
  }
  if (!o.nccl_unique_id) return LOBE_OK;  // no communicator
  NcclApi* api = nccl_api();
  if (!api) {
    *err = "NCCL unavailable";
    return LOBE_E_NCCL;
  }
  const std::string key(static_cast<const char*>(o.nccl_unique_id), sizeof(ncclUniqueId));
  std::lock_guard<std::mutex> lk(g_comm_mu);
  auto k = std::make_tuple(key, o.rank, o.world, o.device);
  auto it = g_nccl_comms.find(k);
  if (it == g_nccl_comms.end()) {
    std::unique_ptr<Comm> c(new Comm());
    c->kind = 1;
    c->rank = o.rank;
    c->world = o.world;
    c->device = o.device;
    ncclUniqueId id;
    std::memcpy(&id, o.nccl_unique_id, sizeof(id));
    if (cudaSetDevice(o.device) != cudaSuccess) {
      *err = "cudaSetDevice";
      return LOBE_E_CUDA;
    }
    const ncclResult_t r = api->CommInitRank(&c->nccl, o.world, id, o.rank);
    if (r != ncclSuccess) {
      *err = nccl_msg("ncclCommInitRank", r);
      return LOBE_E_NCCL;
    }
    it = g_nccl_comms.emplace(k, std::move(c)).first;
  }
  *out = it->second.get();
  return LOBE_OK;
}

bool comm_is_nccl(const Comm* c) { return c && c->kind == 1; }

void comm_release_scene(Comm* c) {
  if (c && c->kind == 2) delete c;  // NCCL comms stay cached (lobe_release_comms)
}

// ============================================================================
// XOps: device memory (NCCL on the stream, or host-staged callbacks)
// ============================================================================
namespace {
struct DeviceOps : XOps {
  Comm* c;
  cudaStream_t st;
  explicit DeviceOps(Comm* cm, cudaStream_t s) : c(cm), st(s) {}
  lobe_status cuda(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return LOBE_OK;
    err = std::string(what) + ": " + cudaGetErrorString(e);
    return LOBE_E_CUDA;
  }
  lobe_status nccl(ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return LOBE_OK;
    err = nccl_msg(what, r);
    return LOBE_E_NCCL;
  }
  lobe_status alloc(void** p, size_t bytes) override { return cuda(cudaMallocAsync(p, bytes, st), "alloc"); }
  void release(void* p) override {
    if (p) cudaFreeAsync(p, st);
  }
  lobe_status copy(void* d, const void* s, size_t b) override {
    return b ? cuda(cudaMemcpyAsync(d, s, b, cudaMemcpyDeviceToDevice, st), "copy") : LOBE_OK;
  }
  lobe_status zero(void* p, size_t b) override { return cuda(cudaMemsetAsync(p, 0, b, st), "memset"); }
  lobe_status or_combine(const uint32_t* g, int W, int nb, size_t words, uint32_t* out, uint32_t* gvis) override {
    return cuda(launch_masks_combine(g, W, nb, (int64_t)words, out, gvis, st), "k_masks_combine");
  }
  lobe_status to_host(void* d, const void* s, size_t b) override {
    if (!b) return LOBE_OK;
    XT(cuda(cudaMemcpyAsync(d, s, b, cudaMemcpyDeviceToHost, st), "d2h"));
    return cuda(cudaStreamSynchronize(st), "sync");
  }
  // ---- transport
  lobe_status all_to_all_v(const void* send, const size_t* sb, const size_t* so, void* recv, const size_t* rb,
                           const size_t* ro) override {
    const uint8_t* s8 = static_cast<const uint8_t*>(send);
    uint8_t* r8 = static_cast<uint8_t*>(recv);
    const int r = c->rank;
    if (rb[r] != sb[r]) {
      err = "all_to_all_v: self sizes differ";
      return LOBE_E_STATE;
    }
    XT(copy(r8 + ro[r], s8 + so[r], sb[r]));  // own part: a local copy
    if (c->world == 1) return LOBE_OK;
    if (c->kind == 1) {
      NcclApi* a = nccl_api();
      XT(nccl(a->GroupStart(), "ncclGroupStart"));
      for (int j = 0; j < c->world; ++j) {
        if (j == r) continue;
        if (sb[j]) XT(nccl(a->Send(s8 + so[j], sb[j], ncclUint8, j, c->nccl, st), "ncclSend"));
        if (rb[j]) XT(nccl(a->Recv(r8 + ro[j], rb[j], ncclUint8, j, c->nccl, st), "ncclRecv"));
      }
      return nccl(a->GroupEnd(), "ncclGroupEnd");
    }
    // host-staged: whole send buffer down, callbacks, received parts up
    size_t stot = 0, rtot = 0;
    for (int j = 0; j < c->world; ++j) {
      stot = std::max(stot, so[j] + sb[j]);
      rtot = std::max(rtot, ro[j] + rb[j]);
    }
    std::vector<uint8_t> hs(std::max<size_t>(stot, 1)), hr(std::max<size_t>(rtot, 1));
    XT(to_host(hs.data(), send, stot));
    if (c->host.all_to_all_v(c->host.ctx, hs.data(), sb, so, hr.data(), rb, ro) != 0) {
      err = "host_comm all_to_all_v failed";
      return LOBE_E_NCCL;
    }
    for (int j = 0; j < c->world; ++j)
      if (j != r && rb[j])
        XT(cuda(cudaMemcpyAsync(r8 + ro[j], hr.data() + ro[j], rb[j], cudaMemcpyHostToDevice, st), "h2d"));
    return cuda(cudaStreamSynchronize(st), "sync");  // hr is freed on return
  }
  lobe_status all_gather(const void* send, void* recv, size_t bytes) override {
    if (c->kind == 1) return nccl(nccl_api()->AllGather(send, recv, bytes, ncclUint8, c->nccl, st), "ncclAllGather");
    std::vector<uint8_t> hs(std::max<size_t>(bytes, 1)), hr(std::max<size_t>(bytes * c->world, 1));
    XT(to_host(hs.data(), send, bytes));
    if (c->host.all_gather(c->host.ctx, hs.data(), hr.data(), bytes) != 0) {
      err = "host_comm all_gather failed";
      return LOBE_E_NCCL;
    }
    XT(cuda(cudaMemcpyAsync(recv, hr.data(), bytes * c->world, cudaMemcpyHostToDevice, st), "h2d"));
    return cuda(cudaStreamSynchronize(st), "sync");
  }
  lobe_status all_reduce_u64(uint64_t* buf, size_t n) override {
    if (c->kind == 1)
      return nccl(nccl_api()->AllReduce(buf, buf, n, ncclUint64, ncclSum, c->nccl, st), "ncclAllReduce");
    std::vector<uint64_t> h(std::max<size_t>(n, 1));
    XT(to_host(h.data(), buf, n * 8));
    if (c->host.all_reduce_u64(c->host.ctx, h.data(), n) != 0) {
      err = "host_comm all_reduce_u64 failed";
      return LOBE_E_NCCL;
    }
    XT(cuda(cudaMemcpyAsync(buf, h.data(), n * 8, cudaMemcpyHostToDevice, st), "h2d"));
    return cuda(cudaStreamSynchronize(st), "sync");
  }
};

// host memory + host callbacks (no GPU): the CPU tests' path
struct HostOps : XOps {
  lobe_host_comm h;
  int rank, world;
  HostOps(const lobe_host_comm& hc, int r, int w) : h(hc), rank(r), world(w) {}
  lobe_status alloc(void** p, size_t b) override {
    *p = std::malloc(std::max<size_t>(b, 1));
    if (!*p) {
      err = "malloc";
      return LOBE_E_OOM;
    }
    return LOBE_OK;
  }
  void release(void* p) override { std::free(p); }
  lobe_status copy(void* d, const void* s, size_t b) override {
    if (b) std::memmove(d, s, b);
    return LOBE_OK;
  }
  lobe_status zero(void* p, size_t b) override {
    std::memset(p, 0, b);
    return LOBE_OK;
  }
  lobe_status or_combine(const uint32_t* g, int W, int nb, size_t words, uint32_t* out, uint32_t* gvis) override {
    for (int k = 0; k < nb; ++k) {
      uint32_t cnt = 0;
      for (size_t w = 0; w < words; ++w) {
        uint32_t m = 0;
        for (int r = 0; r < W; ++r) m |= g[((size_t)r * nb + k) * words + w];
        out[(size_t)k * words + w] = m;
        cnt += (uint32_t)__builtin_popcount(m);
      }
      gvis[k] += cnt;
    }
    return LOBE_OK;
  }
  lobe_status to_host(void* d, const void* s, size_t b) override { return copy(d, s, b); }
  lobe_status all_to_all_v(const void* send, const size_t* sb, const size_t* so, void* recv, const size_t* rb,
                           const size_t* ro) override {
    if (h.all_to_all_v(h.ctx, send, sb, so, recv, rb, ro) != 0) {
      err = "host_comm all_to_all_v failed";
      return LOBE_E_NCCL;
    }
    return LOBE_OK;
  }
  lobe_status all_gather(const void* send, void* recv, size_t bytes) override {
    if (h.all_gather(h.ctx, send, recv, bytes) != 0) {
      err = "host_comm all_gather failed";
      return LOBE_E_NCCL;
    }
    return LOBE_OK;
  }
  lobe_status all_reduce_u64(uint64_t* buf, size_t n) override {
    if (h.all_reduce_u64(h.ctx, buf, n) != 0) {
      err = "host_comm all_reduce_u64 failed";
      return LOBE_E_NCCL;
    }
    return LOBE_OK;
  }
};
}  // namespace

XOps* comm_device_ops(Comm* c, int device, cudaStream_t st) {
  (void)device;
  return new DeviceOps(c, st);
}

}  // namespace lobe

// ============================================================================
// exports
// ============================================================================
extern "C" {

lobe_status lobe_nccl_unique_id(void* out) {
  if (!out) return LOBE_E_INVALID_CONFIG;
  lobe::NcclApi* a = lobe::nccl_api();
  if (!a) return LOBE_E_NCCL;
  ncclUniqueId id;
  if (a->GetUniqueId(&id) != ncclSuccess) return LOBE_E_NCCL;
  std::memcpy(out, &id, sizeof(id));
  return LOBE_OK;
}

void lobe_release_comms(void) {
  std::lock_guard<std::mutex> lk(lobe::g_comm_mu);
  lobe::NcclApi* a = lobe::nccl_api();
  for (auto& kv : lobe::g_nccl_comms)
    if (a && kv.second->nccl) a->CommDestroy(kv.second->nccl);
  lobe::g_nccl_comms.clear();
}

lobe_status lobe_xchg_block_loads_host(const lobe_host_comm* hc, int32_t rank, int32_t world, int32_t B,
                                       size_t words, const uint32_t* partial, const uint64_t* counts_local,
                                       uint32_t* own, uint32_t* g_vis, uint64_t* counts_global) {
  if (!hc || world < 1 || rank < 0 || rank >= world || B < 1 || B > lobe::kMaxBlocks) return LOBE_E_INVALID_CONFIG;
  lobe::HostOps x(*hc, rank, world);
  std::vector<uint64_t> c(counts_local, counts_local + 2 * (size_t)B);
  return lobe::xchg_block_loads(x, rank, world, B, words, partial, c.data(), own, g_vis, counts_global);
}

lobe_status lobe_xchg_all_masks_host(const lobe_host_comm* hc, int32_t rank, int32_t world, int32_t B, size_t words,
                                     const uint32_t* own, uint32_t* all) {
  if (!hc || world < 1 || rank < 0 || rank >= world || B < 1) return LOBE_E_INVALID_CONFIG;
  lobe::HostOps x(*hc, rank, world);
  return lobe::xchg_all_masks(x, rank, world, B, words, own, all);
}

lobe_status lobe_xchg_gather_cameras_host(const lobe_host_comm* hc, int32_t rank, int32_t world, int64_t N,
                                          size_t elem, const void* local, void* out) {
  if (!hc || world < 1 || rank < 0 || rank >= world || N < 0) return LOBE_E_INVALID_CONFIG;
  lobe::HostOps x(*hc, rank, world);
  return lobe::xchg_gather_cameras(x, rank, world, N, elem, local, out);
}

}  // extern "C"
