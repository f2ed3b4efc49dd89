// lobe_comm.h -- the multi-rank exchange of SURVEY.md §8(e) (cameras sharded,
// Gaussians replicated), internal to liblobe.so.
//
// One choreography, written once against XOps (what it needs from a memory
// space + transport), runs in three settings:
//   - DeviceNccl: device buffers, NCCL on the scene's stream (the product path
//     over NVLink / NVSwitch; the library creates and caches its ncclComm from
//     the caller's ncclUniqueId);
//   - DeviceHost: device buffers staged through host memory, the caller's
//     lobe_host_comm callbacks as transport (any process group, e.g. gloo);
//   - HostHost: host buffers and callbacks, no GPU (lobe_xchg_*_host exports:
//     the CPU tests drive the same choreography with oracle partials).
// Per evaluation: rank j owns blocks [floor(jB/W),
// floor((j+1)B/W)); an all-to-all sends every rank the partial masks of its
// blocks, the owner ORs the W partials and popcounts them (k_masks_combine),
// G_vis of the owned blocks is all-gathered and |C^(b)|, I_b are SUM
// all-reduced. NCCL has no bitwise-OR reduction; this moves (W-1)/W of the
// B x G/8 partial masks per rank instead of the W-fold all-gather.
#pragma once
#include <cstddef>
#include <cstdint>
#include <string>

#include <cuda_runtime.h>

#include "../../include/lobe.h"

namespace lobe {

inline int64_t shard_begin(int64_t n, int r, int w) { return (int64_t)r * n / w; }

struct XOps {
  virtual ~XOps() {}
  // scratch in this memory space (zero-filled on request)
  virtual lobe_status alloc(void** p, size_t bytes) = 0;
  virtual void release(void* p) = 0;
  virtual lobe_status copy(void* dst, const void* src, size_t bytes) = 0;
  virtual lobe_status zero(void* p, size_t bytes) = 0;
  // rank j receives sb[j] bytes from send + so[j]; rb[j] bytes from rank j land at recv + ro[j]
  virtual lobe_status all_to_all_v(const void* send, const size_t* sb, const size_t* so, void* recv,
                                   const size_t* rb, const size_t* ro) = 0;
  // recv = world x bytes, rank-major
  virtual lobe_status all_gather(const void* send, void* recv, size_t bytes) = 0;
  virtual lobe_status all_reduce_u64(uint64_t* buf, size_t count) = 0;  // in place, SUM
  // out (nb x words) = OR over W of gathered (W x nb x words); gvis[k] += popcount(out[k]) (gvis zeroed by the caller)
  virtual lobe_status or_combine(const uint32_t* gathered, int W, int nb, size_t words, uint32_t* out,
                                 uint32_t* gvis) = 0;
  // copy to host memory; complete on return
  virtual lobe_status to_host(void* dst, const void* src, size_t bytes) = 0;
  std::string err;
};

// One evaluation's exchange. partial: B x words u32 (this rank's cameras' OR);
// counts: 2B u64 [|C^(b)| | I_b], local in, global out (same memory space);
// own: nb_r x words u32 out (combined masks of this rank's blocks); g_vis_host,
// counts_host: B u32 / 2B u64 host outputs (identical on every rank).
lobe_status xchg_block_loads(XOps& x, int rank, int world, int B, size_t words, const uint32_t* partial,
                             uint64_t* counts, uint32_t* own, uint32_t* g_vis_host, uint64_t* counts_host);
// Every block's combined masks (B x words, block order) from each rank's own blocks.
lobe_status xchg_all_masks(XOps& x, int rank, int world, int B, size_t words, const uint32_t* own, uint32_t* all);
// Per-camera array of N entries of elem bytes; rank r holds its shard (shard_begin) in `local`.
lobe_status xchg_gather_cameras(XOps& x, int rank, int world, int64_t N, size_t elem, const void* local, void* out);

// ---- communicators ---------------------------------------------------------
// A scene's transport: NCCL (cached per unique id / rank / device, created on
// first use, collective) or the caller's host callbacks.
struct Comm;
// creates or reuses; *err set on failure (LOBE_E_NCCL / LOBE_E_INVALID_CONFIG)
lobe_status comm_acquire(const lobe_options& o, Comm** out, std::string* err);
// device-memory ops of a comm on a stream (DeviceNccl or DeviceHost)
XOps* comm_device_ops(Comm* c, int device, cudaStream_t st);
bool comm_is_nccl(const Comm* c);
// a scene's end: host-callback comms are per scene, NCCL comms stay cached
void comm_release_scene(Comm* c);

}  // namespace lobe
