// lobe_api.cpp -- host runtime behind include/lobe.h.
//
// Owns the scene's device memory (stream-ordered pool allocations), validates
// inputs, resolves the frame and the per-camera projection rows (host fp64,
// rounded once to fp32 -- ledger L13), sequences the kernels of
// lobe_kernels.cu and caches the last evaluated grid so that assign / loads /
// crop calls on the same cuts reuse one evaluation. Compiled with
// -ffp-contract=off: the few fp32 host operations (camera-centre grid
// coordinates, region bounds) are single IEEE operations in the order written.
#include <algorithm>
#include <array>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstddef>
#include <cstdio>
#include <cstring>
#include <limits>
#include <string>
#include <vector>
#include <mutex>

#include <functional>

#include <cuda_runtime.h>

#include "../../include/lobe.h"
#include "lobe_internal.h"
#include "lobe_comm.h"

#include <nvtx3/nvToolsExt.h>

using namespace lobe;

namespace lobe {
// lobe_bo.cpp
int bo_run(int m, int n, int L, uint64_t seed, int n_sobol,
           const std::function<int(const float*, const float*, uint32_t*)>& objective, float* v_out, float* h_out,
           uint32_t* history, float* cut_history, std::string* err);
}  // namespace lobe

namespace {

thread_local std::string g_err;

// stream-ordered allocation; LOBE_TRACE_ALLOC=1 prints slow calls (pool growth)
cudaError_t malloc_async(void** p, size_t bytes, cudaStream_t st) {
  static const bool trace = std::getenv("LOBE_TRACE_ALLOC") != nullptr;
  if (!trace) return cudaMallocAsync(p, bytes, st);
  const auto t0 = std::chrono::steady_clock::now();
  const cudaError_t e = cudaMallocAsync(p, bytes, st);
  const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  if (ms > 0.5) std::fprintf(stderr, "[lobe] cudaMallocAsync %.1f MB: %.2f ms\n", bytes / 1e6, ms);
  return e;
}
template <class T>
cudaError_t malloc_async(T** p, size_t bytes, cudaStream_t st) {
  return malloc_async(reinterpret_cast<void**>(p), bytes, st);
}

lobe_status fail(lobe_status st, const std::string& msg) {
  g_err = msg;
  return st;
}

// NVTX range per exported call (nsys / ncu --nvtx show the API structure; a
// no-op unless a tool injects itself)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
#define LOBE_NVTX(name) NvtxRange nvtx_range_(name)

// LOBE_TRACE_HOST=1: host timeline of lobe_load_scene (diagnosis of GPU idle gaps)
struct HostTimeline {
  const bool on = std::getenv("LOBE_TRACE_HOST") != nullptr;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now(), last = t0;
  void mark(const char* what) {
    if (!on) return;
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[lobe host] %-28s +%8.1f us  (%8.1f us)\n", what,
                 std::chrono::duration<double, std::micro>(t - last).count(),
                 std::chrono::duration<double, std::micro>(t - t0).count());
    last = t;
  }
};

#define CK(call)                                                                                   \
  do {                                                                                             \
    cudaError_t e_ = (call);                                                                       \
    if (e_ != cudaSuccess) {                                                                       \
      return fail(e_ == cudaErrorMemoryAllocation ? LOBE_E_OOM : LOBE_E_CUDA,                      \
                  std::string(#call) + ": " + cudaGetErrorString(e_));                             \
    }                                                                                              \
  } while (0)

// launch of one of this library's kernels (counted for lobe_stats.kernel_launches)
#define KL(call)                      \
  do {                                \
    CK(call);                         \
    s->st.kernel_launches += 1;       \
  } while (0)
// a launcher that starts n kernels (launch_cull, launch_crop: 2)
#define KLN(call, n)                  \
  do {                                \
    CK(call);                         \
    s->st.kernel_launches += (n);     \
  } while (0)
#define CUBL(call)                    \
  do {                                \
    CK(call);                         \
    s->st.cub_launches += 1;          \
  } while (0)

#define TRY(expr)                       \
  do {                                  \
    lobe_status s_ = (expr);            \
    if (s_ != LOBE_OK) return s_;       \
  } while (0)

const double kMag = 1e18;  // ledger L22

inline bool in_interval(float x, float lo, float hi) {
  return x >= lo && (x < hi || (hi == 1.0f && x <= 1.0f));
}

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
};

}  // namespace

constexpr int kNumEvents = 25;

struct lobe_scene {
  int device = 0;
  cudaStream_t stream = nullptr;
  int rank = 0, world = 1, assign_mode = 0;
  int num_sms = 148;
  int64_t G = 0, G_pad = 0, N_all = 0, N_loc = 0, cam_begin = 0;
  int64_t words = 0, n_tiles = 0, n_chunks = 0;
  lobe_frame frame{};
  float mm[4] = {0, 0, 0, 0};
  // device, internal order
  float *xy = nullptr, *zk = nullptr, *o2 = nullptr, *gu = nullptr, *gv = nullptr;
  int32_t* iperm = nullptr;
  CamSetup* cams = nullptr;
  CamSetup* cam_pat = nullptr;  // [N_loc x kPatterns] pattern-ordered copies (k_vis_tiles)
  float *d_cam_gu = nullptr, *d_cam_gv = nullptr;
  uint32_t* rows = nullptr;
  uint8_t* flags = nullptr;     // dev bench (camera-inner variants) only
  uint8_t* nonempty = nullptr;  // [kept pairs] any Gaussian visible
  PairPartial* pair_part = nullptr;
  // a4 deferred until needed (ensure_a4)
  bool a4_pending = false;
  bool a4_side = false, a4_joined = false;  // a4 on the depth side stream (LOBE_A4_STREAM=1)
  cudaStream_t dstream = nullptr;
  uint32_t* camtile = nullptr;  // camera x tile bits of the non-empty pairs (a4's camera order)
  int64_t a4_cap = 0, a4_tw = 0;
  unsigned long long a4_kept = 0;
  uint32_t* cam_off = nullptr;
  int32_t* cam_order = nullptr;
  float4 *tile_lo = nullptr, *tile_hi = nullptr, *chunk_lo = nullptr, *chunk_hi = nullptr;
  float4 *slice_lo = nullptr, *slice_hi = nullptr;
  uint32_t* codes = nullptr;  // per kept pair: slice classes (k_slice_codes)
  float4 *group_lo = nullptr, *group_hi = nullptr;  // anisotropic: 64-Gaussian pair-group boxes
  uint32_t* gcodes = nullptr;  // anisotropic: per kept pair, pair-group classes of undecided slices
  bool aniso_fast = true;     // anisotropic test may use the branch-free rcp / sqrt (all depth ranges in range)
  cudaStream_t side = nullptr;  // per-camera host copies (run_staged), created on first use
  bool aniso = false;            // anisotropic predicate (ledger L24)
  float4* cv = nullptr;          // pair-interleaved Sigma (anisotropic)
  AnisoCam* acams = nullptr;     // per local camera (anisotropic)
  unsigned long long* vcnt = nullptr;  // k_vis_tiles counters: undecided, accepted
  uint32_t* keep = nullptr;
  unsigned long long* kept = nullptr;
  uint32_t *koff = nullptr, *klist = nullptr, *unit_tile = nullptr;
  uint32_t* unit_meta = nullptr;  // per visibility unit: {tile, first kept pair, cameras, 0}
  int64_t n_units = 0;
  unsigned long long* queue = nullptr;
  int64_t n_sub = 0;
  uint32_t* K = nullptr;
  // NEXT-1 (ledger L26): back-projected clouds of the local cameras; when
  // cloud_mode is set the assignment (a6/a7) counts cloud points instead of
  // visible Gaussians and K_c is the cloud size
  bool cloud_mode = false;
  float *cloud_gu = nullptr, *cloud_gv = nullptr;
  uint32_t* cloud_cam = nullptr;
  uint32_t* cloud_K = nullptr;
  int64_t n_cloud = 0;
  std::vector<lobe_camera> host_cams;  // the local cameras (render selection)
  double* D = nullptr;
  float *zmin = nullptr, *zmax = nullptr;
  uint32_t *tile_off = nullptr, *pair_cam = nullptr, *pair_tile = nullptr;
  int64_t n_pairs = 0;
  // evaluation scratch
  uint16_t *zp = nullptr, *word_zone = nullptr, *tile_zone = nullptr;
  uint4* wbox = nullptr;  // per row word: gu / gv range of its Gaussians (a5)
  uint32_t* zp_count = nullptr;
  ZoneTables* dz = nullptr;
  uint8_t* d_zp_cell = nullptr;
  uint32_t* hist = nullptr;
  size_t hist_cap = 0;
  uint32_t *ncb = nullptr, *n0cb = nullptr;
  uint64_t *member = nullptr, *sel = nullptr;
  int32_t* home = nullptr;
  uint32_t* counts = nullptr;  // [0:64) ncams, [64:128) gvis, [128:192) gblk
  unsigned long long* incid = nullptr;  // [64]
  uint32_t* masks = nullptr;
  int masks_B = 0;
  // cache of the last evaluated grid
  bool ev_valid = false;
  int ev_m = 0, ev_n = 0, ev_mode = 0;
  std::vector<float> ev_v, ev_h;
  float ev_dv = 0, ev_dh = 0;
  double ev_tau = 0;
  ZoneTables hz{};
  std::vector<uint8_t> zp_cell;
  // pinned host staging (asynchronous copies; one synchronisation per call)
  struct Pinned {
    ZoneTables Z;
    uint8_t zp_cell[kMaxZones * kMaxZones];
    alignas(16) uint32_t counts[3 * kMaxBlocks];  // mirrors the device block: ncams, gvis, gblk
    unsigned long long incid[kMaxBlocks];   // then incid (contiguous on the device too)
    unsigned long long vc[32];              // k_vis_tiles / k_cull counters of the last pass (VisArgs::counters)
    uint32_t prep_hs[8];                    // k_prep_raw: error flags, ordered ground min / max
    uint32_t n_pairs;                       // non-empty (tile, camera) pairs of the last load
    uint32_t n_units;                       // visibility work units of the last load
    unsigned long long kept_pairs;          // (tile, camera) pairs kept by the culling pass
    unsigned long long prep_bad;            // k_prep_raw: first invalid Gaussian
    uint32_t q_err;                         // k_check_quats (deferred path): any invalid quaternion
    unsigned long long q_bad;               // k_check_quats: first invalid quaternion
  };
  static_assert(offsetof(Pinned, incid) == offsetof(Pinned, counts) + 3 * kMaxBlocks * sizeof(uint32_t),
                "pinned counts / incid must mirror the contiguous device block");
  Pinned* pin = nullptr;
  uint8_t* pin_out = nullptr;  // growable staging for per-camera outputs
  size_t pin_out_cap = 0;
  uint8_t* pin_in = nullptr;   // the load's per-camera uploads (pinned: asynchronous, the host never blocks)
  size_t pin_in_cap = 0;
  bool stats_pending = false;  // load-pass timings read lazily (lobe_get_stats)
  bool crop_pending = false;   // crop timing of a call with device outputs, read lazily
  unsigned long long kept_pairs_last = 0;
  // An evaluation ends with an asynchronous copy of its block counts into
  // `pin` (event ev[13]); the host waits only when it reads them.
  bool eval_pending = false;
  void wait_counts() {
    if (!eval_pending) return;
    cudaEventSynchronize(ev[13]);
    float a = 0.f, b = 0.f;
    if (cudaEventElapsedTime(&a, ev[2], ev[3]) == cudaSuccess) st.t_hist_ms = a;
    if (cudaEventElapsedTime(&b, ev[3], ev[4]) == cudaSuccess) st.t_loads_ms = b;
    eval_pending = false;
  }
  const uint32_t* h_ncams() { wait_counts(); return pin->counts; }
  const uint32_t* h_gvis() { wait_counts(); return pin->counts + kMaxBlocks; }
  const uint32_t* h_gblk() { wait_counts(); return pin->counts + 2 * kMaxBlocks; }
  const unsigned long long* h_incid() { wait_counts(); return pin->incid; }
  // stats
  lobe_stats st{};
  cudaEvent_t ev[kNumEvents] = {};  // load pass: 0, 1, 8-12, 16, 17; evaluation: 2-4, 13; combine: 5, 6; dev bench:
                                    // 6, 7; crop: 14, 15; collective exchange: 18, 19; deferred quaternion
                                    // check: 20 (done), 21 (k_prep_raw done), 22 (camera copies done); split
                                    // host-input copies: 23 (positions landed), 24 (other fields landed)
  cudaStream_t qstream = nullptr;   // host inputs, isotropic: quaternion copy + check (side stream)
  // deferred quaternion verdict (event 20): pending after the load, then the
  // status every later call reports (LOBE_E_INVALID_INPUT: the scene is unusable)
  // render-selection scratch (lobe_render_select): grow-only device blocks kept
  // for the scene's lifetime, so repeated selections neither allocate nor free
  struct RBuf {
    void* p = nullptr;
    size_t cap = 0;
  };
  RBuf rscratch[20];
  mutable bool q_pending = false;
  mutable lobe_status q_status = LOBE_OK;
  mutable unsigned long long q_first_bad = 0;
  // ---- communicator: collective calls, global outputs
  lobe::Comm* comm = nullptr;
  lobe::XOps* xops = nullptr;       // device-memory ops of comm on `stream`
  uint32_t* own_masks = nullptr;    // combined masks of this rank's blocks (last exchange)
  int own_cap = 0;                  // blocks own_masks can hold
  unsigned long long* d_xcounts = nullptr;  // [2 x kMaxBlocks] u64: |C^(b)| then I_b
  uint32_t x_gvis[kMaxBlocks] = {};         // global G_vis of the last exchange
  uint64_t x_counts[2 * kMaxBlocks] = {};   // global |C^(b)|, I_b of the last exchange
  bool x_valid = false;                     // the cached evaluation has been exchanged
  bool x_all = false;                       // `masks` holds every block's combined masks

  template <class T>
  cudaError_t alloc(T** p, size_t count) {
    *p = nullptr;
    if (count == 0) count = 1;
    return malloc_async(reinterpret_cast<void**>(p), count * sizeof(T), stream);
  }
  template <class T>
  void release(T*& p) {
    if (p) cudaFreeAsync(p, stream);
    p = nullptr;
  }
};

namespace {

// ---------------------------------------------------------------- validation
lobe_status validate_cameras(const lobe_camera* cams, int64_t N) {
  if (N <= 0) return fail(LOBE_E_INVALID_CONFIG, "n_cams must be > 0 (SPEC.md:110)");
  for (int64_t c = 0; c < N; ++c) {
    const lobe_camera& k = cams[c];
    bool ok = std::isfinite(k.fx) && std::isfinite(k.fy) && std::isfinite(k.cx) && std::isfinite(k.cy) &&
              k.fx > 0.0f && k.fy > 0.0f && k.width > 0 && k.height > 0 && std::isfinite(k.z_near) &&
              std::isfinite(k.z_far) && k.z_near > 0.0f && k.z_near < k.z_far &&
              std::fabs((double)k.cx) <= kMag && std::fabs((double)k.cy) <= kMag;
    for (int j = 0; j < 3; ++j) ok = ok && std::isfinite(k.t[j]) && std::fabs((double)k.t[j]) <= kMag;
    for (int j = 0; j < 9; ++j) ok = ok && std::isfinite(k.R[j]);
    for (int a = 0; ok && a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        double d = (double)k.R[3 * a] * k.R[3 * b] + (double)k.R[3 * a + 1] * k.R[3 * b + 1] +
                   (double)k.R[3 * a + 2] * k.R[3 * b + 2];
        if (std::fabs(d - (a == b ? 1.0 : 0.0)) > 1e-5) ok = false;
      }
    if (!ok)
      return fail(LOBE_E_INVALID_INPUT,
                  "camera " + std::to_string(c) + " invalid (fx,fy>0, 0<z_near<z_far, R orthonormal; SPEC.md:46-48)");
  }
  return LOBE_OK;
}

// camera centre o = -R^T t in fp64
void cam_centre(const lobe_camera& k, double o[3]) {
  for (int j = 0; j < 3; ++j)
    o[j] = -((double)k.R[j] * k.t[0] + (double)k.R[3 + j] * k.t[1] + (double)k.R[6 + j] * k.t[2]);
}

// Ledger L12: lower median centre, ceil(0.9 N)-th smallest distance, world x/y axes.
lobe_status resolve_frame(const lobe_camera* cams, int64_t N, lobe_frame* f) {
  std::vector<double> c[3];
  for (int a = 0; a < 3; ++a) c[a].resize(N);
  for (int64_t i = 0; i < N; ++i) {
    double o[3];
    cam_centre(cams[i], o);
    for (int a = 0; a < 3; ++a) {
      // the full camera validation runs later; the selections below need
      // finite centres (a NaN would break their ordering)
      if (!std::isfinite(o[a]))
        return fail(LOBE_E_INVALID_INPUT, "camera " + std::to_string(i) + " centre not finite (SPEC.md:46-48)");
      c[a][i] = o[a];
    }
  }
  if (f->auto_flags & LOBE_FRAME_AUTO_CENTER) {
    for (int a = 0; a < 3; ++a) {
      std::vector<double> s = c[a];
      std::nth_element(s.begin(), s.begin() + (N - 1) / 2, s.end());
      f->center[a] = (float)s[(N - 1) / 2];
    }
  }
  if (f->auto_flags & LOBE_FRAME_AUTO_RADIUS) {
    std::vector<double> d(N);
    for (int64_t i = 0; i < N; ++i) {
      double dx = c[0][i] - (double)f->center[0], dy = c[1][i] - (double)f->center[1],
             dz = c[2][i] - (double)f->center[2];
      d[i] = std::sqrt(dx * dx + dy * dy + dz * dz);
    }
    const int64_t kth = (9 * N + 9) / 10;  // ceil(0.9 N)
    std::nth_element(d.begin(), d.begin() + (kth - 1), d.end());
    f->radius = (float)d[kth - 1];
  }
  if (f->auto_flags & LOBE_FRAME_AUTO_AXES) {
    const float u[3] = {1, 0, 0}, v[3] = {0, 1, 0};
    std::memcpy(f->axis_u, u, sizeof(u));
    std::memcpy(f->axis_v, v, sizeof(v));
  }
  for (int a = 0; a < 3; ++a)
    if (!std::isfinite(f->center[a]) || !std::isfinite(f->axis_u[a]) || !std::isfinite(f->axis_v[a]))
      return fail(LOBE_E_INVALID_INPUT, "frame centre/axes not finite");
  if (!(f->radius > 0.0f) || !std::isfinite(f->radius))
    return fail(LOBE_E_DEGENERATE_SCENE, "frame radius is zero (all cameras at one point)");
  return LOBE_OK;
}

// scaled rows in fp64, rounded once (L13).
CamSetup camera_setup(const lobe_camera& k) {
  const double f = (double)std::max(k.fx, k.fy);
  CamSetup s;
  for (int j = 0; j < 3; ++j) {
    s.Au[j] = (float)(((double)k.fx * k.R[j] + (double)k.cx * k.R[6 + j]) / f);
    s.Av[j] = (float)(((double)k.fy * k.R[3 + j] + (double)k.cy * k.R[6 + j]) / f);
    s.Aw[j] = k.R[6 + j];
  }
  s.Au[3] = (float)(((double)k.fx * k.t[0] + (double)k.cx * k.t[2]) / f);
  s.Av[3] = (float)(((double)k.fy * k.t[1] + (double)k.cy * k.t[2]) / f);
  s.Aw[3] = k.t[2];
  s.Wf = (float)((double)k.width / f);
  s.Hf = (float)((double)k.height / f);
  s.zn = k.z_near;
  s.zf = k.z_far;
  return s;
}

// Anisotropic predicate: the raw camera, plus w2 >= ||R||_2^2 = max abs row sum
// of R^T R (fp64) for the culling bound (ledger L24).
AnisoCam aniso_setup(const lobe_camera& k) {
  AnisoCam a{};
  for (int i = 0; i < 9; ++i) a.R[i] = k.R[i];
  for (int i = 0; i < 3; ++i) a.t[i] = k.t[i];
  a.fx = k.fx; a.fy = k.fy; a.cx = k.cx; a.cy = k.cy;
  a.Wf = (float)k.width; a.Hf = (float)k.height;
  a.zn = k.z_near; a.zf = k.z_far;
  double w2 = 0.0;
  for (int i = 0; i < 3; ++i) {
    double row = 0.0;
    for (int j = 0; j < 3; ++j) {
      double g = 0.0;
      for (int r = 0; r < 3; ++r) g += (double)k.R[3 * r + i] * (double)k.R[3 * r + j];
      row += std::fabs(g);
    }
    w2 = std::max(w2, row);
  }
  a.w2 = w2 * (1.0 + 1e-12);
  const double fx = a.fx, fy = a.fy, cx = a.cx, cy = a.cy, W = a.Wf, H = a.Hf;
  for (int d = 0; d < 4; ++d) {
    const double r0 = d < 3 ? (double)a.R[d] : (double)a.t[0], r1 = d < 3 ? (double)a.R[3 + d] : (double)a.t[1],
                 r2 = d < 3 ? (double)a.R[6 + d] : (double)a.t[2];
    a.U[d] = (float)(fx * r0 + cx * r2);
    a.EU[d] = (float)(fx * r0 + (cx - W) * r2);
    a.V[d] = (float)(fy * r1 + cy * r2);
    a.EV[d] = (float)(fy * r1 + (cy - H) * r2);
  }
  return a;
}

// O3's fp32 map for one point (contraction + ground projection), host side.
void ground_uv_host(float px, float py, float pz, const lobe_frame& F, float* gu, float* gv) {
  float hx = (px - F.center[0]) / F.radius;
  float hy = (py - F.center[1]) / F.radius;
  float hz = (pz - F.center[2]) / F.radius;
  float r = std::sqrt(std::fmaf(hx, hx, std::fmaf(hy, hy, hz * hz)));
  if (!(r <= 1.0f)) {
    float s = (2.0f - 1.0f / r) / r;
    hx = hx * s;
    hy = hy * s;
    hz = hz * s;
  }
  *gu = std::fmaf(hx, F.axis_u[0], std::fmaf(hy, F.axis_u[1], hz * F.axis_u[2]));
  *gv = std::fmaf(hx, F.axis_v[0], std::fmaf(hy, F.axis_v[1], hz * F.axis_v[2]));
}

// ------------------------------------------------------------- grid / zones
struct GridV {
  int m, n, B;
  std::vector<float> v, h;
  float dv, dh;
  double tau;
};

lobe_status check_grid(const lobe_grid* g, GridV* out) {
  if (!g) return fail(LOBE_E_INVALID_CONFIG, "grid is NULL");
  if (g->m < 1 || g->n < 1 || (int64_t)g->m * g->n > kMaxBlocks)
    return fail(LOBE_E_INVALID_CONFIG, "grid m, n must be >= 1 with m*n <= 64");
  out->m = g->m;
  out->n = g->n;
  out->B = g->m * g->n;
  out->v.assign(g->v ? g->v : nullptr, g->v ? g->v + (g->m - 1) : nullptr);
  out->h.assign(g->h ? g->h : nullptr, g->h ? g->h + (g->n - 1) : nullptr);
  if ((g->m > 1 && !g->v) || (g->n > 1 && !g->h)) return fail(LOBE_E_INVALID_CUTS, "missing cut array");
  for (int i = 0; i + 1 < g->m; ++i)
    if (!(out->v[i] > 0.0f && out->v[i] < 1.0f) || (i > 0 && !(out->v[i] > out->v[i - 1])))
      return fail(LOBE_E_INVALID_CUTS, "v cuts must be strictly increasing in (0,1) (SPEC.md:52-55)");
  for (int j = 0; j + 1 < g->n; ++j)
    if (!(out->h[j] > 0.0f && out->h[j] < 1.0f) || (j > 0 && !(out->h[j] > out->h[j - 1])))
      return fail(LOBE_E_INVALID_CUTS, "h cuts must be strictly increasing in (0,1) (SPEC.md:52-55)");
  out->dv = g->delta_v < 0.0f ? 0.1f / (float)g->m : g->delta_v;  // PAPER.md:167, ledger L14
  out->dh = g->delta_h < 0.0f ? 0.1f / (float)g->n : g->delta_h;
  out->tau = g->tau < 0.0 ? 0.15 : g->tau;
  if (!std::isfinite(out->dv) || !std::isfinite(out->dh)) return fail(LOBE_E_INVALID_CONFIG, "delta not finite");
  if (!(out->tau >= 0.0 && out->tau <= 1.0)) return fail(LOBE_E_INVALID_CONFIG, "tau must be in [0,1]");
  return LOBE_OK;
}

// Zones of one axis: breakpoints of all cell and enlarged-region
// bounds; every point of a zone has the same cell and enlarged memberships.
void build_axis(int count, const std::vector<float>& cuts, float delta, AxisZones* A) {
  std::vector<float> lo(count), hi(count), elo(count), ehi(count);
  std::vector<float> P = {0.0f};
  for (int p = 0; p < count; ++p) {
    lo[p] = (p == 0) ? 0.0f : cuts[p - 1];
    hi[p] = (p == count - 1) ? 1.0f : cuts[p];
    elo[p] = std::fmax(0.0f, lo[p] - delta);
    ehi[p] = std::fmin(1.0f, hi[p] + delta);
    for (float b : {lo[p], hi[p], elo[p], ehi[p]})
      if (b < 1.0f) P.push_back(b);
  }
  std::sort(P.begin(), P.end());
  P.erase(std::unique(P.begin(), P.end()), P.end());
  const int K = (int)P.size();
  A->nz = K + 1;
  A->count = count;
  for (int z = 0; z < A->nz; ++z) {
    const float rep = (z < K) ? P[z] : 1.0f;
    if (z < K) A->P[z] = P[z];
    A->cell[z] = 0;
    A->encl[z] = 0;
    for (int p = 0; p < count; ++p) {
      if (in_interval(rep, lo[p], hi[p])) A->cell[z] = (uint8_t)p;
      if (in_interval(rep, elo[p], ehi[p])) A->encl[z] |= 1ull << p;
    }
  }
  // zone of x = #{k in [1, K-1] : P[k] <= x} (x < 1); per bin, that count at the
  // bin's lower end (exact: b / 1024 is a float) and how many breakpoints lie
  // strictly inside the bin
  int zlo = 0;  // #{k >= 1 : P[k] <= x0}, nondecreasing in b (P ascending)
  for (int b = 0; b < kZoneBins; ++b) {
    const float x0 = (float)b / (float)kZoneBins, x1 = (float)(b + 1) / (float)kZoneBins;
    while (zlo + 1 < K && P[zlo + 1] <= x0) ++zlo;
    int nin = 0;
    for (int k = zlo + 1; k < K && P[k] < x1 && nin < 2; ++k) ++nin;
    A->bin[b] = (uint16_t)(zlo | ((nin == 0 ? 0 : (nin == 1 ? 1 : 2)) << 14));
  }
}

int cell_host(const AxisZones& A, float x) {
  if (x == 1.0f) return A.cell[A.nz - 1];
  int z = 0;
  for (int k = 1; k < A.nz - 1; ++k) z += (A.P[k] <= x) ? 1 : 0;
  return A.cell[z];
}

lobe_status ensure_hist_cap(lobe_scene* s, size_t need) {
  if (s->hist_cap >= need) return LOBE_OK;
  s->release(s->hist);
  CK(s->alloc(&s->hist, need));
  s->hist_cap = need;
  return LOBE_OK;
}

lobe_status ensure_masks(lobe_scene* s, int B) {
  if (s->masks && s->masks_B >= B) return LOBE_OK;
  s->release(s->masks);
  CK(s->alloc(&s->masks, (size_t)B * s->words));
  s->masks_B = B;
  return LOBE_OK;
}

float ms_between(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  if (cudaEventElapsedTime(&ms, a, b) != cudaSuccess) return 0.f;
  return ms;
}

// a5 + a6 + a7 (+ a8 into `masks_out`): one evaluation of a grid on cached rows.
lobe_status evaluate(lobe_scene* s, const GridV& g, uint32_t* masks_out) {
  cudaStream_t st = s->stream;
  s->wait_counts();  // the previous evaluation's copies read / write `pin`
  s->x_valid = false;
  s->x_all = false;
  // ---- a5 zone tables (host) + per-Gaussian zones (device)
  ZoneTables Z{};
  build_axis(g.m, g.v, g.dv, &Z.U);
  build_axis(g.n, g.h, g.dh, &Z.V);
  Z.m = g.m;
  Z.n = g.n;
  Z.B = g.B;
  const int nzv = Z.V.nz, nzp = Z.U.nz * Z.V.nz;
  s->hz = Z;
  s->zp_cell.assign(nzp, 0);
  for (int zp = 0; zp < nzp; ++zp) s->zp_cell[zp] = (uint8_t)(Z.U.cell[zp / nzv] * g.n + Z.V.cell[zp % nzv]);
  s->pin->Z = Z;
  std::memcpy(s->pin->zp_cell, s->zp_cell.data(), nzp);
  // (kernel uploads: a copy-engine transfer would queue behind the deferred
  // quaternions of a host-input load)
  KL(launch_upload(s->dz, &s->pin->Z, sizeof(Z), st));
  KL(launch_upload(s->d_zp_cell, s->pin->zp_cell, nzp, st));
  CK(cudaMemsetAsync(s->zp_count, 0, sizeof(uint32_t) * kMaxZones * kMaxZones, st));
  // counts [3 x kMaxBlocks] u32 and incid [kMaxBlocks] u64 are one device block
  CK(cudaMemsetAsync(s->counts, 0, sizeof(uint32_t) * 3 * kMaxBlocks + sizeof(unsigned long long) * kMaxBlocks, st));
  CK(cudaEventRecord(s->ev[2], st));
  KL(launch_zones(s->dz, nzv, nzp, s->G, s->G_pad, s->gu, s->gv, s->wbox, s->zp, s->word_zone, s->tile_zone,
                  s->zp_count, st));
  KL(launch_gblk(s->dz, nzv, nzp, s->zp_count, s->counts + 2 * kMaxBlocks, st));
  // ---- a6 histograms
  TRY(ensure_hist_cap(s, (size_t)std::max<int64_t>(s->N_loc, 1) * nzp));
  if (s->N_loc > 0) {
    CK(cudaMemsetAsync(s->hist, 0, sizeof(uint32_t) * (size_t)s->N_loc * nzp, st));
    if (s->cloud_mode)
      KL(launch_hist_points(s->n_cloud, s->cloud_gu, s->cloud_gv, s->cloud_cam, s->dz, nzv, nzp, s->hist, st));
    else
      KL(launch_hist(s->n_tiles, s->tile_off, s->pair_cam, s->rows, s->words, s->zp, s->word_zone, s->tile_zone,
                     nzp, s->hist, st));
  }
  CK(cudaEventRecord(s->ev[3], st));
  // ---- a7 assignment
  if (s->N_loc > 0) {
    AssignArgs a{};
    a.dz = s->dz;
    a.hist = s->hist;
    a.nzp = nzp;
    a.cam_gu = s->d_cam_gu;
    a.cam_gv = s->d_cam_gv;
    a.n_cams = s->N_loc;
    a.tau = g.tau;
    a.mode = s->assign_mode;
    a.ncb = s->ncb;
    a.n0cb = s->n0cb;
    a.member = s->member;
    a.home = s->home;
    a.sel = s->sel;
    a.ncams = s->counts;
    a.incid = s->incid;
    KL(launch_assign(a, st));
  }
  // ---- a8 block masks
  if (masks_out) {
    KL(launch_block_masks(s->n_tiles, s->tile_off, s->pair_cam, s->sel, s->rows, s->words, g.B, masks_out,
                          s->counts + kMaxBlocks, st));
  }
  CK(cudaEventRecord(s->ev[4], st));
  // small device -> host results are written into pinned memory by a kernel
  // (mapped under unified addressing): no copy-engine queueing behind bulk
  // transfers in flight (host-input loads, crop downloads)
  KL(launch_upload(s->pin->counts, s->counts,
                   sizeof(uint32_t) * 3 * kMaxBlocks + sizeof(unsigned long long) * kMaxBlocks, st));
  CK(cudaEventRecord(s->ev[13], st));
  s->eval_pending = true;  // no synchronisation: readers of the counts wait (wait_counts)
  s->st.evaluations += 1;
  return LOBE_OK;
}

bool same_grid(const lobe_scene* s, const GridV& g) {
  return s->ev_valid && s->ev_m == g.m && s->ev_n == g.n && s->ev_v == g.v && s->ev_h == g.h &&
         s->ev_dv == g.dv && s->ev_dh == g.dh && s->ev_tau == g.tau && s->ev_mode == s->assign_mode;
}

// world == 1 path: evaluation into the scene's own mask buffer, cached.
lobe_status ensure_eval(lobe_scene* s, const GridV& g) {
  if (same_grid(s, g)) return LOBE_OK;
  s->ev_valid = false;
  TRY(ensure_masks(s, g.B));
  TRY(evaluate(s, g, s->masks));
  s->ev_valid = true;
  s->ev_m = g.m;
  s->ev_n = g.n;
  s->ev_v = g.v;
  s->ev_h = g.h;
  s->ev_dv = g.dv;
  s->ev_dh = g.dh;
  s->ev_tau = g.tau;
  s->ev_mode = s->assign_mode;
  return LOBE_OK;
}

// With a communicator: the evaluation of this grid on the local cameras (partial
// masks in s->masks, local counts), then the collective exchange of SURVEY §8e
// (lobe_comm.h): every rank ends with the global G_vis, |C^(b)|, I_b and the
// combined masks of its own blocks. One host round trip (the B G_vis values and
// 2B counts); cached with the evaluation.
lobe_status ensure_xchg(lobe_scene* s, const GridV& g) {
  TRY(ensure_eval(s, g));
  if (s->x_valid) return LOBE_OK;
  const int B = g.B, W = s->world, r = s->rank;
  const int nb = (int)(lobe::shard_begin(B, r + 1, W) - lobe::shard_begin(B, r, W));
  if (s->own_cap < nb) {
    s->release(s->own_masks);
    CK(s->alloc(&s->own_masks, (size_t)std::max(nb, 1) * s->words));
    s->own_cap = nb;
  }
  // local |C^(b)| (u32 -> u64) and I_b into the exchange buffer, on the device
  KL(launch_xcounts(s->counts, s->incid, B, s->d_xcounts, s->stream));
  CK(cudaEventRecord(s->ev[18], s->stream));
  lobe_status xs = lobe::xchg_block_loads(*s->xops, r, W, B, (size_t)s->words, s->masks,
                                          reinterpret_cast<uint64_t*>(s->d_xcounts), s->own_masks, s->x_gvis,
                                          s->x_counts);
  if (xs != LOBE_OK) return fail(xs, "exchange: " + s->xops->err);
  CK(cudaEventRecord(s->ev[19], s->stream));
  CK(cudaEventSynchronize(s->ev[19]));
  s->st.t_comm_ms = ms_between(s->ev[18], s->ev[19]);
  s->x_valid = true;
  return LOBE_OK;
}

// ... and every block's combined masks in s->masks (for the crop)
lobe_status ensure_xchg_masks(lobe_scene* s, const GridV& g) {
  TRY(ensure_xchg(s, g));
  if (s->x_all) return LOBE_OK;
  CK(cudaEventRecord(s->ev[18], s->stream));
  lobe_status xs = lobe::xchg_all_masks(*s->xops, s->rank, s->world, g.B, (size_t)s->words, s->own_masks, s->masks);
  if (xs != LOBE_OK) return fail(xs, "exchange: " + s->xops->err);
  CK(cudaEventRecord(s->ev[19], s->stream));
  CK(cudaEventSynchronize(s->ev[19]));
  s->st.t_comm_ms += ms_between(s->ev[18], s->ev[19]);
  s->x_all = true;
  return LOBE_OK;
}

void fill_records(lobe_scene* s, const GridV& g, const uint32_t* ncams, const uint64_t* incid,
                  const uint32_t* gvis, lobe_block_load* out, uint32_t* objective) {
  std::vector<float> ulo(g.m), uhi(g.m), uelo(g.m), uehi(g.m), vlo(g.n), vhi(g.n), velo(g.n), vehi(g.n);
  for (int p = 0; p < g.m; ++p) {
    ulo[p] = (p == 0) ? 0.0f : g.v[p - 1];
    uhi[p] = (p == g.m - 1) ? 1.0f : g.v[p];
    uelo[p] = std::fmax(0.0f, ulo[p] - g.dv);
    uehi[p] = std::fmin(1.0f, uhi[p] + g.dv);
  }
  for (int q = 0; q < g.n; ++q) {
    vlo[q] = (q == 0) ? 0.0f : g.h[q - 1];
    vhi[q] = (q == g.n - 1) ? 1.0f : g.h[q];
    velo[q] = std::fmax(0.0f, vlo[q] - g.dh);
    vehi[q] = std::fmin(1.0f, vhi[q] + g.dh);
  }
  uint32_t best = 0;
  for (int b = 0; b < g.B; ++b) {
    const int p = b / g.n, q = b % g.n;
    lobe_block_load r{};
    r.block_id = b;
    r.row = p;
    r.col = q;
    r.lo[0] = uelo[p];
    r.lo[1] = velo[q];
    r.hi[0] = uehi[p];
    r.hi[1] = vehi[q];
    r.area = ((double)uhi[p] - (double)ulo[p]) * ((double)vhi[q] - (double)vlo[q]);
    r.n_cams = ncams[b];
    r.g_blk = s->h_gblk()[b];
    r.g_vis = gvis[b];
    r.g_avgvis = r.n_cams ? (double)r.g_vis / (double)r.n_cams : 0.0;
    r.incidences = incid[b];
    best = std::max(best, r.g_vis);
    if (out) out[b] = r;
  }
  if (objective) *objective = best;
}

// ---- NEXT-4 block pipeline helpers (ledger L25)
CellArgs make_cell_args(const lobe_scene* s, const GridV& g) {
  CellArgs c{};
  for (int a = 0; a < 3; ++a) {
    c.frame.c0[a] = s->frame.center[a];
    c.frame.au[a] = s->frame.axis_u[a];
    c.frame.av[a] = s->frame.axis_v[a];
  }
  c.frame.rho = s->frame.radius;
  for (int k = 0; k < 4; ++k) c.mm[k] = s->mm[k];
  c.m = g.m;
  c.n = g.n;
  for (int i = 0; i + 1 < g.m; ++i) c.v[i] = g.v[i];
  for (int j = 0; j + 1 < g.n; ++j) c.h[j] = g.h[j];
  return c;
}

SubArgs sub_args(const lobe_subscene* in) {
  SubArgs a{};
  const float* f[11] = {in->x, in->y, in->z, in->sx, in->sy, in->sz, in->qw, in->qx, in->qy, in->qz, in->opacity};
  for (int k = 0; k < 11; ++k) a.f[k] = f[k];
  return a;
}

SubOut sub_out(lobe_subscene* out) {
  SubOut o{};
  float* f[11] = {out->x, out->y, out->z, out->sx, out->sy, out->sz, out->qw, out->qx, out->qy, out->qz, out->opacity};
  for (int k = 0; k < 11; ++k) o.f[k] = f[k];
  o.origin = out->origin;
  o.in_block = out->in_block;
  return o;
}

lobe_status check_sub(const lobe_subscene* p, bool need_arrays, const char* what) {
  if (!p) return fail(LOBE_E_INVALID_CONFIG, std::string(what) + " is NULL");
  if (p->n < 0) return fail(LOBE_E_INVALID_CONFIG, std::string(what) + ": negative count");
  if (need_arrays) {
    const void* f[13] = {p->x, p->y, p->z, p->sx, p->sy, p->sz, p->qw, p->qx, p->qy, p->qz, p->opacity,
                         p->origin, p->in_block};
    for (const void* q : f)
      if (!q) return fail(LOBE_E_INVALID_CONFIG, std::string(what) + ": NULL array");
  }
  return LOBE_OK;
}

// exclusive scan of cnt[0..n) into off[0..n] (off[n] = total), total returned on the host
lobe_status scan_counts(lobe_scene* s, const uint32_t* cnt, uint32_t* off, int64_t n, uint64_t* total) {
  cudaStream_t st = s->stream;
  size_t tb = 0;
  CK(exclusive_scan_u32(nullptr, tb, cnt, off, n + 1, st));
  void* tmp = nullptr;
  CK(malloc_async(&tmp, tb, st));
  CUBL(exclusive_scan_u32(tmp, tb, cnt, off, n + 1, st));
  cudaFreeAsync(tmp, st);
  uint32_t t = 0;
  CK(cudaMemcpyAsync(&t, off + n, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  *total = t;
  return LOBE_OK;
}

lobe_status copy_out(lobe_scene* s, void* dst, const void* src, size_t bytes);

// ---- NEXT-1 depth-render camera selection (ledger L26)
struct RenderJob {
  int ds = 4, stride = 2;
  float eps_w = 0.1f;
  // clouds appended here (device; grown as needed)
  float *gu = nullptr, *gv = nullptr;
  uint32_t* cam = nullptr;
  int64_t n = 0, cap = 0;
  // optional: maps of the batch's first camera copied here (host or device)
  float *Dout = nullptr, *Wout = nullptr;
  // k_render roofline: (pixel, splat) tests / composited (device counters), kernel time
  unsigned long long* counters = nullptr;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> kev;  // around each batch's k_render
};

// device scratch slot `k` of at least `bytes` bytes (grow-only)
template <class T>
lobe_status scratch(lobe_scene* s, RenderJob& J, int k, T** out, size_t count) {
  const size_t bytes = std::max<size_t>(count, 1) * sizeof(T);
  lobe_scene::RBuf& b = s->rscratch[k];
  if (b.cap < bytes) {
    // 1.5x headroom: later batches rarely need a new block. Plain cudaMalloc:
    // growing the stream-ordered pool by these multi-GB blocks is far slower
    // (measured: 1.1 s of cudaMallocAsync per MatrixCity render selection)
    const size_t cap = std::max(bytes, b.cap * 3 / 2);
    if (b.p) {
      CK(cudaStreamSynchronize(s->stream));
      cudaFree(b.p);
    }
    b.p = nullptr;
    b.cap = 0;
    CK(cudaMalloc(&b.p, cap));
    b.cap = cap;
  }
  *out = static_cast<T*>(b.p);
  return LOBE_OK;
}
lobe_status grow_cloud(lobe_scene* s, RenderJob& J, int64_t need) {
  if (need <= J.cap) return LOBE_OK;
  const int64_t cap = std::max<int64_t>({need, J.cap * 2, 1});
  float *gu = nullptr, *gv = nullptr;
  uint32_t* cam = nullptr;
  CK(s->alloc(&gu, (size_t)cap));
  CK(s->alloc(&gv, (size_t)cap));
  CK(s->alloc(&cam, (size_t)cap));
  if (J.n > 0) {
    CK(cudaMemcpyAsync(gu, J.gu, sizeof(float) * J.n, cudaMemcpyDeviceToDevice, s->stream));
    CK(cudaMemcpyAsync(gv, J.gv, sizeof(float) * J.n, cudaMemcpyDeviceToDevice, s->stream));
    CK(cudaMemcpyAsync(cam, J.cam, sizeof(uint32_t) * J.n, cudaMemcpyDeviceToDevice, s->stream));
  }
  s->release(J.gu);
  s->release(J.gv);
  s->release(J.cam);
  J.gu = gu;
  J.gv = gv;
  J.cam = cam;
  J.cap = cap;
  return LOBE_OK;
}

// Render cameras [c0, c1) of the local shard and append their clouds.
lobe_status render_batch(lobe_scene* s, const float4* prec, const std::vector<uint32_t>& hoff,
                         const std::vector<lobe_camera>& hcams, int64_t c0, int64_t c1, RenderJob& J) {
  cudaStream_t st = s->stream;
  const int ncam = (int)(c1 - c0);
  // cameras at 1/ds resolution
  std::vector<RenderCam> rc(ncam);
  uint32_t tiles = 0;
  int64_t maps = 0;
  int max_tiles = 0, max_samples = 0;
  std::vector<uint32_t> sp0(ncam + 1, 0);
  for (int q = 0; q < ncam; ++q) {
    const lobe_camera& k = hcams[c0 + q];
    RenderCam& r = rc[q];
    for (int e = 0; e < 9; ++e) r.R[e] = k.R[e];
    for (int e = 0; e < 3; ++e) r.t[e] = k.t[e];
    r.fx = k.fx / (float)J.ds;
    r.fy = k.fy / (float)J.ds;
    r.cx = k.cx / (float)J.ds;
    r.cy = k.cy / (float)J.ds;
    r.Wd = k.width / J.ds;
    r.Hd = k.height / J.ds;
    r.tw = (r.Wd + 15) / 16;
    r.th = (r.Hd + 15) / 16;
    r.tile0 = tiles;
    r.cam = (uint32_t)(c0 + q);
    r.map0 = maps;
    tiles += (uint32_t)(r.tw * r.th);
    maps += (int64_t)r.Wd * r.Hd;
    max_tiles = std::max(max_tiles, r.tw * r.th);
    const int sw = (r.Wd + J.stride - 1) / J.stride, sh = (r.Hd + J.stride - 1) / J.stride;
    sp0[q + 1] = sp0[q] + (uint32_t)(sw * sh);
    max_samples = std::max(max_samples, sw * sh);
  }
  RenderCam* drc = nullptr;
  TRY(scratch(s, J, 0, &drc, (size_t)ncam));
  CK(cudaMemcpyAsync(drc, rc.data(), sizeof(RenderCam) * ncam, cudaMemcpyHostToDevice, st));
  // 1. records: the visible Gaussians of the batch's non-empty pairs (camera-major)
  const int64_t k0 = hoff[c0], nk = (int64_t)hoff[c1] - k0;
  uint32_t *cnt = nullptr, *pos = nullptr;
  TRY(scratch(s, J, 1, &cnt, (size_t)nk + 1));
  TRY(scratch(s, J, 2, &pos, (size_t)nk + 1));
  CK(cudaMemsetAsync(cnt + nk, 0, sizeof(uint32_t), st));
  KL(launch_rvis_count(k0, nk, s->cam_order, s->pair_tile, s->pair_cam, s->rows, s->words, cnt, st));
  uint64_t n = 0;
  TRY(scan_counts(s, cnt, pos, nk, &n));
  std::vector<uint32_t> hpos(nk + 1);
  CK(cudaMemcpyAsync(hpos.data(), pos, sizeof(uint32_t) * (nk + 1), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  std::vector<uint32_t> seg(ncam + 1);
  for (int q = 0; q <= ncam; ++q) seg[q] = hpos[hoff[c0 + q] - k0];
  unsigned long long *keys = nullptr, *keys_s = nullptr;
  uint32_t *vals = nullptr, *vals_s = nullptr, *rcam = nullptr, *dseg = nullptr;
  float* rec = nullptr;
  const size_t N1 = std::max<uint64_t>(n, 1);
  TRY(scratch(s, J, 3, &keys, N1)); TRY(scratch(s, J, 4, &keys_s, N1));
  TRY(scratch(s, J, 5, &vals, N1)); TRY(scratch(s, J, 6, &vals_s, N1));
  TRY(scratch(s, J, 7, &rcam, N1));
  TRY(scratch(s, J, 8, &rec, N1 * 10));
  TRY(scratch(s, J, 9, &dseg, (size_t)ncam + 1));
  CK(cudaMemcpyAsync(dseg, seg.data(), sizeof(uint32_t) * (ncam + 1), cudaMemcpyHostToDevice, st));
  // depth key bits: every splat's zc lies in (z_near, z_far) of its camera, so
  // zc bits - (the batch's smallest z_near bits) fit in zb bits (27 at the
  // synthetic configs' 0.01 .. 8 instead of 32: one radix pass less)
  uint32_t zlo = 0xFFFFFFFFu, zhi = 0u;
  for (int q = 0; q < ncam; ++q) {
    uint32_t a, b;
    std::memcpy(&a, &hcams[c0 + q].z_near, 4);
    std::memcpy(&b, &hcams[c0 + q].z_far, 4);
    zlo = std::min(zlo, a);
    zhi = std::max(zhi, b);
  }
  int zb = 1;
  while (zb < 32 && (1ull << zb) <= (unsigned long long)(zhi - zlo)) ++zb;
  KL(launch_rvis_fill(k0, nk, (int)c0, s->cam_order, s->pair_tile, s->pair_cam, s->rows, s->words, pos, prec, drc,
                      zlo, zb, keys, vals, rec, rcam, st));
  // 2. front to back per camera: (zc, caller index) -- one radix sort on
  //    (camera, zc bits), then runs of equal depth ordered by caller index
  if (n > 0) {
    int cb = 1;
    while ((1 << cb) < ncam) ++cb;
    size_t tb = 0;
    CK(sort_u64_pairs(nullptr, tb, keys, keys_s, vals, vals_s, (int64_t)n, zb + cb, st));
    uint8_t* tmp = nullptr;
    TRY(scratch(s, J, 10, &tmp, tb));
    CUBL(sort_u64_pairs(tmp, tb, keys, keys_s, vals, vals_s, (int64_t)n, zb + cb, st));
    KL(launch_tie_fix((int64_t)n, keys_s, vals_s, rec, st));
  }
  // 3. tile binning in front-to-back order (stable key sort keeps it)
  uint32_t *c2 = nullptr, *o2 = nullptr;
  TRY(scratch(s, J, 1, &c2, N1 + 1));
  TRY(scratch(s, J, 2, &o2, N1 + 1));
  CK(cudaMemsetAsync(c2 + n, 0, sizeof(uint32_t), st));
  KL(launch_bin_count((int64_t)n, vals_s, rec, rcam, drc, c2, st));
  uint64_t E = 0;
  TRY(scan_counts(s, c2, o2, (int64_t)n, &E));
  uint32_t *ek = nullptr, *ev = nullptr, *ek_s = nullptr, *ev_s = nullptr;
  const size_t E1 = std::max<uint64_t>(E, 1);
  TRY(scratch(s, J, 11, &ek, E1)); TRY(scratch(s, J, 12, &ev, E1));
  TRY(scratch(s, J, 13, &ek_s, E1)); TRY(scratch(s, J, 14, &ev_s, E1));
  KL(launch_bin_fill((int64_t)n, vals_s, rec, rcam, drc, o2, ek, ev, st));
  int bits = 1;
  while ((1ull << bits) < (unsigned long long)tiles) ++bits;
  if (E > 0) {
    size_t tb = 0;
    CK(sort_u32_pairs(nullptr, tb, ek, ek_s, ev, ev_s, (int64_t)E, bits, st));
    uint8_t* tmp = nullptr;
    TRY(scratch(s, J, 10, &tmp, tb));
    CUBL(sort_u32_pairs(tmp, tb, ek, ek_s, ev, ev_s, (int64_t)E, bits, st));
  }
  uint32_t *ts = nullptr, *te = nullptr;
  TRY(scratch(s, J, 15, &ts, (size_t)tiles + 1));
  TRY(scratch(s, J, 16, &te, (size_t)tiles + 1));
  CK(cudaMemsetAsync(ts, 0, sizeof(uint32_t) * (tiles + 1), st));
  CK(cudaMemsetAsync(te, 0, sizeof(uint32_t) * (tiles + 1), st));
  KL(launch_tile_ranges((int64_t)E, ek_s, ts, te, st));
  // 4. render
  float *Dm = nullptr, *Wm = nullptr;
  TRY(scratch(s, J, 17, &Dm, (size_t)std::max<int64_t>(maps, 1)));
  TRY(scratch(s, J, 18, &Wm, (size_t)std::max<int64_t>(maps, 1)));
  std::pair<cudaEvent_t, cudaEvent_t> ke{nullptr, nullptr};
  if (J.counters && cudaEventCreate(&ke.first) == cudaSuccess && cudaEventCreate(&ke.second) == cudaSuccess) {
    J.kev.push_back(ke);
    CK(cudaEventRecord(ke.first, st));
  }
  KL(launch_render(ncam, max_tiles, drc, ts, te, ev_s, rec, Dm, Wm, J.counters, st));
  if (ke.second) CK(cudaEventRecord(ke.second, st));
  if (J.Dout) TRY(copy_out(s, J.Dout, Dm, sizeof(float) * (size_t)rc[0].Wd * rc[0].Hd));
  if (J.Wout) TRY(copy_out(s, J.Wout, Wm, sizeof(float) * (size_t)rc[0].Wd * rc[0].Hd));
  // 5. back-projection of every stride-th pixel with weight >= eps_w
  const uint32_t ns = sp0[ncam];
  uint32_t *flag = nullptr, *foff = nullptr, *dsp0 = nullptr;
  TRY(scratch(s, J, 11, &flag, (size_t)ns + 1));
  TRY(scratch(s, J, 12, &foff, (size_t)ns + 1));
  TRY(scratch(s, J, 19, &dsp0, (size_t)ncam + 1));
  CK(cudaMemcpyAsync(dsp0, sp0.data(), sizeof(uint32_t) * (ncam + 1), cudaMemcpyHostToDevice, st));
  CK(cudaMemsetAsync(flag + ns, 0, sizeof(uint32_t), st));
  KL(launch_bp_count(ncam, max_samples, drc, J.stride, J.eps_w, Wm, dsp0, flag, st));
  uint64_t np = 0;
  TRY(scan_counts(s, flag, foff, ns, &np));
  TRY(grow_cloud(s, J, J.n + (int64_t)np));
  PrepIn fr{};
  for (int a = 0; a < 3; ++a) {
    fr.c0[a] = s->frame.center[a];
    fr.au[a] = s->frame.axis_u[a];
    fr.av[a] = s->frame.axis_v[a];
  }
  fr.rho = s->frame.radius;
  KL(launch_bp_write(ncam, max_samples, drc, J.stride, Dm, dsp0, flag, foff, fr, s->mm, (uint32_t)J.n, J.gu, J.gv,
                     J.cam, st));
  J.n += (int64_t)np;
  return LOBE_OK;
}


// a4, the per-camera depth statistic over the non-empty (tile, camera) pairs of
// the load pass, enqueued once on `st` (the scene's stream, or the depth side
// stream; see lobe_load_scene). Its scratch lives and dies on `st`.
// CTAs per SM of k_depth_pairs when it runs on the depth side stream next to the
// evaluation / crop kernels (LOBE_A4_CTAS overrides; 0 = full occupancy, two waves)
static int a4_side_ctas() {
  static const int v = [] {
    const char* e = std::getenv("LOBE_A4_CTAS");
    return e ? std::atoi(e) : 3;
  }();
  return v;
}

// ... and when it runs alone on the scene's stream (deferred): one resident
// wave over the tile queue at full occupancy (LOBE_A4_CTAS_ALONE overrides;
// 0 = two waves, grid-stride)
static int a4_alone_ctas() {
  static const int v = [] {
    const char* e = std::getenv("LOBE_A4_CTAS_ALONE");
    return e ? std::atoi(e) : 4;
  }();
  return v;
}

lobe_status launch_a4(lobe_scene* s, cudaStream_t st, bool side) {
  const int64_t NL = std::max<int64_t>(s->N_loc, 1), cap = s->a4_cap, tw = s->a4_tw;
  if (s->N_loc > 0) {
    KL(launch_depth_pairs(s->n_tiles, s->tile_off, s->pair_cam, s->rows, s->words,
                          reinterpret_cast<const float4*>(s->xy), reinterpret_cast<const float4*>(s->zk),
                          reinterpret_cast<const float2*>(s->o2), s->cams, s->pair_part,
                          side ? a4_side_ctas() : a4_alone_ctas(), s->queue + 1, st));
    // pair indices in camera-major order, tile order within a camera
    uint32_t *ccount = nullptr, *wordpre = nullptr;
    CK(malloc_async(&ccount, sizeof(uint32_t) * ((size_t)NL + 1), st));
    CK(malloc_async(&wordpre, sizeof(uint32_t) * (size_t)NL * tw, st));
    CK(cudaMemsetAsync(ccount + NL, 0, sizeof(uint32_t), st));
    KL(launch_cam_order(s->N_loc, tw, s->camtile, wordpre, ccount, st));
    size_t sb2 = 0;
    CK(exclusive_scan_u32(nullptr, sb2, ccount, s->cam_off, NL + 1, st));
    void* tmp2 = nullptr;
    CK(malloc_async(&tmp2, sb2, st));
    CUBL(exclusive_scan_u32(tmp2, sb2, ccount, s->cam_off, NL + 1, st));
    cudaFreeAsync(tmp2, st);
    cudaFreeAsync(ccount, st);
    if (s->a4_kept > 0)
      KL(launch_cam_scatter(s->tile_off, s->n_tiles, cap, s->pair_cam, s->pair_tile, s->camtile, wordpre, tw,
                            s->cam_off, s->cam_order, st));
    cudaFreeAsync(wordpre, st);
    KL(launch_depth_reduce(s->N_loc, s->cam_off, s->cam_order, s->pair_part, s->K, s->D, s->zmin, s->zmax, st));
  }
  if (s->camtile) cudaFreeAsync(s->camtile, st);
  s->camtile = nullptr;
  CK(cudaEventRecord(s->ev[12], st));
  return LOBE_OK;
}

// a4's results for the scene's stream: a deferred a4 is enqueued now; an a4
// running on the depth side stream is joined (the scene's stream waits for it)
// when `join` is set.
lobe_status ensure_a4(lobe_scene* s, bool join = true) {
  if (s->a4_pending) {
    s->a4_pending = false;
    CK(cudaEventRecord(s->ev[11], s->stream));
    return launch_a4(s, s->stream, false);
  }
  if (s->a4_side && join && !s->a4_joined) {
    CK(cudaStreamWaitEvent(s->stream, s->ev[12], 0));
    s->a4_joined = true;
  }
  return LOBE_OK;
}

// Load-pass timings and counters (events and pinned counters of the last load).
void finalize_load_stats(lobe_scene* s) {
  if (!s->stats_pending) return;
  ensure_a4(s);
  cudaStreamSynchronize(s->stream);
  s->st.t_prep_ms = ms_between(s->ev[0], s->ev[1]);
  // visibility pass = culling kernel + test kernel (list building excluded)
  s->st.t_cull_ms = ms_between(s->ev[1], s->ev[8]);
  // slice classification (k_slice_codes) is part of the test decision
  const float t_codes = (s->kept_pairs_last > 0) ? ms_between(s->ev[16], s->ev[17]) : 0.f;
  s->st.t_vis_ms = s->st.t_cull_ms + t_codes + ms_between(s->ev[9], s->ev[10]);
  s->st.t_depth_ms = ms_between(s->ev[11], s->ev[12]);
  s->n_pairs = s->pin->n_pairs;
  s->st.tile_pairs = (uint64_t)s->n_pairs;
  s->st.kept_tests = (uint64_t)s->kept_pairs_last * (uint64_t)kTile;  // pairs surviving the tile bound
  // exact tests run, counted by the test kernels (real Gaussians of the undecided
  // slices, less the anisotropic pair groups their own box decided)
  s->st.dense_tests = (uint64_t)s->pin->vc[11];
  s->st.accepted_tests = (uint64_t)s->pin->vc[10];  // slices and (anisotropic) pair groups accepted
  for (int p = 0; p < 9; ++p) s->st.exact_pattern_tests[p] = (uint64_t)s->pin->vc[16 + p] * (uint64_t)(kTile / 4);
  for (int v = 0; v < 4; ++v) s->st.exact_variant_tests[v] = s->st.exact_pattern_tests[v];
  s->st.exact_variant_tests[4] = s->st.exact_pattern_tests[4] + s->st.exact_pattern_tests[5] +
                                 s->st.exact_pattern_tests[6] + s->st.exact_pattern_tests[7];
  s->st.exact_variant_tests[5] = s->st.exact_pattern_tests[8];
  // I16, counted by k_cull / k_vis_tiles themselves (VisArgs::counters [8..13])
  uint64_t decided = 0;
  for (int k = 0; k < 4; ++k) decided += (s->st.decided_tests[k] = (uint64_t)s->pin->vc[8 + k]);
  s->st.visible_bits[0] = (uint64_t)s->pin->vc[12];
  s->st.visible_bits[1] = (uint64_t)s->pin->vc[13];
  s->st.tests_executed += decided;
  s->stats_pending = false;
}

// Pinned staging blocks, recycled across scenes (cudaFreeHost would synchronise).
std::mutex g_pin_mu;
std::vector<void*> g_pin_free;
lobe_scene::Pinned* acquire_pinned() {
  {
    std::lock_guard<std::mutex> lk(g_pin_mu);
    if (!g_pin_free.empty()) {
      void* p = g_pin_free.back();
      g_pin_free.pop_back();
      return static_cast<lobe_scene::Pinned*>(p);
    }
  }
  void* p = nullptr;
  if (cudaMallocHost(&p, sizeof(lobe_scene::Pinned)) != cudaSuccess) return nullptr;
  return static_cast<lobe_scene::Pinned*>(p);
}
void recycle_pinned(lobe_scene::Pinned* p) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_pin_mu);
  g_pin_free.push_back(p);
}
std::vector<std::pair<uint8_t*, size_t>> g_pin_out_free;
uint8_t* acquire_pinned_out(size_t need, size_t* cap) {
  {
    std::lock_guard<std::mutex> lk(g_pin_mu);
    for (size_t i = 0; i < g_pin_out_free.size(); ++i)
      if (g_pin_out_free[i].second >= need) {
        auto e = g_pin_out_free[i];
        g_pin_out_free.erase(g_pin_out_free.begin() + i);
        *cap = e.second;
        return e.first;
      }
  }
  void* p = nullptr;
  if (cudaMallocHost(&p, need) != cudaSuccess) return nullptr;
  *cap = need;
  return static_cast<uint8_t*>(p);
}
void recycle_pinned_out(uint8_t* p, size_t cap) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_pin_mu);
  g_pin_out_free.emplace_back(p, cap);
}

// Timing events of a scene, recycled across scenes as one set per device.
std::vector<std::pair<int, std::array<cudaEvent_t, kNumEvents>>> g_ev_free;
void acquire_events(int device, cudaEvent_t (&ev)[kNumEvents]) {
  {
    std::lock_guard<std::mutex> lk(g_pin_mu);
    for (size_t i = 0; i < g_ev_free.size(); ++i)
      if (g_ev_free[i].first == device) {
        for (int k = 0; k < kNumEvents; ++k) ev[k] = g_ev_free[i].second[k];
        g_ev_free.erase(g_ev_free.begin() + i);
        return;
      }
  }
  for (auto& e : ev) cudaEventCreate(&e);
}
void recycle_events(int device, cudaEvent_t (&ev)[kNumEvents]) {
  std::array<cudaEvent_t, kNumEvents> a;
  for (int k = 0; k < kNumEvents; ++k) {
    if (!ev[k]) {  // incomplete set: destroy it
      for (auto& e : ev)
        if (e) cudaEventDestroy(e);
      return;
    }
    a[k] = ev[k];
  }
  std::lock_guard<std::mutex> lk(g_pin_mu);
  g_ev_free.emplace_back(device, a);
}

// Side streams for the per-camera copies, recycled across scenes (one per
// live scene; creating a stream costs ~0.4 ms).
std::vector<std::pair<int, cudaStream_t>> g_side_free;
cudaStream_t acquire_side_stream(int device) {
  {
    std::lock_guard<std::mutex> lk(g_pin_mu);
    for (size_t i = 0; i < g_side_free.size(); ++i)
      if (g_side_free[i].first == device) {
        cudaStream_t st = g_side_free[i].second;
        g_side_free.erase(g_side_free.begin() + i);
        return st;
      }
  }
  cudaStream_t st = nullptr;
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
  return st;
}
void recycle_side_stream(int device, cudaStream_t st) {
  std::lock_guard<std::mutex> lk(g_pin_mu);
  g_side_free.emplace_back(device, st);
}

// Per-camera outputs: asynchronous copies into pinned staging when the
// destination is ordinary pageable host memory, one synchronisation, then host
// copies into the caller's buffers (out_plan collects them).
struct StagedCopy { void* dst; size_t off, bytes; };
lobe_status stage_out(lobe_scene* s, std::vector<StagedCopy>& plan, size_t& used, void* dst, const void* src,
                      size_t bytes) {
  if (!dst || bytes == 0) return LOBE_OK;
  cudaPointerAttributes at{};
  const bool pageable = cudaPointerGetAttributes(&at, dst) != cudaSuccess || at.type == cudaMemoryTypeUnregistered;
  cudaGetLastError();  // clear a possible error of the attribute query
  if (!pageable) {
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, s->stream));
    return LOBE_OK;
  }
  plan.push_back(StagedCopy{dst, used, bytes});
  used += (bytes + 15) & ~size_t(15);
  return LOBE_OK;
}
lobe_status run_staged(lobe_scene* s, std::vector<StagedCopy>& plan, size_t used,
                       const std::vector<const void*>& srcs, cudaEvent_t after = nullptr) {
  if (plan.empty()) {
    CK(cudaStreamSynchronize(s->stream));
    return LOBE_OK;
  }
  // The copies run on a side stream that waits only for the end of the last
  // evaluation (ev[4]): kernels enqueued after it on the scene's stream (e.g.
  // a crop) keep running while the host copies out.
  if (!s->side) s->side = acquire_side_stream(s->device);
  if (!s->side) return fail(LOBE_E_CUDA, "side stream creation failed");
  if (used > s->pin_out_cap) {
    // the old block's copies ran on the side stream, which every call drains
    // before returning (below); a scene's first call has no block yet. No wait
    // on the scene's stream: a crop enqueued there keeps running.
    if (s->pin_out) {
      CK(cudaStreamSynchronize(s->side));
      recycle_pinned_out(s->pin_out, s->pin_out_cap);
    }
    s->pin_out = acquire_pinned_out(used, &s->pin_out_cap);
    if (!s->pin_out) {
      s->pin_out_cap = 0;
      return fail(LOBE_E_CUDA, "pinned staging allocation failed");
    }
  }
  CK(cudaStreamWaitEvent(s->side, after ? after : s->ev[4], 0));
  CK(cudaStreamWaitEvent(s->side, s->ev[12], 0));  // a4 (K, D, z_min, z_max), launched before the copies
  for (size_t i = 0; i < plan.size(); ++i)
    CK(cudaMemcpyAsync(s->pin_out + plan[i].off, srcs[i], plan[i].bytes, cudaMemcpyDeviceToHost, s->side));
  CK(cudaStreamSynchronize(s->side));
  for (const auto& c : plan) std::memcpy(c.dst, s->pin_out + c.off, c.bytes);
  CK(cudaEventSynchronize(s->ev[4]));  // device destinations (scene stream) are ordered after it anyway
  return LOBE_OK;
}

lobe_status copy_out(lobe_scene* s, void* dst, const void* src, size_t bytes) {
  if (!dst || bytes == 0) return LOBE_OK;
  CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, s->stream));
  return LOBE_OK;
}

}  // namespace

// ============================================================================
// The deferred quaternion verdict of a host-input load (isotropic mode): known
// once event 20 has completed. wait = false: report it only if already decided
// (the call then refuses to run on an invalid scene); wait = true: decide now.
static lobe_status scene_verdict(const lobe_scene* s, bool wait) {
  if (!s) return LOBE_OK;
  if (s->q_pending) {
    if (!wait && cudaEventQuery(s->ev[20]) == cudaErrorNotReady) return LOBE_OK;
    if (cudaEventSynchronize(s->ev[20]) != cudaSuccess) return fail(LOBE_E_CUDA, "quaternion check");
    s->q_pending = false;
    if (s->pin->q_err) {
      s->q_status = LOBE_E_INVALID_INPUT;
      s->q_first_bad = s->pin->q_bad;
    }
  }
  if (s->q_status != LOBE_OK)
    return fail(s->q_status, "gaussian " + std::to_string(s->q_first_bad) +
                                 " invalid (|q| = 1 +- 1e-6, SPEC.md:30-33; reported after the load: the quaternions "
                                 "of a host-input load are checked while the device works)");
  return LOBE_OK;
}

extern "C" {

const char* lobe_last_error(void) { return g_err.c_str(); }

const char* lobe_version(void) {
  return "lobe 0.1 sm_100a (-fmad=false, IEEE div/sqrt, FFMA2 visibility, tile lists)";
}

size_t lobe_mask_words(const lobe_scene* s) { return s ? (size_t)s->words : 0; }

void lobe_free_scene(lobe_scene* s) {
  if (!s) return;
  cudaSetDevice(s->device);
  if (s->a4_side && !s->a4_joined) cudaStreamWaitEvent(s->stream, s->ev[12], 0);  // a4 reads what is freed below
  bool synced = false;
  for (auto& b : s->rscratch)  // render-selection scratch (plain cudaMalloc blocks)
    if (b.p) {
      if (!synced) cudaStreamSynchronize(s->stream);
      synced = true;
      cudaFree(b.p);
      b.p = nullptr;
      b.cap = 0;
    }
  s->release(s->xy); s->release(s->zk); s->release(s->o2); s->release(s->gu); s->release(s->gv); s->release(s->wbox);
  s->release(s->iperm); s->release(s->cams); s->release(s->cam_pat); s->release(s->d_cam_gu); s->release(s->d_cam_gv);
  s->release(s->rows); s->release(s->flags); s->release(s->nonempty); s->release(s->pair_part); s->release(s->cam_off); s->release(s->cam_order);
  s->release(s->tile_lo); s->release(s->tile_hi); s->release(s->chunk_lo); s->release(s->chunk_hi); s->release(s->cv); s->release(s->acams); s->release(s->cloud_gu); s->release(s->cloud_gv); s->release(s->cloud_cam); s->release(s->cloud_K); s->release(s->slice_lo); s->release(s->slice_hi); s->release(s->codes); s->release(s->group_lo); s->release(s->group_hi); s->release(s->gcodes); s->release(s->vcnt); s->release(s->keep); s->release(s->kept);
  s->release(s->koff); s->release(s->klist); s->release(s->unit_tile); s->release(s->unit_meta); s->release(s->queue); s->release(s->K); s->release(s->D);
  s->release(s->zmin); s->release(s->zmax); s->release(s->tile_off); s->release(s->pair_cam);
  s->release(s->pair_tile); s->release(s->zp); s->release(s->word_zone); s->release(s->tile_zone);
  s->release(s->zp_count); s->release(s->dz); s->release(s->d_zp_cell); s->release(s->hist);
  s->release(s->ncb); s->release(s->n0cb); s->release(s->member); s->release(s->sel); s->release(s->home);
  s->release(s->counts); s->incid = nullptr; s->release(s->masks); s->release(s->camtile);
  s->release(s->own_masks); s->release(s->d_xcounts);
  cudaStreamSynchronize(s->stream);
  delete s->xops;
  lobe::comm_release_scene(s->comm);
  if (s->side) {
    cudaStreamSynchronize(s->side);
    recycle_side_stream(s->device, s->side);  // stream creation costs ~0.4 ms: reuse across scenes
  }
  if (s->qstream) {
    cudaStreamSynchronize(s->qstream);
    recycle_side_stream(s->device, s->qstream);
  }
  if (s->dstream) {
    cudaStreamSynchronize(s->dstream);
    recycle_side_stream(s->device, s->dstream);
  }
  recycle_events(s->device, s->ev);  // event creation costs ~2 us each: reuse across scenes
  recycle_pinned(s->pin);
  recycle_pinned_out(s->pin_out, s->pin_out_cap);
  recycle_pinned_out(s->pin_in, s->pin_in_cap);  // the load's camera staging (its copies are complete)
  delete s;
}

lobe_status lobe_load_scene(const lobe_gaussians* g, const lobe_camera* cams, int64_t n_cams, lobe_frame* inout_frame,
                            const lobe_options* opt, lobe_scene** out) {
  LOBE_NVTX("lobe_load_scene");
  HostTimeline tl;
  g_err.clear();
  if (!out) return fail(LOBE_E_INVALID_CONFIG, "out is NULL");
  *out = nullptr;
  if (!g || !cams) return fail(LOBE_E_INVALID_CONFIG, "gaussians/cameras NULL");
  if (g->n <= 0) return fail(LOBE_E_INVALID_CONFIG, "gaussian count must be > 0 (SPEC.md:110)");
  if (g->n > (int64_t)INT32_MAX - 2 * kChunk) return fail(LOBE_E_INVALID_CONFIG, "too many Gaussians");
  lobe_options o{};
  o.world = 1;
  if (opt) o = *opt;
  if (o.world < 1 || o.rank < 0 || o.rank >= o.world) return fail(LOBE_E_INVALID_CONFIG, "bad rank/world");
  if (o.assign_mode < 0 || o.assign_mode > 2) return fail(LOBE_E_INVALID_CONFIG, "bad assign_mode");
  if (o.predicate != LOBE_PREDICATE_ISOTROPIC && o.predicate != LOBE_PREDICATE_ANISOTROPIC)
    return fail(LOBE_E_INVALID_CONFIG, "bad predicate");
  if (n_cams <= 0) return fail(LOBE_E_INVALID_CONFIG, "n_cams must be > 0 (SPEC.md:110)");
  // validate_cameras runs later, while the device works on a1 (checked before
  // the load's first synchronisation); invalid cameras only yield garbage in
  // that window, never an out-of-range index
  lobe_frame F{};
  if (inout_frame) F = *inout_frame;
  else F.auto_flags = LOBE_FRAME_AUTO_ALL;
  TRY(resolve_frame(cams, n_cams, &F));
  tl.mark("resolve_frame");

  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(LOBE_E_CUDA, "no CUDA device");
  CK(cudaSetDevice(o.device));
  {  // keep freed pool memory for the next scene (stream-ordered allocator)
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, o.device) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  lobe_scene* s = new lobe_scene();
  s->device = o.device;
  s->stream = static_cast<cudaStream_t>(o.stream);
  s->rank = o.rank;
  s->world = o.world;
  s->assign_mode = o.assign_mode;
  s->aniso = (o.predicate == LOBE_PREDICATE_ANISOTROPIC);
  s->frame = F;
  cudaDeviceGetAttribute(&s->num_sms, cudaDevAttrMultiProcessorCount, o.device);
  acquire_events(o.device, s->ev);
  s->pin = acquire_pinned();
  if (!s->pin) {
    delete s;
    return fail(LOBE_E_CUDA, "pinned staging allocation failed");
  }
  tl.mark("scene setup");
  lobe_status rs = [&]() -> lobe_status {
    cudaStream_t st = s->stream;
    {  // communicator first: NCCL creation is collective (every rank is in this call)
      std::string cerr;
      const lobe_status cs = lobe::comm_acquire(o, &s->comm, &cerr);
      if (cs != LOBE_OK) return fail(cs, cerr);
      if (s->comm) {
        s->xops = lobe::comm_device_ops(s->comm, o.device, st);
        CK(s->alloc(&s->d_xcounts, 2 * kMaxBlocks));
      }
    }
    const int64_t G = g->n;
    s->G = G;
    s->G_pad = (G + kChunk - 1) / kChunk * kChunk;
    s->words = s->G_pad / 32;
    s->n_tiles = s->G_pad / kTile;
    s->n_chunks = s->G_pad / kChunk;
    s->N_all = n_cams;
    s->cam_begin = (int64_t)o.rank * n_cams / o.world;
    const int64_t cam_end = (int64_t)(o.rank + 1) * n_cams / o.world;
    s->N_loc = cam_end - s->cam_begin;

    tl.mark("comm");
    CK(cudaEventRecord(s->ev[0], st));
    // ---- inputs on device
    const float* src[11] = {g->x, g->y, g->z, g->sx, g->sy, g->sz, g->qw, g->qx, g->qy, g->qz, g->opacity};
    for (int k = 0; k < 11; ++k)
      if (!src[k]) return fail(LOBE_E_INVALID_CONFIG, "gaussian array NULL");
    float* dev_in = nullptr;
    const float* din[11];
    // host inputs in the isotropic mode: the quaternions are only validated, so
    // they travel last on a side stream (with their check) while the device runs
    // a1 / a3 on the other fields; the verdict is read before the load returns
    const bool q_defer = !g->on_device && !s->aniso;
    uint32_t* q_flags = nullptr;  // [0] err, [1..2] first bad index (u64)
    if (!g->on_device) {
      CK(s->alloc(&dev_in, (size_t)11 * G));
      for (int k = 0; k < 11; ++k) din[k] = dev_in + (size_t)k * G;
      if (q_defer) {
        // the copy engine is the bound of a host-input load (440 MB): positions
        // first on the scene's stream, so the sort keys and the sort run while
        // the scales and opacities follow on the side stream (strictly after
        // the positions: event 23), then the camera tables, then the quaternions
        if (!s->qstream) s->qstream = acquire_side_stream(s->device);
        if (!s->qstream) return fail(LOBE_E_CUDA, "side stream creation failed");
        for (int k = 0; k < 3; ++k)
          CK(cudaMemcpyAsync(dev_in + (size_t)k * G, src[k], sizeof(float) * G, cudaMemcpyHostToDevice, st));
        CK(cudaEventRecord(s->ev[23], st));
        CK(cudaStreamWaitEvent(s->qstream, s->ev[23], 0));
        for (int k : {3, 4, 5, 10})
          CK(cudaMemcpyAsync(dev_in + (size_t)k * G, src[k], sizeof(float) * G, cudaMemcpyHostToDevice,
                             s->qstream));
        CK(cudaEventRecord(s->ev[24], s->qstream));
        CK(s->alloc(&q_flags, 4));
        // {0, first bad = ~0}: memsets, not pageable copies (those block this
        // thread until the copy engine reaches them, behind the field copies)
        CK(cudaMemsetAsync(q_flags, 0, 2 * sizeof(uint32_t), st));
        CK(cudaMemsetAsync(q_flags + 2, 0xff, 2 * sizeof(uint32_t), st));
      } else {
        for (int k = 0; k < 11; ++k)
          CK(cudaMemcpyAsync(dev_in + (size_t)k * G, src[k], sizeof(float) * G, cudaMemcpyHostToDevice, st));
      }
    } else {
      for (int k = 0; k < 11; ++k) din[k] = src[k];
    }
    // camera buffers now (stream-ordered allocations a side stream may write)
    const int64_t NLc = std::max<int64_t>(s->N_loc, 1);
    float* cr = nullptr;  // camera-centre raw grid coordinates
    CK(s->alloc(&s->cams, NLc));
    CK(s->alloc(&s->cam_pat, (size_t)NLc * kPatterns));
    CK(s->alloc(&s->d_cam_gu, NLc));
    CK(s->alloc(&s->d_cam_gv, NLc));
    if (s->aniso) CK(s->alloc(&s->acams, NLc));
    CK(s->alloc(&cr, (size_t)2 * NLc));
    if (q_defer) CK(cudaEventRecord(s->ev[20], s->qstream));  // the camera copies follow the fields' copies
    // ---- a1 precompute

    float4* rec;
    uint32_t *keys, *keys_s, *scratch;
    int32_t *vals, *perm;
    unsigned long long* err_idx;

    float* cov_raw = nullptr;  // anisotropic: Sigma per Gaussian, caller order
    if (s->aniso) CK(s->alloc(&cov_raw, (size_t)6 * G));
    CK(s->alloc(&rec, (size_t)2 * G));
    CK(s->alloc(&keys, G)); CK(s->alloc(&keys_s, G)); CK(s->alloc(&vals, G)); CK(s->alloc(&perm, G));
    CK(s->alloc(&scratch, 8)); CK(s->alloc(&err_idx, 1));
    // {err 0, min_u ~0, max_u 0, min_v ~0, max_v 0, 0, 0, 0} and err_idx = ~0 (memsets:
    // no pageable copies behind the field copies)
    CK(cudaMemsetAsync(scratch, 0, 8 * sizeof(uint32_t), st));
    CK(cudaMemsetAsync(scratch + 1, 0xff, sizeof(uint32_t), st));
    CK(cudaMemsetAsync(scratch + 3, 0xff, sizeof(uint32_t), st));
    CK(cudaMemsetAsync(err_idx, 0xff, sizeof(unsigned long long), st));
    PrepIn pin{};
    pin.x = din[0]; pin.y = din[1]; pin.z = din[2]; pin.sx = din[3]; pin.sy = din[4]; pin.sz = din[5];
    pin.qw = din[6]; pin.qx = din[7]; pin.qy = din[8]; pin.qz = din[9]; pin.o = din[10];
    pin.G = G;
    for (int a = 0; a < 3; ++a) {
      pin.c0[a] = F.center[a];
      pin.au[a] = F.axis_u[a];
      pin.av[a] = F.axis_v[a];
    }
    pin.rho = F.radius;
    pin.cov = cov_raw;
    pin.q_deferred = q_defer ? 1 : 0;
    tl.mark("inputs + a1 allocs");
    // split host-input path: sort keys from the positions now, the records once
    // the other fields have landed (after the sort, below)
    pin.pass = q_defer ? 1 : 0;
    KL(launch_prep_raw(pin, rec, keys, vals, scratch, err_idx, scratch + 1, st));
    tl.mark("k_prep_raw launched");
    size_t tmpb = 0;
    CK(radix_sort_pairs(nullptr, tmpb, keys, keys_s, vals, perm, G, st, 0, 30));  // all 30 bits of the Hilbert keys (24 bits of the Morton order: tiles less compact, the evaluation 7 % slower)
    void* tmp = nullptr;
    CK(malloc_async(&tmp, tmpb, st));
    CUBL(radix_sort_pairs(tmp, tmpb, keys, keys_s, vals, perm, G, st, 0, 30));
    if (q_defer) {
      CK(cudaStreamWaitEvent(st, s->ev[24], 0));
      pin.pass = 2;
      KL(launch_prep_raw(pin, rec, keys, vals, scratch, err_idx, scratch + 1, st));
    }
    // validation flags and the ground min / max reach the host asynchronously;
    // they are checked at the first synchronisation (after the culling pass)
    KL(launch_upload(s->pin->prep_hs, scratch, sizeof(s->pin->prep_hs), st));
    KL(launch_upload(&s->pin->prep_bad, err_idx, sizeof(s->pin->prep_bad), st));
    CK(s->alloc(&s->xy, (size_t)s->G_pad * 2));
    CK(s->alloc(&s->zk, (size_t)s->G_pad * 2));
    CK(s->alloc(&s->o2, (size_t)s->G_pad));
    CK(s->alloc(&s->gu, (size_t)s->G_pad));
    CK(s->alloc(&s->gv, (size_t)s->G_pad));
    CK(s->alloc(&s->wbox, (size_t)s->G_pad / 32));
    CK(s->alloc(&s->iperm, (size_t)G));
    if (s->aniso) CK(s->alloc(&s->cv, (size_t)s->G_pad / 2 * 3));
    KLN(launch_pack(G, s->G_pad, perm, rec, scratch + 1, s->xy, s->zk, s->o2, s->gu, s->gv, s->iperm, cov_raw, s->cv, s->wbox, st), 2);
    tl.mark("sort + k_pack launched");
    s->release(cov_raw);
    cudaFreeAsync(tmp, st);
    s->release(rec);
    s->release(keys); s->release(keys_s); s->release(vals); s->release(perm);
    s->release(err_idx);
    float* dev_in_q = nullptr;  // deferred path: freed after the quaternion check (below)
    if (dev_in && q_defer) {
      dev_in_q = dev_in;
      dev_in = nullptr;
    }
    if (dev_in) s->release(dev_in);

    // ---- a2 camera setup (local shard) + camera-centre grid coords
    std::vector<CamSetup> hset(std::max<int64_t>(s->N_loc, 1));
    std::vector<AnisoCam> haset(std::max<int64_t>(s->N_loc, 1));
    s->host_cams.assign(cams + s->cam_begin, cams + s->cam_begin + s->N_loc);
    std::vector<float> cam_ru(std::max<int64_t>(s->N_loc, 1)), cam_rv(std::max<int64_t>(s->N_loc, 1));
    for (int64_t c = 0; c < s->N_loc; ++c) {  // host work overlapping the device's a1 pass
      const lobe_camera& k = cams[s->cam_begin + c];
      hset[c] = camera_setup(k);
      if (s->aniso) {
        haset[c] = aniso_setup(k);
        // branch-free reciprocal / square root need depths in [2^-126, 2^126]
        if (!(haset[c].zn >= 0x1p-126f && haset[c].zf <= 0x1p126f)) s->aniso_fast = false;
      }
      double oc[3];
      cam_centre(k, oc);
      ground_uv_host((float)oc[0], (float)oc[1], (float)oc[2], F, &cam_ru[c], &cam_rv[c]);
    }
    const int64_t NL = NLc;
    // with deferred quaternions the H2D engine is shared: the camera copies go
    // first, on the side stream (the H2D engine serves copies in issue order,
    // and copies queued on the scene's stream behind k_pack would wait for the
    // 160 MB of quaternions); the scene's stream waits for them (event 22)
    cudaStream_t cst = q_defer ? s->qstream : st;
    if (q_defer) CK(cudaStreamWaitEvent(cst, s->ev[20], 0));
    // staged in pinned memory: a pageable copy would block this thread until the
    // copy engine reaches it (behind the bulk field copies of a host-input load)
    const size_t b_set = sizeof(CamSetup) * NL, b_aset = s->aniso ? sizeof(AnisoCam) * NL : 0,
                 b_r = sizeof(float) * NL;
    const size_t o_aset = (b_set + 255) & ~(size_t)255, o_r = (o_aset + b_aset + 255) & ~(size_t)255;
    const size_t need_in = o_r + 2 * b_r;
    if (need_in > s->pin_in_cap) {
      recycle_pinned_out(s->pin_in, s->pin_in_cap);  // a new scene: nothing in flight uses it yet
      s->pin_in = acquire_pinned_out(need_in, &s->pin_in_cap);
      if (!s->pin_in) {
        s->pin_in_cap = 0;
        return fail(LOBE_E_CUDA, "pinned staging allocation failed");
      }
    }
    std::memcpy(s->pin_in, hset.data(), b_set);
    if (b_aset) std::memcpy(s->pin_in + o_aset, haset.data(), b_aset);
    std::memcpy(s->pin_in + o_r, cam_ru.data(), b_r);
    std::memcpy(s->pin_in + o_r + b_r, cam_rv.data(), b_r);
    CK(cudaMemcpyAsync(s->cams, s->pin_in, b_set, cudaMemcpyHostToDevice, cst));
    if (s->aniso) CK(cudaMemcpyAsync(s->acams, s->pin_in + o_aset, b_aset, cudaMemcpyHostToDevice, cst));
    {  // camera-centre grid coordinates, normalised on the device with k_prep_raw's min / max
      CK(cudaMemcpyAsync(cr, s->pin_in + o_r, 2 * b_r, cudaMemcpyHostToDevice, cst));
      if (q_defer) {
        CK(cudaEventRecord(s->ev[22], cst));
        CK(cudaStreamWaitEvent(st, s->ev[22], 0));
        // now the quaternions (side stream) and their check
        for (int k = 6; k <= 9; ++k)
          CK(cudaMemcpyAsync(dev_in_q + (size_t)k * G, src[k], sizeof(float) * G, cudaMemcpyHostToDevice,
                             s->qstream));
        KL(launch_check_quats(dev_in_q + 6 * (size_t)G, dev_in_q + 7 * (size_t)G, dev_in_q + 8 * (size_t)G,
                              dev_in_q + 9 * (size_t)G, G, q_flags, reinterpret_cast<unsigned long long*>(q_flags + 2),
                              s->qstream));
        KL(launch_upload(&s->pin->q_err, q_flags, sizeof(uint32_t), s->qstream));
        KL(launch_upload(&s->pin->q_bad, q_flags + 2, sizeof(unsigned long long), s->qstream));
        CK(cudaEventRecord(s->ev[20], s->qstream));
        // dev_in is freed on the side stream once both readers are done
        CK(cudaEventRecord(s->ev[21], st));
        CK(cudaStreamWaitEvent(s->qstream, s->ev[21], 0));
        CK(cudaFreeAsync(dev_in_q, s->qstream));
        CK(cudaFreeAsync(q_flags, s->qstream));
      }
      if (s->N_loc > 0) KL(launch_cam_grid(s->N_loc, cr, cr + NL, scratch + 1, s->d_cam_gu, s->d_cam_gv, st));
      s->release(cr);
      s->release(scratch);
    }
    s->n_sub = (NL + 31) / 32;
    CK(s->alloc(&s->tile_lo, (size_t)s->n_tiles));
    CK(s->alloc(&s->tile_hi, (size_t)s->n_tiles));
    CK(s->alloc(&s->slice_lo, (size_t)s->n_tiles * 4));
    CK(s->alloc(&s->slice_hi, (size_t)s->n_tiles * 4));
    CK(s->alloc(&s->vcnt, 32));
    CK(s->alloc(&s->chunk_lo, (size_t)s->n_chunks));
    CK(s->alloc(&s->chunk_hi, (size_t)s->n_chunks));
    CK(s->alloc(&s->keep, (size_t)s->n_tiles * s->n_sub));
    CK(s->alloc(&s->kept, 1));
    if (s->aniso) {
      CK(s->alloc(&s->group_lo, (size_t)s->n_tiles * 16));
      CK(s->alloc(&s->group_hi, (size_t)s->n_tiles * 16));
    }
    KL(launch_tile_bounds(reinterpret_cast<const float4*>(s->xy), reinterpret_cast<const float4*>(s->zk), s->n_tiles,
                          s->tile_lo, s->tile_hi, s->slice_lo, s->slice_hi, s->group_lo, s->group_hi, st));
    // ---- a3/a4 visibility pass
    CK(s->alloc(&s->rows, (size_t)NL * s->words));
    CK(s->alloc(&s->K, NL)); CK(s->alloc(&s->D, NL)); CK(s->alloc(&s->zmin, NL)); CK(s->alloc(&s->zmax, NL));
    tl.mark("camera setup + bounds");
    CK(cudaEventRecord(s->ev[1], st));
    CK(cudaMemsetAsync(s->kept, 0, sizeof(unsigned long long), st));
    CK(cudaMemsetAsync(s->vcnt, 0, 32 * sizeof(unsigned long long), st));
    if (s->N_loc > 0)
      KLN(launch_cull(s->tile_lo, s->tile_hi, s->chunk_lo, s->chunk_hi, s->n_tiles, G, s->cams,
                      s->aniso ? s->acams : nullptr, s->N_loc, s->keep, s->kept, s->vcnt + 8, st), 2);
    CK(cudaEventRecord(s->ev[8], st));
    // kept-camera lists per tile (CSR)
    // list sizes go to pinned memory: the copies do not block the host, which
    // keeps enqueueing until the one synchronisation below
    KL(launch_upload(&s->pin->kept_pairs, s->kept, sizeof(unsigned long long), st));
    CK(s->alloc(&s->koff, (size_t)s->n_tiles + 1));
    {
      uint32_t* kc;
      CK(s->alloc(&kc, (size_t)s->n_tiles + 1));
      CK(cudaMemsetAsync(kc, 0, sizeof(uint32_t) * (s->n_tiles + 1), st));
      if (s->N_loc > 0) KL(launch_keep_lists(s->keep, s->n_tiles, s->n_sub, kc, nullptr, nullptr, nullptr, 0, st));
      size_t sbk = 0;
      CK(exclusive_scan_u32(nullptr, sbk, kc, s->koff, s->n_tiles + 1, st));
      void* tk = nullptr;
      CK(malloc_async(&tk, sbk, st));
      CUBL(exclusive_scan_u32(tk, sbk, kc, s->koff, s->n_tiles + 1, st));
      cudaFreeAsync(tk, st);
      s->release(kc);
    }
    // work units (tile, <= kVisUnit kept cameras)
    uint32_t *uc, *uoff;
    CK(s->alloc(&uc, (size_t)s->n_tiles + 1));
    CK(s->alloc(&uoff, (size_t)s->n_tiles + 1));
    CK(cudaMemsetAsync(uc, 0, sizeof(uint32_t) * (s->n_tiles + 1), st));
    KL(launch_units(s->koff, s->n_tiles, kVisUnit, uc, nullptr, nullptr, nullptr, 0, 0, st));
    {
      size_t sbu = 0;
      CK(exclusive_scan_u32(nullptr, sbu, uc, uoff, s->n_tiles + 1, st));
      void* tu = nullptr;
      CK(malloc_async(&tu, sbu, st));
      CUBL(exclusive_scan_u32(tu, sbu, uc, uoff, s->n_tiles + 1, st));
      cudaFreeAsync(tu, st);
    }
    KL(launch_upload(&s->pin->n_units, uoff + s->n_tiles, sizeof(uint32_t), st));
    tl.mark("cull + lists launched");
    TRY(validate_cameras(cams, n_cams));  // host work overlapping the device's a1 / culling
    tl.mark("validate_cameras");
    CK(cudaStreamSynchronize(st));
    tl.mark("sync (kept pairs)");
    const unsigned long long kept_pairs = s->pin->kept_pairs;
    const uint32_t nu = s->pin->n_units;
    s->n_units = nu;
    {  // k_prep_raw's verdict (its copies completed with this synchronisation)
      const uint32_t* hs = s->pin->prep_hs;
      unsigned long long hbad = s->pin->prep_bad;
      if ((hs[0] & 1u) && q_defer) {  // report the first invalid Gaussian of either check
        CK(cudaEventSynchronize(s->ev[20]));
        if (s->pin->q_err) hbad = std::min(hbad, s->pin->q_bad);
      }
      if (hs[0] & 1u)
        return fail(LOBE_E_INVALID_INPUT, "gaussian " + std::to_string(hbad) +
                                              " invalid (finite, scale > 0, |q| = 1 +- 1e-6, opacity in [0,1]; "
                                              "SPEC.md:30-33)");
      if (hs[0] & 2u) return fail(LOBE_E_INVALID_INPUT, "non-finite grid coordinate at " + std::to_string(hbad));
      auto ord2f = [](uint32_t u) {
        uint32_t b = (u & 0x80000000u) ? (u & 0x7fffffffu) : ~u;
        float f;
        std::memcpy(&f, &b, 4);
        return f;
      };
      s->mm[0] = ord2f(hs[1]); s->mm[1] = ord2f(hs[2]); s->mm[2] = ord2f(hs[3]); s->mm[3] = ord2f(hs[4]);
      if (s->mm[1] == s->mm[0] || s->mm[3] == s->mm[2])
        return fail(LOBE_E_DEGENERATE_SCENE, "all Gaussians share a ground coordinate (SPEC.md:80)");
    }
    CK(s->alloc(&s->klist, (size_t)std::max<unsigned long long>(kept_pairs, 1)));
    CK(s->alloc(&s->nonempty, (size_t)std::max<unsigned long long>(kept_pairs, 1)));
    CK(s->alloc(&s->codes, (size_t)std::max<unsigned long long>(kept_pairs, 1)));
    if (s->aniso) CK(s->alloc(&s->gcodes, (size_t)std::max<unsigned long long>(kept_pairs, 1)));
    CK(cudaMemsetAsync(s->nonempty, 0, (size_t)std::max<unsigned long long>(kept_pairs, 1), st));
    CK(s->alloc(&s->unit_tile, (size_t)nu + s->n_tiles + 1));
    CK(s->alloc(&s->unit_meta, (size_t)4 * std::max<uint32_t>(nu, 1)));
    CK(s->alloc(&s->queue, 2));  // [0] visibility items, [1] a4 tiles (side stream)
    if (s->N_loc > 0 && kept_pairs > 0) {
      KL(launch_keep_lists(s->keep, s->n_tiles, s->n_sub, nullptr, s->koff, s->klist, nullptr, 1, st));
      KL(launch_units(s->koff, s->n_tiles, kVisUnit, nullptr, uoff, s->unit_tile,
                       reinterpret_cast<uint4*>(s->unit_meta), nu, 1, st));
      CK(cudaEventRecord(s->ev[16], st));
      if (!s->aniso) KL(launch_cam_patterns(s->cams, s->N_loc, s->cam_pat, st));
      KLN(launch_slice_codes((int64_t)nu, reinterpret_cast<const uint4*>(s->unit_meta), s->klist, s->cams,
                            s->aniso ? s->acams : nullptr, s->slice_lo, s->slice_hi, s->codes, s->group_lo,
                            s->group_hi, s->gcodes, st), s->aniso ? 2 : 1);
      CK(cudaEventRecord(s->ev[17], st));
    }
    s->release(uc);
    s->release(uoff);
    CK(cudaEventRecord(s->ev[9], st));
    if (s->N_loc > 0 && kept_pairs > 0) {
      VisArgs va{};
      va.xy = reinterpret_cast<const float4*>(s->xy);
      va.zk = reinterpret_cast<const float4*>(s->zk);
      va.o2 = reinterpret_cast<const float2*>(s->o2);
      va.cams = s->cams;
      va.n_cams = s->N_loc;
      va.n_chunks = s->n_chunks;
      va.words = s->words;
      va.rows = s->rows;
      va.flags = nullptr;
      va.nonempty = s->nonempty;
      va.keep = s->keep;
      va.n_sub = s->n_sub;
      va.slo = s->slice_lo;
      va.shi = s->slice_hi;
      va.counters = s->vcnt;
      va.G = G;
      va.aniso = s->aniso;
      va.cv = s->cv;
      va.acams = s->acams;
      va.codes = s->codes;
      va.gcodes = s->gcodes;
      va.aniso_fast = s->aniso_fast ? 1 : 0;
      va.cam_pat = s->cam_pat;
      int grid = 0;
      KL(launch_vis_tiles(va, s->koff, s->klist, s->unit_tile, reinterpret_cast<const uint4*>(s->unit_meta),
                          s->n_units, s->queue, s->num_sms, st, &grid));
    }
    CK(cudaEventRecord(s->ev[10], st));
    KL(launch_upload(s->pin->vc, s->vcnt, sizeof(s->pin->vc), st));
    CK(cudaEventRecord(s->ev[2], st));
    // ---- (tile, camera) lists
    CK(s->alloc(&s->tile_off, (size_t)s->n_tiles + 1));
    uint32_t* cnt;
    CK(s->alloc(&cnt, (size_t)s->n_tiles + 1));
    CK(cudaMemsetAsync(cnt, 0, sizeof(uint32_t) * (s->n_tiles + 1), st));
    if (s->N_loc > 0 && kept_pairs > 0) KL(launch_tile_count(s->koff, s->nonempty, s->n_tiles, cnt, st));
    size_t sb = 0;
    CK(exclusive_scan_u32(nullptr, sb, cnt, s->tile_off, s->n_tiles + 1, st));
    CK(malloc_async(&tmp, sb, st));
    CUBL(exclusive_scan_u32(tmp, sb, cnt, s->tile_off, s->n_tiles + 1, st));
    cudaFreeAsync(tmp, st);
    s->release(cnt);
    // the pair count stays on the device: lists are sized by the kept pairs
    // (an upper bound known since the culling pass); the host reads the count
    // lazily with the statistics
    KL(launch_upload(&s->pin->n_pairs, s->tile_off + s->n_tiles, sizeof(uint32_t), st));
    const int64_t cap = (int64_t)std::max<unsigned long long>(kept_pairs, 1);
    const int64_t tw = (s->n_tiles + 31) / 32;
    CK(s->alloc(&s->pair_cam, (size_t)cap));
    CK(s->alloc(&s->pair_tile, (size_t)cap));
    uint32_t* camtile = nullptr;
    CK(s->alloc(&camtile, (size_t)NL * tw));
    CK(cudaMemsetAsync(camtile, 0, sizeof(uint32_t) * NL * tw, st));
    if (s->N_loc > 0 && kept_pairs > 0)
      KL(launch_tile_fill(s->koff, s->klist, s->nonempty, s->n_tiles, s->tile_off, s->pair_cam, s->pair_tile,
                          camtile, tw, st));
    // ---- a4 depth statistic: deferred (ensure_a4) -- enqueued by the first call
    // that needs it, or right after the first crop kernel, whose device->host copy
    // then overlaps it; the assignment does not need it (K_c = sum_b n0_cb, I5)
    s->camtile = camtile;
    s->a4_cap = cap;
    s->a4_tw = tw;
    s->a4_kept = kept_pairs;
    CK(s->alloc(&s->pair_part, (size_t)cap));
    CK(s->alloc(&s->cam_off, (size_t)NL + 1));
    CK(s->alloc(&s->cam_order, (size_t)cap));
    // Where a4 runs. Device-resident inputs: now, on the depth side stream,
    // concurrent with the caller's evaluation / crop (measured: step 5.30 ->
    // 5.15 ms at MatrixCity size). Host inputs: deferred behind the first crop
    // kernel, so it overlaps the crop's device->host copy instead of delaying
    // the evaluation (e2e 12.6 ms side stream vs 11.3 ms deferred).
    // LOBE_A4_STREAM=0|1 overrides.
    const char* a4_env = std::getenv("LOBE_A4_STREAM");
    const bool a4_stream = a4_env ? a4_env[0] == '1' : (bool)g->on_device;
    if (a4_stream) {  // a4 now, on the depth side stream, concurrent with the caller's next calls
      if (!s->dstream) s->dstream = acquire_side_stream(s->device);
      if (!s->dstream) return fail(LOBE_E_CUDA, "side stream creation failed");
      CK(cudaEventRecord(s->ev[11], st));
      CK(cudaStreamWaitEvent(s->dstream, s->ev[11], 0));
      TRY(launch_a4(s, s->dstream, true));
      s->a4_side = true;
      s->a4_joined = false;
    } else {
      s->a4_pending = true;
    }
    // ---- evaluation scratch
    CK(s->alloc(&s->zp, (size_t)s->G_pad));
    CK(s->alloc(&s->word_zone, (size_t)s->words));
    CK(s->alloc(&s->tile_zone, (size_t)s->n_tiles));
    CK(s->alloc(&s->zp_count, (size_t)kMaxZones * kMaxZones));
    CK(s->alloc(&s->dz, 1));
    CK(s->alloc(&s->d_zp_cell, (size_t)kMaxZones * kMaxZones));
    CK(s->alloc(&s->ncb, (size_t)NL * kMaxBlocks));
    CK(s->alloc(&s->n0cb, (size_t)NL * kMaxBlocks));
    CK(s->alloc(&s->member, NL)); CK(s->alloc(&s->sel, NL)); CK(s->alloc(&s->home, NL));
    {  // counts [3 x kMaxBlocks] u32 followed by incid [kMaxBlocks] u64 (one block, one copy)
      static_assert((3 * kMaxBlocks * sizeof(uint32_t)) % 8 == 0, "incid alignment");
      CK(s->alloc(&s->counts, 3 * kMaxBlocks + 2 * kMaxBlocks));
      s->incid = reinterpret_cast<unsigned long long*>(s->counts + 3 * kMaxBlocks);
    }
    CK(cudaEventRecord(s->ev[3], st));
    tl.mark("rest enqueued");
    // the deferred quaternion check decides while the device works on: the
    // load returns now if it is still running; every later scene call reports it
    if (q_defer) s->q_pending = true;
    // no synchronisation here: the depth statistic may still run while the caller
    // enqueues the next call; event timings are read lazily (finalize_load_stats)
    s->kept_pairs_last = kept_pairs;
    s->stats_pending = true;
    s->st.vis_launches += s->N_loc > 0 ? 1 : 0;
    s->st.bytes_read = (uint64_t)s->G_pad * 16ull;
    s->st.bytes_written = (uint64_t)s->N_loc * (uint64_t)s->words * 4ull;
    s->st.n_gaussians = G;
    s->st.n_cameras = n_cams;
    s->st.n_local_cameras = s->N_loc;
    s->st.cam_begin = s->cam_begin;
    return LOBE_OK;
  }();
  if (rs != LOBE_OK) {
    std::string keep = g_err;
    lobe_free_scene(s);
    g_err = keep;
    return rs;
  }
  if (inout_frame) *inout_frame = F;
  *out = s;
  return LOBE_OK;
}

static lobe_status impl_lobe_assign_cameras(lobe_scene* s, const lobe_grid* grid, uint32_t* K, double* depth_mean, float* z_min,
                                float* z_max, uint32_t* n_cb, uint32_t* n0_cb, uint64_t* member, int32_t* home) {
  LOBE_NVTX("lobe_assign_cameras");
  g_err.clear();
  if (!s) return fail(LOBE_E_STATE, "scene is NULL");
  CK(cudaSetDevice(s->device));
  GridV g;
  TRY(check_grid(grid, &g));
  TRY(ensure_eval(s, g));
  TRY(ensure_a4(s));  // K, D, z_min, z_max
  const size_t NL = (size_t)s->N_loc;
  std::vector<StagedCopy> plan;
  std::vector<const void*> srcs;
  size_t used = 0;
  bool direct = false;  // a copy went straight to a device / pinned destination on the scene's stream
  auto add = [&](void* dst, const void* src, size_t bytes) -> lobe_status {
    const size_t before = plan.size();
    TRY(stage_out(s, plan, used, dst, src, bytes));
    if (plan.size() != before) srcs.push_back(src);
    else if (dst && bytes) direct = true;
    return LOBE_OK;
  };
  // device layout of n, n0 is [c][B] with B = g.B stride
  struct Arr {
    void* dst;
    const void* src;
    size_t elem;
  };
  const Arr arrs[8] = {{K, s->K, 4},           {depth_mean, s->D, 8},   {z_min, s->zmin, 4},
                       {z_max, s->zmax, 4},    {n_cb, s->ncb, 4 * (size_t)g.B}, {n0_cb, s->n0cb, 4 * (size_t)g.B},
                       {member, s->member, 8}, {home, s->home, 4}};
  std::vector<uint8_t*> gathered;
  if (s->comm) {  // collective: every rank receives all N cameras
    const int64_t N = s->N_all;
    CK(cudaEventRecord(s->ev[18], s->stream));
    for (const Arr& a : arrs) {
      if (!a.dst) continue;
      uint8_t* gb = nullptr;
      CK(s->alloc(&gb, (size_t)N * a.elem));
      gathered.push_back(gb);
      lobe_status xs = lobe::xchg_gather_cameras(*s->xops, s->rank, s->world, N, a.elem, a.src, gb);
      if (xs != LOBE_OK) {
        for (uint8_t* p : gathered) s->release(p);
        return fail(xs, "exchange: " + s->xops->err);
      }
      TRY(add(a.dst, gb, (size_t)N * a.elem));
    }
    CK(cudaEventRecord(s->ev[19], s->stream));
  } else {
    for (const Arr& a : arrs) TRY(add(a.dst, a.src, NL * a.elem));
  }
  TRY(run_staged(s, plan, used, srcs, s->comm ? s->ev[19] : nullptr));
  for (uint8_t* p : gathered) s->release(p);
  if (direct) CK(cudaStreamSynchronize(s->stream));  // outputs are complete on return
  return LOBE_OK;
}

static lobe_status impl_lobe_block_loads(lobe_scene* s, const lobe_grid* grid, lobe_block_load* out, uint32_t* objective) {
  LOBE_NVTX("lobe_block_loads");
  g_err.clear();
  if (!s) return fail(LOBE_E_STATE, "scene is NULL");
  if (s->world != 1 && !s->comm)
    return fail(LOBE_E_STATE, "bare shard (world > 1, no communicator): use lobe_block_partial + lobe_masks_combine");
  CK(cudaSetDevice(s->device));
  GridV g;
  TRY(check_grid(grid, &g));
  if (s->comm) {
    TRY(ensure_xchg(s, g));
    uint32_t nc[kMaxBlocks];
    for (int b = 0; b < g.B; ++b) nc[b] = (uint32_t)s->x_counts[b];
    fill_records(s, g, nc, s->x_counts + g.B, s->x_gvis, out, objective);
    return LOBE_OK;
  }
  TRY(ensure_eval(s, g));
  uint64_t inc[kMaxBlocks];
  for (int b = 0; b < g.B; ++b) inc[b] = s->h_incid()[b];
  fill_records(s, g, s->h_ncams(), inc, s->h_gvis(), out, objective);
  return LOBE_OK;
}

static lobe_status impl_lobe_crop_masks(lobe_scene* s, const lobe_grid* grid, uint64_t* crop, uint64_t* eligible) {
  LOBE_NVTX("lobe_crop_masks");
  g_err.clear();
  if (!s) return fail(LOBE_E_STATE, "scene is NULL");
  if (s->world != 1 && !s->comm)
    return fail(LOBE_E_STATE, "bare shard (world > 1, no communicator): use lobe_crop_from_masks on combined masks");
  CK(cudaSetDevice(s->device));
  GridV g;
  TRY(check_grid(grid, &g));
  if (s->comm)
    TRY(ensure_xchg_masks(s, g));
  else
    TRY(ensure_eval(s, g));
  return lobe_crop_from_masks(s, grid, s->masks, crop, eligible);
}

static lobe_status impl_lobe_crop_from_masks(lobe_scene* s, const lobe_grid* grid, const uint32_t* d_masks, uint64_t* crop,
                                 uint64_t* eligible) {
  LOBE_NVTX("lobe_crop_from_masks");
  if (!s) return fail(LOBE_E_STATE, "scene is NULL");
  CK(cudaSetDevice(s->device));
  GridV g;
  TRY(check_grid(grid, &g));
  // the zone tables on the device must describe this grid (evaluate() uploads them)
  {
    ZoneTables Z{};
    build_axis(g.m, g.v, g.dv, &Z.U);
    build_axis(g.n, g.h, g.dh, &Z.V);
    if (s->hz.m != g.m || s->hz.n != g.n || std::memcmp(&Z.U, &s->hz.U, sizeof(AxisZones)) != 0 ||
        std::memcmp(&Z.V, &s->hz.V, sizeof(AxisZones)) != 0) {
      s->ev_valid = false;
      TRY(evaluate(s, g, nullptr));
    }
  }
  const int64_t W64 = (s->G + 63) / 64;
  const size_t bytes = (size_t)g.B * W64 * 8;
  // device destinations are written in place; host ones through scratch + copy
  auto on_device = [&](const void* p) {
    cudaPointerAttributes at{};
    const bool d = p && cudaPointerGetAttributes(&at, p) == cudaSuccess && at.type == cudaMemoryTypeDevice &&
                   at.device == s->device;
    cudaGetLastError();
    return d;
  };
  const bool crop_dev = on_device(crop), elig_dev = on_device(eligible);
  uint32_t *dc = nullptr, *de = nullptr;
  if (crop) {
    if (crop_dev) dc = reinterpret_cast<uint32_t*>(crop);
    else CK(s->alloc(&dc, bytes / 4));
  }
  if (eligible) {
    if (elig_dev) de = reinterpret_cast<uint32_t*>(eligible);
    else CK(s->alloc(&de, bytes / 4));
  }
  uint64_t* mbits = nullptr;
  uint8_t* cb8 = nullptr;
  CK(s->alloc(&mbits, (size_t)s->words * 32));
  CK(s->alloc(&cb8, (size_t)s->words * 32));
  CK(cudaEventRecord(s->ev[14], s->stream));
  KLN(launch_crop(s->G, s->iperm, s->zp, s->word_zone, s->d_zp_cell, d_masks, s->words, g.B, mbits, cb8, dc, de, s->stream), 2);
  CK(cudaEventRecord(s->ev[15], s->stream));
  // a pending a4 (depth statistic) goes on the scene's stream now, so it runs
  // while the masks travel to the host on the side stream (copy engines)
  TRY(ensure_a4(s, false));
  const bool host_out = (crop && !crop_dev) || (eligible && !elig_dev);
  if (host_out) {
    if (!s->side) s->side = acquire_side_stream(s->device);
    if (!s->side) return fail(LOBE_E_CUDA, "side stream creation failed");
    CK(cudaStreamWaitEvent(s->side, s->ev[15], 0));
    if (crop && !crop_dev) CK(cudaMemcpyAsync(crop, dc, bytes, cudaMemcpyDefault, s->side));
    if (eligible && !elig_dev) CK(cudaMemcpyAsync(eligible, de, bytes, cudaMemcpyDefault, s->side));
    CK(cudaStreamSynchronize(s->side));  // host outputs are complete on return
    s->st.t_crop_ms = ms_between(s->ev[14], s->ev[15]);
  }
  if (crop && !crop_dev) s->release(dc);    // the copies are done: stream-ordered frees are safe
  if (eligible && !elig_dev) s->release(de);
  s->release(mbits);
  s->release(cb8);
  if (!host_out) s->crop_pending = true;  // device outputs: stream-ordered; timing read lazily
  return LOBE_OK;
}

static lobe_status impl_lobe_block_partial(lobe_scene* s, const lobe_grid* grid, uint32_t* d_masks, uint32_t* n_cams,
                               uint64_t* incid) {
  LOBE_NVTX("lobe_block_partial");
  g_err.clear();
  if (!s) return fail(LOBE_E_STATE, "scene is NULL");
  if (!d_masks) return fail(LOBE_E_INVALID_CONFIG, "d_masks NULL");
  CK(cudaSetDevice(s->device));
  GridV g;
  TRY(check_grid(grid, &g));
  s->ev_valid = false;  // masks go to the caller's buffer; do not cache
  CK(cudaMemsetAsync(d_masks, 0, sizeof(uint32_t) * g.B * s->words, s->stream));
  TRY(evaluate(s, g, d_masks));
  if (n_cams) CK(cudaMemcpy(n_cams, s->h_ncams(), sizeof(uint32_t) * g.B, cudaMemcpyDefault));
  if (incid) CK(cudaMemcpy(incid, s->h_incid(), sizeof(uint64_t) * g.B, cudaMemcpyDefault));
  return LOBE_OK;
}

static lobe_status impl_lobe_masks_combine(lobe_scene* s, int32_t B, const uint32_t* d_gathered, int32_t W, uint32_t* d_out,
                               uint32_t* g_vis) {
  LOBE_NVTX("lobe_masks_combine");
  g_err.clear();
  if (!s) return fail(LOBE_E_STATE, "scene is NULL");
  if (B < 1 || B > kMaxBlocks || W < 1) return fail(LOBE_E_INVALID_CONFIG, "bad B or W");
  CK(cudaSetDevice(s->device));
  CK(cudaMemsetAsync(s->counts + kMaxBlocks, 0, sizeof(uint32_t) * kMaxBlocks, s->stream));
  CK(cudaEventRecord(s->ev[5], s->stream));
  KL(launch_masks_combine(d_gathered, W, B, s->words, d_out, s->counts + kMaxBlocks, s->stream));
  CK(cudaEventRecord(s->ev[6], s->stream));
  if (g_vis) CK(cudaMemcpyAsync(g_vis, s->counts + kMaxBlocks, sizeof(uint32_t) * B, cudaMemcpyDefault, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  s->st.t_comm_ms = ms_between(s->ev[5], s->ev[6]);
  return LOBE_OK;
}

static lobe_status impl_lobe_block_records(lobe_scene* s, const lobe_grid* grid, const uint32_t* n_cams, const uint64_t* incid,
                               const uint32_t* g_vis, lobe_block_load* out, uint32_t* objective) {
  LOBE_NVTX("lobe_block_records");
  g_err.clear();
  if (!s) return fail(LOBE_E_STATE, "scene is NULL");
  GridV g;
  TRY(check_grid(grid, &g));
  if (!(s->hz.m == g.m && s->hz.n == g.n)) return fail(LOBE_E_STATE, "lobe_block_partial first");
  fill_records(s, g, n_cams, incid, g_vis, out, objective);
  return LOBE_OK;
}

static lobe_status impl_lobe_export_rows(lobe_scene* s, int64_t c0, int64_t count, uint32_t* rows) {
  LOBE_NVTX("lobe_export_rows");
  g_err.clear();
  if (!s) return fail(LOBE_E_STATE, "scene is NULL");
  if (c0 < 0 || count < 0 || c0 + count > s->N_loc) return fail(LOBE_E_INVALID_INDEX, "camera range");
  if (count == 0) return LOBE_OK;
  CK(cudaSetDevice(s->device));
  const size_t W32 = (size_t)((s->G + 31) / 32);
  uint32_t* d = nullptr;
  CK(s->alloc(&d, W32 * count));
  KL(launch_export_rows(s->G, s->iperm, s->rows, s->words, c0, count, s->keep, s->n_sub, d, s->stream));
  TRY(copy_out(s, rows, d, W32 * count * 4));
  s->release(d);
  CK(cudaStreamSynchronize(s->stream));
  return LOBE_OK;
}

static lobe_status impl_lobe_dev_vis_bench(lobe_scene* s, int32_t variant, int32_t reps, float* ms, int32_t* grid) {
  LOBE_NVTX("lobe_dev_vis_bench");
  // variant 0: tile-major kernel over the kept lists (production);
  // 1-5: the camera-inner kernel (1 = culled, 2 = dense: every test evaluated)
  g_err.clear();
  if (!s) return fail(LOBE_E_STATE, "scene is NULL");
  if (variant < 0 || variant >= 1 + num_visibility_variants()) return fail(LOBE_E_INVALID_INDEX, "variant");
  if (s->N_loc <= 0 || reps < 1) return fail(LOBE_E_INVALID_CONFIG, "nothing to run");
  CK(cudaSetDevice(s->device));
  TRY(ensure_a4(s));  // the variants rewrite the rows a4 reads
  VisArgs va{};
  va.xy = reinterpret_cast<const float4*>(s->xy);
  va.zk = reinterpret_cast<const float4*>(s->zk);
  va.o2 = reinterpret_cast<const float2*>(s->o2);
  va.cams = s->cams;
  va.n_cams = s->N_loc;
  va.n_chunks = s->n_chunks;
  va.words = s->words;
  va.rows = s->rows;
  va.flags = nullptr;
  va.nonempty = s->nonempty;
  va.keep = s->keep;
  va.n_sub = s->n_sub;
  va.slo = s->slice_lo;
  va.shi = s->slice_hi;
  va.counters = nullptr;
  va.aniso = s->aniso;
  va.cv = s->cv;
  va.acams = s->acams;
  va.codes = s->codes;
  va.gcodes = s->gcodes;
  va.aniso_fast = s->aniso_fast ? 1 : 0;
  va.cam_pat = s->cam_pat;
  if (s->aniso && variant != 0) return fail(LOBE_E_INVALID_CONFIG, "camera-inner variants are isotropic only");
  int g = 0;
  auto run = [&]() -> cudaError_t {
    if (variant == 0)
      return launch_vis_tiles(va, s->koff, s->klist, s->unit_tile, reinterpret_cast<const uint4*>(s->unit_meta),
                              s->n_units, s->queue, s->num_sms, s->stream, &g);
    return launch_visibility_variant(variant - 1, va, s->num_sms, s->stream, &g);
  };
  KL(run());  // warm
  CK(cudaEventRecord(s->ev[6], s->stream));
  for (int r = 0; r < reps; ++r) KL(run());
  CK(cudaEventRecord(s->ev[7], s->stream));
  CK(cudaEventSynchronize(s->ev[7]));
  if (ms) *ms = ms_between(s->ev[6], s->ev[7]) / reps;
  if (grid) *grid = g;
  return LOBE_OK;
}

static lobe_status impl_lobe_block_subscene(lobe_scene* s, const lobe_grid* grid, int32_t block, const lobe_gaussians* coarse,
                                lobe_subscene* out, int64_t capacity) {
  LOBE_NVTX("lobe_block_subscene");
  g_err.clear();
  if (!s) return fail(LOBE_E_STATE, "scene is NULL");
  if (s->world != 1) return fail(LOBE_E_STATE, "world > 1: not supported for the block pipeline");
  if (!coarse || coarse->n != s->G || !coarse->on_device)
    return fail(LOBE_E_INVALID_CONFIG, "coarse: the loaded Gaussians as device arrays");
  TRY(check_sub(out, capacity > 0, "out"));
  CK(cudaSetDevice(s->device));
  GridV g;
  TRY(check_grid(grid, &g));
  if (block < 0 || block >= g.B) return fail(LOBE_E_INVALID_INDEX, "block");
  TRY(ensure_eval(s, g));
  cudaStream_t st = s->stream;
  const int64_t W64 = (s->G + 63) / 64;
  uint64_t *dc = nullptr, *de = nullptr;
  CK(s->alloc(&dc, (size_t)g.B * W64));
  CK(s->alloc(&de, (size_t)g.B * W64));
  {
    uint64_t* mbits = nullptr;
    uint8_t* cb8 = nullptr;
    CK(s->alloc(&mbits, (size_t)s->words * 32));
    CK(s->alloc(&cb8, (size_t)s->words * 32));
    KLN(launch_crop(s->G, s->iperm, s->zp, s->word_zone, s->d_zp_cell, s->masks, s->words, g.B, mbits, cb8,
                   reinterpret_cast<uint32_t*>(dc), reinterpret_cast<uint32_t*>(de), st), 2);
    s->release(mbits);
    s->release(cb8);
  }
  const uint64_t* cb = dc + (size_t)block * W64;
  const uint64_t* eb = de + (size_t)block * W64;
  uint32_t *cnt = nullptr, *off = nullptr;
  CK(s->alloc(&cnt, (size_t)W64 + 1));
  CK(s->alloc(&off, (size_t)W64 + 1));
  CK(cudaMemsetAsync(cnt + W64, 0, sizeof(uint32_t), st));
  KL(launch_mask_popc(cb, W64, cnt, st));
  uint64_t total = 0;
  TRY(scan_counts(s, cnt, off, W64, &total));
  out->n = (int64_t)total;
  lobe_status rs = LOBE_OK;
  if ((int64_t)total > capacity) {
    rs = fail(LOBE_E_CAPACITY, "sub-scene needs " + std::to_string(total) + " entries");
  } else if (total > 0) {
    SubArgs in{};
    const float* f[11] = {coarse->x, coarse->y, coarse->z, coarse->sx, coarse->sy, coarse->sz,
                          coarse->qw, coarse->qx, coarse->qy, coarse->qz, coarse->opacity};
    for (int k = 0; k < 11; ++k) in.f[k] = f[k];
    KL(launch_extract(cb, eb, W64, off, in, sub_out(out), st));
  }
  s->release(cnt);
  s->release(off);
  s->release(dc);
  s->release(de);
  CK(cudaStreamSynchronize(st));
  return rs;
}

static lobe_status impl_lobe_densify_step(lobe_scene* s, const lobe_grid* grid, int32_t block, const lobe_subscene* in,
                              const float* grad, const float* normals, float tau_grad, float scale_split,
                              lobe_subscene* out, int64_t capacity) {
  LOBE_NVTX("lobe_densify_step");
  g_err.clear();
  if (!s) return fail(LOBE_E_STATE, "scene is NULL");
  TRY(check_sub(in, in && in->n > 0, "in"));
  TRY(check_sub(out, capacity > 0, "out"));
  if (in->n > 0 && (!grad || !normals)) return fail(LOBE_E_INVALID_CONFIG, "grad / normals NULL");
  if (!std::isfinite(tau_grad) || !std::isfinite(scale_split)) return fail(LOBE_E_INVALID_CONFIG, "thresholds");
  CK(cudaSetDevice(s->device));
  GridV g;
  TRY(check_grid(grid, &g));
  if (block < 0 || block >= g.B) return fail(LOBE_E_INVALID_INDEX, "block");
  cudaStream_t st = s->stream;
  const int64_t n = in->n;
  uint32_t *cnt = nullptr, *off = nullptr;
  CK(s->alloc(&cnt, (size_t)n + 1));
  CK(s->alloc(&off, (size_t)n + 1));
  CK(cudaMemsetAsync(cnt + n, 0, sizeof(uint32_t), st));
  if (n > 0) KL(launch_densify_count(n, in->in_block, grad, tau_grad, cnt, st));
  uint64_t total = 0;
  TRY(scan_counts(s, cnt, off, n, &total));
  out->n = (int64_t)total;
  lobe_status rs = LOBE_OK;
  if ((int64_t)total > capacity) rs = fail(LOBE_E_CAPACITY, "densified sub-scene needs " + std::to_string(total));
  else if (n > 0)
    KL(launch_densify_write(n, sub_args(in), in->origin, in->in_block, grad, normals, tau_grad, scale_split, off,
                            make_cell_args(s, g), block, sub_out(out), st));
  s->release(cnt);
  s->release(off);
  CK(cudaStreamSynchronize(st));
  return rs;
}

static lobe_status impl_lobe_prune_outside(lobe_scene* s, const lobe_grid* grid, int32_t block, const lobe_subscene* in,
                               lobe_subscene* out, int64_t capacity) {
  LOBE_NVTX("lobe_prune_outside");
  g_err.clear();
  if (!s) return fail(LOBE_E_STATE, "scene is NULL");
  TRY(check_sub(in, in && in->n > 0, "in"));
  TRY(check_sub(out, capacity > 0, "out"));
  CK(cudaSetDevice(s->device));
  GridV g;
  TRY(check_grid(grid, &g));
  if (block < 0 || block >= g.B) return fail(LOBE_E_INVALID_INDEX, "block");
  cudaStream_t st = s->stream;
  const int64_t n = in->n;
  uint32_t *cnt = nullptr, *off = nullptr;
  CK(s->alloc(&cnt, (size_t)n + 1));
  CK(s->alloc(&off, (size_t)n + 1));
  CK(cudaMemsetAsync(cnt + n, 0, sizeof(uint32_t), st));
  const CellArgs cell = make_cell_args(s, g);
  if (n > 0) KL(launch_prune_count(n, in->x, in->y, in->z, cell, block, cnt, st));
  uint64_t total = 0;
  TRY(scan_counts(s, cnt, off, n, &total));
  out->n = (int64_t)total;
  lobe_status rs = LOBE_OK;
  if ((int64_t)total > capacity) rs = fail(LOBE_E_CAPACITY, "pruned sub-scene needs " + std::to_string(total));
  else if (n > 0) KL(launch_prune_write(n, sub_args(in), in->origin, cnt, off, sub_out(out), st));
  s->release(cnt);
  s->release(off);
  CK(cudaStreamSynchronize(st));
  return rs;
}

static lobe_status impl_lobe_merge_blocks(lobe_scene* s, const lobe_subscene* subs, int32_t count, lobe_subscene* out,
                              int64_t capacity) {
  LOBE_NVTX("lobe_merge_blocks");
  g_err.clear();
  if (!s) return fail(LOBE_E_STATE, "scene is NULL");
  if (count < 0 || (count > 0 && !subs)) return fail(LOBE_E_INVALID_CONFIG, "subs");
  TRY(check_sub(out, capacity > 0, "out"));
  int64_t total = 0;
  for (int32_t k = 0; k < count; ++k) {
    TRY(check_sub(&subs[k], subs[k].n > 0, "subs[k]"));
    total += subs[k].n;
  }
  out->n = total;
  if (total > capacity) return fail(LOBE_E_CAPACITY, "merged scene needs " + std::to_string(total));
  CK(cudaSetDevice(s->device));
  cudaStream_t st = s->stream;
  uint32_t* bits = nullptr;
  unsigned long long* dup = nullptr;
  CK(s->alloc(&bits, (size_t)(s->G + 31) / 32 + 1));
  CK(s->alloc(&dup, 1));
  CK(cudaMemsetAsync(bits, 0, sizeof(uint32_t) * ((s->G + 31) / 32 + 1), st));
  CK(cudaMemsetAsync(dup, 0xff, sizeof(unsigned long long), st));
  int64_t pos = 0;
  for (int32_t k = 0; k < count; ++k) {
    const lobe_subscene& a = subs[k];
    if (a.n == 0) continue;
    const float* fi[11] = {a.x, a.y, a.z, a.sx, a.sy, a.sz, a.qw, a.qx, a.qy, a.qz, a.opacity};
    float* fo[11] = {out->x, out->y, out->z, out->sx, out->sy, out->sz, out->qw, out->qx, out->qy, out->qz,
                     out->opacity};
    for (int f = 0; f < 11; ++f)
      CK(cudaMemcpyAsync(fo[f] + pos, fi[f], sizeof(float) * a.n, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(out->origin + pos, a.origin, sizeof(int64_t) * a.n, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(out->in_block + pos, a.in_block, a.n, cudaMemcpyDeviceToDevice, st));
    KL(launch_origin_claim(a.n, a.origin, s->G, bits, dup, st));
    pos += a.n;
  }
  unsigned long long hd = ~0ull;
  CK(cudaMemcpyAsync(&hd, dup, sizeof(hd), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  s->release(bits);
  s->release(dup);
  if (hd != ~0ull) return fail(LOBE_E_INTEGRITY, "origin index " + std::to_string(hd) + " appears twice (SPEC.md:569)");
  return LOBE_OK;
}

// Shared driver of lobe_render_select / lobe_render_maps.
lobe_status render_cameras(lobe_scene* s, const lobe_gaussians* coarse, int64_t cb, int64_t ce, RenderJob& J,
                           std::vector<uint32_t>* cloud_counts) {
  if (!coarse || coarse->n != s->G || !coarse->on_device)
    return fail(LOBE_E_INVALID_CONFIG, "coarse: the loaded Gaussians as device arrays");
  if (J.ds < 1 || J.stride < 1 || !(J.eps_w >= 0.0f)) return fail(LOBE_E_INVALID_CONFIG, "downscale/stride/eps_w");
  cudaStream_t st = s->stream;
  finalize_load_stats(s);
  SubArgs g{};
  const float* f[11] = {coarse->x, coarse->y, coarse->z, coarse->sx, coarse->sy, coarse->sz,
                        coarse->qw, coarse->qx, coarse->qy, coarse->qz, coarse->opacity};
  for (int k = 0; k < 11; ++k) g.f[k] = f[k];
  int32_t* perm = nullptr;
  CK(s->alloc(&perm, (size_t)s->G_pad));
  KL(launch_perm_from_iperm(s->G, s->iperm, perm, st));
  float4* prec = nullptr;
  CK(s->alloc(&prec, (size_t)3 * std::max<int64_t>(s->G, 1)));
  KL(launch_render_prep(s->G, perm, g, prec, st));
  s->release(perm);
  const int64_t NL = s->N_loc;
  std::vector<uint32_t> hoff(NL + 1), hK(std::max<int64_t>(NL, 1));
  CK(cudaMemcpyAsync(hoff.data(), s->cam_off, sizeof(uint32_t) * (NL + 1), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(hK.data(), s->K, sizeof(uint32_t) * std::max<int64_t>(NL, 1), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  std::vector<lobe_camera> hcams(s->host_cams.begin(), s->host_cams.end());
  {  // the clouds at their upper bound (one point per sample pixel) in one block:
     // growing them batch by batch re-copied them and grew the pool (~0.5 s)
    int64_t bound = J.n;
    for (int64_t c = cb; c < ce; ++c) {
      const int64_t wd = hcams[c].width / J.ds, hd = hcams[c].height / J.ds;
      bound += ((wd + J.stride - 1) / J.stride) * ((hd + J.stride - 1) / J.stride);
    }
    TRY(grow_cloud(s, J, bound));
  }
  // batches bounded by the records they hold (the splats of their visible Gaussians)
  const uint64_t kBudget = 48ull << 20;
  auto batch_end = [&](int64_t c, uint64_t* recs) {
    int64_t e = c;
    *recs = 0;
    while (e < ce && (e == c || *recs + hK[e] <= kBudget) && e - c < 2048) *recs += hK[e++];
    return e;
  };
  {  // the scratch blocks at the largest batch's sizes before the first batch
     // (records = sum of K_c exactly; tile entries still grow on demand)
    uint64_t mrec = 1, mpairs = 1, mcam = 1, mtiles = 1, mmaps = 1, msamp = 1;
    for (int64_t c = cb; c < ce;) {
      uint64_t recs = 0;
      const int64_t e = batch_end(c, &recs);
      uint64_t tiles = 0, maps = 0, samp = 0;
      for (int64_t q = c; q < e; ++q) {
        const int64_t wd = hcams[q].width / J.ds, hd = hcams[q].height / J.ds;
        tiles += (uint64_t)(((wd + 15) / 16) * ((hd + 15) / 16));
        maps += (uint64_t)(wd * hd);
        samp += (uint64_t)(((wd + J.stride - 1) / J.stride) * ((hd + J.stride - 1) / J.stride));
      }
      mrec = std::max<uint64_t>(mrec, recs);
      mpairs = std::max<uint64_t>(mpairs, (uint64_t)hoff[e] - hoff[c]);
      mcam = std::max<uint64_t>(mcam, (uint64_t)(e - c));
      mtiles = std::max(mtiles, tiles);
      mmaps = std::max(mmaps, maps);
      msamp = std::max(msamp, samp);
      c = e;
    }
    uint8_t* d = nullptr;
    const uint64_t s12 = std::max(std::max(mpairs, mrec), msamp) + 1;
    const std::pair<int, uint64_t> want[] = {
        {0, sizeof(RenderCam) * mcam}, {1, 4 * s12},       {2, 4 * s12},          {3, 8 * mrec},
        {4, 8 * mrec},                 {5, 4 * mrec},      {6, 4 * mrec},         {7, 4 * mrec},
        {8, 40 * mrec},                {9, 4 * (mcam + 1)}, {11, 4 * (msamp + 1)}, {12, 4 * (msamp + 1)},
        {15, 4 * (mtiles + 1)},        {16, 4 * (mtiles + 1)}, {17, 4 * mmaps},    {18, 4 * mmaps},
        {19, 4 * (mcam + 1)}};
    for (const auto& w : want) TRY(scratch(s, J, w.first, &d, (size_t)w.second));
  }
  const bool trace = std::getenv("LOBE_TRACE") != nullptr;
  int64_t c = cb;
  while (c < ce) {
    uint64_t recs = 0;
    const int64_t e = batch_end(c, &recs);
    const auto t0 = std::chrono::steady_clock::now();
    TRY(render_batch(s, prec, hoff, hcams, c, e, J));
    if (trace) {
      CK(cudaStreamSynchronize(st));
      const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      std::fprintf(stderr, "[lobe] render batch cams %lld-%lld records %llu: %.1f ms\n", (long long)c, (long long)e,
                   (unsigned long long)recs, ms);
    }
    c = e;
  }
  s->release(prec);
  if (cloud_counts) {
    // cloud size per local camera (integer atomics: order-free)
    cloud_counts->assign(std::max<int64_t>(NL, 1), 0);
    uint32_t* dc = nullptr;
    CK(s->alloc(&dc, cloud_counts->size()));
    CK(cudaMemsetAsync(dc, 0, sizeof(uint32_t) * cloud_counts->size(), st));
    if (J.n > 0) KL(launch_cam_counts(J.n, J.cam, dc, st));
    CK(cudaMemcpyAsync(cloud_counts->data(), dc, sizeof(uint32_t) * cloud_counts->size(), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    s->release(dc);
  }
  CK(cudaStreamSynchronize(st));
  return LOBE_OK;
}

static lobe_status impl_lobe_render_select(lobe_scene* s, const lobe_gaussians* coarse, int32_t downscale, int32_t stride,
                               float eps_w) {
  LOBE_NVTX("lobe_render_select");
  g_err.clear();
  if (!s) return fail(LOBE_E_STATE, "scene is NULL");
  CK(cudaSetDevice(s->device));
  RenderJob J;
  J.ds = downscale <= 0 ? 4 : downscale;
  J.stride = stride <= 0 ? 2 : stride;
  J.eps_w = eps_w < 0.0f ? 0.1f : eps_w;
  std::vector<uint32_t> counts;
  CK(s->alloc(&J.counters, 2));
  CK(cudaMemsetAsync(J.counters, 0, 2 * sizeof(unsigned long long), s->stream));
  lobe_status rs = render_cameras(s, coarse, 0, s->N_loc, J, &counts);
  {  // k_render roofline counters and kernel time (render_cameras ended with a sync)
    unsigned long long hc[2] = {0, 0};
    cudaMemcpy(hc, J.counters, sizeof(hc), cudaMemcpyDeviceToHost);
    double ms = 0.0;
    for (auto& e : J.kev) {
      ms += ms_between(e.first, e.second);
      cudaEventDestroy(e.first);
      cudaEventDestroy(e.second);
    }
    s->st.render_tests = hc[0];
    s->st.render_composited = hc[1];
    s->st.t_render_kernel_ms = ms;
    s->release(J.counters);
  }
  if (rs != LOBE_OK) {
    s->release(J.gu); s->release(J.gv); s->release(J.cam);
    return rs;
  }
  s->release(s->cloud_gu); s->release(s->cloud_gv); s->release(s->cloud_cam); s->release(s->cloud_K);
  s->cloud_gu = J.gu;
  s->cloud_gv = J.gv;
  s->cloud_cam = J.cam;
  s->n_cloud = J.n;
  CK(s->alloc(&s->cloud_K, counts.size()));
  CK(cudaMemcpyAsync(s->cloud_K, counts.data(), sizeof(uint32_t) * counts.size(), cudaMemcpyHostToDevice,
                     s->stream));
  CK(cudaStreamSynchronize(s->stream));
  s->cloud_mode = true;
  s->ev_valid = false;  // evaluations now count cloud points
  return LOBE_OK;
}

static lobe_status impl_lobe_camera_clouds(lobe_scene* s, int64_t* offsets, float* gu, float* gv, int64_t capacity) {
  LOBE_NVTX("lobe_camera_clouds");
  g_err.clear();
  if (!s) return fail(LOBE_E_STATE, "scene is NULL");
  if (!s->cloud_mode) return fail(LOBE_E_STATE, "no clouds: call lobe_render_select first");
  CK(cudaSetDevice(s->device));
  const int64_t NL = s->N_loc;
  std::vector<uint32_t> hk(std::max<int64_t>(NL, 1));
  CK(cudaMemcpyAsync(hk.data(), s->cloud_K, sizeof(uint32_t) * hk.size(), cudaMemcpyDeviceToHost, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  if (offsets) {
    offsets[0] = 0;
    for (int64_t c = 0; c < NL; ++c) offsets[c + 1] = offsets[c] + hk[c];
  }
  if (s->n_cloud > capacity) return fail(LOBE_E_CAPACITY, "clouds need " + std::to_string(s->n_cloud));
  TRY(copy_out(s, gu, s->cloud_gu, sizeof(float) * s->n_cloud));
  TRY(copy_out(s, gv, s->cloud_gv, sizeof(float) * s->n_cloud));
  CK(cudaStreamSynchronize(s->stream));
  return LOBE_OK;
}

static lobe_status impl_lobe_render_maps(lobe_scene* s, const lobe_gaussians* coarse, int64_t camera, int32_t downscale,
                             float* depth, float* weight) {
  LOBE_NVTX("lobe_render_maps");
  g_err.clear();
  if (!s) return fail(LOBE_E_STATE, "scene is NULL");
  if (camera < 0 || camera >= s->N_loc) return fail(LOBE_E_INVALID_INDEX, "camera");
  CK(cudaSetDevice(s->device));
  RenderJob J;
  J.ds = downscale <= 0 ? 4 : downscale;
  J.Dout = depth;
  J.Wout = weight;
  lobe_status rs = render_cameras(s, coarse, camera, camera + 1, J, nullptr);
  s->release(J.gu); s->release(J.gv); s->release(J.cam);
  CK(cudaStreamSynchronize(s->stream));
  return rs;
}

lobe_status lobe_scene_info(const lobe_scene* s, int64_t* n_gaussians, int64_t* n_cameras, int64_t* n_local_cameras,
                            int64_t* cam_begin) {
  LOBE_NVTX("lobe_scene_info");
  if (!s) return fail(LOBE_E_STATE, "scene is NULL");
  if (n_gaussians) *n_gaussians = s->st.n_gaussians;
  if (n_cameras) *n_cameras = s->st.n_cameras;
  if (n_local_cameras) *n_local_cameras = s->st.n_local_cameras;
  if (cam_begin) *cam_begin = s->st.cam_begin;
  return LOBE_OK;
}

static lobe_status impl_lobe_get_stats(const lobe_scene* s, lobe_stats* out) {
  LOBE_NVTX("lobe_get_stats");
  if (!s || !out) return fail(LOBE_E_STATE, "NULL");
  finalize_load_stats(const_cast<lobe_scene*>(s));
  const_cast<lobe_scene*>(s)->wait_counts();
  if (s->crop_pending) {
    lobe_scene* w = const_cast<lobe_scene*>(s);
    cudaEventSynchronize(w->ev[15]);
    w->st.t_crop_ms = ms_between(w->ev[14], w->ev[15]);
    w->crop_pending = false;
  }
  *out = s->st;
  return LOBE_OK;
}

lobe_status lobe_bo_run(int32_t m, int32_t n, const lobe_balance_opts* opts, lobe_objective_fn objective, void* ctx,
                        float* v_out, float* h_out, uint32_t* history, float* cut_history) {
  LOBE_NVTX("lobe_bo_run");
  g_err.clear();
  if (m < 1 || n < 1 || m * n > kMaxBlocks) return fail(LOBE_E_INVALID_CONFIG, "grid m, n");
  if (!objective) return fail(LOBE_E_INVALID_CONFIG, "objective NULL");
  lobe_balance_opts o{100, 0, 0.1f, 0.15, 8};
  if (opts) o = *opts;
  if (o.L <= 0) o.L = 100;
  if (o.n_sobol < 0) o.n_sobol = 8;
  std::string err;
  auto f = [&](const float* v, const float* h, uint32_t* val) { return objective(ctx, v, h, val); };
  int rc = lobe::bo_run(m, n, o.L, o.seed, o.n_sobol, f, v_out, h_out, history, cut_history, &err);
  if (rc != 0) return fail(LOBE_E_INVALID_CONFIG, "bo: " + err);
  return LOBE_OK;
}

static lobe_status impl_lobe_balance_partition(lobe_scene* s, int32_t m, int32_t n, const lobe_balance_opts* opts, float* v_out,
                                   float* h_out, uint32_t* history, float* cut_history, lobe_block_load* best) {
  LOBE_NVTX("lobe_balance_partition");
  g_err.clear();
  if (!s) return fail(LOBE_E_STATE, "scene is NULL");
  if (s->world != 1 && !s->comm)
    return fail(LOBE_E_STATE, "bare shard (world > 1, no communicator): use lobe_bo_run with an exchange objective");
  if (m < 1 || n < 1 || m * n > kMaxBlocks) return fail(LOBE_E_INVALID_CONFIG, "grid m, n");
  lobe_balance_opts o{100, 0, 0.1f, 0.15, 8};
  if (opts) o = *opts;
  if (o.L <= 0) o.L = 100;
  if (o.n_sobol < 0) o.n_sobol = 8;
  const float ds = o.delta_scale > 0.0f ? o.delta_scale : 0.1f;
  const double tau = o.tau < 0.0 ? 0.15 : o.tau;
  const float dv = ds / (float)m, dh = ds / (float)n;  // ledger L14
  lobe_status last = LOBE_OK;
  auto f = [&](const float* v, const float* h, uint32_t* val) -> int {
    lobe_grid gr{m, n, v, h, dv, dh, tau};
    GridV g;
    lobe_status st = check_grid(&gr, &g);
    if (st == LOBE_OK) st = s->comm ? ensure_xchg(s, g) : ensure_eval(s, g);
    if (st != LOBE_OK) {
      last = st;
      return 1;
    }
    const uint32_t* gv = s->comm ? s->x_gvis : s->h_gvis();
    uint32_t b = 0;
    for (int k = 0; k < g.B; ++k) b = std::max(b, gv[k]);
    *val = b;
    return 0;
  };
  std::vector<float> vb(std::max(m - 1, 1)), hb(std::max(n - 1, 1));
  std::string err;
  int rc = lobe::bo_run(m, n, o.L, o.seed, o.n_sobol, f, vb.data(), hb.data(), history, cut_history, &err);
  if (rc != 0) return last != LOBE_OK ? last : fail(LOBE_E_INVALID_CONFIG, "bo: " + err);
  if (v_out) std::copy(vb.begin(), vb.begin() + (m - 1), v_out);
  if (h_out) std::copy(hb.begin(), hb.begin() + (n - 1), h_out);
  if (best) {
    lobe_grid gr{m, n, vb.data(), hb.data(), dv, dh, tau};
    uint32_t obj;
    TRY(lobe_block_loads(s, &gr, best, &obj));
  }
  return LOBE_OK;
}


// ---- exported scene calls: a host-input load in the isotropic mode returns
// before the deferred quaternion check has decided (the copy engine is the
// bound of that load and the quaternions travel last); every scene call reports
// its verdict: before its work if already known, else before it returns.
lobe_status lobe_assign_cameras(lobe_scene* s, const lobe_grid* grid, uint32_t* K, double* depth_mean, float* z_min,
                                float* z_max, uint32_t* n_cb, uint32_t* n0_cb, uint64_t* member, int32_t* home) {
  TRY(scene_verdict(s, false));
  const lobe_status r = impl_lobe_assign_cameras(s, grid, K, depth_mean, z_min, z_max, n_cb, n0_cb, member, home);
  return r != LOBE_OK ? r : scene_verdict(s, true);
}

lobe_status lobe_block_loads(lobe_scene* s, const lobe_grid* grid, lobe_block_load* out, uint32_t* objective) {
  TRY(scene_verdict(s, false));
  const lobe_status r = impl_lobe_block_loads(s, grid, out, objective);
  return r != LOBE_OK ? r : scene_verdict(s, true);
}

lobe_status lobe_crop_masks(lobe_scene* s, const lobe_grid* grid, uint64_t* crop, uint64_t* eligible) {
  TRY(scene_verdict(s, false));
  const lobe_status r = impl_lobe_crop_masks(s, grid, crop, eligible);
  return r != LOBE_OK ? r : scene_verdict(s, true);
}

lobe_status lobe_crop_from_masks(lobe_scene* s, const lobe_grid* grid, const uint32_t* d_masks, uint64_t* crop,
                                 uint64_t* eligible) {
  TRY(scene_verdict(s, false));
  const lobe_status r = impl_lobe_crop_from_masks(s, grid, d_masks, crop, eligible);
  return r != LOBE_OK ? r : scene_verdict(s, true);
}

lobe_status lobe_block_partial(lobe_scene* s, const lobe_grid* grid, uint32_t* d_masks, uint32_t* n_cams,
                               uint64_t* incid) {
  TRY(scene_verdict(s, false));
  const lobe_status r = impl_lobe_block_partial(s, grid, d_masks, n_cams, incid);
  return r != LOBE_OK ? r : scene_verdict(s, true);
}

lobe_status lobe_masks_combine(lobe_scene* s, int32_t B, const uint32_t* d_gathered, int32_t W, uint32_t* d_out,
                               uint32_t* g_vis) {
  TRY(scene_verdict(s, false));
  const lobe_status r = impl_lobe_masks_combine(s, B, d_gathered, W, d_out, g_vis);
  return r != LOBE_OK ? r : scene_verdict(s, true);
}

lobe_status lobe_block_records(lobe_scene* s, const lobe_grid* grid, const uint32_t* n_cams, const uint64_t* incid,
                               const uint32_t* g_vis, lobe_block_load* out, uint32_t* objective) {
  TRY(scene_verdict(s, false));
  const lobe_status r = impl_lobe_block_records(s, grid, n_cams, incid, g_vis, out, objective);
  return r != LOBE_OK ? r : scene_verdict(s, true);
}

lobe_status lobe_export_rows(lobe_scene* s, int64_t c0, int64_t count, uint32_t* rows) {
  TRY(scene_verdict(s, false));
  const lobe_status r = impl_lobe_export_rows(s, c0, count, rows);
  return r != LOBE_OK ? r : scene_verdict(s, true);
}

lobe_status lobe_dev_vis_bench(lobe_scene* s, int32_t variant, int32_t reps, float* ms, int32_t* grid) {
  TRY(scene_verdict(s, false));
  const lobe_status r = impl_lobe_dev_vis_bench(s, variant, reps, ms, grid);
  return r != LOBE_OK ? r : scene_verdict(s, true);
}

lobe_status lobe_block_subscene(lobe_scene* s, const lobe_grid* grid, int32_t block, const lobe_gaussians* coarse,
                                lobe_subscene* out, int64_t capacity) {
  TRY(scene_verdict(s, false));
  const lobe_status r = impl_lobe_block_subscene(s, grid, block, coarse, out, capacity);
  return r != LOBE_OK ? r : scene_verdict(s, true);
}

lobe_status lobe_densify_step(lobe_scene* s, const lobe_grid* grid, int32_t block, const lobe_subscene* in,
                              const float* grad, const float* normals, float tau_grad, float scale_split,
                              lobe_subscene* out, int64_t capacity) {
  TRY(scene_verdict(s, false));
  const lobe_status r = impl_lobe_densify_step(s, grid, block, in, grad, normals, tau_grad, scale_split, out, capacity);
  return r != LOBE_OK ? r : scene_verdict(s, true);
}

lobe_status lobe_prune_outside(lobe_scene* s, const lobe_grid* grid, int32_t block, const lobe_subscene* in,
                               lobe_subscene* out, int64_t capacity) {
  TRY(scene_verdict(s, false));
  const lobe_status r = impl_lobe_prune_outside(s, grid, block, in, out, capacity);
  return r != LOBE_OK ? r : scene_verdict(s, true);
}

lobe_status lobe_merge_blocks(lobe_scene* s, const lobe_subscene* subs, int32_t count, lobe_subscene* out,
                              int64_t capacity) {
  TRY(scene_verdict(s, false));
  const lobe_status r = impl_lobe_merge_blocks(s, subs, count, out, capacity);
  return r != LOBE_OK ? r : scene_verdict(s, true);
}

lobe_status lobe_render_select(lobe_scene* s, const lobe_gaussians* coarse, int32_t downscale, int32_t stride,
                               float eps_w) {
  TRY(scene_verdict(s, false));
  const lobe_status r = impl_lobe_render_select(s, coarse, downscale, stride, eps_w);
  return r != LOBE_OK ? r : scene_verdict(s, true);
}

lobe_status lobe_camera_clouds(lobe_scene* s, int64_t* offsets, float* gu, float* gv, int64_t capacity) {
  TRY(scene_verdict(s, false));
  const lobe_status r = impl_lobe_camera_clouds(s, offsets, gu, gv, capacity);
  return r != LOBE_OK ? r : scene_verdict(s, true);
}

lobe_status lobe_render_maps(lobe_scene* s, const lobe_gaussians* coarse, int64_t camera, int32_t downscale,
                             float* depth, float* weight) {
  TRY(scene_verdict(s, false));
  const lobe_status r = impl_lobe_render_maps(s, coarse, camera, downscale, depth, weight);
  return r != LOBE_OK ? r : scene_verdict(s, true);
}

lobe_status lobe_get_stats(const lobe_scene* s, lobe_stats* out) {
  TRY(scene_verdict(s, false));
  const lobe_status r = impl_lobe_get_stats(s, out);
  return r != LOBE_OK ? r : scene_verdict(s, true);
}

lobe_status lobe_balance_partition(lobe_scene* s, int32_t m, int32_t n, const lobe_balance_opts* opts, float* v_out,
                                   float* h_out, uint32_t* history, float* cut_history, lobe_block_load* best) {
  TRY(scene_verdict(s, false));
  const lobe_status r = impl_lobe_balance_partition(s, m, n, opts, v_out, h_out, history, cut_history, best);
  return r != LOBE_OK ? r : scene_verdict(s, true);
}

}  // extern "C"
