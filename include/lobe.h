/* lobe.h -- C ABI of the B200 visibility engine for LoBE-GS (arXiv 2510.01767).
 *
 * The engine computes, for a coarse 3D-Gaussian model and a set of camera views,
 * the quantities the paper's partitioner needs (§4.1-§4.3):
 *   - which Gaussians each camera sees (frustum + 3-sigma footprint culling,
 *     SPEC.md:243, :298-299; ledger L1/L2 in DESIGN.md);
 *   - a per-camera depth statistic (opacity-weighted mean camera depth, L4);
 *   - the camera->block assignment C^(b) = {c | V_{c,b} >= tau}
 *     (Eq. 3), over enlarged regions
 *     B^(b) = [v_{i-1}-dv, v_i+dv] x [h_{j-1}-dh, h_j+dh];
 *   - per-block loads A, |C|, G_blk, G_vis, G_avgvis and the
 *     objective max_b G_vis^(b) (Eq. 2);
 *   - visibility-cropping and selective-densification masks;
 *   - the load-balanced cuts by Bayesian optimisation (L = 100).
 *
 * Conventions (all calls):
 *   - Status codes, never exceptions. lobe_last_error() returns a thread-local
 *     message valid until the next lobe_* call on the calling thread. After a
 *     failed call outputs are unspecified and the scene handle stays valid.
 *   - Ownership: the caller owns every pointer it passes. lobe_load_scene copies
 *     its inputs; the caller may free them on return (exception: the quaternion
 *     arrays of a host-input load in the isotropic mode, see lobe_load_scene).
 *     Outputs are caller-allocated
 *     with the sizes stated per call. The scene handle owns its device memory and
 *     is released by lobe_free_scene.
 *   - Pointers: output (and, with on_device, input) pointers may be host or
 *     device pointers (unified addressing decides); device writes are issued on
 *     lobe_options.stream. Host outputs are complete when a call returns; device
 *     outputs of lobe_crop_masks are stream-ordered (the call returns without
 *     waiting, like a kernel launch), every other call's outputs are complete on
 *     return.
 *   - Index conventions: Gaussian i is the caller's index; camera c is the
 *     caller's array index. Block b = p*n + q (0-based), p indexes the v cuts
 *     (first ground axis), q the h cuts (PAPER.md:165 garbled index read as
 *     b = (i-1) n + j, ledger L9). B = m*n <= 64. Mask bit (i mod 64) of u64 word
 *     floor(i/64) is Gaussian i.
 *   - Multi-GPU: options.rank / options.world select this
 *     process's camera shard [floor(rN/W), floor((r+1)N/W)) (cameras sharded,
 *     Gaussians replicated). With a communicator (options.nccl_unique_id or
 *     options.host_comm) ALL ranks call every function collectively (MPI style,
 *     same arguments), the library runs the exchange itself (NCCL on the scene's
 *     stream, or the caller's host callbacks), and every output is GLOBAL and
 *     identical on every rank: per-camera outputs cover all N cameras. Without a
 *     communicator and world > 1 the scene is a bare camera shard: per-camera
 *     outputs cover the local shard and the block-level results come from the
 *     exchange points below (lobe_block_partial, lobe_masks_combine, ...).
 *     With world == 1 and no communicator every call is complete on its own.
 *   - Concurrency: a handle is not thread-safe; distinct handles are. Every call
 *     is deterministic (identical inputs give identical bytes, for any world).
 */
#ifndef LOBE_H_
#define LOBE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  LOBE_OK = 0,
  LOBE_E_INVALID_INPUT = 1,     /* non-finite / out-of-range field */
  LOBE_E_INVALID_CONFIG = 2,    /* zero counts, bad grid, B > 64, bad tau/delta */
  LOBE_E_INVALID_CUTS = 3,      /* cuts not strictly increasing in (0,1) */
  LOBE_E_INVALID_INDEX = 4,     /* bad block / camera index */
  LOBE_E_DEGENERATE_SCENE = 5,  /* all points identical on a ground axis, zero radius */
  LOBE_E_CUDA = 6,              /* CUDA runtime error or no device */
  LOBE_E_NCCL = 7,              /* collective failure: NCCL error / library missing, or a host_comm callback failed */
  LOBE_E_OOM = 8,               /* device allocation failed */
  LOBE_E_STATE = 9,             /* call out of order (e.g. combine before partial) */
  LOBE_E_CAPACITY = 10,         /* output capacity too small (the needed count is reported) */
  LOBE_E_INTEGRITY = 11         /* merge: an origin index appears in two blocks */
} lobe_status;

typedef struct lobe_scene lobe_scene; /* opaque */

/* Coarse Gaussians, SoA fp32, caller order (SPEC.md:28-33 Gaussian3D).
 * s* are per-axis standard deviations (> 0), q* a unit quaternion (|q| = 1
 * within 1e-6), opacity in [0,1]. |position|, scale <= 1e18 (ledger L22).
 * on_device != 0: the arrays are device pointers. */
typedef struct {
  int64_t n;
  const float *x, *y, *z, *sx, *sy, *sz, *qw, *qx, *qy, *qz, *opacity;
  int32_t on_device;
} lobe_gaussians;

/* Pinhole camera (SPEC.md:44-49 CameraView): world->camera rotation R (row
 * major) and translation t, p_cam = R p + t, looking along +z_cam; image
 * width x height pixels; 0 < z_near < z_far. */
typedef struct {
  int32_t id;
  float fx, fy, cx, cy;
  int32_t width, height;
  float R[9];
  float t[3];
  float z_near, z_far;
} lobe_camera;

/* Normalisation frame for the spherical contraction and ground plane (ledger
 * L12). auto_flags bit0: centre = component-wise lower median
 * of camera centres; bit1: radius = ceil(0.9 N)-th smallest camera distance;
 * bit2: axes = world x, y. Resolved values are written back. */
#define LOBE_FRAME_AUTO_CENTER 1u
#define LOBE_FRAME_AUTO_RADIUS 2u
#define LOBE_FRAME_AUTO_AXES 4u
#define LOBE_FRAME_AUTO_ALL 7u
typedef struct {
  float center[3];
  float radius;
  float axis_u[3], axis_v[3];
  uint32_t auto_flags;
} lobe_frame;

/* C^(b) selection (ledger L8): RATIO = {c : V_{c,b} >= tau} (PAPER.md:179,
 * default), HOME = {c : home_c = b}, UNION = both. */
#define LOBE_ASSIGN_RATIO 0
#define LOBE_ASSIGN_HOME 1
#define LOBE_ASSIGN_UNION 2

/* Caller-provided collectives over HOST buffers (any transport: gloo, MPI, ...).
 * Each returns 0 on success; every rank calls them in the same order.
 *   all_gather: recv (world x bytes, rank-major) = every rank's `bytes` of send;
 *   all_reduce_u64: element-wise SUM over ranks, in place;
 *   all_to_all_v: send_bytes[j] bytes at send + send_off[j] go to rank j; the
 *     recv_bytes[j] bytes from rank j land at recv + recv_off[j]. */
typedef struct {
  void* ctx;
  int (*all_gather)(void* ctx, const void* send, void* recv, size_t bytes);
  int (*all_reduce_u64)(void* ctx, uint64_t* buf, size_t count);
  int (*all_to_all_v)(void* ctx, const void* send, const size_t* send_bytes, const size_t* send_off, void* recv,
                      const size_t* recv_bytes, const size_t* recv_off);
} lobe_host_comm;

typedef struct {
  int32_t device;       /* CUDA device ordinal */
  int32_t rank, world;  /* camera shard; world >= 1 */
  void* stream;         /* cudaStream_t; NULL = legacy default stream */
  int32_t assign_mode;  /* LOBE_ASSIGN_* */
  int32_t predicate;    /* LOBE_PREDICATE_* (0 = isotropic, the default) */
  /* Communicator; at most one, both NULL = none.
   * nccl_unique_id: 128 bytes (an ncclUniqueId from lobe_nccl_unique_id on rank 0,
   *   broadcast by the caller); the library creates one ncclComm per (id, rank,
   *   device) on first use -- collectively, so every rank must load its scene --
   *   and reuses it for later scenes with the same id (lobe_release_comms frees).
   * host_comm: host collectives (copied; must outlive the scene's calls). */
  const void* nccl_unique_id;
  const lobe_host_comm* host_comm;
} lobe_options;

/* NCCL unique id for options.nccl_unique_id (rank 0 calls this and broadcasts the
 * 128 bytes). LOBE_E_NCCL if libnccl.so.2 cannot be loaded. Needs no scene. */
lobe_status lobe_nccl_unique_id(void* out_128_bytes);
/* Destroy the cached NCCL communicators (collective over each communicator). */
void lobe_release_comms(void);

/* Visibility predicate. ISOTROPIC: SPEC.md:299's culling bound, footprint radius
 * 3 max(s) max(fx, fy) / z (the measured path). ANISOTROPIC: the
 * projected-covariance footprint of SPEC.md:338/:387 (EWA: Sigma' = J W Sigma
 * W^T J^T + 0.3 I, radius 3 sqrt(lambda_max(Sigma')), Sigma from the rotation
 * and scales, DESIGN.md ledger L24 pins the fp32 op order).
 * Everything downstream (depth statistic, assignment, loads, crop) is shared. */
#define LOBE_PREDICATE_ISOTROPIC 0
#define LOBE_PREDICATE_ANISOTROPIC 1

/* Grid cuts (GridCuts SPEC.md:51-56). v: m-1 cuts on the first
 * ground axis, h: n-1 cuts on the second, strictly increasing in (0,1).
 * delta_v/delta_h < 0 select the paper's (0.1/m, 0.1/n) in fp32 (PAPER.md:167,
 * ledger L14); tau < 0 selects 0.15. tau is compared in fp64
 * (ledger L6). */
typedef struct {
  int32_t m, n;
  const float* v;
  const float* h;
  float delta_v, delta_h;
  double tau;
} lobe_grid;

/* Per-block record (§3.2; BlockLoadStats SPEC.md:232-237).
 * lo/hi: enlarged region B^(b) (fp32, clamped to [0,1]); area: delta = 0 cell
 * area in fp64; incidences: sum_c n0_{c,b}. */
typedef struct {
  int32_t block_id, row, col;
  float lo[2], hi[2];
  double area;
  uint32_t n_cams, g_blk, g_vis;
  double g_avgvis;
  uint64_t incidences;
} lobe_block_load;

/* BO options. L <= 0 -> 100; n_sobol < 0 -> 8;
 * delta_scale <= 0 -> 0.1 (delta = delta_scale/m, delta_scale/n); tau < 0 -> 0.15. */
typedef struct {
  int32_t L;
  uint64_t seed;
  float delta_scale;
  double tau;
  int32_t n_sobol;
} lobe_balance_opts;

/* Stage timings of the last call (CUDA events on options.stream), cumulative
 * logical Gaussian-camera tests decided by the visibility kernels (I16: counted
 * inside k_cull / k_vis_tiles, see decided_tests), and algorithmic bytes of the
 * last visibility pass. */
typedef struct {
  double t_prep_ms, t_vis_ms, t_hist_ms, t_loads_ms, t_comm_ms, t_crop_ms;
  uint64_t tests_executed, bytes_read, bytes_written;
  uint64_t vis_launches, evaluations;
  int64_t n_gaussians, n_cameras, n_local_cameras, cam_begin;
  uint64_t tile_pairs; /* (tile, camera) pairs with any visible Gaussian */
  uint64_t dense_tests;     /* exact per-Gaussian tests run in the last visibility pass; the other logical
                               tests (G x N_local) are decided by box bounds:
                               rejected tiles/slices (no Gaussian visible) or accepted slices (every
                               non-gated Gaussian visible) -- identical results, see k_vis_tiles */
  double t_cull_ms;         /* tile-culling kernel of the last visibility pass (included in t_vis_ms,
                               which is culling + slice classification + test kernels) */
  double t_depth_ms;        /* depth statistic over the non-empty (tile, camera) pairs (a4) */
  uint64_t kernel_launches; /* cumulative launches of this library's own kernels */
  uint64_t cub_launches;    /* cumulative CUB primitive calls (radix sort, scan) */
  uint64_t kept_tests;      /* tests in (tile, camera) pairs the tile bound did not reject (last pass) */
  uint64_t accepted_tests;  /* tests in (slice, camera) pairs the slice bound accepted (last pass) */
  uint64_t exact_variant_tests[6]; /* exact tests by the conditions left open: left edge only, top edge only,
                                      right edge only, bottom edge only, the four edges, all six */
  uint64_t decided_tests[4]; /* I16, measured by the kernels of the last visibility pass: the logical
                                tests over REAL Gaussians (padding excluded) decided by [0] the chunk / tile bound
                                (k_cull, rejected), [1] the slice bound rejecting, [2] the slice bound accepting,
                                [3] the exact per-Gaussian test; they add up to G x N_local when every pair is
                                decided exactly once. tests_executed accumulates their sum over loads. */
  uint64_t visible_bits[2];  /* visible (Gaussian, camera) bits written by the last pass for accepted / exact-tested
                                slices; their sum equals sum_c K_c of the local cameras */
  uint64_t exact_pattern_tests[9]; /* isotropic exact tests by open-condition pattern (k_vis_tiles): left, top,
                                      right, bottom edge; top-left, top-right, bottom-left corner; the four edges;
                                      all six -- 3, 3, 7, 7, 6, 10, 10, 11, 11 FFMA per test (issued flop) */
  uint64_t render_tests;      /* last lobe_render_select: (pixel, splat) footprint tests in k_render (11 flop each) */
  uint64_t render_composited; /* ... of which composited (inside the 3-sigma ellipse: + 28 flop incl. the pinned exp) */
  double t_render_kernel_ms;  /* ... k_render's CUDA-event time summed over the batches */
} lobe_stats;

/* ---- scene --------------------------------------------------------------- */

/* Validate, resolve the frame, precompute per-Gaussian data (contraction,
 * grid coords, footprint radius, opacity gate, spatial sort) and per-camera
 * projection rows, then run the visibility pass once for the local cameras
 * (rows). Everything after this reuses the cached rows ("the back-projection
 * is computed once and reused"); the depth statistic (K_c, D_c,
 * z_min, z_max) is enqueued after the first crop kernel or by the first call
 * that needs it. Every input is validated, and the error names the first
 * invalid Gaussian. Host inputs in the isotropic mode (the quaternions are only
 * validated there): the positions are copied first (the spatial sort runs while
 * the other fields travel), the quaternions last, on a side stream, with their
 * own check, and this call returns without waiting for that check: its verdict
 * (LOBE_E_INVALID_INPUT, naming the first invalid quaternion) is the status of
 * the scene's next call, and of every call after it. The quaternion arrays of
 * such a load are read after the call returns: keep them valid and unmodified
 * until the scene's next call has returned (or lobe_free_scene). Every other
 * input is consumed before the call returns. With a communicator this call is
 * collective (NCCL communicators are created here on first use). inout_frame
 * may be NULL (= LOBE_FRAME_AUTO_ALL). */
lobe_status lobe_load_scene(const lobe_gaussians* gaussians, const lobe_camera* cameras, int64_t n_cams,
                            lobe_frame* inout_frame, const lobe_options* options, lobe_scene** out);
void lobe_free_scene(lobe_scene* scene);
const char* lobe_last_error(void);

/* ---- per-camera outputs: N entries (global) with a communicator or world == 1;
 *      a bare shard's n_local entries (see lobe_scene_info) otherwise -------- */

/* K_c, depth mean D_c = sum(o w)/sum(o) over V_c (0 if K_c = 0, ledger L4/L7),
 * z_min/z_max over V_c (+inf/-inf if K_c = 0); n_cb/n0_cb: N x B counts of
 * V_c inside the enlarged regions / delta = 0 cells;
 * member: bit b set iff K_c > 0 and n_cb >= tau K_c;
 * home: lowest b maximising n0_cb, camera-centre cell if K_c = 0 (ledger L7/L8).
 * Any output pointer may be NULL; host or device pointers. The outputs are
 * complete on return. Copies into pageable host memory wait only for the end of
 * the evaluation, not for later work on the scene's stream (e.g. a crop). */
lobe_status lobe_assign_cameras(lobe_scene* scene, const lobe_grid* grid, uint32_t* K, double* depth_mean,
                                float* z_min, float* z_max, uint32_t* n_cb, uint32_t* n0_cb, uint64_t* member,
                                int32_t* home);

/* ---- block loads (world == 1 or with a communicator: complete) ---------- */

/* out: B records; objective: max_b g_vis. */
lobe_status lobe_block_loads(lobe_scene* scene, const lobe_grid* grid, lobe_block_load* out, uint32_t* objective);

/* crop, eligible: B x ceil(G/64) u64, caller order. crop_b = union of the rows
 * of C^(b) (visibility cropping); eligible_b = crop_b and
 * "centre in the delta = 0 cell of b" (selective densification).
 * Either may be NULL. Host outputs are complete on return; device outputs (on
 * the scene's device) are written in the order of the scene's stream -- the
 * call returns without waiting, like a kernel launch. */
lobe_status lobe_crop_masks(lobe_scene* scene, const lobe_grid* grid, uint64_t* crop, uint64_t* eligible);

/* Load-balanced cuts: uniform cuts first, then n_sobol
 * scrambled Sobol points, then GP (Matern-5/2 ARD) + expected improvement, L
 * evaluations in total, each cut bounded to move at most halfway to its
 * neighbours. v_out: m-1, h_out: n-1 floats; history: L objective values
 * (may be NULL); cut_history: L x (m+n-2) floats (may be NULL); best: B records
 * at the returned cuts (may be NULL). With a communicator every evaluation is a
 * collective exchange; the deterministic BO then proposes the same cuts on every
 * rank (identical objective values), so no broadcast is needed. A bare shard
 * (world > 1, no communicator) returns LOBE_E_STATE. */
lobe_status lobe_balance_partition(lobe_scene* scene, int32_t m, int32_t n, const lobe_balance_opts* opts,
                                   float* v_out, float* h_out, uint32_t* history, float* cut_history,
                                   lobe_block_load* best);

/* Host-only BO driver with a caller objective (the same driver the call above
 * uses). objective(ctx, v, h, out_value) returns 0 on success. Needs no GPU. */
typedef int (*lobe_objective_fn)(void* ctx, const float* v, const float* h, uint32_t* out_value);
lobe_status lobe_bo_run(int32_t m, int32_t n, const lobe_balance_opts* opts, lobe_objective_fn objective, void* ctx,
                        float* v_out, float* h_out, uint32_t* history, float* cut_history);

/* ---- multi-rank exchange points (bare shards: world > 1 without a communicator) */

/* Rank-local part of lobe_block_loads: d_masks (DEVICE, B x lobe_mask_words
 * u32, internal Gaussian order) receives OR over the LOCAL cameras of C^(b);
 * n_cams / incid (B entries, host or device) the local counts. */
size_t lobe_mask_words(const lobe_scene* scene);
lobe_status lobe_block_partial(lobe_scene* scene, const lobe_grid* grid, uint32_t* d_masks, uint32_t* n_cams,
                               uint64_t* incid);
/* OR the W gathered partial mask sets (DEVICE, W x B x lobe_mask_words u32,
 * rank-major) into d_out (DEVICE, B x words) and popcount each block into g_vis
 * (B entries). d_out may alias d_gathered. */
lobe_status lobe_masks_combine(lobe_scene* scene, int32_t B, const uint32_t* d_gathered, int32_t W, uint32_t* d_out,
                               uint32_t* g_vis);
/* Assemble B records from global counts (areas, regions, G_blk from the scene). */
lobe_status lobe_block_records(lobe_scene* scene, const lobe_grid* grid, const uint32_t* n_cams,
                               const uint64_t* incid, const uint32_t* g_vis, lobe_block_load* out,
                               uint32_t* objective);
/* Crop / eligible masks (caller order) from combined masks d_masks (DEVICE). */
lobe_status lobe_crop_from_masks(lobe_scene* scene, const lobe_grid* grid, const uint32_t* d_masks, uint64_t* crop,
                                 uint64_t* eligible);

/* The exchange of SURVEY §8(e) on HOST buffers with host collectives (no GPU):
 * the same choreography the collective calls run (lib-internal xchg_*), exported
 * so a CPU process group can drive it (tests: gloo with oracle partials).
 * block loads: partial B x words u32, counts_local 2B u64 [|C^(b)| | I_b] ->
 *   own (this rank's blocks [floor(rB/W), floor((r+1)B/W)) x words, the OR of all
 *   ranks' partials), g_vis (B), counts_global (2B);
 * all masks: own -> all (B x words); gather cameras: N entries of elem bytes. */
lobe_status lobe_xchg_block_loads_host(const lobe_host_comm* comm, int32_t rank, int32_t world, int32_t B,
                                       size_t words, const uint32_t* partial, const uint64_t* counts_local,
                                       uint32_t* own, uint32_t* g_vis, uint64_t* counts_global);
lobe_status lobe_xchg_all_masks_host(const lobe_host_comm* comm, int32_t rank, int32_t world, int32_t B, size_t words,
                                     const uint32_t* own, uint32_t* all);
lobe_status lobe_xchg_gather_cameras_host(const lobe_host_comm* comm, int32_t rank, int32_t world, int64_t N,
                                          size_t elem, const void* local, void* out);

/* ---- introspection / tests ----------------------------------------------- */

/* ---------------------------------------------------------------------------
 * Block pipeline after the path (PAPER.md:156
 * "prune regions outside each block and merge", :185-187 visibility cropping and
 * selective densification; DESIGN.md ledger L25).
 *
 * A sub-scene: device SoA arrays of one block's Gaussians. origin: caller index
 * of the coarse Gaussian (-1 for Gaussians created by densification);
 * in_block: centre inside the block's delta = 0 half-open cell. Outputs are
 * written into caller-allocated device arrays of `capacity` entries; out->n
 * receives the count. If the count exceeds capacity nothing is written, out->n
 * is the needed count and the call returns LOBE_E_CAPACITY. Block indices are
 * b = p n + q of the grid (ledger L9); point-in-cell tests use the scene's
 * frame and min/max (O3), normalised coordinates clamped to [0,1] (L25). */
typedef struct {
  int64_t n;
  float *x, *y, *z, *sx, *sy, *sz, *qw, *qx, *qy, *qz, *opacity;
  int64_t* origin;
  uint8_t* in_block;
} lobe_subscene;

/* visibility_crop: the Gaussians of block b's crop mask M_b
 * (visible from some camera of C^(b)) in ascending caller index,
 * gathered from `coarse` (the loaded Gaussians, device pointers, caller order);
 * in_block = the eligible mask bit. Single-rank scenes. */
lobe_status lobe_block_subscene(lobe_scene* s, const lobe_grid* grid, int32_t block, const lobe_gaussians* coarse,
                                lobe_subscene* out, int64_t capacity);

/* simulate_densify_step: Gaussians with in_block and
 * grad >= tau_grad are cloned (max(s) < scale_split: two copies at
 * mu + (0.1 s) * n_k, the first keeps its origin) or split (two children at
 * mu + R(q)(s * n_k) with scale s / 1.6, origin -1), n_1 = normals[6 i .. 6 i + 2],
 * n_2 = normals[6 i + 3 .. 6 i + 5] (device, caller-drawn standard normals);
 * moved and new Gaussians get a fresh in-block test; every other Gaussian is
 * copied field for field; output in input order (each selected Gaussian
 * replaced in place by its two results). grad: device, in->n floats. */
lobe_status lobe_densify_step(lobe_scene* s, const lobe_grid* grid, int32_t block, const lobe_subscene* in,
                              const float* grad, const float* normals, float tau_grad, float scale_split,
                              lobe_subscene* out, int64_t capacity);

/* prune_outside: the Gaussians whose centre lies in block b's
 * delta = 0 cell (fresh test), in order; in_block = 1 for all of them. */
lobe_status lobe_prune_outside(lobe_scene* s, const lobe_grid* grid, int32_t block, const lobe_subscene* in,
                               lobe_subscene* out, int64_t capacity);

/* merge_blocks: concatenation of `count` sub-scenes in order.
 * LOBE_E_INTEGRITY if a non-negative origin index appears twice (the merged
 * arrays are still written). */
lobe_status lobe_merge_blocks(lobe_scene* s, const lobe_subscene* subs, int32_t count, lobe_subscene* out,
                              int64_t capacity);

/* ---------------------------------------------------------------------------
 * Paper-exact camera selection (SPEC.md:
 * 335-353, :383-387; DESIGN.md ledger L26). Renders, for every local camera, the
 * alpha-blended depth D = sum d_i a_i prod_{j<i}(1 - a_j) of its visible Gaussians
 * (EWA splats, front to back by centre depth, 3-sigma support, stop at
 * T < 1e-4) at 1/downscale resolution, back-projects every stride-th pixel with
 * weight >= eps_w to the ground grid and from then on assigns cameras by the
 * fraction of their cloud points inside each enlarged block (V_{c,b} >= tau,
 * K_c = cloud size) in every lobe_assign_cameras / lobe_block_loads /
 * lobe_balance_partition call; visibility rows, depth statistic and G_vis are
 * unchanged. coarse: the loaded Gaussians as device arrays (their rotations and
 * scales give the splats). downscale <= 0 -> 4, stride <= 0 -> 2, eps_w < 0 -> 0.1. */
lobe_status lobe_render_select(lobe_scene* s, const lobe_gaussians* coarse, int32_t downscale, int32_t stride,
                               float eps_w);
/* The clouds of the last lobe_render_select: offsets[N_local + 1] (host),
 * gu / gv (host or device, capacity entries), camera-major, row-major samples. */
lobe_status lobe_camera_clouds(lobe_scene* s, int64_t* offsets, float* gu, float* gv, int64_t capacity);
/* Depth and weight maps of one local camera ((height / ds) x (width / ds) floats,
 * host or device), rendered as lobe_render_select does. */
lobe_status lobe_render_maps(lobe_scene* s, const lobe_gaussians* coarse, int64_t camera, int32_t downscale,
                             float* depth, float* weight);

/* Sizes of a loaded scene without waiting for its work to finish (lobe_get_stats
 * synchronises the scene's stream to read the load-pass timings): total
 * Gaussians and cameras, this rank's camera count and first camera. Any output
 * pointer may be NULL. Errors: LOBE_E_STATE if s is NULL. */
lobe_status lobe_scene_info(const lobe_scene* s, int64_t* n_gaussians, int64_t* n_cameras, int64_t* n_local_cameras,
                            int64_t* cam_begin);

/* Visibility rows of local cameras [c0, c0 + count) in caller Gaussian order:
 * count x ceil(G/32) u32, bit (i mod 32) of word i/32 (for parity tests). */
lobe_status lobe_export_rows(lobe_scene* scene, int64_t c0, int64_t count, uint32_t* rows);
lobe_status lobe_get_stats(const lobe_scene* scene, lobe_stats* out);
/* Tuning: re-run the visibility kernel (a3) of this scene with kernel variant
 * `variant` (0 = default; all variants produce identical bytes) `reps` times on
 * options.stream; *ms = mean CUDA-event time per launch, *grid = CTAs launched.
 * LOBE_E_INVALID_INDEX for an unknown variant. */
lobe_status lobe_dev_vis_bench(lobe_scene* scene, int32_t variant, int32_t reps, float* ms, int32_t* grid);
/* Library build info string (arch, flags). */
const char* lobe_version(void);

#ifdef __cplusplus
}
#endif
#endif /* LOBE_H_ */
