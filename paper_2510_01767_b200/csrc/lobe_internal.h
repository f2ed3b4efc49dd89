// lobe_internal.h -- internal types shared by the host runtime (lobe_api.cpp)
// and the sm_100a kernels (lobe_kernels.cu). Not part of the public ABI.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace lobe {

// Geometry of the internal layout.
constexpr int kTile = 1024;                 // Gaussians per smem stage / per row tile (32 u32 words)
constexpr int kTileWords = kTile / 32;      // 32
constexpr int kChunk = 16384;               // Gaussians per visibility work item (fixed: world-size invariance)
constexpr int kTilesPerChunk = kChunk / kTile;
constexpr int kMaxBlocks = 64;              // B <= 64 (member mask is one u64)
constexpr int kMaxZones = 4 * kMaxBlocks + 2;  // per-axis zones upper bound
constexpr uint16_t kMixed = 0xFFFF;

// Per-camera projection rows: 16 floats, 64 B.
struct __align__(16) CamSetup {
  float Au[4];  // Au[0..2], au
  float Av[4];  // Av[0..2], av
  float Aw[4];  // Aw[0..2], aw
  float Wf, Hf, zn, zf;
};
static_assert(sizeof(CamSetup) == 64, "CamSetup layout");

// Per non-empty (tile, camera) pair: partial depth statistics (a4).
struct __align__(16) PairPartial {
  double S, O;       // sum o*w, sum o over the visible Gaussians of the pair
  float zmin, zmax;  // min/max w
  uint32_t K, pad;
};
static_assert(sizeof(PairPartial) == 32, "PairPartial layout");

// Zone tables for one grid (a5): per axis, sorted breakpoints P[0..nz-2] with
// P[0] = 0; zone z < nz-1 is [P[z], P[z+1]) (P[nz-1] := 1), zone nz-1 is {1}.
constexpr int kZoneBins = 1024;  // zone lookup bins per axis: bin b = [b / 1024, (b + 1) / 1024)
struct AxisZones {
  int nz;                      // number of zones including the top zone {1}
  int count;                   // intervals on this axis (m or n)
  float P[kMaxZones];          // breakpoints (nz-1 of them)
  uint8_t cell[kMaxZones];     // delta=0 interval of the zone
  uint64_t encl[kMaxZones];    // bitmask of enlarged intervals containing the zone
  // zone of x by bin (exact, replaces the binary search): low 12 bits = zone of the
  // bin's lower end; bits 14-15 = 0: no breakpoint strictly inside the bin, 1: one
  // (the zone is +1 from it on), 2: several (binary search)
  uint16_t bin[kZoneBins];
};
struct ZoneTables {
  AxisZones U, V;
  int m, n, B;
};

// ---- kernel launchers (lobe_kernels.cu) ------------------------------------
struct PrepIn {
  const float *x, *y, *z, *sx, *sy, *sz, *qw, *qx, *qy, *qz, *o;
  int64_t G;
  float c0[3], rho, au[3], av[3];
  float* cov;  // anisotropic predicate: 6 floats per Gaussian (caller order), else NULL
  int q_deferred;  // 1: the quaternions are validated by k_check_quats (host inputs, isotropic)
  // 0: one pass over every field; split passes for host inputs (the positions
  // arrive first, so the sort runs while the other fields are still in flight):
  // 1: positions only -> sort keys / values, ground min / max, position checks;
  // 2: the records (every field; keys, values and the min / max untouched)
  int pass;
};
// |q| = 1 +- 1e-6, the check k_prep_raw applies, for the deferred
// path: err |= 1 and err_idx = min index of an invalid quaternion
cudaError_t launch_check_quats(const float* qw, const float* qx, const float* qy, const float* qz, int64_t G,
                               uint32_t* err, unsigned long long* err_idx, cudaStream_t st);

// Anisotropic predicate (ledger L24): the raw camera parameters of the EWA
// footprint test, plus w2 >= ||R||_2^2 (host: max absolute row sum of R^T R in
// fp64) for the culling bound.
struct __align__(16) AnisoCam {
  float R[9], t[3];
  float fx, fy, cx, cy;
  float Wf, Hf, zn, zf;
  double w2, pad;
  // the depth-multiplied pixel forms of the box bound (box_class_aniso) as
  // affine forms of the world position, computed in fp64 and rounded once:
  // U = fx xc + cx zc, EU = fx xc + (cx - W) zc, V = fy yc + cy zc, EV = fy yc + (cy - H) zc
  float U[4], EU[4], V[4], EV[4];
};
static_assert(sizeof(AnisoCam) == 160, "AnisoCam layout");
// Validation + per-Gaussian raw ground coords and footprint radius (isotropic:
// k = 3 max(s); anisotropic: k = trace(Sigma) and Sigma into in.cov). err[0] =
// error class bits, err_idx = first bad index; mm_ord: ordered-int min/max.
// Also writes the 3D Hilbert sort key of the contracted centre and identity values.
cudaError_t launch_prep_raw(const PrepIn& in, float4* rec, uint32_t* keys, int32_t* vals, uint32_t* err,
                            unsigned long long* err_idx, uint32_t* mm_ord, cudaStream_t st);
// Normalise the ground coordinates to [0,1].
cudaError_t launch_cam_grid(int64_t N, const float* ru, const float* rv, const uint32_t* mm_ord, float* gu, float* gv,
                            cudaStream_t st);

// stable LSD radix sort of (key, value) pairs on key bits [begin_bit, end_bit)
cudaError_t radix_sort_pairs(void* tmp, size_t& tmp_bytes, const uint32_t* kin, uint32_t* kout, const int32_t* vin,
                             int32_t* vout, int64_t n, cudaStream_t st, int begin_bit = 0, int end_bit = 32);
// Gather into the internal pair-interleaved layout, build the inverse permutation;
// anisotropic: also Sigma, cv[3 (32 g + l) + {0,1,2}] = {S00A,S00B,S01A,S01B},
// {S02A,S02B,S11A,S11B}, {S12A,S12B,S22A,S22B}.
// wbox (may be NULL): per 32-Gaussian row word, the {min, max} of its real
// Gaussians' gu and gv as float bits {umin, umax, vmin, vmax} (a padding-only
// word: {~0, 0, ~0, 0}); a5 resolves zone-uniform words from it
cudaError_t launch_pack(int64_t G, int64_t G_pad, const int32_t* perm, const float4* rec, const uint32_t* mm_ord,
                        float* xy, float* zk, float* o2, float* gu, float* gv, int32_t* iperm, const float* cov_raw,
                        float4* cv, uint4* wbox, cudaStream_t st);

// a3: visibility tests -> rows, tile flags, per-(chunk,camera) partials.
struct VisArgs {
  const float4* xy;
  const float4* zk;
  const float2* o2;
  const CamSetup* cams;
  int64_t n_cams;      // local cameras
  int64_t n_chunks;
  int64_t words;       // row stride in u32 words (G_pad / 32)
  uint32_t* rows;
  uint8_t* flags;      // camera-inner variants only (may be NULL): [n_tiles x n_cams] any-visible flags
  uint8_t* nonempty;   // k_vis_tiles: [kept pairs], zeroed before the pass; 1 = some Gaussian visible
  const uint32_t* keep;  // [n_tiles x n_sub] camera masks surviving tile culling (NULL: dense)
  int64_t n_sub;         // ceil(n_cams / 32)
  const float4* slo;     // [n_tiles x 4] slice boxes (256 Gaussians) for k_vis_tiles
  const float4* shi;
  unsigned long long* counters;  // [32]: k_vis_tiles: [0] undecided, [1] accepted (slice, camera) pairs; I16
                                 // (measured, weighted by the slice's real Gaussians): [9] slice-rejected, [10]
                                 // slice-accepted, [11] exact-tested tests, [12] / [13] visible bits written for
                                 // accepted / exact-tested slices ([8]: k_cull's tile-rejected tests);
                                 // [16 + p]: exact-tested (slice, camera) pairs by open-condition pattern p
                                 // (isotropic; 9 patterns, see k_vis_tiles); may be NULL
  int64_t G;                     // real Gaussians (the rest of G_pad is padding)
  int aniso;                     // 1: anisotropic predicate (ledger L24)
  const float4* cv;              // anisotropic: pair-interleaved Sigma
  const AnisoCam* acams;         // anisotropic: per local camera
  const uint32_t* codes;         // k_vis_tiles (isotropic): per kept pair, the 4 slices' box_class codes (8 bits each)
  int aniso_fast;                // anisotropic: every camera's depth range within [2^-126, 2^126] (branch-free rcp/sqrt)
  const uint32_t* gcodes;        // k_vis_tiles_aniso: per kept pair, byte q = the classes (2 bits each) of
                                 // slice q's four 64-Gaussian pair groups when the slice is undecided
  const CamSetup* cam_pat;       // k_vis_tiles (isotropic): per local camera, kPatterns copies of its
                                 // CamSetup with the fields in each open-condition pattern's test order
};

// Tile culling: per camera the five linear forms of the
// test (w, u, v, eu, ev as c . p + c0, fp64 from the fp32 setup) and the depth
// range; per tile the AABB of its non-gated Gaussian centres and max k.
// tile boxes and 256-Gaussian slice boxes: lo = {x, y, z, kmin}, hi = {x, y, z, kmax}
// glo / ghi (may be NULL; the anisotropic mode's finer bound): the boxes of the
// 64-Gaussian pair groups, [n_tiles x 16]
cudaError_t launch_tile_bounds(const float4* xy, const float4* zk, int64_t n_tiles, float4* tlo, float4* thi,
                               float4* slo, float4* shi, float4* glo, float4* ghi, cudaStream_t st);
// hierarchical: chunk boxes (clo/chi scratch, n_tiles/16 each) then tile boxes
// rej_tests (may be NULL): += the real Gaussians of every (tile, camera) pair the
// chunk or tile bound rejects (I16, measured in the kernel)
cudaError_t launch_cull(const float4* tlo, const float4* thi, float4* clo, float4* chi, int64_t n_tiles, int64_t G,
                        const CamSetup* cams, const AnisoCam* acams, int64_t n_cams, uint32_t* keep, unsigned long long* kept_pairs,
                        unsigned long long* rej_tests, cudaStream_t st);
// kept-camera lists per tile: phase 0 counts, phase 1 fills (after a scan of the counts)
// per kept (tile, camera) pair (klist order): byte q = box_class of slice q
// (0 reject, 2 accept, 1 | need << 2 undecided), so the test kernel loads
// camera parameters only for undecided slices
// kPatterns pattern-ordered copies of every camera's CamSetup (k_vis_tiles stages
// the copy of a slice's open-condition pattern as is)
constexpr int kPatterns = 9;
cudaError_t launch_cam_patterns(const CamSetup* cams, int64_t n_cams, CamSetup* cam_pat, cudaStream_t st);
cudaError_t launch_slice_codes(int64_t n_units, const uint4* unit_meta, const uint32_t* klist, const CamSetup* cams,
                               const AnisoCam* acams, const float4* slo, const float4* shi, uint32_t* codes,
                               const float4* glo, const float4* ghi, uint32_t* gcodes, cudaStream_t st);
cudaError_t launch_keep_lists(const uint32_t* keep, int64_t n_tiles, int64_t n_sub, uint32_t* counts,
                              const uint32_t* offs, uint32_t* list, uint32_t* tlist, int phase, cudaStream_t st);
// tile-major visibility over the kept lists: work units = (tile, <= kVisUnit cameras)
constexpr int kVisUnit = 64;
cudaError_t launch_units(const uint32_t* koff, int64_t n_tiles, int cmax, uint32_t* uc, const uint32_t* uoff,
                         uint32_t* unit_tile, uint4* unit_meta, int64_t n_units, int phase, cudaStream_t st);
cudaError_t launch_vis_tiles(const VisArgs& a, const uint32_t* koff, const uint32_t* klist, const uint32_t* unit_tile,
                             const uint4* unit_meta, int64_t n_units, unsigned long long* queue, int num_sms,
                             cudaStream_t st, int* grid_out);
// tuning variants of the same kernel (bit-identical outputs)
int num_visibility_variants();
cudaError_t launch_visibility_variant(int variant, const VisArgs& a, int num_sms, cudaStream_t st, int* grid_out);
// a4: depth statistic per non-empty (tile, camera) pair, then per camera in tile order.
cudaError_t launch_depth_pairs(int64_t n_tiles, const uint32_t* tile_off, const uint32_t* pair_cam,
                               const uint32_t* rows, int64_t words, const float4* xy, const float4* zk,
                               const float2* o2, const CamSetup* cams, PairPartial* out, int ctas_per_sm,
                               unsigned long long* tile_queue, cudaStream_t st);
cudaError_t launch_cam_counts(int64_t n_pairs, const uint32_t* pair_cam, uint32_t* counts, cudaStream_t st);
// copy from pinned (mapped) host memory by a kernel, not the copy engine
cudaError_t launch_upload(void* dst, const void* src_pinned, size_t bytes, cudaStream_t st);
cudaError_t launch_iota(int32_t* v, int64_t n, cudaStream_t st);
cudaError_t launch_depth_reduce(int64_t n_cams, const uint32_t* cam_off, const int32_t* order, const PairPartial* part,
                                uint32_t* K, double* D, float* zmin, float* zmax, cudaStream_t st);
// tile -> camera lists (CSR) of the non-empty pairs, from the kept lists and nonempty bytes.
cudaError_t launch_tile_count(const uint32_t* koff, const uint8_t* nonempty, int64_t n_tiles, uint32_t* counts,
                              cudaStream_t st);
cudaError_t exclusive_scan_u32(void* tmp, size_t& tmp_bytes, const uint32_t* in, uint32_t* out, int64_t n,
                               cudaStream_t st);
cudaError_t launch_tile_fill(const uint32_t* koff, const uint32_t* klist, const uint8_t* nonempty, int64_t n_tiles,
                             const uint32_t* offsets, uint32_t* pair_cam, uint32_t* pair_tile, uint32_t* camtile,
                             int64_t tw, cudaStream_t st);
cudaError_t launch_cam_order(int64_t n_cams, int64_t tw, const uint32_t* camtile, uint32_t* wordpre,
                             uint32_t* counts, cudaStream_t st);
cudaError_t launch_cam_scatter(const uint32_t* tile_off, int64_t n_tiles, int64_t cap, const uint32_t* pair_cam,
                               const uint32_t* pair_tile, const uint32_t* camtile, const uint32_t* wordpre,
                               int64_t tw, const uint32_t* cam_off, int32_t* cam_order, cudaStream_t st);

// a5: per-Gaussian zone pair, per-word / per-tile uniform zone, per-zone counts.
// zp is written only for the words whose box straddles a zone boundary (the
// others are resolved from their word box: word_zone != kMixed there)
cudaError_t launch_zones(const ZoneTables* dz, int nzv, int nzp, int64_t G, int64_t G_pad, const float* gu,
                         const float* gv, const uint4* wbox, uint16_t* zp, uint16_t* word_zone, uint16_t* tile_zone,
                         uint32_t* zp_count, cudaStream_t st);
// a6: zone-pair histograms per camera from the (tile, camera) pairs.
// a6 per (tile, batch of 32 cameras of the tile's non-empty list)
cudaError_t launch_hist(int64_t n_tiles, const uint32_t* tile_off, const uint32_t* pair_cam, const uint32_t* rows,
                        int64_t words, const uint16_t* zp, const uint16_t* word_zone, const uint16_t* tile_zone,
                        int nzp, uint32_t* hist, cudaStream_t st);
// a7: n, n0, member, home, selection mask, |C^(b)|, I_b.
struct AssignArgs {
  const ZoneTables* dz;
  const uint32_t* hist;
  int nzp;
  const float* cam_gu;
  const float* cam_gv;
  int64_t n_cams;
  double tau;
  int mode;
  uint32_t* ncb;
  uint32_t* n0cb;
  uint64_t* member;
  int32_t* home;
  uint64_t* sel;
  uint32_t* ncams;       // [B]
  unsigned long long* incid;  // [B]
};
cudaError_t launch_assign(const AssignArgs& a, cudaStream_t st);
// a8: per-block OR of selected rows -> masks (internal order) + popcounts.
cudaError_t launch_block_masks(int64_t n_tiles, const uint32_t* tile_off, const uint32_t* pair_cam,
                               const uint64_t* sel, const uint32_t* rows, int64_t words, int B, uint32_t* masks,
                               uint32_t* gvis, cudaStream_t st);
cudaError_t launch_masks_combine(const uint32_t* gathered, int W, int B, int64_t words, uint32_t* out,
                                 uint32_t* gvis, cudaStream_t st);
// exchange buffer of the local block counts: out[b] = ncams[b] (u64), out[B + b] = incid[b]
cudaError_t launch_xcounts(const uint32_t* ncams, const unsigned long long* incid, int B, unsigned long long* out,
                           cudaStream_t st);
// a9: caller-order crop / eligible masks.
// mt: scratch, B x words u32 (word-major transpose of masks)
// a9: per-Gaussian block bits (scratch mbits, cb8: words * 32 entries each), then the caller-order gather
cudaError_t launch_crop(int64_t G, const int32_t* iperm, const uint16_t* zp, const uint16_t* word_zone,
                        const uint8_t* zp_cellblock,
                        const uint32_t* masks, int64_t words, int B, uint64_t* mbits, uint8_t* cb8, uint32_t* crop32,
                        uint32_t* elig32, cudaStream_t st);
cudaError_t launch_export_rows(int64_t G, const int32_t* iperm, const uint32_t* rows, int64_t words, int64_t c0,
                               int64_t count, const uint32_t* keep, int64_t n_sub, uint32_t* out, cudaStream_t st);
// G_blk from per-zone-pair counts.
cudaError_t launch_gblk(const ZoneTables* dz, int nzv, int nzp, const uint32_t* zp_count, uint32_t* gblk,
                        cudaStream_t st);

// ---- NEXT-4 block pipeline (ledger L25) -------------------------------------
struct SubArgs {  // 11 input float fields: x y z sx sy sz qw qx qy qz opacity
  const float* f[11];
};
struct SubOut {
  float* f[11];
  int64_t* origin;
  uint8_t* in_block;
};
struct CellArgs {  // delta = 0 cell of a position: frame (O3), min/max, cuts
  PrepIn frame;    // only c0, rho, au, av are used
  float mm[4];
  int m, n;
  float v[64], h[64];
};
cudaError_t launch_mask_popc(const uint64_t* mask, int64_t W64, uint32_t* cnt, cudaStream_t st);
cudaError_t launch_extract(const uint64_t* crop, const uint64_t* elig, int64_t W64, const uint32_t* off,
                           const SubArgs& in, const SubOut& out, cudaStream_t st);
cudaError_t launch_densify_count(int64_t n, const uint8_t* in_block, const float* grad, float tau, uint32_t* cnt,
                                 cudaStream_t st);
cudaError_t launch_densify_write(int64_t n, const SubArgs& in, const int64_t* origin, const uint8_t* in_block,
                                 const float* grad, const float* normals, float tau, float split, const uint32_t* off,
                                 const CellArgs& cell, int block, const SubOut& out, cudaStream_t st);
cudaError_t launch_prune_count(int64_t n, const float* x, const float* y, const float* z, const CellArgs& cell,
                               int block, uint32_t* cnt, cudaStream_t st);
cudaError_t launch_prune_write(int64_t n, const SubArgs& in, const int64_t* origin, const uint32_t* cnt,
                               const uint32_t* off, const SubOut& out, cudaStream_t st);
cudaError_t launch_origin_claim(int64_t n, const int64_t* origin, int64_t G, uint32_t* bits, unsigned long long* dup,
                                cudaStream_t st);

// ---- NEXT-1 depth-render camera selection (ledger L26) ---------------------
struct RenderCam {
  float R[9], t[3];
  float fx, fy, cx, cy;  // intrinsics at 1/downscale (fp32 divisions, as the oracle)
  int Wd, Hd, tw, th;    // image and tile-grid size (16 x 16 tiles)
  uint32_t tile0;        // first tile key of this camera within the batch
  uint32_t cam;          // local camera index
  int64_t map0;          // offset of its maps in the batch's D / W buffers
};
cudaError_t launch_perm_from_iperm(int64_t G, const int32_t* iperm, int32_t* perm, cudaStream_t st);
cudaError_t launch_rvis_count(int64_t k0, int64_t nk, const int32_t* cam_order, const uint32_t* pair_tile,
                              const uint32_t* pair_cam, const uint32_t* rows, int64_t words, uint32_t* cnt,
                              cudaStream_t st);
cudaError_t launch_rvis_fill(int64_t k0, int64_t nk, int c0, const int32_t* cam_order, const uint32_t* pair_tile,
                             const uint32_t* pair_cam, const uint32_t* rows, int64_t words, const uint32_t* pos,
                             const float4* prec, const RenderCam* rc, uint32_t zlo, int zb, unsigned long long* keys,
                             uint32_t* vals, float* rec, uint32_t* rcam, cudaStream_t st);
cudaError_t launch_render_prep(int64_t G, const int32_t* perm, const SubArgs& g, float4* prec, cudaStream_t st);
cudaError_t seg_sort_u64(void* tmp, size_t& tmp_bytes, const unsigned long long* kin, unsigned long long* kout,
                         const uint32_t* vin, uint32_t* vout, int64_t n, int nseg, const uint32_t* seg_begin,
                         const uint32_t* seg_end, cudaStream_t st);
cudaError_t sort_u64_pairs(void* tmp, size_t& tmp_bytes, const unsigned long long* kin, unsigned long long* kout,
                           const uint32_t* vin, uint32_t* vout, int64_t n, int end_bit, cudaStream_t st);
cudaError_t launch_tie_fix(int64_t n, const unsigned long long* key, uint32_t* val, const float* rec, cudaStream_t st);
cudaError_t sort_u32_pairs(void* tmp, size_t& tmp_bytes, const uint32_t* kin, uint32_t* kout, const uint32_t* vin,
                           uint32_t* vout, int64_t n, int end_bit, cudaStream_t st);
cudaError_t launch_bin_count(int64_t n, const uint32_t* svals, const float* rec, const uint32_t* rcam,
                             const RenderCam* rc, uint32_t* cnt, cudaStream_t st);
cudaError_t launch_bin_fill(int64_t n, const uint32_t* svals, const float* rec, const uint32_t* rcam,
                            const RenderCam* rc, const uint32_t* off, uint32_t* ekey, uint32_t* eval, cudaStream_t st);
cudaError_t launch_tile_ranges(int64_t n, const uint32_t* skey, uint32_t* start, uint32_t* end, cudaStream_t st);
cudaError_t launch_render(int ncam, int max_tiles, const RenderCam* rc, const uint32_t* start, const uint32_t* end,
                          const uint32_t* sval, const float* rec, float* Dmap, float* Wmap,
                          unsigned long long* counters, cudaStream_t st);
cudaError_t launch_bp_count(int ncam, int max_samples, const RenderCam* rc, int stride, float eps_w, const float* Wmap,
                            const uint32_t* sp0, uint32_t* flag, cudaStream_t st);
cudaError_t launch_bp_write(int ncam, int max_samples, const RenderCam* rc, int stride, const float* Dmap,
                            const uint32_t* sp0, const uint32_t* flag, const uint32_t* off, const PrepIn& frame,
                            const float* mm, uint32_t cloud0, float* pgu, float* pgv, uint32_t* pcam,
                            cudaStream_t st);
cudaError_t launch_hist_points(int64_t n, const float* pgu, const float* pgv, const uint32_t* pcam,
                               const ZoneTables* dz, int nzv, int nzp, uint32_t* hist, cudaStream_t st);

}  // namespace lobe
