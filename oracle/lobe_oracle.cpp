// lobe_oracle.cpp -- plain, slow, obviously-correct CPU oracle for the LoBE-GS
// visibility engine (arXiv 2510.01767).
//
// TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference leg may load this library. It shares no code,
// header, table or constant generator with the CUDA path
// (paper_2510_01767_b200/csrc) and neither side includes the other.
//
// What it computes: the steps O1-O11 of SURVEY.md §8(c), which restate the
// paper's definitions:
//   * visible set / frustum + footprint culling
//   * V_{c,b} = (1/K) sum_k 1[p_{c,k} in B^(b)]    PAPER.md:176-178 (§4.2, Eq. 3)
//   * C^(b) = { c | V_{c,b} >= tau }, tau = 0.15   PAPER.md:179 (§4.2)
//   * B^(b) = [v_{i-1}-dv, v_i+dv] x [h_{j-1}-dh, h_j+dh], (dv,dh)=(0.1/m,0.1/n)
//                                                  PAPER.md:167 (§4.1)
//   * G_vis^(b) = |{g visible from some c in C^(b)}|   PAPER.md:129, :185 (§3.2, §4.3)
//   * objective max_b G_vis^(b)                    PAPER.md:160-164 (§4.1, Eq. 2)
//   * A, C, G_blk, G_vis, G_avgvis                 PAPER.md:124-130 (§3.2)
//   * visibility cropping / selective densification masks  PAPER.md:185-187 (§4.3)
// with the readings of the DESIGN.md ledger (L1-L22): Gaussian-resolution
// back-projected cloud (L3), fp64 tau comparison (L6), half-open intervals
// closed at 1 (L11), spherical contraction frame (L12), fp64 camera setup (L13).
//
// Arithmetic contract (SURVEY.md §8c "Build flags"): every float operation is a
// single IEEE-754 binary32 operation in round-to-nearest-even; std::fmaf appears
// exactly where the contract writes fmaf; compiled with -ffp-contract=off
// -fno-fast-math so the compiler fuses nothing. No blocking, sorting, tiling or
// reordering: loops run in index order.
//
// Parity pins (tests/test_oracle_*.py): hand cases H1-H12 (tests/golden/), the
// float64 SPEC-formula brute force B1 (oracle/brute.py), set-level enumeration
// and the invariants I1-I16 / special cases P1-P6 of SURVEY.md §8(c).
// D_c (O7) has no paper value: it is pinned by hand case H7, invariants and a
// float64 recomputation from the caller's extrinsics (tests/test_oracle_props.py;
// "parity partially pinned" -- see DESIGN.md, ledger L3/L4).

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

namespace {

enum {
  O_OK = 0,
  O_E_INVALID_INPUT = 1,
  O_E_INVALID_CONFIG = 2,
  O_E_INVALID_CUTS = 3,
  O_E_INVALID_INDEX = 4,
  O_E_DEGENERATE_SCENE = 5,
};

// Largest magnitude accepted for positions / translations / scales (ledger L22):
// keeps every O6 intermediate finite so the predicate never sees inf - inf.
const double MAG_MAX = 1e18;

struct Cam {  // SPEC.md:44-49 CameraView; R = world_to_cam rotation, row major
  float fx, fy, cx, cy;
  int32_t width, height;
  float R[9];
  float t[3];
  float z_near, z_far;
};

// Per-camera setup, SURVEY.md §8c O4 (ledger L13).
struct Setup {
  float Au[3], au, Av[3], av, Aw[3], aw, Wf, Hf, zn, zf;
};

inline bool finite_f(float a) { return std::isfinite(a); }

// ---------------------------------------------------------------- O5 regions
// Interval membership on one axis: x in [lo, hi) or, when hi == 1, [lo, 1]
// (SPEC.md:89 and :125 half-open convention, ledger L11).
inline bool in_interval(float x, float lo, float hi) {
  return x >= lo && (x < hi || (hi == 1.0f && x <= 1.0f));
}

struct Axis {
  int count;
  std::vector<float> lo, hi, elo, ehi;
};

// cuts c[0..count-2]; delta is the fp32 enlargement on this axis.
Axis make_axis(int count, const float* cuts, float delta) {
  Axis a;
  a.count = count;
  for (int p = 0; p < count; ++p) {
    float lo = (p == 0) ? 0.0f : cuts[p - 1];
    float hi = (p == count - 1) ? 1.0f : cuts[p];
    a.lo.push_back(lo);
    a.hi.push_back(hi);
    a.elo.push_back(std::fmax(0.0f, lo - delta));
    a.ehi.push_back(std::fmin(1.0f, hi + delta));
  }
  return a;
}

// δ=0 cell index along an axis (the unique interval containing x).
int cell_of(const Axis& a, float x) {
  for (int p = 0; p < a.count; ++p)
    if (in_interval(x, a.lo[p], a.hi[p])) return p;
  return -1;  // unreachable for x in [0,1]
}

int check_grid(int m, int n, const float* v, const float* h, float dv, float dh, double tau) {
  if (m < 1 || n < 1 || (int64_t)m * n > 64) return O_E_INVALID_CONFIG;
  if (!(dv >= 0.0f) || !(dh >= 0.0f) || !std::isfinite(dv) || !std::isfinite(dh)) return O_E_INVALID_CONFIG;
  if (!(tau >= 0.0 && tau <= 1.0)) return O_E_INVALID_CONFIG;
  for (int i = 0; i + 1 < m; ++i) {
    if (!(v[i] > 0.0f && v[i] < 1.0f)) return O_E_INVALID_CUTS;
    if (i > 0 && !(v[i] > v[i - 1])) return O_E_INVALID_CUTS;
  }
  for (int j = 0; j + 1 < n; ++j) {
    if (!(h[j] > 0.0f && h[j] < 1.0f)) return O_E_INVALID_CUTS;
    if (j > 0 && !(h[j] > h[j - 1])) return O_E_INVALID_CUTS;
  }
  return O_OK;
}

inline uint32_t get_bit(const uint32_t* row, int64_t i) { return (row[i >> 5] >> (i & 31)) & 1u; }

template <class F>
void parallel_for(int64_t n, int nthreads, F f) {
  if (nthreads <= 1 || n <= 1) {
    for (int64_t i = 0; i < n; ++i) f(i);
    return;
  }
  int T = (int)std::min<int64_t>(nthreads, n);
  std::vector<std::thread> th;
  for (int t = 0; t < T; ++t) {
    int64_t b = n * t / T, e = n * (t + 1) / T;
    th.emplace_back([=, &f]() {
      for (int64_t i = b; i < e; ++i) f(i);
    });
  }
  for (auto& x : th) x.join();
}

}  // namespace

extern "C" {

// ------------------------------------------------------------------ O1 validate
// SPEC.md:30-33 (Gaussian3D invariants) and ledger L22 magnitude bound.
// Returns status; *bad = first offending index.
int oracle_validate_gaussians(int64_t G, const float* x, const float* y, const float* z, const float* sx,
                              const float* sy, const float* sz, const float* qw, const float* qx, const float* qy,
                              const float* qz, const float* o, int64_t* bad) {
  *bad = -1;
  if (G <= 0) return O_E_INVALID_CONFIG;  // zero counts
  for (int64_t i = 0; i < G; ++i) {
    bool ok = finite_f(x[i]) && finite_f(y[i]) && finite_f(z[i]) && std::fabs((double)x[i]) <= MAG_MAX &&
              std::fabs((double)y[i]) <= MAG_MAX && std::fabs((double)z[i]) <= MAG_MAX;
    ok = ok && finite_f(sx[i]) && finite_f(sy[i]) && finite_f(sz[i]) && sx[i] > 0.0f && sy[i] > 0.0f &&
         sz[i] > 0.0f && (double)sx[i] <= MAG_MAX && (double)sy[i] <= MAG_MAX && (double)sz[i] <= MAG_MAX;
    double qn = std::sqrt((double)qw[i] * qw[i] + (double)qx[i] * qx[i] + (double)qy[i] * qy[i] +
                          (double)qz[i] * qz[i]);
    ok = ok && std::isfinite(qn) && std::fabs(qn - 1.0) <= 1e-6;
    ok = ok && finite_f(o[i]) && o[i] >= 0.0f && o[i] <= 1.0f;
    if (!ok) {
      *bad = i;
      return O_E_INVALID_INPUT;
    }
  }
  return O_OK;
}

// SPEC.md:46-48 (CameraView invariants).
int oracle_validate_cameras(int64_t N, const Cam* cams, int64_t* bad) {
  *bad = -1;
  if (N <= 0) return O_E_INVALID_CONFIG;
  for (int64_t c = 0; c < N; ++c) {
    const Cam& k = cams[c];
    bool ok = finite_f(k.fx) && finite_f(k.fy) && finite_f(k.cx) && finite_f(k.cy) && k.fx > 0.0f &&
              k.fy > 0.0f && k.width > 0 && k.height > 0 && finite_f(k.z_near) && finite_f(k.z_far) &&
              k.z_near > 0.0f && k.z_near < k.z_far && std::fabs((double)k.cx) <= MAG_MAX &&
              std::fabs((double)k.cy) <= MAG_MAX;
    for (int j = 0; j < 3; ++j) ok = ok && finite_f(k.t[j]) && std::fabs((double)k.t[j]) <= MAG_MAX;
    for (int j = 0; j < 9; ++j) ok = ok && finite_f(k.R[j]);
    if (ok) {  // R R^T = I within 1e-5
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) {
          double d = 0;
          for (int j = 0; j < 3; ++j) d += (double)k.R[3 * a + j] * (double)k.R[3 * b + j];
          if (std::fabs(d - (a == b ? 1.0 : 0.0)) > 1e-5) ok = false;
        }
    }
    if (!ok) {
      *bad = c;
      return O_E_INVALID_INPUT;
    }
  }
  return O_OK;
}

// --------------------------------------------------------------------- O2 frame
// Ledger L12 / SPEC.md:123: centre = component-wise lower median of camera
// centres o_c = -R^T t (fp64, rounded once to fp32); radius = the ceil(0.9 N)-th
// smallest |o_c - c0| (fp64, rounded to fp32); axes default to world x, y.
// flags bit0: compute centre, bit1: compute radius, bit2: default axes.
int oracle_frame(int64_t N, const Cam* cams, uint32_t flags, float* c0, float* rho, float* au, float* av) {
  std::vector<double> ox(N), oy(N), oz(N);
  for (int64_t c = 0; c < N; ++c) {
    const float* R = cams[c].R;
    const float* t = cams[c].t;
    // o = -R^T t
    ox[c] = -((double)R[0] * t[0] + (double)R[3] * t[1] + (double)R[6] * t[2]);
    oy[c] = -((double)R[1] * t[0] + (double)R[4] * t[1] + (double)R[7] * t[2]);
    oz[c] = -((double)R[2] * t[0] + (double)R[5] * t[1] + (double)R[8] * t[2]);
  }
  if (flags & 1u) {
    std::vector<double>* comp[3] = {&ox, &oy, &oz};
    for (int a = 0; a < 3; ++a) {
      std::vector<double> s = *comp[a];
      std::sort(s.begin(), s.end());
      c0[a] = (float)s[(size_t)((N - 1) / 2)];  // lower median
    }
  }
  if (flags & 2u) {
    std::vector<double> d(N);
    for (int64_t c = 0; c < N; ++c) {
      double dx = ox[c] - (double)c0[0], dy = oy[c] - (double)c0[1], dz = oz[c] - (double)c0[2];
      d[c] = std::sqrt(dx * dx + dy * dy + dz * dz);
    }
    std::sort(d.begin(), d.end());
    int64_t kth = (9 * N + 9) / 10;  // ceil(0.9 N), 1-based
    *rho = (float)d[(size_t)(kth - 1)];
  }
  if (flags & 4u) {
    au[0] = 1.0f; au[1] = 0.0f; au[2] = 0.0f;
    av[0] = 0.0f; av[1] = 1.0f; av[2] = 0.0f;
  }
  for (int a = 0; a < 3; ++a)
    if (!finite_f(c0[a]) || !finite_f(au[a]) || !finite_f(av[a])) return O_E_INVALID_INPUT;
  if (!(*rho > 0.0f) || !finite_f(*rho)) return O_E_DEGENERATE_SCENE;
  return O_OK;
}

// ------------------------------------------------------------ O3 per Gaussian
// Contraction and ground projection + tight normalisation
// (SPEC.md:76-84). One fp32 operation per step, fmaf where written.
static void ground_uv(float px, float py, float pz, const float* c0, float rho, const float* au, const float* av,
                      float* gu, float* gv) {
  float dx = px - c0[0], dy = py - c0[1], dz = pz - c0[2];
  float hx = dx / rho, hy = dy / rho, hz = dz / rho;
  float r2 = std::fmaf(hx, hx, std::fmaf(hy, hy, hz * hz));
  float r = std::sqrt(r2);
  float yx = hx, yy = hy, yz = hz;
  if (!(r <= 1.0f)) {  // f(x) = (2 - 1/|x|) x/|x| outside the unit ball
    float s = (2.0f - 1.0f / r) / r;
    yx = hx * s;
    yy = hy * s;
    yz = hz * s;
  }
  *gu = std::fmaf(yx, au[0], std::fmaf(yy, au[1], yz * au[2]));
  *gv = std::fmaf(yx, av[0], std::fmaf(yy, av[1], yz * av[2]));
}

// Outputs k_i = 3 max(s), gate_i = (o_i >= 0.005),
// grid coords gu, gv in [0,1] and mm = {min_u, max_u, min_v, max_v}.
int oracle_prep(int64_t G, const float* x, const float* y, const float* z, const float* sx, const float* sy,
                const float* sz, const float* o, const float* c0, float rho, const float* au, const float* av,
                float* k, uint8_t* gate, float* gu, float* gv, float* mm) {
  std::vector<float> ru(G), rv(G);
  for (int64_t i = 0; i < G; ++i) {
    k[i] = 3.0f * std::fmax(std::fmax(sx[i], sy[i]), sz[i]);
    gate[i] = (o[i] >= 0.005f) ? 1 : 0;
    ground_uv(x[i], y[i], z[i], c0, rho, au, av, &ru[i], &rv[i]);
  }
  float mnu = ru[0], mxu = ru[0], mnv = rv[0], mxv = rv[0];
  for (int64_t i = 1; i < G; ++i) {
    mnu = std::min(mnu, ru[i]);
    mxu = std::max(mxu, ru[i]);
    mnv = std::min(mnv, rv[i]);
    mxv = std::max(mxv, rv[i]);
  }
  mm[0] = mnu; mm[1] = mxu; mm[2] = mnv; mm[3] = mxv;
  if (!std::isfinite(mnu) || !std::isfinite(mxu) || !std::isfinite(mnv) || !std::isfinite(mxv))
    return O_E_INVALID_INPUT;
  if (mxu == mnu || mxv == mnv) return O_E_DEGENERATE_SCENE;
  float du = mxu - mnu, dv = mxv - mnv;
  for (int64_t i = 0; i < G; ++i) {
    gu[i] = (ru[i] - mnu) / du;
    gv[i] = (rv[i] - mnv) / dv;
  }
  return O_OK;
}

// ----------------------------------------------------------- O4 camera setup
// Scaled projection rows in fp64 from the fp32 inputs, rounded once (L13).
// setup: 16 floats per camera, {Au[3], au, Av[3], av, Aw[3], aw, Wf, Hf, zn, zf}.
// cam_gu/cam_gv: camera centre mapped by O3 and clamped to [0,1] (K=0 home, L7).
int oracle_cam_setup(int64_t N, const Cam* cams, const float* c0, float rho, const float* au, const float* av,
                     const float* mm, float* setup, float* cam_gu, float* cam_gv) {
  for (int64_t c = 0; c < N; ++c) {
    const Cam& k = cams[c];
    double f = (double)std::max(k.fx, k.fy);
    Setup s;
    for (int j = 0; j < 3; ++j) {
      s.Au[j] = (float)(((double)k.fx * k.R[j] + (double)k.cx * k.R[6 + j]) / f);
      s.Av[j] = (float)(((double)k.fy * k.R[3 + j] + (double)k.cy * k.R[6 + j]) / f);
      s.Aw[j] = k.R[6 + j];
    }
    s.au = (float)(((double)k.fx * k.t[0] + (double)k.cx * k.t[2]) / f);
    s.av = (float)(((double)k.fy * k.t[1] + (double)k.cy * k.t[2]) / f);
    s.aw = k.t[2];
    s.Wf = (float)((double)k.width / f);
    s.Hf = (float)((double)k.height / f);
    s.zn = k.z_near;
    s.zf = k.z_far;
    std::memcpy(setup + 16 * c, &s, sizeof(Setup));
    static_assert(sizeof(Setup) == 64, "setup layout");
    // camera centre o_c = -R^T t in fp64, rounded to fp32, then O3's fp32 map
    const float* R = k.R;
    const float* t = k.t;
    float ox = (float)(-((double)R[0] * t[0] + (double)R[3] * t[1] + (double)R[6] * t[2]));
    float oy = (float)(-((double)R[1] * t[0] + (double)R[4] * t[1] + (double)R[7] * t[2]));
    float oz = (float)(-((double)R[2] * t[0] + (double)R[5] * t[1] + (double)R[8] * t[2]));
    float ru, rv;
    ground_uv(ox, oy, oz, c0, rho, au, av, &ru, &rv);
    float gu = (ru - mm[0]) / (mm[1] - mm[0]);
    float gv = (rv - mm[2]) / (mm[3] - mm[2]);
    cam_gu[c] = std::fmin(1.0f, std::fmax(0.0f, gu));
    cam_gv[c] = std::fmin(1.0f, std::fmax(0.0f, gv));
  }
  return O_OK;
}

// ---------------------------------------------------------- O6/O7 visibility
// For each selected camera c (sel[j], or j itself if sel == nullptr) and each
// Gaussian i in index order: the pinned predicate of SURVEY §8c O6, which in
// real arithmetic is SPEC.md:243's depth-in-(zn,zf) and pixel-in-dilated-image
// test with r = 3 max(s) max(fx,fy)/z. rows: camera-major,
// ceil(G/32) u32 words per selected camera, bit (i mod 32) of word i/32.
// K: |V_c|; S = sum o w, Om = sum o over V_c (fp64, index order);
// zmin/zmax over w (+inf/-inf when K = 0).
int oracle_visibility(int64_t G, const float* x, const float* y, const float* z, const float* k,
                      const uint8_t* gate, const float* o, int64_t nsel, const int64_t* sel, const float* setup,
                      uint32_t* rows, uint32_t* K, double* S, double* Om, float* zmin, float* zmax, int nthreads) {
  const int64_t words = (G + 31) / 32;
  parallel_for(nsel, nthreads, [&](int64_t j) {
    int64_t c = sel ? sel[j] : j;
    Setup s;
    std::memcpy(&s, setup + 16 * c, sizeof(Setup));
    uint32_t* row = rows + j * words;
    std::fill(row, row + words, 0u);
    uint32_t cnt = 0;
    double sum_ow = 0.0, sum_o = 0.0;
    float mn = INFINITY, mx = -INFINITY;
    for (int64_t i = 0; i < G; ++i) {
      float w = std::fmaf(s.Aw[0], x[i], std::fmaf(s.Aw[1], y[i], std::fmaf(s.Aw[2], z[i], s.aw)));
      float u = std::fmaf(s.Au[0], x[i], std::fmaf(s.Au[1], y[i], std::fmaf(s.Au[2], z[i], s.au)));
      float v = std::fmaf(s.Av[0], x[i], std::fmaf(s.Av[1], y[i], std::fmaf(s.Av[2], z[i], s.av)));
      float eu = std::fmaf(-s.Wf, w, u);
      float ev = std::fmaf(-s.Hf, w, v);
      float ki = k[i];
      bool visible = gate[i] && w > s.zn && w < s.zf && u >= -ki && eu <= ki && v >= -ki && ev <= ki;
      if (visible) {
        row[i >> 5] |= 1u << (i & 31);
        cnt += 1;
        sum_ow += (double)o[i] * (double)w;
        sum_o += (double)o[i];
        mn = std::min(mn, w);
        mx = std::max(mx, w);
      }
    }
    K[j] = cnt;
    S[j] = sum_ow;
    Om[j] = sum_o;
    zmin[j] = mn;
    zmax[j] = mx;
  });
  return O_OK;
}

// ------------------------------------------------ O6a anisotropic predicate
// SURVEY §8f NEXT-2 / ledger L24: the projected-covariance footprint of SPEC.md
// :338 and :387 (EWA: Sigma' = J W Sigma W^T J^T + 0.3 I, radius 3 sqrt(lambda_max),
// S:299's "3 sigma footprint from projected covariance") replaces the isotropic
// bound; depth range and opacity gate as in O6.
//
// Per Gaussian (oracle_cov): rotation from the quaternion as given (validated
// unit norm, not renormalised), M = R diag(s), Sigma = M M^T:
//   r00 = 1 - 2(y y + z z), r01 = 2(x y - w z), r02 = 2(x z + w y),
//   r10 = 2(x y + w z), r11 = 1 - 2(x x + z z), r12 = 2(y z - w x),
//   r20 = 2(x z - w y), r21 = 2(y z + w x), r22 = 1 - 2(x x + y y),
//   M_ij = r_ij s_j, Sigma_ij = fma(M_i0, M_j0, fma(M_i1, M_j1, M_i2 M_j2)).
// cov: 6 floats per Gaussian {S00, S01, S02, S11, S12, S22}; trace out (for the
// GPU's culling bound it is not needed here).
int oracle_cov(int64_t G, const float* sx, const float* sy, const float* sz, const float* qw, const float* qx,
               const float* qy, const float* qz, float* cov) {
  for (int64_t i = 0; i < G; ++i) {
    const float w = qw[i], x = qx[i], y = qy[i], z = qz[i];
    float r[9];
    r[0] = 1.0f - 2.0f * (y * y + z * z);
    r[1] = 2.0f * (x * y - w * z);
    r[2] = 2.0f * (x * z + w * y);
    r[3] = 2.0f * (x * y + w * z);
    r[4] = 1.0f - 2.0f * (x * x + z * z);
    r[5] = 2.0f * (y * z - w * x);
    r[6] = 2.0f * (x * z - w * y);
    r[7] = 2.0f * (y * z + w * x);
    r[8] = 1.0f - 2.0f * (x * x + y * y);
    const float s[3] = {sx[i], sy[i], sz[i]};
    float M[9];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) M[3 * a + b] = r[3 * a + b] * s[b];
    auto sig = [&](int a, int b) {
      return std::fmaf(M[3 * a], M[3 * b], std::fmaf(M[3 * a + 1], M[3 * b + 1], M[3 * a + 2] * M[3 * b + 2]));
    };
    float* c = cov + 6 * i;
    c[0] = sig(0, 0); c[1] = sig(0, 1); c[2] = sig(0, 2);
    c[3] = sig(1, 1); c[4] = sig(1, 2); c[5] = sig(2, 2);
  }
  return O_OK;
}

// Per (camera c, Gaussian i), with the camera's raw fp32 R (rows), t, fx, fy,
// cx, cy, W, H, z_near, z_far (no pre-scaling):
//   xc = fma(R00, x, fma(R01, y, fma(R02, z, t0)))      (yc, zc: rows 1, 2)
//   depth ok: zc > zn && zc < zf      (invisible otherwise; nothing else evaluated)
//   iz = 1 / zc;  a = xc iz;  b = yc iz;  upix = fma(fx, a, cx);  vpix = fma(fy, b, cy)
//   j00 = fx iz;  j11 = fy iz;  j02 = -(j00 a);  j12 = -(j11 b)
//   T0k = fma(j00, R0k, j02 R2k);  T1k = fma(j11, R1k, j12 R2k)          (T = J W)
//   V0i = fma(Si0, T00, fma(Si1, T01, Si2 T02)), V1i likewise with T1   (V = Sigma T^T)
//   A = fma(T00, V00, fma(T01, V01, T02 V02)) + 0.3
//   B = fma(T10, V00, fma(T11, V01, T12 V02))
//   C = fma(T10, V10, fma(T11, V11, T12 V12)) + 0.3
//   mid = 0.5 (A + C);  d = 0.5 (A - C);  disc = fma(d, d, B B)
//   r = 3 sqrt(mid + sqrt(disc))
//   visible = gate && depth ok && upix >= -r && upix <= W + r && vpix >= -r && vpix <= H + r
// (all IEEE binary32, round to nearest; division and square roots correctly
// rounded). The depth statistic uses w = zc (the same fma chain as O6's w).
int oracle_visibility_aniso(int64_t G, const float* x, const float* y, const float* z, const float* cov,
                            const uint8_t* gate, const float* o, int64_t nsel, const int64_t* sel, const Cam* cams,
                            uint32_t* rows, uint32_t* K, double* S, double* Om, float* zmin, float* zmax,
                            int nthreads) {
  const int64_t words = (G + 31) / 32;
  parallel_for(nsel, nthreads, [&](int64_t j) {
    const int64_t c = sel ? sel[j] : j;
    const Cam& k = cams[c];
    const float* R = k.R;
    const float Wf = (float)k.width, Hf = (float)k.height;
    uint32_t* row = rows + j * words;
    std::fill(row, row + words, 0u);
    uint32_t cnt = 0;
    double sum_ow = 0.0, sum_o = 0.0;
    float mn = INFINITY, mx = -INFINITY;
    for (int64_t i = 0; i < G; ++i) {
      const float xc = std::fmaf(R[0], x[i], std::fmaf(R[1], y[i], std::fmaf(R[2], z[i], k.t[0])));
      const float yc = std::fmaf(R[3], x[i], std::fmaf(R[4], y[i], std::fmaf(R[5], z[i], k.t[1])));
      const float zc = std::fmaf(R[6], x[i], std::fmaf(R[7], y[i], std::fmaf(R[8], z[i], k.t[2])));
      if (!gate[i] || !(zc > k.z_near && zc < k.z_far)) continue;
      const float iz = 1.0f / zc;
      const float a = xc * iz, b = yc * iz;
      const float upix = std::fmaf(k.fx, a, k.cx), vpix = std::fmaf(k.fy, b, k.cy);
      const float j00 = k.fx * iz, j11 = k.fy * iz;
      const float j02 = -(j00 * a), j12 = -(j11 * b);
      float T0[3], T1[3];
      for (int q = 0; q < 3; ++q) {
        T0[q] = std::fmaf(j00, R[q], j02 * R[6 + q]);
        T1[q] = std::fmaf(j11, R[3 + q], j12 * R[6 + q]);
      }
      const float* cv = cov + 6 * i;
      const float Sg[3][3] = {{cv[0], cv[1], cv[2]}, {cv[1], cv[3], cv[4]}, {cv[2], cv[4], cv[5]}};
      float V0[3], V1[3];
      for (int q = 0; q < 3; ++q) {
        V0[q] = std::fmaf(Sg[q][0], T0[0], std::fmaf(Sg[q][1], T0[1], Sg[q][2] * T0[2]));
        V1[q] = std::fmaf(Sg[q][0], T1[0], std::fmaf(Sg[q][1], T1[1], Sg[q][2] * T1[2]));
      }
      const float A = std::fmaf(T0[0], V0[0], std::fmaf(T0[1], V0[1], T0[2] * V0[2])) + 0.3f;
      const float B = std::fmaf(T1[0], V0[0], std::fmaf(T1[1], V0[1], T1[2] * V0[2]));
      const float C = std::fmaf(T1[0], V1[0], std::fmaf(T1[1], V1[1], T1[2] * V1[2])) + 0.3f;
      const float mid = 0.5f * (A + C), d = 0.5f * (A - C);
      const float disc = std::fmaf(d, d, B * B);
      const float r = 3.0f * std::sqrt(mid + std::sqrt(disc));
      const bool visible = upix >= -r && upix <= Wf + r && vpix >= -r && vpix <= Hf + r;
      if (visible) {
        row[i >> 5] |= 1u << (i & 31);
        cnt += 1;
        sum_ow += (double)o[i] * (double)zc;
        sum_o += (double)o[i];
        mn = std::min(mn, zc);
        mx = std::max(mx, zc);
      }
    }
    K[j] = cnt;
    S[j] = sum_ow;
    Om[j] = sum_o;
    zmin[j] = mn;
    zmax[j] = mx;
  });
  return O_OK;
}

// ------------------------------------------------------------- O8 assignment
// n[c][b] = |{i in V_c : (gu_i, gv_i) in B^(b)}| over the enlarged regions
// (PAPER.md:167, :176-178); n0 over the delta=0 cells. member bit b set iff
// K_c > 0 and (double)n >= tau * (double)K (one fp64 multiply, ledger L6,
// PAPER.md:179). home = lowest b maximising n0 (L16); K_c = 0 -> cell of the
// camera centre (L7).
int oracle_assign(int64_t G, const float* gu, const float* gv, int64_t nsel, const uint32_t* rows,
                  const uint32_t* K, const float* cam_gu, const float* cam_gv, int m, int n, const float* vcuts,
                  const float* hcuts, float dv, float dh, double tau, uint32_t* ncb, uint32_t* n0cb,
                  uint64_t* member, int32_t* home, int nthreads) {
  int st = check_grid(m, n, vcuts, hcuts, dv, dh, tau);
  if (st) return st;
  const int B = m * n;
  const int64_t words = (G + 31) / 32;
  Axis U = make_axis(m, vcuts, dv), V = make_axis(n, hcuts, dh);
  parallel_for(nsel, nthreads, [&](int64_t j) {
    const uint32_t* row = rows + j * words;
    uint32_t* nj = ncb + j * B;
    uint32_t* n0j = n0cb + j * B;
    for (int b = 0; b < B; ++b) nj[b] = n0j[b] = 0;
    for (int64_t i = 0; i < G; ++i) {
      if (!get_bit(row, i)) continue;
      for (int p = 0; p < m; ++p)
        for (int q = 0; q < n; ++q) {
          if (in_interval(gu[i], U.elo[p], U.ehi[p]) && in_interval(gv[i], V.elo[q], V.ehi[q])) nj[p * n + q] += 1;
          if (in_interval(gu[i], U.lo[p], U.hi[p]) && in_interval(gv[i], V.lo[q], V.hi[q])) n0j[p * n + q] += 1;
        }
    }
    uint64_t mem = 0;
    if (K[j] > 0)
      for (int b = 0; b < B; ++b)
        if ((double)nj[b] >= tau * (double)K[j]) mem |= (uint64_t)1 << b;
    member[j] = mem;
    int hb;
    if (K[j] > 0) {
      hb = 0;
      for (int b = 1; b < B; ++b)
        if (n0j[b] > n0j[hb]) hb = b;
    } else {
      hb = cell_of(U, cam_gu[j]) * n + cell_of(V, cam_gv[j]);
    }
    home[j] = hb;
  });
  return O_OK;
}

// ------------------------------------------------------------- O9 block loads
// mode 0 = RATIO (C^(b) = {c : b in member_c}), 1 = HOME,
// 2 = RATIO u HOME (ledger L8). M (out, may be null): B x ceil(G/64) u64 masks,
// caller order. Per block: n_cams = |C^(b)|, g_vis = popcount(M_b) (L18),
// g_blk = #{i : cell(i) = b} over all Gaussians (L19), incid = sum_c n0[c][b],
// area = (hi_p - lo_p)(hi_q - lo_q) in fp64 of the delta=0 cell,
// g_avgvis = g_vis / n_cams or 0, lohi = enlarged region
// {elo_p, elo_q, ehi_p, ehi_q}. objective = max_b g_vis.
int oracle_block_loads(int64_t G, const float* gu, const float* gv, int64_t N, const uint32_t* rows,
                       const uint64_t* member, const int32_t* home, const uint32_t* n0cb, int m, int n,
                       const float* vcuts, const float* hcuts, float dv, float dh, int mode, uint32_t* n_cams,
                       uint32_t* g_blk, uint32_t* g_vis, uint64_t* incid, double* area, double* g_avgvis,
                       float* lohi, uint64_t* M, uint32_t* objective) {
  int st = check_grid(m, n, vcuts, hcuts, dv, dh, 0.0);
  if (st) return st;
  if (mode < 0 || mode > 2) return O_E_INVALID_CONFIG;
  const int B = m * n;
  const int64_t words = (G + 31) / 32;
  const int64_t words64 = (G + 63) / 64;
  Axis U = make_axis(m, vcuts, dv), V = make_axis(n, hcuts, dh);
  std::vector<uint32_t> cellblk(G);
  for (int64_t i = 0; i < G; ++i) cellblk[i] = cell_of(U, gu[i]) * n + cell_of(V, gv[i]);
  uint32_t best = 0;
  for (int b = 0; b < B; ++b) {
    std::vector<uint32_t> acc(words, 0u);
    uint32_t nc = 0;
    uint64_t inc = 0;
    for (int64_t c = 0; c < N; ++c) {
      inc += n0cb[c * B + b];
      bool in_ratio = (member[c] >> b) & 1u;
      bool in_home = home[c] == b;
      bool sel = (mode == 0) ? in_ratio : (mode == 1) ? in_home : (in_ratio || in_home);
      if (!sel) continue;
      nc += 1;
      const uint32_t* row = rows + c * words;
      for (int64_t w = 0; w < words; ++w) acc[w] |= row[w];
    }
    uint32_t gvis = 0;
    for (int64_t i = 0; i < G; ++i) gvis += get_bit(acc.data(), i);
    uint32_t gb = 0;
    for (int64_t i = 0; i < G; ++i) gb += (cellblk[i] == (uint32_t)b);
    int p = b / n, q = b % n;
    n_cams[b] = nc;
    g_vis[b] = gvis;
    g_blk[b] = gb;
    incid[b] = inc;
    area[b] = ((double)U.hi[p] - (double)U.lo[p]) * ((double)V.hi[q] - (double)V.lo[q]);
    g_avgvis[b] = nc ? (double)gvis / (double)nc : 0.0;
    lohi[4 * b + 0] = U.elo[p];
    lohi[4 * b + 1] = V.elo[q];
    lohi[4 * b + 2] = U.ehi[p];
    lohi[4 * b + 3] = V.ehi[q];
    best = std::max(best, gvis);
    if (M) {
      uint64_t* Mb = M + (int64_t)b * words64;
      for (int64_t w = 0; w < words64; ++w) Mb[w] = 0;
      for (int64_t i = 0; i < G; ++i)
        if (get_bit(acc.data(), i)) Mb[i >> 6] |= (uint64_t)1 << (i & 63);
    }
  }
  *objective = best;
  return O_OK;
}

// ------------------------------------------------------------------ O10 crop
// crop_b = M_b (PAPER.md:185 G_vis^(b)); eligible_b = M_b and cell_b
// ("restricts densification to Gaussians strictly within the
// block").
int oracle_crop(int64_t G, const float* gu, const float* gv, int m, int n, const float* vcuts, const float* hcuts,
                const uint64_t* M, uint64_t* crop, uint64_t* eligible) {
  int st = check_grid(m, n, vcuts, hcuts, 0.0f, 0.0f, 0.0);
  if (st) return st;
  const int B = m * n;
  const int64_t words64 = (G + 63) / 64;
  Axis U = make_axis(m, vcuts, 0.0f), V = make_axis(n, hcuts, 0.0f);
  for (int b = 0; b < B; ++b)
    for (int64_t w = 0; w < words64; ++w) {
      crop[(int64_t)b * words64 + w] = M[(int64_t)b * words64 + w];
      eligible[(int64_t)b * words64 + w] = 0;
    }
  for (int64_t i = 0; i < G; ++i) {
    int b = cell_of(U, gu[i]) * n + cell_of(V, gv[i]);
    uint64_t bit = (uint64_t)1 << (i & 63);
    if (M[(int64_t)b * words64 + (i >> 6)] & bit) eligible[(int64_t)b * words64 + (i >> 6)] |= bit;
  }
  return O_OK;
}

// ------------------------------------------- NEXT-4 block pipeline (L25)
// Block of arbitrary points (densified children, moved clones): O3's map with
// the scene's frame and min/max, normalised coordinates clamped to [0,1]
// (ledger L25), then the delta = 0 half-open cells (L11). block[i] = p n + q.
int oracle_block_of_points(int64_t N, const float* x, const float* y, const float* z, const float* c0, float rho,
                           const float* au, const float* av, const float* mm, int m, int n, const float* vcuts,
                           const float* hcuts, int32_t* block) {
  int st = check_grid(m, n, vcuts, hcuts, 0.0f, 0.0f, 0.0);
  if (st) return st;
  Axis U = make_axis(m, vcuts, 0.0f), V = make_axis(n, hcuts, 0.0f);
  const float du = mm[1] - mm[0], dv = mm[3] - mm[2];
  for (int64_t i = 0; i < N; ++i) {
    float ru, rv;
    ground_uv(x[i], y[i], z[i], c0, rho, au, av, &ru, &rv);
    float gu = (ru - mm[0]) / du, gv = (rv - mm[2]) / dv;
    gu = std::fmin(1.0f, std::fmax(0.0f, gu));
    gv = std::fmin(1.0f, std::fmax(0.0f, gv));
    block[i] = cell_of(U, gu) * n + cell_of(V, gv);
  }
  return O_OK;
}

// ------------------------------------- NEXT-1 depth-render camera selection (L26)
// SURVEY §8f NEXT-1; PAPER.md:175-179 (alpha-blended depth D = sum d_i a_i
// prod_{j<i}(1 - a_j), back-projected to a point cloud, V_{c,b} ratios);
// SPEC.md:335-353, :383-387 (downscale 4, stride 2, weight floor 0.1,
// front-to-back by centre depth, EWA covariance + 0.3 px^2, stop at T < 1e-4).
//
// exp for the footprint weight, x in [-4.5, 0]: 2^n p(r), n = nearest(x log2 e),
// r = x - n ln2 (two-step Cody-Waite), p = degree-7 Taylor polynomial in Horner
// form with fmaf; the scaling by 2^n is exact (ledger L26).
float exp_l26(float x) {
  const float n = std::nearbyintf(x * 1.44269504f);
  float r = std::fmaf(n, -0.693145752f, x);
  r = std::fmaf(n, -1.42860677e-06f, r);
  float p = 1.98412701e-04f;
  p = std::fmaf(p, r, 1.38888892e-03f);
  p = std::fmaf(p, r, 8.33333377e-03f);
  p = std::fmaf(p, r, 4.16666679e-02f);
  p = std::fmaf(p, r, 1.66666672e-01f);
  p = std::fmaf(p, r, 0.5f);
  p = std::fmaf(p, r, 1.0f);
  p = std::fmaf(p, r, 1.0f);
  return std::ldexp(p, (int)n);
}

// Render one camera at 1/ds resolution from its visible Gaussians (vis: caller
// indices, any order; sorted here by (zc, index)), then back-project every
// stride-th pixel (row-major) with weight >= eps_w. Per Gaussian (O6a's
// sequence with fx' = fx/ds, fy' = fy/ds, cx' = cx/ds, cy' = cy/ds): upix, vpix,
// A, B, C; det = A C - B B (skip if det <= 0); conic ca = C/det, cb = -(B/det),
// cc = A/det. Per pixel centre (px + 0.5, py + 0.5): dx = px + 0.5 - upix,
// dy likewise, power = -0.5 ((ca dx) dx + (cc dy) dy) - (cb dx) dy; a Gaussian
// contributes iff power >= -4.5 (inside its 3-sigma ellipse):
// alpha = o exp_l26(min(power, 0)); w = alpha T; D += zc w; W += w;
// T *= (1 - alpha); stop when T < 1e-4. Back-projection: xn = (u - cx')/fx',
// yn = (v - cy')/fy', Pc = (xn D, yn D, D), world_k = fma(R0k, q0, fma(R1k, q1,
// R2k q2)) with q = Pc - t, then O3's map, min/max normalisation, clamp to [0,1].
// Outputs: D, W maps (H' x W', W' = width / ds), cloud points (pu, pv, up to
// ceil(H'/stride) ceil(W'/stride)), *K.
int oracle_render_camera(int64_t G, const float* x, const float* y, const float* z, const float* cov,
                         const float* o, const Cam* cam, int64_t nvis, const int64_t* vis, int ds, int stride,
                         float eps_w, const float* c0, float rho, const float* au, const float* av, const float* mm,
                         float* Dmap, float* Wmap, float* pu, float* pv, int64_t* K) {
  const Cam& k = *cam;
  const float* R = k.R;
  const float fx = k.fx / (float)ds, fy = k.fy / (float)ds, cx = k.cx / (float)ds, cy = k.cy / (float)ds;
  const int Wd = k.width / ds, Hd = k.height / ds;
  struct Rec { float zc; int64_t i; float up, vp, ca, cb, cc, o; bool ok; };
  std::vector<Rec> g(nvis);
  for (int64_t n = 0; n < nvis; ++n) {
    const int64_t i = vis[n];
    Rec& e = g[n];
    e.i = i;
    const float xc = std::fmaf(R[0], x[i], std::fmaf(R[1], y[i], std::fmaf(R[2], z[i], k.t[0])));
    const float yc = std::fmaf(R[3], x[i], std::fmaf(R[4], y[i], std::fmaf(R[5], z[i], k.t[1])));
    const float zc = std::fmaf(R[6], x[i], std::fmaf(R[7], y[i], std::fmaf(R[8], z[i], k.t[2])));
    e.zc = zc;
    const float iz = 1.0f / zc;
    const float a = xc * iz, b = yc * iz;
    e.up = std::fmaf(fx, a, cx);
    e.vp = std::fmaf(fy, b, cy);
    const float j00 = fx * iz, j11 = fy * iz;
    const float j02 = -(j00 * a), j12 = -(j11 * b);
    float T0[3], T1[3];
    for (int q = 0; q < 3; ++q) {
      T0[q] = std::fmaf(j00, R[q], j02 * R[6 + q]);
      T1[q] = std::fmaf(j11, R[3 + q], j12 * R[6 + q]);
    }
    const float* cv = cov + 6 * i;
    const float Sg[3][3] = {{cv[0], cv[1], cv[2]}, {cv[1], cv[3], cv[4]}, {cv[2], cv[4], cv[5]}};
    float V0[3], V1[3];
    for (int q = 0; q < 3; ++q) {
      V0[q] = std::fmaf(Sg[q][0], T0[0], std::fmaf(Sg[q][1], T0[1], Sg[q][2] * T0[2]));
      V1[q] = std::fmaf(Sg[q][0], T1[0], std::fmaf(Sg[q][1], T1[1], Sg[q][2] * T1[2]));
    }
    const float A = std::fmaf(T0[0], V0[0], std::fmaf(T0[1], V0[1], T0[2] * V0[2])) + 0.3f;
    const float B = std::fmaf(T1[0], V0[0], std::fmaf(T1[1], V0[1], T1[2] * V0[2]));
    const float C = std::fmaf(T1[0], V1[0], std::fmaf(T1[1], V1[1], T1[2] * V1[2])) + 0.3f;
    const float p1 = A * C, p2 = B * B;
    const float det = p1 - p2;
    e.ok = det > 0.0f;
    e.ca = C / det;
    e.cb = -(B / det);
    e.cc = A / det;
    e.o = o[i];
  }
  std::stable_sort(g.begin(), g.end(), [](const Rec& a, const Rec& b) {
    return a.zc < b.zc || (a.zc == b.zc && a.i < b.i);
  });
  for (int py = 0; py < Hd; ++py)
    for (int px = 0; px < Wd; ++px) {
      float D = 0.0f, Wt = 0.0f, T = 1.0f;
      const float u = (float)px + 0.5f, v = (float)py + 0.5f;
      for (const Rec& e : g) {
        if (!e.ok) continue;
        const float dx = u - e.up, dy = v - e.vp;
        const float t1 = (e.ca * dx) * dx, t2 = (e.cc * dy) * dy, t3 = (e.cb * dx) * dy;
        const float power = -0.5f * (t1 + t2) - t3;
        if (!(power >= -4.5f)) continue;
        const float alpha = e.o * exp_l26(std::fmin(power, 0.0f));
        const float w = alpha * T;
        D = D + e.zc * w;
        Wt = Wt + w;
        T = T * (1.0f - alpha);
        if (T < 1e-4f) break;
      }
      Dmap[(int64_t)py * Wd + px] = D;
      Wmap[(int64_t)py * Wd + px] = Wt;
    }
  int64_t cnt = 0;
  const float du = mm[1] - mm[0], dvv = mm[3] - mm[2];
  for (int py = 0; py < Hd; py += stride)
    for (int px = 0; px < Wd; px += stride) {
      const float Wt = Wmap[(int64_t)py * Wd + px];
      if (!(Wt >= eps_w)) continue;
      const float D = Dmap[(int64_t)py * Wd + px];
      const float u = (float)px + 0.5f, v = (float)py + 0.5f;
      const float xn = (u - cx) / fx, yn = (v - cy) / fy;
      const float q0 = xn * D - k.t[0], q1 = yn * D - k.t[1], q2 = D - k.t[2];
      const float wx = std::fmaf(R[0], q0, std::fmaf(R[3], q1, R[6] * q2));
      const float wy = std::fmaf(R[1], q0, std::fmaf(R[4], q1, R[7] * q2));
      const float wz = std::fmaf(R[2], q0, std::fmaf(R[5], q1, R[8] * q2));
      float ru, rv;
      ground_uv(wx, wy, wz, c0, rho, au, av, &ru, &rv);
      float gu = (ru - mm[0]) / du, gv = (rv - mm[2]) / dvv;
      pu[cnt] = std::fmin(1.0f, std::fmax(0.0f, gu));
      pv[cnt] = std::fmin(1.0f, std::fmax(0.0f, gv));
      ++cnt;
    }
  *K = cnt;
  return O_OK;
}

// O8 over explicit point clouds (CSR off[0..ns]): n over the enlarged regions,
// n0 over the delta = 0 cells, member iff K > 0 and (double)n >= tau (double)K,
// home = lowest argmax n0 (K = 0: the camera centre's cell).
int oracle_assign_points(int64_t ns, const int64_t* off, const float* pu, const float* pv, const float* cam_gu,
                         const float* cam_gv, int m, int n, const float* vcuts, const float* hcuts, float dv, float dh,
                         double tau, uint32_t* ncb, uint32_t* n0cb, uint64_t* member, int32_t* home) {
  int st = check_grid(m, n, vcuts, hcuts, dv, dh, tau);
  if (st) return st;
  const int B = m * n;
  Axis U = make_axis(m, vcuts, dv), V = make_axis(n, hcuts, dh);
  for (int64_t j = 0; j < ns; ++j) {
    uint32_t* nj = ncb + j * B;
    uint32_t* n0j = n0cb + j * B;
    for (int b = 0; b < B; ++b) nj[b] = n0j[b] = 0;
    const int64_t K = off[j + 1] - off[j];
    for (int64_t e = off[j]; e < off[j + 1]; ++e)
      for (int p = 0; p < m; ++p)
        for (int q = 0; q < n; ++q) {
          if (in_interval(pu[e], U.elo[p], U.ehi[p]) && in_interval(pv[e], V.elo[q], V.ehi[q])) nj[p * n + q] += 1;
          if (in_interval(pu[e], U.lo[p], U.hi[p]) && in_interval(pv[e], V.lo[q], V.hi[q])) n0j[p * n + q] += 1;
        }
    uint64_t mem = 0;
    if (K > 0)
      for (int b = 0; b < B; ++b)
        if ((double)nj[b] >= tau * (double)K) mem |= (uint64_t)1 << b;
    member[j] = mem;
    int hb;
    if (K > 0) {
      hb = 0;
      for (int b = 1; b < B; ++b)
        if (n0j[b] > n0j[hb]) hb = b;
    } else {
      hb = cell_of(U, cam_gu[j]) * n + cell_of(V, cam_gv[j]);
    }
    home[j] = hb;
  }
  return O_OK;
}

}  // extern "C"
