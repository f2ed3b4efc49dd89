// Microbenchmark: cycles per (64-test, camera) step of candidate formulations
// of the visibility inner loop, data resident in shared
// memory, 16 warps x 2 cameras per CTA as in k_visibility. Not product code.
//   F0: camera coefficients in vector registers (current kernel)
//   F1: coefficients read from __constant__ with uniform addresses (per-warp
//       template specialisation), re-read once per tile
//   F2: scalar FFMA instead of FFMA2
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

struct __align__(16) Cam { float Au[4], Av[4], Aw[4], Wf, Hf, zn, zf; };
__constant__ Cam c_cams[1024];
__device__ Cam g_cams[1024];
__device__ long long g_cyc[4096];
__device__ unsigned g_sink[1 << 20];
constexpr int TILE = 1024, NW = 16, CW = 2;

__device__ __forceinline__ float2 bc2(float a) { return make_float2(a, a); }
__device__ __forceinline__ float max3f(float a, float b, float c) {
  float d; asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c)); return d; }

template <int F>
__device__ __forceinline__ void test_pair(const Cam& c, float4 P0, float4 P1, uint32_t& b0, uint32_t& b1) {
  bool pa, pb;
  if (F != 2) {
    const float2 x2 = make_float2(P0.x, P0.y), y2 = make_float2(P0.z, P0.w), z2 = make_float2(P1.x, P1.y);
    const float2 w = __ffma2_rn(x2, bc2(c.Aw[0]), __ffma2_rn(y2, bc2(c.Aw[1]), __ffma2_rn(z2, bc2(c.Aw[2]), bc2(c.Aw[3]))));
    const float2 u = __ffma2_rn(x2, bc2(c.Au[0]), __ffma2_rn(y2, bc2(c.Au[1]), __ffma2_rn(z2, bc2(c.Au[2]), bc2(c.Au[3]))));
    const float2 v = __ffma2_rn(x2, bc2(c.Av[0]), __ffma2_rn(y2, bc2(c.Av[1]), __ffma2_rn(z2, bc2(c.Av[2]), bc2(c.Av[3]))));
    const float2 eu = __ffma2_rn(w, bc2(-c.Wf), u);
    const float2 ev = __ffma2_rn(w, bc2(-c.Hf), v);
    pa = (w.x > c.zn) & (w.x < c.zf) & (max3f(-u.x, eu.x, -v.x) <= P1.z) & (ev.x <= P1.z);
    pb = (w.y > c.zn) & (w.y < c.zf) & (max3f(-u.y, eu.y, -v.y) <= P1.w) & (ev.y <= P1.w);
  } else {
    const float wa = __fmaf_rn(c.Aw[0], P0.x, __fmaf_rn(c.Aw[1], P0.z, __fmaf_rn(c.Aw[2], P1.x, c.Aw[3])));
    const float wb = __fmaf_rn(c.Aw[0], P0.y, __fmaf_rn(c.Aw[1], P0.w, __fmaf_rn(c.Aw[2], P1.y, c.Aw[3])));
    const float ua = __fmaf_rn(c.Au[0], P0.x, __fmaf_rn(c.Au[1], P0.z, __fmaf_rn(c.Au[2], P1.x, c.Au[3])));
    const float ub = __fmaf_rn(c.Au[0], P0.y, __fmaf_rn(c.Au[1], P0.w, __fmaf_rn(c.Au[2], P1.y, c.Au[3])));
    const float va = __fmaf_rn(c.Av[0], P0.x, __fmaf_rn(c.Av[1], P0.z, __fmaf_rn(c.Av[2], P1.x, c.Av[3])));
    const float vb = __fmaf_rn(c.Av[0], P0.y, __fmaf_rn(c.Av[1], P0.w, __fmaf_rn(c.Av[2], P1.y, c.Av[3])));
    const float eua = __fmaf_rn(-c.Wf, wa, ua), eub = __fmaf_rn(-c.Wf, wb, ub);
    const float eva = __fmaf_rn(-c.Hf, wa, va), evb = __fmaf_rn(-c.Hf, wb, vb);
    pa = (wa > c.zn) & (wa < c.zf) & (max3f(-ua, eua, -va) <= P1.z) & (eva <= P1.z);
    pb = (wb > c.zn) & (wb < c.zf) & (max3f(-ub, eub, -vb) <= P1.w) & (evb <= P1.w);
  }
  b0 = __ballot_sync(0xffffffffu, pa);
  b1 = __ballot_sync(0xffffffffu, pb);
}

template <int F, int W>
__device__ void consumer(const float4* tile, uint32_t* words, int reps, int cam0) {
  const int lane = threadIdx.x & 31;
  uint32_t* mw = words + W * CW * 32;
  uint32_t acc = 0;
  Cam cr[CW];
  if (F != 1) {
#pragma unroll
    for (int j = 0; j < CW; ++j) cr[j] = g_cams[cam0 + W * CW + j];
  }
  for (int r = 0; r < reps; ++r) {
    Cam cc[CW];
#pragma unroll
    for (int j = 0; j < CW; ++j) cc[j] = (F == 1) ? c_cams[(cam0 + W * CW + j) & 1023] : cr[j];
#pragma unroll 4
    for (int step = 0; step < TILE / 64; step += 2) {
      uint32_t bal[CW][4];
      float4 P0[2], P1[2];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        P0[q] = tile[(step + q) * 64 + lane];
        P1[q] = tile[(step + q) * 64 + 32 + lane];
      }
#pragma unroll
      for (int j = 0; j < CW; ++j)
#pragma unroll
        for (int q = 0; q < 2; ++q) test_pair<F>(cc[j], P0[q], P1[q], bal[j][2 * q], bal[j][2 * q + 1]);
      uint32_t anyb = 0;
#pragma unroll
      for (int j = 0; j < CW; ++j) {
        *reinterpret_cast<uint4*>(&mw[j * 32 + 2 * step]) = make_uint4(bal[j][0], bal[j][1], bal[j][2], bal[j][3]);
        anyb |= bal[j][0] | bal[j][1] | bal[j][2] | bal[j][3];
      }
      if (anyb) acc += __popc(anyb) + lane;
    }
    __syncwarp();
    acc += mw[lane];
    __syncwarp();
  }
  g_sink[(blockIdx.x * blockDim.x + threadIdx.x) & ((1 << 20) - 1)] = acc;
}

template <int F>
__global__ void __launch_bounds__(NW * 32, 1) kern(int reps) {
  __shared__ __align__(16) float4 tile[TILE / 2 * 2];
  __shared__ __align__(16) uint32_t words[NW * CW * 32];
  for (int i = threadIdx.x; i < TILE; i += blockDim.x) {
    int grp = i / 64, l = i % 32, h = (i % 64) / 32;
    float xi = -10.f + 20.f * (float)i / TILE, yi = 0.1f * ((i * 37) % 17 - 8) / 8.f, zi = 5.0f + 0.01f * (i % 13);
    float* t = reinterpret_cast<float*>(&tile[grp * 64 + l]);
    float* t2 = reinterpret_cast<float*>(&tile[grp * 64 + 32 + l]);
    t[h] = xi; t[2 + h] = yi; t2[h] = zi; t2[2 + h] = 0.01f;
  }
  __syncthreads();
  const int cam0 = (blockIdx.x * NW * CW) & 1023;
  long long t0 = clock64();
  switch (threadIdx.x >> 5) {
#define C(W) case W: consumer<F, W>(tile, words, reps, cam0); break;
    C(0) C(1) C(2) C(3) C(4) C(5) C(6) C(7) C(8) C(9) C(10) C(11) C(12) C(13) C(14) C(15)
#undef C
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) g_cyc[blockIdx.x] = t1 - t0;
}

template <int F>
void run(const char* name, int reps) {
  kern<F><<<148, NW * 32>>>(2);
  kern<F><<<148, NW * 32>>>(reps);
  cudaDeviceSynchronize();
  long long cyc[148];
  cudaMemcpyFromSymbol(cyc, g_cyc, sizeof(cyc));
  double m = 0; for (int i = 0; i < 148; ++i) m += cyc[i]; m /= 148;
  double camsteps_per_smsp = (double)reps * (TILE / 64) * NW * CW / 4.0;
  printf("%-44s %.1f cycles per 64-test camera step per SMSP  -> %.1f%% of FP32 peak  err=%s\n", name,
         m / camsteps_per_smsp, 100.0 * (64.0 * 22 / 2 / 32) / (m / camsteps_per_smsp) * 1.0,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  Cam h[1024];
  for (int c = 0; c < 1024; ++c) {
    float tx = -10.f + 20.f * c / 1024.f;
    h[c] = Cam{{1, 0, 0.5f, -tx}, {0, 1, 0.5f, 0}, {0, 0, 1, 0}, 1.f, 1.f, 0.01f, 100.f};
  }
  cudaMemcpyToSymbol(c_cams, h, sizeof(h));
  cudaMemcpyToSymbol(g_cams, h, sizeof(h));
  for (int it = 0; it < 2; ++it) {
    run<0>("F0 FFMA2, coefficients in vector regs", 200);
    run<1>("F1 FFMA2, coefficients from __constant__", 200);
    run<2>("F2 scalar FFMA, coefficients in regs", 200);
  }
}
