// Microbenchmark: dispatch floor of the visibility instruction mix (no memory,
// no branches): per (Gaussian pair, camera) 11 FFMA2 + compares + 2 ballots,
// 4 independent pair groups per lane, 16 warps per SM. Variants strip parts of
// the mix to locate the bottleneck. Not product code.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

struct __align__(16) Cam { float Au[4], Av[4], Aw[4], Wf, Hf, zn, zf; };
__device__ long long g_cyc[4096];
__device__ unsigned g_sink[1 << 20];
constexpr int NW = 16, PG = 4, NCAM = 32;

__device__ __forceinline__ float2 bc2(float a) { return make_float2(a, a); }
__device__ __forceinline__ float max3f(float a, float b, float c) {
  float d; asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c)); return d; }

template <int V>
__global__ void __launch_bounds__(NW * 32, 1) kern(const Cam* __restrict__ cams, int reps) {
  __shared__ Cam sc[NCAM];
  if (threadIdx.x < NCAM) sc[threadIdx.x] = cams[threadIdx.x];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  float4 P0[PG], P1[PG];
  for (int k = 0; k < PG; ++k) {
    float x = -1.f + 0.1f * k + 0.003f * lane;
    P0[k] = make_float4(x, x + 0.01f, 0.2f * k, 0.2f * k + 0.01f);
    P1[k] = make_float4(5.f, 5.1f, 0.01f, 0.011f);
  }
  uint32_t acc = 0;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll 1
    for (int j = 0; j < NCAM; ++j) {
      const Cam c = sc[j];
      uint32_t b[2 * PG];
#pragma unroll
      for (int k = 0; k < PG; ++k) {
        const float2 x2 = make_float2(P0[k].x, P0[k].y), y2 = make_float2(P0[k].z, P0[k].w);
        const float2 z2 = make_float2(P1[k].x, P1[k].y);
        const float2 w = __ffma2_rn(x2, bc2(c.Aw[0]), __ffma2_rn(y2, bc2(c.Aw[1]), __ffma2_rn(z2, bc2(c.Aw[2]), bc2(c.Aw[3]))));
        const float2 u = __ffma2_rn(x2, bc2(c.Au[0]), __ffma2_rn(y2, bc2(c.Au[1]), __ffma2_rn(z2, bc2(c.Au[2]), bc2(c.Au[3]))));
        const float2 v = __ffma2_rn(x2, bc2(c.Av[0]), __ffma2_rn(y2, bc2(c.Av[1]), __ffma2_rn(z2, bc2(c.Av[2]), bc2(c.Av[3]))));
        const float2 eu = __ffma2_rn(w, bc2(-c.Wf), u);
        const float2 ev = __ffma2_rn(w, bc2(-c.Hf), v);
        bool pa, pb;
        if (V == 0) {  // full mix
          pa = (w.x > c.zn) & (w.x < c.zf) & (max3f(-u.x, eu.x, -v.x) <= P1[k].w) & (ev.x <= P1[k].w);
          pb = (w.y > c.zn) & (w.y < c.zf) & (max3f(-u.y, eu.y, -v.y) <= P1[k].z) & (ev.y <= P1[k].z);
        } else if (V == 1) {  // FFMA2 floor: one compare per Gaussian consuming all results
          pa = (w.x + u.x + v.x + eu.x + ev.x) > 0.f;
          pb = (w.y + u.y + v.y + eu.y + ev.y) > 0.f;
        } else if (V == 2) {  // compares only on a cheap value (no FFMA2 chain except one)
          pa = (w.x > c.zn) & (w.x < c.zf) & (max3f(-w.x, w.x, -w.x) <= P1[k].w) & (w.x <= P1[k].w);
          pb = (w.y > c.zn) & (w.y < c.zf) & (max3f(-w.y, w.y, -w.y) <= P1[k].z) & (w.y <= P1[k].z);
        } else {  // V == 3: full mix, ballots replaced by predicate accumulation
          pa = (w.x > c.zn) & (w.x < c.zf) & (max3f(-u.x, eu.x, -v.x) <= P1[k].w) & (ev.x <= P1[k].w);
          pb = (w.y > c.zn) & (w.y < c.zf) & (max3f(-u.y, eu.y, -v.y) <= P1[k].z) & (ev.y <= P1[k].z);
        }
        if (V == 3) {
          b[2 * k] = pa; b[2 * k + 1] = pb;
        } else {
          b[2 * k] = __ballot_sync(0xffffffffu, pa);
          b[2 * k + 1] = __ballot_sync(0xffffffffu, pb);
        }
      }
#pragma unroll
      for (int k = 0; k < 2 * PG; ++k) acc ^= b[k] + k;
    }
  }
  long long t1 = clock64();
  g_sink[(blockIdx.x * blockDim.x + threadIdx.x) & ((1 << 20) - 1)] = acc;
  if (threadIdx.x == 0) g_cyc[blockIdx.x] = t1 - t0;
}

template <int V>
void run(const char* name, const Cam* d, int reps) {
  kern<V><<<148, NW * 32>>>(d, 2);
  kern<V><<<148, NW * 32>>>(d, reps);
  cudaDeviceSynchronize();
  long long cyc[148];
  cudaMemcpyFromSymbol(cyc, g_cyc, sizeof(cyc));
  double m = 0; for (int i = 0; i < 148; ++i) m += cyc[i]; m /= 148;
  // cam-steps per SMSP: reps * NCAM * PG pair groups * NW warps / 4 SMSPs  (1 cam-step = 64 tests = 1 pair group x 1 camera)
  double cs = (double)reps * NCAM * PG * NW / 4.0;
  printf("%-52s %.1f cycles per 64-test camera step per SMSP  (FP32 frac %.1f%%)  err=%s\n", name, m / cs,
         100.0 * 22.0 / (m / cs), cudaGetErrorString(cudaGetLastError()));
}

int main() {
  Cam h[NCAM];
  for (int c = 0; c < NCAM; ++c) h[c] = Cam{{1, 0, 0.5f, 0.01f * c}, {0, 1, 0.5f, 0}, {0, 0, 1, 0}, 1.f, 1.f, 0.01f, 100.f};
  Cam* d; cudaMalloc(&d, sizeof(h)); cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  for (int it = 0; it < 2; ++it) {
    run<0>("V0 full mix (11 FFMA2 + 4 FSETP + FMNMX3 + 2 VOTE)", d, 400);
    run<1>("V1 FFMA2 floor (11 FFMA2 + adds + 1 FSETP + VOTE)", d, 400);
    run<2>("V2 compares on 3 FFMA2", d, 400);
    run<3>("V3 full mix without VOTE", d, 400);
  }
}
