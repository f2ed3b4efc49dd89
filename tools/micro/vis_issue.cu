// Microbenchmark: issue/pipe throughput of candidate inner loops for the
// visibility test. Not part of the product; evidence for
// the kernel design choices in DESIGN.md (packed FFMA2 vs scalar FFMA, camera
// coefficients in uniform registers, FMNMX3 compare folding).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

struct Cam { float Aw[4], Au[4], Av[4], lim[4]; };  // lim = {Wf, Hf, zn, zf}
__constant__ Cam c_cams[1024];

#define T_TILE 4096
#define NWARP 16

__device__ __forceinline__ float2 bc(float a) { return make_float2(a, a); }

template <int PACK, int CW, int CMP, int UR>
__global__ void __launch_bounds__(NWARP * 32, 1)
mb(int reps, unsigned long long* sink, double* dsink) {
  extern __shared__ float4 tile[];
  __shared__ unsigned words[NWARP][CW][32];
  for (int i = threadIdx.x; i < T_TILE; i += blockDim.x) {
    float xi = -10.f + 20.f * (float)i / T_TILE;
    float k = (i % 1000 == 7) ? -__int_as_float(0x7f800000) : 0.01f;
    float yi = 0.1f * ((i * 37) % 17 - 8) / 8.f, zi = 5.0f + 0.01f * (i % 13);
    int grp = i / 64, l = i % 32, h = (i % 64) / 32;
    float* t = reinterpret_cast<float*>(&tile[grp * 64 + 2 * l]);
    t[0 + h] = xi; t[2 + h] = yi; t[4 + h] = zi; t[6 + h] = k;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cam0 = UR ? (blockIdx.x * CW) & 1023 : ((blockIdx.x * NWARP + warp) * CW) & 1023;
  unsigned long long acc = 0;
  double S[CW], O[CW];
  float zmn[CW], zmx[CW];
#pragma unroll
  for (int j = 0; j < CW; ++j) { S[j] = 0; O[j] = 0; zmn[j] = 1e30f; zmx[j] = -1e30f; }
  Cam C[CW];
#pragma unroll
  for (int j = 0; j < CW; ++j) C[j] = c_cams[cam0 + j];
  for (int r = 0; r < reps; ++r) {
    for (int s = 0; s < T_TILE / 64; ++s) {
      float4 P0 = tile[s * 64 + 2 * lane], P1 = tile[s * 64 + 2 * lane + 1];
      float4 A = make_float4(P0.x, P0.z, P1.x, P1.z), B = make_float4(P0.y, P0.w, P1.y, P1.w);
#pragma unroll
      for (int j = 0; j < CW; ++j) {
        bool pa, pb;
        float wa, wb;
        if (PACK) {
          float2 x = make_float2(P0.x, P0.y), y = make_float2(P0.z, P0.w), z = make_float2(P1.x, P1.y);
          float2 w = __ffma2_rn(x, bc(C[j].Aw[0]), __ffma2_rn(y, bc(C[j].Aw[1]), __ffma2_rn(z, bc(C[j].Aw[2]), bc(C[j].Aw[3]))));
          float2 u = __ffma2_rn(x, bc(C[j].Au[0]), __ffma2_rn(y, bc(C[j].Au[1]), __ffma2_rn(z, bc(C[j].Au[2]), bc(C[j].Au[3]))));
          float2 v = __ffma2_rn(x, bc(C[j].Av[0]), __ffma2_rn(y, bc(C[j].Av[1]), __ffma2_rn(z, bc(C[j].Av[2]), bc(C[j].Av[3]))));
          float2 eu = __ffma2_rn(w, bc(-C[j].lim[0]), u);
          float2 ev = __ffma2_rn(w, bc(-C[j].lim[1]), v);
          if (CMP) {
            float ma, mb_;
            asm("max.f32 %0, %1, %2, %3;" : "=f"(ma) : "f"(-u.x), "f"(eu.x), "f"(-v.x));
            asm("max.f32 %0, %1, %2, %3;" : "=f"(mb_) : "f"(-u.y), "f"(eu.y), "f"(-v.y));
            pa = (w.x > C[j].lim[2]) & (w.x < C[j].lim[3]) & (ma <= A.w) & (ev.x <= A.w);
            pb = (w.y > C[j].lim[2]) & (w.y < C[j].lim[3]) & (mb_ <= B.w) & (ev.y <= B.w);
          } else {
            pa = (w.x > C[j].lim[2]) & (w.x < C[j].lim[3]) & (u.x >= -A.w) & (eu.x <= A.w) & (v.x >= -A.w) & (ev.x <= A.w);
            pb = (w.y > C[j].lim[2]) & (w.y < C[j].lim[3]) & (u.y >= -B.w) & (eu.y <= B.w) & (v.y >= -B.w) & (ev.y <= B.w);
          }
          wa = w.x; wb = w.y;
        } else {
          float w0 = __fmaf_rn(C[j].Aw[0], A.x, __fmaf_rn(C[j].Aw[1], A.y, __fmaf_rn(C[j].Aw[2], A.z, C[j].Aw[3])));
          float u0 = __fmaf_rn(C[j].Au[0], A.x, __fmaf_rn(C[j].Au[1], A.y, __fmaf_rn(C[j].Au[2], A.z, C[j].Au[3])));
          float v0 = __fmaf_rn(C[j].Av[0], A.x, __fmaf_rn(C[j].Av[1], A.y, __fmaf_rn(C[j].Av[2], A.z, C[j].Av[3])));
          float w1 = __fmaf_rn(C[j].Aw[0], B.x, __fmaf_rn(C[j].Aw[1], B.y, __fmaf_rn(C[j].Aw[2], B.z, C[j].Aw[3])));
          float u1 = __fmaf_rn(C[j].Au[0], B.x, __fmaf_rn(C[j].Au[1], B.y, __fmaf_rn(C[j].Au[2], B.z, C[j].Au[3])));
          float v1 = __fmaf_rn(C[j].Av[0], B.x, __fmaf_rn(C[j].Av[1], B.y, __fmaf_rn(C[j].Av[2], B.z, C[j].Av[3])));
          float eu0 = __fmaf_rn(-C[j].lim[0], w0, u0), ev0 = __fmaf_rn(-C[j].lim[1], w0, v0);
          float eu1 = __fmaf_rn(-C[j].lim[0], w1, u1), ev1 = __fmaf_rn(-C[j].lim[1], w1, v1);
          pa = (w0 > C[j].lim[2]) & (w0 < C[j].lim[3]) & (u0 >= -A.w) & (eu0 <= A.w) & (v0 >= -A.w) & (ev0 <= A.w);
          pb = (w1 > C[j].lim[2]) & (w1 < C[j].lim[3]) & (u1 >= -B.w) & (eu1 <= B.w) & (v1 >= -B.w) & (ev1 <= B.w);
          wa = w0; wb = w1;
        }
        unsigned b0 = __ballot_sync(~0u, pa), b1 = __ballot_sync(~0u, pb);
        *reinterpret_cast<uint2*>(&words[warp][j][(2 * s) & 31]) = make_uint2(b0, b1);
        if (b0 | b1) {
          if (pa) { S[j] += (double)0.5f * (double)wa; O[j] += 0.5; zmn[j] = fminf(zmn[j], wa); zmx[j] = fmaxf(zmx[j], wa); }
          if (pb) { S[j] += (double)0.5f * (double)wb; O[j] += 0.5; zmn[j] = fminf(zmn[j], wb); zmx[j] = fmaxf(zmx[j], wb); }
        }
      }
      if ((s & 15) == 15) {
        __syncwarp();
#pragma unroll
        for (int j = 0; j < CW; ++j) acc += words[warp][j][lane];
        __syncwarp();
      }
    }
  }
  double d = 0;
#pragma unroll
  for (int j = 0; j < CW; ++j) d += S[j] + O[j] + zmn[j] + zmx[j];
  dsink[blockIdx.x * blockDim.x + threadIdx.x] = d;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int PACK, int CW, int CMP, int UR>
void run(const char* name, int grid, int reps, unsigned long long* sink, double* dsink) {
  auto k = mb<PACK, CW, CMP, UR>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, T_TILE * 16);
  k<<<grid, NWARP * 32, T_TILE * 16>>>(1, sink, dsink);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k<<<grid, NWARP * 32, T_TILE * 16>>>(reps, sink, dsink);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double tests = (double)grid * NWARP * CW * (double)reps * T_TILE;
  printf("%-28s grid=%d  %.3f ms  %.3e tests/s  %.1f%% of 74.45TF@22flop  err=%s\n", name, grid, ms,
         tests / (ms * 1e-3), 100.0 * tests * 22 / (ms * 1e-3) / 74.45e12, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  Cam h[1024];
  for (int c = 0; c < 1024; ++c) {
    float tx = -10.f + 20.f * c / 1024.f;
    // identity rotation, f=100, cx=50: u = x' + 0.5 z', with x' = x - tx
    h[c] = Cam{{0, 0, 1, 0}, {1, 0, 0.5f, -tx}, {0, 1, 0.5f, 0}, {1.f, 1.f, 0.01f, 100.f}};
  }
  cudaMemcpyToSymbol(c_cams, h, sizeof(h));
  unsigned long long* sink; double* dsink;
  int grid = 148 * 2;
  cudaMalloc(&sink, grid * 512 * 8); cudaMalloc(&dsink, grid * 512 * 8);
  int reps = 40;
  for (int it = 0; it < 2; ++it) {
    run<0, 1, 0, 0>("scalar CW1 fsetp reg", grid, reps, sink, dsink);
    run<0, 2, 0, 0>("scalar CW2 fsetp reg", grid, reps, sink, dsink);
    run<0, 2, 0, 1>("scalar CW2 fsetp UR", grid, reps, sink, dsink);
    run<1, 1, 0, 0>("ffma2 CW1 fsetp reg", grid, reps, sink, dsink);
    run<1, 2, 0, 0>("ffma2 CW2 fsetp reg", grid, reps, sink, dsink);
    run<1, 2, 0, 1>("ffma2 CW2 fsetp UR", grid, reps, sink, dsink);
    run<1, 1, 1, 0>("ffma2 CW1 fmnmx3 reg", grid, reps, sink, dsink);
    run<1, 2, 1, 0>("ffma2 CW2 fmnmx3 reg", grid, reps, sink, dsink);
    run<1, 2, 1, 1>("ffma2 CW2 fmnmx3 UR", grid, reps, sink, dsink);
    run<1, 3, 1, 0>("ffma2 CW3 fmnmx3 reg", grid, reps, sink, dsink);
    run<1, 3, 1, 1>("ffma2 CW3 fmnmx3 UR", grid, reps, sink, dsink);
    run<1, 4, 1, 0>("ffma2 CW4 fmnmx3 reg", grid, reps, sink, dsink);
  }
  return 0;
}
