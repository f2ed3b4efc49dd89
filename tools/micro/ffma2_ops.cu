// Microbenchmark: FFMA2 throughput vs. number of distinct register operands, and
// overlap of FFMA2 with ALU-pipe FSETP/FMNMX3. Evidence for DESIGN.md §4.
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 1024
__device__ float g_sink[1 << 20];
__device__ long long g_cyc[1024];
__device__ __forceinline__ unsigned long long pk(float a, float b) {
  unsigned long long r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r; }

template <int OP>
__global__ void __launch_bounds__(512) kern(float s0, int iters) {
  const int t = threadIdx.x;
  unsigned long long x[4], acc[4], cp[4];
  float sc[8];
  for (int i = 0; i < 4; ++i) { x[i] = pk(1.0f + t * 1e-7f + i, 2.0f + i); acc[i] = pk(0.5f + i, 0.25f * i); cp[i] = pk(0.1f * i, 0.2f); }
  for (int i = 0; i < 8; ++i) sc[i] = s0 + i * 1e-3f + t * 1e-9f;
  float f[8]; for (int i = 0; i < 8; ++i) f[i] = sc[i] * 0.5f;
  unsigned pred = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (OP == 0) {  // FFMA2 d = a_pair * s + c_pair (5 distinct regs: x, s, acc -> new acc)
        asm volatile("{.reg .b64 s; mov.b64 s, {%2,%2}; fma.rn.f32x2 %0, %1, s, %0;}" : "+l"(acc[i]) : "l"(x[i]), "f"(sc[i]));
      } else if (OP == 1) {  // FFMA2 d = a_pair * s1 + s2 (4 regs)
        asm volatile("{.reg .b64 s, u; mov.b64 s, {%2,%2}; mov.b64 u, {%3,%3}; fma.rn.f32x2 %0, %1, s, u;}" : "=l"(acc[i]) : "l"(x[i] ^ acc[i]), "f"(sc[i]), "f"(sc[i + 4]));
      } else if (OP == 2) {  // scalar FFMA, 3 distinct sources
        asm volatile("fma.rn.f32 %0, %1, %2, %0;" : "+f"(f[i]) : "f"(sc[i]), "f"(sc[i + 4]));
        asm volatile("fma.rn.f32 %0, %1, %2, %0;" : "+f"(f[i + 4]) : "f"(sc[i + 4]), "f"(sc[i]));
      } else if (OP == 3) {  // FFMA2 (5 regs) + 2 independent FSETP-like ALU ops
        asm volatile("{.reg .b64 s; mov.b64 s, {%2,%2}; fma.rn.f32x2 %0, %1, s, %0;}" : "+l"(acc[i]) : "l"(x[i]), "f"(sc[i]));
        unsigned q;
        asm volatile("{.reg .pred p, r; setp.le.f32 p, %1, %2; setp.gt.and.f32 r, %3, %2, p; selp.u32 %0, 1, 0, r;}" : "=r"(q) : "f"(f[i]), "f"(sc[i]), "f"(f[i+4]));
        pred += q;
      } else if (OP == 4) {  // FMNMX3 x2 (ALU only)
        asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(f[i]) : "f"(sc[i]), "f"(sc[i + 4]));
        asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(f[i + 4]) : "f"(sc[i + 4]), "f"(sc[i]));
      } else if (OP == 6) {  // FFMA2 a_pair * s(UR, kernel param) + c_pair (4 vector regs)
        asm volatile("{.reg .b64 s; mov.b64 s, {%2,%2}; fma.rn.f32x2 %0, %1, s, %0;}" : "+l"(acc[i]) : "l"(x[i]), "f"(s0));
      } else if (OP == 7) {  // FMNMX3 with all-even sources vs mixed: a.x, b.x, c.x of pairs
        float a0 = __uint_as_float((unsigned)x[i]), a1 = __uint_as_float((unsigned)acc[i]), a2 = __uint_as_float((unsigned)cp[i]);
        float r; asm volatile("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a0), "f"(a1), "f"(a2));
        f[i] += r;
      } else if (OP == 5) {  // FFMA2 (5 regs) + FMNMX3
        asm volatile("{.reg .b64 s; mov.b64 s, {%2,%2}; fma.rn.f32x2 %0, %1, s, %0;}" : "+l"(acc[i]) : "l"(x[i]), "f"(sc[i]));
        asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(f[i]) : "f"(sc[i]), "f"(sc[i + 4]));
      }
    }
  }
  long long t1 = clock64();
  float s = pred;
  for (int i = 0; i < 4; ++i) s += __uint_as_float((unsigned)acc[i]) + __uint_as_float((unsigned)(acc[i] >> 32));
  for (int i = 0; i < 8; ++i) s += f[i];
  g_sink[(blockIdx.x * blockDim.x + t) & ((1 << 20) - 1)] = s;
  if (t == 0) g_cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int threads, double instr_per_inner) {
  kern<OP><<<148, threads>>>(1.0f, 8);
  kern<OP><<<148, threads>>>(1.0f, ITERS);
  cudaDeviceSynchronize();
  long long cyc[148];
  cudaMemcpyFromSymbol(cyc, g_cyc, sizeof(cyc));
  double m = 0; for (int i = 0; i < 148; ++i) m += cyc[i]; m /= 148;
  double warps = threads / 32.0;
  double instr = warps * ITERS * 4 * instr_per_inner;  // per SM
  printf("%-40s thr=%4d  %.3f warp-instr/clk/SMSP  (%.1f cyc per inner per warp-SMSP)  err=%s\n", name, threads,
         instr / m / 4, m / (ITERS * 4) / (warps / 4), cudaGetErrorString(cudaGetLastError()));
}
int main() {
  for (int t : {256, 512}) {
    run<0>("FFMA2 a_pair*s+c_pair (5 regs)", t, 1);
    run<1>("FFMA2 a_pair*s1+s2 (4 regs)", t, 1);
    run<2>("2x FFMA scalar 3 regs", t, 2);
    run<3>("FFMA2(5) + 2 FSETP (3 instr)", t, 3);
    run<4>("2x FMNMX3", t, 2);
    run<5>("FFMA2(5) + FMNMX3", t, 2);
    run<6>("FFMA2 a_pair*UR+c_pair (4 vector regs)", t, 1);
    run<7>("FMNMX3 3 even regs + FADD", t, 2);
  }
}
