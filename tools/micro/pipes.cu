// Microbenchmark: per-SM throughput (ops/clk/SM) of the instructions the
// visibility test is built from, measured with clock64.
// Evidence for DESIGN.md's issue/pipe model. Not part of the product.
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 2048
#define NC 8
__device__ float g_sink[1 << 20];
__device__ long long g_cyc[1024];

template <int OP>
__global__ void __launch_bounds__(1024) kern(float a0, float b0, float c0, int iters) {
  float acc[NC]; unsigned long long acc2[NC];
#pragma unroll
  for (int i = 0; i < NC; ++i) { acc[i] = a0 + i + threadIdx.x; acc2[i] = __double_as_longlong((double)(a0 + i)); }
  float b = b0 + threadIdx.x * 1e-9f, c = c0 + threadIdx.x * 1e-9f;
  unsigned p = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      if (OP == 0) {  // FFMA 3-reg
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(acc[i]) : "f"(b), "f"(c));
      } else if (OP == 1) {  // FFMA2 with scalar broadcast
        asm volatile("{.reg .b64 t; mov.b64 t, {%1,%1}; fma.rn.f32x2 %0, %0, t, %0;}" : "+l"(acc2[i]) : "f"(b));
      } else if (OP == 2) {  // FSETP chain-free
        unsigned q;
        asm volatile("{.reg .pred P; setp.le.f32 P, %1, %2; selp.u32 %0, 1, 0, P;}" : "=r"(q) : "f"(acc[i]), "f"(b));
        p += q;
      } else if (OP == 3) {  // FMNMX3
        asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(acc[i]) : "f"(b), "f"(c));
      } else if (OP == 4) {  // FFMA2 + FSETP interleaved 1:1
        asm volatile("{.reg .b64 t; mov.b64 t, {%1,%1}; fma.rn.f32x2 %0, %0, t, %0;}" : "+l"(acc2[i]) : "f"(b));
        asm volatile("{.reg .pred P; setp.le.and.f32 P, %1, %2, 1; @P add.u32 %0, %0, 1;}" : "+r"(p) : "f"(acc[i]), "f"(b));
      } else if (OP == 5) {  // FFMA 2-reg+const-ish (imm)
        asm volatile("fma.rn.f32 %0, %0, %1, 0f3F800001;" : "+f"(acc[i]) : "f"(b));
      } else if (OP == 6) {  // FFMA2 with two scalars (innermost form)
        asm volatile("{.reg .b64 t, s; mov.b64 t, {%1,%1}; mov.b64 s, {%2,%2}; fma.rn.f32x2 %0, %0, t, s;}" : "+l"(acc2[i]) : "f"(b), "f"(c));
      } else if (OP == 7) {  // VOTE
        unsigned v = __ballot_sync(~0u, acc[i] > b);
        p ^= v;
        acc[i] += 1.0f;
      }
    }
  }
  long long t1 = clock64();
  float s = p;
#pragma unroll
  for (int i = 0; i < NC; ++i) s += acc[i] + (float)__longlong_as_double(acc2[i]);
  g_sink[(blockIdx.x * blockDim.x + threadIdx.x) & ((1 << 20) - 1)] = s;
  if (threadIdx.x == 0) g_cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int threads, double ops_per_iter_per_thread) {
  kern<OP><<<148, threads>>>(1.0f, 0.999f, 0.5f, 16);
  kern<OP><<<148, threads>>>(1.0f, 0.999f, 0.5f, ITERS);
  cudaDeviceSynchronize();
  long long cyc[148];
  cudaMemcpyFromSymbol(cyc, g_cyc, sizeof(cyc));
  double m = 0; for (int i = 0; i < 148; ++i) m += cyc[i]; m /= 148;
  double ops = (double)threads * ITERS * NC * ops_per_iter_per_thread;
  printf("%-34s thr=%4d  %.1f lane-ops/clk/SM  (%.2f warp-instr/clk/SMSP)  err=%s\n", name, threads, ops / m,
         ops / m / 32 / 4, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  for (int t : {256, 512, 1024}) {
    run<0>("FFMA r,r,r,r", t, 1);
    run<5>("FFMA r,r,imm,r", t, 1);
    run<1>("FFMA2 pair,scalar,pair (fma count)", t, 2);
    run<6>("FFMA2 pair,scalar,scalar (fma count)", t, 2);
    run<2>("FSETP+SEL+IADD (3 instr)", t, 1);
    run<3>("FMNMX3", t, 1);
    run<4>("FFMA2 + FSETP.AND + @P IADD", t, 1);
    run<7>("VOTE + LOP + FADD", t, 1);
  }
}
