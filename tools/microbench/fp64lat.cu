// FP64 latency / ILP microbenchmark on B200: how many independent FP64
// instructions per SMSP keep the DADD pipe full, and what a mix of FP64 +
// ALU/FMA instructions (the crossing kernel's per-pair mix) sustains.
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 2048

template <int ILP>
__global__ void chain(double *out, double s, int iters) {
  double x[ILP];
#pragma unroll
  for (int k = 0; k < ILP; ++k) x[k] = threadIdx.x * 1e-3 + k;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < ILP; ++k) x[k] = __dadd_rn(x[k], s);
  }
  double a = 0;
#pragma unroll
  for (int k = 0; k < ILP; ++k) a += x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = a;
}

// per "pair": 11 FP64 (DADD/DMUL), 2 FMUL, 4 ISETP + 2 FSETP chained, 1 predicated add
template <int ILP>
__global__ void mix(double *out, double s, int iters, int r0, int r1) {
  double a[ILP], b[ILP];
  unsigned cnt = 0;
  int q0 = threadIdx.x, q1 = threadIdx.x * 3;
#pragma unroll
  for (int k = 0; k < ILP; ++k) { a[k] = threadIdx.x * 1e-3 + k; b[k] = 1.0 + k * 1e-3; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < ILP; ++k) {
      double d1 = __dsub_rn(s, a[k]);
      double d2 = __dsub_rn(s, b[k]);
      double c2 = __dsub_rn(__dmul_rn(a[k], d2), __dmul_rn(b[k], d1));
      double c3 = __dsub_rn(__dmul_rn(s, a[k]), __dmul_rn(s, b[k]));
      double c4 = __dsub_rn(__dmul_rn(d1, b[k]), __dmul_rn(d2, a[k]));
      float p = __fmul_rn(__int_as_float(__double2hiint(c2)), __int_as_float(__double2hiint(c3)));
      float p2 = __fmul_rn(__int_as_float(__double2hiint(c4)), 1.5f);
      asm("{\n\t.reg .pred p;\n\t"
          "setp.ge.s32 p, %1, %2;\n\t"
          "setp.ge.and.s32 p, %3, %2, p;\n\t"
          "setp.ge.and.s32 p, %1, %4, p;\n\t"
          "setp.ge.and.s32 p, %3, %4, p;\n\t"
          "setp.le.and.f32 p, %5, 0f00000000, p;\n\t"
          "setp.le.and.f32 p, %6, 0f00000000, p;\n\t"
          "@p add.u32 %0, %0, 1;\n\t}"
          : "+r"(cnt) : "r"(q0), "r"(r0), "r"(q1), "r"(r1), "f"(p), "f"(p2));
      a[k] = c2; b[k] = c4;   // carry a dependency into the next iteration
    }
  }
  double acc = cnt;
#pragma unroll
  for (int k = 0; k < ILP; ++k) acc += a[k] + b[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <class F>
float timeit(F f) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  f(); cudaDeviceSynchronize();
  cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); return ms;
}

int main() {
  double *out; cudaMalloc(&out, 1 << 26);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double f = clk * 1e3;  // Hz (max)
  printf("clock %.0f MHz\n", f / 1e6);
  // latency: 1 warp per SM, 1 chain
  float ms = timeit([&] { chain<1><<<148, 32>>>(out, 1.0000001, 1 << 16); });
  printf("DADD dependent latency ~ %.1f cycles\n", ms * 1e-3 * f / (1 << 16));
  for (int w : {1, 2, 3, 4, 6, 8, 16}) {
    for (int ilp : {1, 2, 4, 8}) {
      int iters = 4096;
      float t;
      if (ilp == 1) t = timeit([&] { chain<1><<<148, 32 * w>>>(out, 1.0000001, iters); });
      if (ilp == 2) t = timeit([&] { chain<2><<<148, 32 * w>>>(out, 1.0000001, iters); });
      if (ilp == 4) t = timeit([&] { chain<4><<<148, 32 * w>>>(out, 1.0000001, iters); });
      if (ilp == 8) t = timeit([&] { chain<8><<<148, 32 * w>>>(out, 1.0000001, iters); });
      double lanes = 148.0 * 32 * w * ilp * iters / (t * 1e-3) / (148 * f);
      printf("DADD warps/SM=%2d ilp=%d: %.1f lanes/clk/SM\n", w, ilp, lanes);
    }
  }
  for (int w : {4, 8, 12, 16, 24, 32}) {
    for (int ilp : {1, 2, 4}) {
      int iters = 1024;
      float t;
      if (ilp == 1) t = timeit([&] { mix<1><<<148, 32 * w>>>(out, 1.0000001, iters, 5, 7); });
      if (ilp == 2) t = timeit([&] { mix<2><<<148, 32 * w>>>(out, 1.0000001, iters, 5, 7); });
      if (ilp == 4) t = timeit([&] { mix<4><<<148, 32 * w>>>(out, 1.0000001, iters, 5, 7); });
      double pairs = 148.0 * 32 * w * ilp * iters / (t * 1e-3);
      printf("MIX warps/SM=%2d ilp=%d: %.3e pairs/s  fp64 lanes/clk/SM %.1f\n", w, ilp, pairs,
             pairs * 11 / (148 * f));
    }
  }
  return 0;
}
