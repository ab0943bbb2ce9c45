// Register-file operand bandwidth of packed FP32 (FFMA2) on B200: throughput
// of FFMA2 by operand form (P = 64-bit register pair, S = 32-bit scalar used
// as a broadcast pair) with distinct registers in consecutive instructions
// (no operand-reuse-cache hits) and 8 independent accumulator chains, at
// 1/2/4 warps per scheduler.  Also the filter's ALU companions.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o rfbench rfbench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define ILP 8
#define ITERS 2048

__device__ __forceinline__ uint64_t pk(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ uint64_t mul2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

template <int OP>
__global__ void kern(float *out, const float *in) {
  const int t = threadIdx.x;
  uint64_t acc[ILP], P[ILP], Q[ILP], S[ILP];
  unsigned cnt = 0, mn = 0xffffffffu;
#pragma unroll
  for (int k = 0; k < ILP; ++k) {
    float a = in[(t + k) & 63], b = in[(t + 3 * k + 1) & 63], c = in[(t + 5 * k + 2) & 63];
    P[k] = pk(a, b);
    Q[k] = pk(b, c);
    S[k] = pk(c, c);  // broadcast scalar
    acc[k] = pk(a * 0.5f, c * 0.25f);
  }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int k = 0; k < ILP; ++k) {
      if (OP == 0) acc[k] = fma2(P[k], S[k], acc[k]);                  // P-S-P (c1 outer)
      if (OP == 1) acc[k] = fma2(S[k], P[k], S[(k + 1) % ILP]);        // S-P-S (c3 inner)
      if (OP == 2) acc[k] = fma2(P[k], Q[k], acc[k]);                  // P-P-P
      if (OP == 3) acc[k] = fma2(P[k], acc[k], S[k]);                  // P-P-S (product)
      if (OP == 4) acc[k] = fma2(P[0], S[k], acc[k]);                  // P common, S-P distinct
      if (OP == 5) acc[k] = mul2(P[k], acc[k]);                        // P-P mul
      if (OP == 6) {                                                   // P-S-P + 1 ALU per FFMA2
        acc[k] = fma2(P[k], S[k], acc[k]);
        cnt += (unsigned)acc[k] >> 31;
      }
      if (OP == 7) {                                                   // P-S-P + 2 ALU per FFMA2
        acc[k] = fma2(P[k], S[k], acc[k]);
        cnt += (unsigned)acc[k] >> 31;
        mn = min(mn, (unsigned)(acc[k] >> 32));
      }
    }
  }
  float r = 0.f;
#pragma unroll
  for (int k = 0; k < ILP; ++k) r += __uint_as_float((unsigned)acc[k]) + __uint_as_float((unsigned)(acc[k] >> 32));
  out[blockIdx.x * blockDim.x + t] = r + (float)cnt + (float)mn;
}

template <int OP>
void run(const char *name, int nsm, int wps, const float *in, float *out, int clk) {
  const int threads = 128, blocks = nsm * wps;  // wps warps per scheduler
  kern<OP><<<blocks, threads>>>(out, in);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<OP><<<blocks, threads>>>(out, in);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  // FFMA2 instructions per scheduler: warps/SMSP x ITERS x ILP
  const double inst = (double)wps * ITERS * ILP;
  const double cycles = ms * 1e-3 * clk * 1e6;
  printf("%-28s warps/SMSP %d  %6.3f ms  %.2f cycles per FFMA2 per scheduler\n", name, wps, ms,
         cycles / inst);
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  const int n = p.multiProcessorCount, clk = 1965;
  printf("%s SMs=%d (cycles at %d MHz)\n", p.name, n, clk);
  float *in, *out;
  cudaMalloc(&in, 64 * sizeof(float));
  float h[64];
  for (int i = 0; i < 64; ++i) h[i] = 1.0f + i * 1e-3f;
  cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaMalloc(&out, sizeof(float) * n * 16 * 128);
  for (int w : {1, 2, 4, 8}) {
    run<0>("FFMA2 P-S-P", n, w, in, out, clk);
    run<1>("FFMA2 S-P-S", n, w, in, out, clk);
    run<2>("FFMA2 P-P-P", n, w, in, out, clk);
    run<3>("FFMA2 P-P-S", n, w, in, out, clk);
    run<4>("FFMA2 Pc-S-P", n, w, in, out, clk);
    run<5>("FMUL2 P-P", n, w, in, out, clk);
    run<6>("FFMA2 P-S-P + LEA.HI", n, w, in, out, clk);
    run<7>("FFMA2 P-S-P + LEA.HI + IMNMX", n, w, in, out, clk);
  }
  return 0;
}
