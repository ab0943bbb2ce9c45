// Throughput of packed FP32 (FADD2/FMUL2/FFMA2) vs scalar FFMA and the ALU
// ops of the filter's tail, in lanes/clk/SM (a packed op counts 2 lanes per
// thread).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o packed packed.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ILP 8
#define ITERS 4096

__device__ __forceinline__ uint64_t pk(float a, float b) { uint64_t r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ uint64_t add2(uint64_t a, uint64_t b) { uint64_t r; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ uint64_t mul2(uint64_t a, uint64_t b) { uint64_t r; asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) { uint64_t r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }
__device__ __forceinline__ float ffma(float a, float b, float c) { float r; asm volatile("fma.rn.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c)); return r; }
__device__ __forceinline__ float fmx(float a, float b) { float r; asm volatile("max.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b)); return r; }

template <int OP>
__global__ void kern(float* out, float s0, float s1) {
  uint64_t x[ILP]; float f[ILP];
  const uint64_t c = pk(s1, s1), d = pk(s0, s1 * 0.5f);
#pragma unroll
  for (int k = 0; k < ILP; ++k) { f[k] = s0 + threadIdx.x * 1e-7f + k; x[k] = pk(f[k], f[k] * 0.5f); }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int k = 0; k < ILP; ++k) {
      if (OP == 0) x[k] = add2(x[k], c);
      if (OP == 1) x[k] = mul2(x[k], c);
      if (OP == 2) x[k] = fma2(x[k], c, d);
      if (OP == 3) f[k] = ffma(f[k], s1, s0);
      if (OP == 4) f[k] = fmx(f[k], s1 + k);
      if (OP == 5) { x[k] = add2(x[k], c); f[k] = fmx(f[k], s1 + k); }  // FMA-pipe + ALU co-issue
      if (OP == 6) x[k] = add2(pk(s1, s1), x[k]);                        // broadcast operand form
      if (OP == 7) x[k] = add2(x[k], x[(k + 1) % ILP]);                   // reg-reg
      if (OP == 8) x[k] = fma2(x[k], x[(k + 1) % ILP], x[(k + 2) % ILP]); // reg-reg-reg
      if (OP == 9) x[k] = mul2(x[k], x[(k + 1) % ILP]);
    }
  }
  float acc = 0.f;
#pragma unroll
  for (int k = 0; k < ILP; ++k) acc += __uint_as_float((unsigned)x[k]) + __uint_as_float((unsigned)(x[k] >> 32)) + f[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int OP>
void run(const char* name, int nsm, double lanes_per_thread_op, int clk_mhz) {
  int blocks = nsm * 4, threads = 256;
  float* out; cudaMalloc(&out, sizeof(float) * blocks * threads);
  kern<OP><<<blocks, threads>>>(out, 1.0f, 1.0000001f);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<OP><<<blocks, threads>>>(out, 1.0f, 1.0000001f);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double ops = (double)blocks * threads * ITERS * ILP * lanes_per_thread_op;
  double per_s = ops / (ms * 1e-3);
  printf("%-34s %8.3f ms  %.3e lane-op/s  %.1f lanes/clk/SM @%d MHz\n", name, ms, per_s,
         per_s / (nsm * clk_mhz * 1e6), clk_mhz);
  cudaFree(out);
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int n = p.multiProcessorCount, clk = 1965;
  printf("%s SMs=%d\n", p.name, n);
  run<0>("FADD2 (2 lanes/op)", n, 2, clk);
  run<1>("FMUL2 (2 lanes/op)", n, 2, clk);
  run<2>("FFMA2 (2 lanes/op)", n, 2, clk);
  run<3>("FFMA 3-reg", n, 1, clk);
  run<4>("FMNMX", n, 1, clk);
  run<5>("FADD2 + FMNMX (per FADD2 lanes)", n, 2, clk);
  run<6>("FADD2 broadcast operand", n, 2, clk);
  run<7>("FADD2 reg-reg", n, 2, clk);
  run<8>("FFMA2 reg-reg-reg", n, 2, clk);
  run<9>("FMUL2 reg-reg", n, 2, clk);
  return 0;
}
