// Pipe-throughput microbenchmark for the FP64 all-pairs kernels: how many
// lanes/clk/SM does B200 retire for DADD, DMUL, DFMA, DSETP, FP32 and INT ops.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipes pipes.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ILP 8
#define ITERS 4096

struct Stamp { unsigned long long c0, c1, t0, t1; };

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t;
}

template <int OP>
__global__ void kern(double* out, Stamp* st, double s0, double s1) {
  double x[ILP]; float f[ILP]; unsigned u[ILP]; int cnt = 0;
#pragma unroll
  for (int k = 0; k < ILP; ++k) { x[k] = s0 + threadIdx.x * 1e-9 + k; f[k] = (float)x[k]; u[k] = threadIdx.x + k; }
  __syncthreads();
  unsigned long long c0 = clock64(), t0 = gtimer();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int k = 0; k < ILP; ++k) {
      if (OP == 0) x[k] = __dadd_rn(x[k], s1);
      if (OP == 1) x[k] = __dmul_rn(x[k], s1);
      if (OP == 2) x[k] = __fma_rn(x[k], s1, s0);
      if (OP == 3) { cnt += (x[k] < s1) ? 1 : 0; x[k] = __dadd_rn(x[k], s1); }  // DSETP+DADD
      if (OP == 4) f[k] = __fadd_rn(f[k], (float)s1);
      if (OP == 5) f[k] = __fmul_rn(f[k], (float)s1);
      if (OP == 6) u[k] = (u[k] + 0x9e3779b9u) ^ (u[k] >> 3);  // IADD + LOP/SHF
      if (OP == 7) { x[k] = __dmul_rn(x[k], s1); u[k] = (u[k] + 0x9e3779b9u) ^ (u[k] >> 3); } // FP64 + INT co-issue
      if (OP == 8) { x[k] = __dmul_rn(x[k], s1); f[k] = __fmul_rn(f[k], (float)s1); }       // FP64 + FP32 co-issue
    }
  }
  unsigned long long c1 = clock64(), t1 = gtimer();
  double acc = cnt;
#pragma unroll
  for (int k = 0; k < ILP; ++k) acc += x[k] + f[k] + u[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) st[blockIdx.x] = Stamp{c0, c1, t0, t1};
}

template <int OP>
void run(const char* name, int nsm, double ops_per_elem) {
  int blocks = nsm * 4, threads = 256;
  double* out; Stamp* st;
  cudaMalloc(&out, sizeof(double) * blocks * threads);
  cudaMalloc(&st, sizeof(Stamp) * blocks);
  kern<OP><<<blocks, threads>>>(out, st, 1.0, 1.0000001);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<OP><<<blocks, threads>>>(out, st, 1.0, 1.0000001);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  Stamp* h = new Stamp[blocks];
  cudaMemcpy(h, st, sizeof(Stamp) * blocks, cudaMemcpyDeviceToHost);
  double cyc = 0, ns = 0;
  for (int b = 0; b < blocks; ++b) { cyc += h[b].c1 - h[b].c0; ns += h[b].t1 - h[b].t0; }
  double mhz = cyc / ns * 1e3;
  double ops = (double)blocks * threads * ITERS * ILP * ops_per_elem;
  double per_s = ops / (ms * 1e-3);
  double lanes_clk_sm = per_s / (nsm * mhz * 1e6);
  printf("%-22s %8.3f ms  %.3e op/s  sm_clk %.0f MHz  %.1f lanes/clk/SM\n", name, ms, per_s, mhz, lanes_clk_sm);
  cudaFree(out); cudaFree(st); delete[] h;
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("%s SMs=%d cc=%d.%d\n", p.name, p.multiProcessorCount, p.major, p.minor);
  int n = p.multiProcessorCount;
  run<0>("DADD", n, 1);
  run<1>("DMUL", n, 1);
  run<2>("DFMA", n, 1);
  run<3>("DSETP+DADD (2 ops)", n, 2);
  run<4>("FADD", n, 1);
  run<5>("FMUL", n, 1);
  run<6>("IADD+LOP+SHF (~2-3)", n, 1);
  run<7>("DMUL + INT (per DMUL)", n, 1);
  run<8>("DMUL + FMUL (per DMUL)", n, 1);
  return 0;
}
