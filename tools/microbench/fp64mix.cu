// Is the FP64 pipe slower for interleaved DMUL/DADD than for either alone?
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void __launch_bounds__(128) k(double *out, double s, double t, int iters) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) x[i] = __dadd_rn(x[i], t);
      if (MODE == 1) x[i] = __dmul_rn(x[i], s);
      if (MODE == 2) x[i] = (i & 1) ? __dmul_rn(x[i], s) : __dadd_rn(x[i], t);
      if (MODE == 3) x[i] = (i & 1) ? __dmul_rn(x[i], x[i ^ 1]) : __dadd_rn(x[i], x[i ^ 1]);  // reg-reg
      if (MODE == 4) x[i] = __dsub_rn(__dmul_rn(x[i], s), __dmul_rn(x[(i + 1) & 7], t));   // c = p - q
    }
  }
  double a = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) a += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = a;
}
int main() {
  double *out; cudaMalloc(&out, 148 * 16 * 128 * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4096;
  auto run = [&](auto kern, const char *name, double ops_per) {
    kern<<<148 * 4, 128>>>(out, 1.0000001, 1e-9, iters);
    cudaEventRecord(e0);
    kern<<<148 * 4, 128>>>(out, 1.0000001, 1e-9, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = 148.0 * 4 * 128 * 8 * iters * ops_per;
    printf("%-28s %.1f FP64 lanes/clk/SM (at 1965 MHz)\n", name, ops / (ms * 1e-3) / (148 * 1.965e9));
  };
  run(k<0>, "DADD only", 1);
  run(k<1>, "DMUL only", 1);
  run(k<2>, "DADD/DMUL interleaved", 1);
  run(k<3>, "interleaved reg-reg", 1);
  run(k<4>, "DMUL,DMUL,DSUB pattern", 3);
  return 0;
}
