// Stepwise reconstruction of the crossing kernel's j-loop to find where the
// FP64 issue rate is lost (FP64 pipe 97% in a register-only mix vs 67% in
// cross_pairs_kernel).  Variants:
//  A  register-only mix (11 FP64 + 2 FMUL + 6 setp + pred add per pair)
//  B  A with j-data broadcast from shared memory (3 LDS.128 per j)
//  C  B with the exact pair body of pair_row_fast (no run refresh)
//  D  C plus the run-refresh branch (flag pattern ~15% of j)
#include <cstdio>
#include <cuda_runtime.h>

constexpr int KMIX = 2;
constexpr int TILE = 256;

struct __align__(16) JRec { double dx, dy, cdx, cdy; int r0, r1, r2, r3; };

__device__ inline float hv(double c) { return __int_as_float(__double2hiint(c)); }

__device__ inline void tail(unsigned &cnt, int jx1, int ix0, int ix1, int jx0, int jy1, int iy0,
                            int iy1, int jy0, float p12, float p34) {
  asm("{\n\t.reg .pred p;\n\t"
      "setp.ge.s32 p, %1, %2;\n\t"
      "setp.ge.and.s32 p, %3, %4, p;\n\t"
      "setp.ge.and.s32 p, %5, %6, p;\n\t"
      "setp.ge.and.s32 p, %7, %8, p;\n\t"
      "setp.le.and.f32 p, %9, 0f00000000, p;\n\t"
      "setp.le.and.f32 p, %10, 0f00000000, p;\n\t"
      "@p add.u32 %0, %0, 1;\n\t}"
      : "+r"(cnt)
      : "r"(jx1), "r"(ix0), "r"(ix1), "r"(jx0), "r"(jy1), "r"(iy0), "r"(iy1), "r"(jy0),
        "f"(p12), "f"(p34));
}

__constant__ JRec cj[TILE];

template <int V, int K = 2, int MINB = 4>
__global__ void __launch_bounds__(128, MINB) loop(const JRec *g, const double2 *gc, const unsigned char *gf,
                                               int reps, unsigned *out) {
  __shared__ JRec sj[TILE];
  __shared__ double2 sc[TILE];
  __shared__ unsigned char sf[TILE];
  for (int q = threadIdx.x; q < TILE; q += 128) { sj[q] = g[q]; sc[q] = gc[q]; sf[q] = gf[q]; }
  __syncthreads();
  double ax[K], ay[K], bx[K], by[K], abx[K], aby[K];
  int r0[K], r1[K], r2[K], r3[K];
  double dcx[K], dcy[K], ebx[K], eby[K];
  float f1[K];
  unsigned cnt[K];
  for (int k = 0; k < K; ++k) {
    const JRec &r = g[(threadIdx.x * K + k) % TILE];
    ax[k] = r.dx; ay[k] = r.dy; bx[k] = r.dx + 1; by[k] = r.dy - 1;
    abx[k] = r.cdx; aby[k] = r.cdy;
    r0[k] = r.r0; r1[k] = r.r1; r2[k] = r.r2; r3[k] = r.r3;
    dcx[k] = ax[k] - 0.5; dcy[k] = ay[k] - 0.25; ebx[k] = bx[k] - 0.5; eby[k] = by[k] - 0.25;
    f1[k] = hv(abx[k] * dcy[k] - aby[k] * dcx[k]);
    cnt[k] = 0;
  }
  for (int rep = 0; rep < reps; ++rep) {
#pragma unroll 4
    for (int jj = 0; jj < TILE; ++jj) {
      double dx, dy, cdx, cdy;
      int j0, j1, j2, j3;
      if (V == 0) {
        dx = ax[0] + jj; dy = ay[1] - jj; cdx = 1.0 + jj; cdy = 2.0 - jj;
        j0 = jj; j1 = jj + 7; j2 = jj; j3 = jj + 9;
      } else if (V == 5) {
        dx = cj[jj].dx; dy = cj[jj].dy; cdx = cj[jj].cdx; cdy = cj[jj].cdy;
        j0 = cj[jj].r0; j1 = cj[jj].r1; j2 = cj[jj].r2; j3 = cj[jj].r3;
      } else {
        const double4 d4 = reinterpret_cast<const double4 *>(sj + jj)[0];
        const int4 rk = reinterpret_cast<const int4 *>(sj + jj)[2];
        dx = d4.x; dy = d4.y; cdx = d4.z; cdy = d4.w;
        j0 = rk.x; j1 = rk.y; j2 = rk.z; j3 = rk.w;
      }
      if (V == 3 && sf[jj]) {
        const double2 c = sc[jj];
#pragma unroll
        for (int k = 0; k < K; ++k) {
          dcx[k] = __dsub_rn(c.x, ax[k]);
          dcy[k] = __dsub_rn(c.y, ay[k]);
          ebx[k] = __dsub_rn(bx[k], c.x);
          eby[k] = __dsub_rn(by[k], c.y);
          f1[k] = hv(__dsub_rn(__dmul_rn(abx[k], dcy[k]), __dmul_rn(aby[k], dcx[k])));
        }
      }
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const double ddx = __dsub_rn(dx, ax[k]);
        const double ddy = __dsub_rn(dy, ay[k]);
        const double c2 = __dsub_rn(__dmul_rn(abx[k], ddy), __dmul_rn(aby[k], ddx));
        const double c3 = __dsub_rn(__dmul_rn(cdy, dcx[k]), __dmul_rn(cdx, dcy[k]));
        const double c4 = __dsub_rn(__dmul_rn(cdx, eby[k]), __dmul_rn(cdy, ebx[k]));
        const float p12 = __fmul_rn(f1[k], hv(c2));
        const float p34 = __fmul_rn(hv(c3), hv(c4));
        if (V == 6) {          // G: no tail, keep results live with one IADD3
          cnt[k] += __float_as_uint(p12) ^ __float_as_uint(p34);
        } else if (V == 8) {   // G2: no FMUL either: xor of the c hi words
          cnt[k] += (unsigned)__double2hiint(c2) ^ (unsigned)__double2hiint(c3) ^ (unsigned)__double2hiint(c4);
        } else if (V == 7) {   // H: sign tail only (no bbox ISETP)
          asm("{\n\t.reg .pred p;\n\tsetp.le.f32 p, %1, 0f00000000;\n\t"
              "setp.le.and.f32 p, %2, 0f00000000, p;\n\t@p add.u32 %0, %0, 1;\n\t}"
              : "+r"(cnt[k]) : "f"(p12), "f"(p34));
        } else {
          tail(cnt[k], j1, r0[k], r1[k], j0, j3, r2[k], r3[k], j2, p12, p34);
        }
      }
    }
  }
  unsigned s = 0;
  for (int k = 0; k < K; ++k) s += cnt[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// E: the fp64lat "mix" body (11 FP64 with constant operands) at the same shape
template <int K = KMIX>
__global__ void __launch_bounds__(128, 4) mixk(double s, int iters, int r0, int r1, unsigned *out) {
  double a[K], b[K];
  unsigned cnt = 0;
  int q0 = threadIdx.x, q1 = threadIdx.x * 3;
  for (int k = 0; k < K; ++k) { a[k] = threadIdx.x * 1e-3 + k; b[k] = 1.0 + k * 1e-3; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll 4
    for (int jj = 0; jj < TILE; ++jj) {
#pragma unroll
      for (int k = 0; k < K; ++k) {
        double d1 = __dsub_rn(s, a[k]);
        double d2 = __dsub_rn(s, b[k]);
        double c2 = __dsub_rn(__dmul_rn(a[k], d2), __dmul_rn(b[k], d1));
        double c3 = __dsub_rn(__dmul_rn(s, a[k]), __dmul_rn(s, b[k]));
        double c4 = __dsub_rn(__dmul_rn(d1, b[k]), __dmul_rn(d2, a[k]));
        float p = __fmul_rn(hv(c2), hv(c3));
        float p2 = __fmul_rn(hv(c4), 1.5f);
        tail(cnt, q0, r0, q1, r0, q0, r1, q1, r1, p, p2);
        a[k] = c2; b[k] = c4;
      }
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = cnt + (unsigned)(a[0] + b[1]);
}

int main() {
  JRec h[TILE]; double2 hc[TILE]; unsigned char hf[TILE];
  for (int i = 0; i < TILE; ++i) {
    h[i] = JRec{1.0 * i, 2.0 * i, 0.5 * i, -0.25 * i, i, i + 100, i, i + 100};
    hc[i] = make_double2(0.3 * i, 0.7 * i);
    hf[i] = (i * 37 % 100) < 15;
  }
  JRec *g; double2 *gc; unsigned char *gf; unsigned *out;
  cudaMalloc(&g, sizeof(h)); cudaMalloc(&gc, sizeof(hc)); cudaMalloc(&gf, sizeof(hf));
  cudaMalloc(&out, 148 * 4 * 128 * 4);
  cudaMemcpy(g, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaMemcpy(gc, hc, sizeof(hc), cudaMemcpyHostToDevice);
  cudaMemcpy(gf, hf, sizeof(hf), cudaMemcpyHostToDevice);
  const int reps = 200;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaFree(out); cudaMalloc(&out, 148 * 16 * 128 * 4);
  auto run = [&](auto kern, const char *name, int kk = 2, int minb = 4) {
    kern<<<148 * minb, 128>>>(g, gc, gf, reps, out);
    cudaEventRecord(e0);
    kern<<<148 * minb, 128>>>(g, gc, gf, reps, out);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double pairs = 148.0 * minb * 128 * kk * TILE * (double)reps;
    printf("%-40s %.3e pairs/s  fp64(11/pair) %.0f%%\n", name, pairs / (ms * 1e-3),
           100.0 * pairs / (ms * 1e-3) * 11 / (64.0 * 148 * 1.965e9));
  };
  run(loop<0>, "A regs only");
  run(loop<1>, "B smem j-data");
  run(loop<3>, "D smem + refresh branch (15%)");
  cudaMemcpyToSymbol(cj, h, sizeof(h));
  run(loop<5>, "F constant-memory j-data");
  run(loop<6>, "G smem, no tail");
  run(loop<7>, "H smem, sign tail only");
  run(loop<1, 1, 6>, "B K=1 minb6", 1, 6);
  run(loop<1, 1, 8>, "B K=1 minb8", 1, 8);
  run(loop<1, 2, 5>, "B K=2 minb5", 2, 5);
  run(loop<1, 2, 6>, "B K=2 minb6", 2, 6);
  run(loop<1, 4, 2>, "B K=4 minb2", 4, 2);
  run(loop<1, 4, 3>, "B K=4 minb3", 4, 3);
  run(loop<6, 1, 8>, "G K=1 minb8", 1, 8);
  run(loop<8>, "G2 no FMUL, no tail");
  run(loop<6, 2, 6>, "G K=2 minb6", 2, 6);
  {
    mixk<KMIX><<<148 * 4, 128>>>(1.0000001, reps, 5, 7, out);
    cudaEventRecord(e0);
    mixk<KMIX><<<148 * 4, 128>>>(1.0000001, reps, 5, 7, out);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double pairs = 148.0 * 4 * 128 * KMIX * TILE * (double)reps;
    printf("%-40s %.3e pairs/s  fp64(11/pair) %.0f%%\n", "E mix (const operands)", pairs / (ms * 1e-3),
           100.0 * pairs / (ms * 1e-3) * 11 / (64.0 * 148 * 1.965e9));
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
