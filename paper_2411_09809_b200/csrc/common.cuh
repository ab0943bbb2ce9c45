// Shared plumbing for the glare_b200 kernels: error reporting, launch
// accounting, stream-ordered scratch, deterministic block reductions.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <cstdarg>
#include <string>

#include "../../include/glare_b200.h"

namespace glr {

constexpr int kNumSmB200 = 148;

// Thread-local last-error message (glr_last_error).
std::string &last_error();
void set_error(const char *fmt, ...);
// Per-thread launch counter (glr_take_launch_count).
void count_launch(uint64_t n = 1);

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// Returns GLR_ECUDA with a message if the last launch / call failed.
inline int check_cuda(cudaError_t e, const char *what) {
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return GLR_ECUDA;
  }
  return GLR_OK;
}

#define GLR_CUDA(call)                                      \
  do {                                                      \
    int _rc = ::glr::check_cuda((call), #call);             \
    if (_rc != GLR_OK) return _rc;                          \
  } while (0)

#define GLR_LAUNCHED(name)                                  \
  do {                                                      \
    ::glr::count_launch();                                  \
    int _rc = ::glr::check_cuda(cudaGetLastError(), name);  \
    if (_rc != GLR_OK) return _rc;                          \
  } while (0)

// Keep freed stream-ordered scratch in the device's default pool instead of
// returning it to the driver at every synchronisation (release threshold 0
// by default), so repeated calls do not re-map hundreds of MB each time.
// Only cudaMallocAsync users (this library) draw from this pool; torch's
// caching allocator is separate.
inline void retain_scratch_pool() {
  static thread_local int done_dev = -1;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev == done_dev) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done_dev = dev;
}

// RAII stream-ordered scratch allocation (cudaMallocAsync / cudaFreeAsync).
struct Scratch {
  void *ptr = nullptr;
  cudaStream_t stream = nullptr;
  cudaError_t err = cudaSuccess;
  Scratch(size_t bytes, cudaStream_t s) : stream(s) {
    if (bytes) {
      retain_scratch_pool();
      err = cudaMallocAsync(&ptr, bytes, s);
    }
  }
  ~Scratch() {
    if (ptr) cudaFreeAsync(ptr, stream);
  }
  Scratch(const Scratch &) = delete;
  Scratch &operator=(const Scratch &) = delete;
  template <class T>
  T *as() const { return reinterpret_cast<T *>(ptr); }
};

inline int sm_count() {
  static int n = [] {
    int dev = 0, v = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return kNumSmB200;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      return kNumSmB200;
    return v;
  }();
  return n;
}

// Upper-triangular tile-pair enumeration shared by the all-pairs kernels:
// units are (ti, tj) with 0 <= ti <= tj < T in row-major order.
__host__ __device__ inline uint64_t tri_units(uint64_t T) { return T * (T + 1) / 2; }

__host__ __device__ inline uint64_t tri_row_start(uint64_t ti, uint64_t T) {
  return ti * T - ti * (ti - 1) / 2;  // ti*(2T-ti+1)/2, valid for ti >= 0
}

// (ti, tj) of unit u; double-precision guess corrected with exact integers.
__host__ __device__ inline void tri_unit_coords(uint64_t u, uint64_t T, uint64_t *ti,
                                                uint64_t *tj) {
  double b = 2.0 * (double)T + 1.0;
  double disc = b * b - 8.0 * (double)u;
  long long t = (long long)((b - sqrt(disc > 0 ? disc : 0.0)) * 0.5);
  if (t < 0) t = 0;
  if ((uint64_t)t >= T) t = (long long)T - 1;
  while (t > 0 && tri_row_start((uint64_t)t, T) > u) --t;
  while ((uint64_t)t + 1 < T && tri_row_start((uint64_t)t + 1, T) <= u) ++t;
  *ti = (uint64_t)t;
  *tj = (uint64_t)t + (u - tri_row_start((uint64_t)t, T));
}

// Banded enumeration of the same unit set, used by the crossing pass so that
// CTAs running at the same time share j-tiles in L2: units are ordered by
// (band of tj, ti, tj) with bands of W consecutive j-tiles.  Within band b
// (tj in [bW, e), w = e - bW): first the full rows ti < bW (w units each),
// then the triangle ti, tj in [bW, e).  W >= T gives the row-major order.
__host__ __device__ inline uint64_t band_units_before(uint64_t b, uint64_t W) {
  // all bands before b are full: unit count of band k = k*W*W + W(W+1)/2
  return W * W * (b * (b - 1) / 2) + b * (W * (W + 1) / 2);
}

__host__ __device__ inline void band_unit_coords(uint64_t u, uint64_t T, uint64_t W,
                                                 uint64_t *ti, uint64_t *tj) {
  const uint64_t nb = (T + W - 1) / W;
  uint64_t lo = 0, hi = nb - 1;  // last band whose prefix <= u
  while (lo < hi) {
    const uint64_t mid = (lo + hi + 1) >> 1;
    if (band_units_before(mid, W) <= u) lo = mid; else hi = mid - 1;
  }
  const uint64_t b = lo, b0 = b * W, e = (b0 + W < T) ? b0 + W : T, w = e - b0;
  const uint64_t local = u - band_units_before(b, W);
  if (local < b0 * w) {
    *ti = local / w;
    *tj = b0 + local % w;
  } else {
    uint64_t a, c;
    tri_unit_coords(local - b0 * w, w, &a, &c);
    *ti = b0 + a;
    *tj = b0 + c;
  }
}

// inverse of band_unit_coords
__host__ __device__ inline uint64_t band_unit_index(uint64_t ti, uint64_t tj, uint64_t T,
                                                    uint64_t W) {
  const uint64_t b = tj / W, b0 = b * W, e = (b0 + W < T) ? b0 + W : T, w = e - b0;
  const uint64_t base = band_units_before(b, W);
  if (ti < b0) return base + ti * w + (tj - b0);
  return base + b0 * w + tri_row_start(ti - b0, w) + (tj - ti);
}

// next unit in banded order
__host__ __device__ inline void band_advance(uint64_t T, uint64_t W, uint64_t *ti,
                                             uint64_t *tj) {
  const uint64_t b0 = (*tj / W) * W, e = (b0 + W < T) ? b0 + W : T;
  if (++*tj < e) return;
  ++*ti;
  if (*ti < b0) {
    *tj = b0;
  } else if (*ti < e) {
    *tj = *ti;
  } else {  // next band
    *ti = 0;
    *tj = e;
  }
}

// Block-wide sum of a double (deterministic: fixed shuffle tree + fixed
// warp order).  All threads must call; result valid in thread 0.
template <int NT>
__device__ inline double block_sum(double v, double *sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < NT / 32; ++i) r += sh[i];
  return r;
}

template <int NT>
__device__ inline unsigned long long block_sum_u64(unsigned long long v,
                                                   unsigned long long *sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  unsigned long long r = 0;
  if (threadIdx.x == 0)
    for (int i = 0; i < NT / 32; ++i) r += sh[i];
  return r;
}

// Kahan-compensated sequential sum of per-block partials, one thread.
__device__ inline double kahan_sum(const double *p, int64_t n) {
  double s = 0.0, c = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double y = p[i] - c;
    double t = s + y;
    c = (t - s) - y;
    s = t;
  }
  return s;
}

}  // namespace glr
