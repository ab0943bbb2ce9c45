// Node occlusion N_c: the O(|V|^2) all-pairs pass.
//
// Replaces the numpy body of the reference's node_occlusion
// (/root/reference/pkg/src/glare/metrics/exact.py:55-74): the number of
// unordered vertex pairs with fl(fl(dx*dx) + fl(dy*dy)) < thr, strict, no FMA,
// over every vertex (isolated ones included).  thr = (2.0*r)**2 is computed by
// the caller with the reference's own Python expression (exact.py:63).
//
// FP64 budget per pair: 2 DADD + 2 DMUL + 1 DADD = 5.  The comparison runs on
// the ALU pipe: s = fl(dx^2 + dy^2) is +0 or positive (or +inf), so
// s < thr  <=>  bits(s) < bits(thr) as unsigned 64-bit integers.
//
// Tiling mirrors crossing.cu: vertex tiles of kThreads*kK, upper-triangular
// tile-pair units, persistent CTAs over a contiguous unit range, i-vertices in
// registers, the j-tile in shared memory.
#include <cub/cub.cuh>

#include "common.cuh"

namespace glr {
namespace {

constexpr int kThreads = 128;
constexpr int kK = 8;
constexpr int kTile = kThreads * kK;
constexpr int kMinBlocks = 4;

inline int64_t pad_vertices(int64_t n) { return ((n + kTile - 1) / kTile) * kTile; }

template <bool DIAG>
__device__ inline void occ_row(const double (&xi)[kK], const double (&yi)[kK], double2 pj, int jj,
                               unsigned long long thr_bits, unsigned (&cnt)[kK]) {
#pragma unroll
  for (int k = 0; k < kK; ++k) {
    const double dx = __dsub_rn(xi[k], pj.x);
    const double dy = __dsub_rn(yi[k], pj.y);
    const double s = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
    const int diag_ok = DIAG ? (jj > (int)threadIdx.x + k * kThreads) : 1;
    // s < thr as a 64-bit unsigned compare of bit patterns, then a predicated
    // add (PTX keeps it to 2 ISETP + 1 IADD)
    asm("{\n\t.reg .pred p;\n\t"
        "setp.lt.u64 p, %1, %2;\n\t"
        "setp.ne.and.s32 p, %3, 0, p;\n\t"
        "@p add.u32 %0, %0, 1;\n\t}"
        : "+r"(cnt[k])
        : "l"((unsigned long long)__double_as_longlong(s)), "l"(thr_bits), "r"(diag_ok));
  }
}

__global__ void __launch_bounds__(kThreads, kMinBlocks)
occlusion_pairs_kernel(const double2 *__restrict__ xy, int64_t n, const int2 *__restrict__ ulist,
                       uint64_t T, uint64_t ubeg, uint64_t uend, unsigned long long thr_bits,
                       unsigned long long *__restrict__ cta_cnt) {
  // ulist == nullptr: units are the implicit upper triangle of tile pairs;
  // otherwise unit u is the explicit tile pair ulist[u] (culled candidates).
  __shared__ __align__(16) double2 sj[kTile];
  __shared__ unsigned long long red[kThreads / 32];
  const uint64_t span = uend - ubeg;
  const uint64_t b = ubeg + span * blockIdx.x / gridDim.x;
  const uint64_t e = ubeg + span * (blockIdx.x + 1) / gridDim.x;
  // padding vertices sit at +inf (i side) / -inf (j side): every difference
  // with them is +-inf, whose square sum is +inf -- never below a threshold
  const double PAD = __longlong_as_double(0x7ff0000000000000ll);
  unsigned long long total = 0;
  double xi[kK], yi[kK];
  uint64_t ti = 0, tj = 0, cur = ~0ull;
  if (b < e && ulist == nullptr) tri_unit_coords(b, T, &ti, &tj);
  for (uint64_t u = b; u < e; ++u) {
    if (ulist != nullptr) {
      const int2 p = ulist[u];
      ti = (uint64_t)p.x;
      tj = (uint64_t)p.y;
    }
    if (ti != cur) {
#pragma unroll
      for (int k = 0; k < kK; ++k) {
        const int64_t v = (int64_t)ti * kTile + threadIdx.x + k * kThreads;
        double2 p = v < n ? xy[v] : make_double2(PAD, PAD);
        xi[k] = p.x;
        yi[k] = p.y;
      }
      cur = ti;
    }
    __syncthreads();
    for (int q = threadIdx.x; q < kTile; q += kThreads) {
      const int64_t v = (int64_t)tj * kTile + q;
      sj[q] = v < n ? xy[v] : make_double2(-PAD, -PAD);
    }
    __syncthreads();
    unsigned cnt[kK];
#pragma unroll
    for (int k = 0; k < kK; ++k) cnt[k] = 0;
    if (ti == tj) {
      for (int jj = 0; jj < kTile; ++jj) occ_row<true>(xi, yi, sj[jj], jj, thr_bits, cnt);
    } else {
#pragma unroll 4
      for (int jj = 0; jj < kTile; ++jj) occ_row<false>(xi, yi, sj[jj], jj, thr_bits, cnt);
    }
    unsigned c = 0;
#pragma unroll
    for (int k = 0; k < kK; ++k) c += cnt[k];
    total += c;
    if (ulist == nullptr && ++tj == T) { ++ti; tj = ti; }
  }
  unsigned long long bc = block_sum_u64<kThreads>(total, red);
  if (threadIdx.x == 0) cta_cnt[blockIdx.x] = bc;
}

__global__ void occ_finalize_kernel(const unsigned long long *cta_cnt, int ncta, double *out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    unsigned long long c = 0;
    for (int i = 0; i < ncta; ++i) c += cta_cnt[i];
    out[0] = (double)c;
  }
}

// ---- culled candidate list -------------------------------------------------

// per vertex tile: (min x, max x, min y, max y) over real vertices
__global__ void __launch_bounds__(256)
vtile_box_kernel(const double2 *__restrict__ xy, int64_t n, double4 *__restrict__ box) {
  __shared__ double4 red[8];
  const double INF = __longlong_as_double(0x7ff0000000000000ll);
  double x0 = INF, x1 = -INF, y0 = INF, y1 = -INF;
  for (int q = threadIdx.x; q < kTile; q += 256) {
    const int64_t v = (int64_t)blockIdx.x * kTile + q;
    if (v < n) {
      const double2 p = xy[v];
      x0 = fmin(x0, p.x); x1 = fmax(x1, p.x);
      y0 = fmin(y0, p.y); y1 = fmax(y1, p.y);
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    x0 = fmin(x0, __shfl_down_sync(0xffffffffu, x0, o));
    x1 = fmax(x1, __shfl_down_sync(0xffffffffu, x1, o));
    y0 = fmin(y0, __shfl_down_sync(0xffffffffu, y0, o));
    y1 = fmax(y1, __shfl_down_sync(0xffffffffu, y1, o));
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = make_double4(x0, x1, y0, y1);
  __syncthreads();
  if (threadIdx.x == 0) {
    double4 b = red[0];
    for (int w = 1; w < 8; ++w) {
      b.x = fmin(b.x, red[w].x); b.y = fmax(b.y, red[w].y);
      b.z = fmin(b.z, red[w].z); b.w = fmax(b.w, red[w].w);
    }
    box[blockIdx.x] = b;
  }
}

// A tile pair can hold an occluding pair only if neither axis gap reaches 2r.
// Exactness: for i in A, j in B with fl(minB - maxA) >= 2r, monotone rounding
// gives |fl(x_i - x_j)| >= 2r, hence fl(dx*dx) >= fl((2r)^2) = thr and the
// pair fails (same argument as the oracle's x-sorted sweep).  Empty tiles
// (+inf/-inf boxes) give infinite gaps.
__device__ inline bool may_occlude(double4 a, double4 b, double reach) {
  return !(__dsub_rn(b.x, a.y) >= reach || __dsub_rn(a.x, b.y) >= reach ||
           __dsub_rn(b.z, a.w) >= reach || __dsub_rn(a.z, b.w) >= reach);
}

template <bool FILL>
__global__ void vtile_pairs_kernel(const double4 *__restrict__ box, int64_t T, double reach,
                                   unsigned long long *__restrict__ counts,
                                   const unsigned long long *__restrict__ offs, int2 *list) {
  for (int64_t ti = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; ti < T;
       ti += (int64_t)gridDim.x * blockDim.x) {
    const double4 a = box[ti];
    unsigned long long c = 0, o = FILL ? offs[ti] : 0;
    for (int64_t tj = ti; tj < T; ++tj) {
      if (may_occlude(a, box[tj], reach)) {
        if (FILL) list[o + c] = make_int2((int)ti, (int)tj);
        ++c;
      }
    }
    if (!FILL) counts[ti] = c;
  }
}

int occ_blocks(int64_t work) {
  int64_t b = (work + 127) / 128;
  const int64_t cap = (int64_t)sm_count() * 16;
  if (b > cap) b = cap;
  return (int)(b < 1 ? 1 : b);
}

int occlusion_run(const double *d_xy, int64_t n, double thr, const int2 *d_list,
                  uint64_t list_len, uint64_t ubeg, uint64_t uend, double *d_out,
                  cudaStream_t st, const char *who) {
  if (d_out == nullptr || n < 0 || (n > 0 && d_xy == nullptr)) {
    set_error("%s: invalid arguments", who);
    return GLR_EARG;
  }
  const uint64_t T = (uint64_t)(pad_vertices(n < 1 ? 1 : n) / kTile);
  const uint64_t U = d_list != nullptr ? list_len : tri_units(T);
  if (ubeg > uend || uend > U) {
    set_error("%s: unit range [%llu, %llu) outside [0, %llu)", who, (unsigned long long)ubeg,
              (unsigned long long)uend, (unsigned long long)U);
    return GLR_EARG;
  }
  if (n < 2 || ubeg == uend || !(thr > 0.0)) {
    GLR_CUDA(cudaMemsetAsync(d_out, 0, sizeof(double), st));
    return GLR_OK;
  }
  uint64_t g = (uint64_t)sm_count() * kMinBlocks;
  if (uend - ubeg < g) g = uend - ubeg;
  const int grid = (int)g;
  Scratch scr((size_t)grid * sizeof(unsigned long long), st);
  GLR_CUDA(scr.err);
  unsigned long long thr_bits;
  memcpy(&thr_bits, &thr, sizeof(thr));
  occlusion_pairs_kernel<<<grid, kThreads, 0, st>>>(reinterpret_cast<const double2 *>(d_xy), n,
                                                    d_list, T, ubeg, uend, thr_bits,
                                                    scr.as<unsigned long long>());
  GLR_LAUNCHED("occlusion_pairs_kernel");
  occ_finalize_kernel<<<1, 32, 0, st>>>(scr.as<unsigned long long>(), grid, d_out);
  GLR_LAUNCHED("occ_finalize_kernel");
  return GLR_OK;
}

}  // namespace
}  // namespace glr

extern "C" {

int glr_occlusion_tile(void) { return glr::kTile; }

uint64_t glr_occlusion_units(int64_t n) {
  const int64_t np = glr::pad_vertices(n < 1 ? 1 : n);
  return glr::tri_units((uint64_t)(np / glr::kTile));
}

int glr_occlusion_count(const double *d_xy, int64_t n, double thr, uint64_t unit_begin,
                        uint64_t unit_end, double *d_out, void *stream) {
  return glr::occlusion_run(d_xy, n, thr, nullptr, 0, unit_begin, unit_end, d_out,
                            glr::as_stream(stream), "glr_occlusion_count");
}

int glr_occlusion_candidates(const double *d_xy, int64_t n, double reach, void *d_list,
                             uint64_t capacity, uint64_t *h_count, void *stream) {
  using namespace glr;
  cudaStream_t st = as_stream(stream);
  if (h_count == nullptr || n < 0 || (n > 0 && d_xy == nullptr) || !(reach > 0.0)) {
    set_error("glr_occlusion_candidates: invalid arguments");
    return GLR_EARG;
  }
  const int64_t T = pad_vertices(n < 1 ? 1 : n) / kTile;
  size_t t_scan = 0;
  GLR_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t_scan, (unsigned long long *)nullptr,
                                         (unsigned long long *)nullptr, (int)(T + 1), st));
  const size_t a_box = ((size_t)T * sizeof(double4) + 255) & ~(size_t)255;
  const size_t a_cnt = ((size_t)(T + 1) * sizeof(unsigned long long) + 255) & ~(size_t)255;
  Scratch scr(a_box + 2 * a_cnt + t_scan, st);
  GLR_CUDA(scr.err);
  char *p = scr.as<char>();
  double4 *box = reinterpret_cast<double4 *>(p);
  unsigned long long *counts = reinterpret_cast<unsigned long long *>(p + a_box);
  unsigned long long *offs = reinterpret_cast<unsigned long long *>(p + a_box + a_cnt);
  void *tmp = p + a_box + 2 * a_cnt;
  vtile_box_kernel<<<(unsigned)T, 256, 0, st>>>(reinterpret_cast<const double2 *>(d_xy), n, box);
  GLR_LAUNCHED("vtile_box_kernel");
  GLR_CUDA(cudaMemsetAsync(counts + T, 0, sizeof(unsigned long long), st));
  vtile_pairs_kernel<false><<<occ_blocks(T), 128, 0, st>>>(box, T, reach, counts, nullptr, nullptr);
  GLR_LAUNCHED("vtile_pairs_kernel<count>");
  size_t tb = t_scan;
  GLR_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, counts, offs, (int)(T + 1), st));
  count_launch(2);
  unsigned long long total = 0;
  GLR_CUDA(cudaMemcpyAsync(&total, offs + T, sizeof(total), cudaMemcpyDeviceToHost, st));
  GLR_CUDA(cudaStreamSynchronize(st));
  *h_count = total;
  if (d_list != nullptr && capacity >= total && total > 0) {
    vtile_pairs_kernel<true><<<occ_blocks(T), 128, 0, st>>>(box, T, reach, nullptr, offs,
                                                            reinterpret_cast<int2 *>(d_list));
    GLR_LAUNCHED("vtile_pairs_kernel<fill>");
  }
  return GLR_OK;
}

int glr_occlusion_count_list(const double *d_xy, int64_t n, double thr, const void *d_list,
                             uint64_t list_len, uint64_t unit_begin, uint64_t unit_end,
                             double *d_out, void *stream) {
  if (list_len == 0) {
    if (unit_begin != 0 || unit_end != 0) {
      glr::set_error("glr_occlusion_count_list: unit range outside an empty list");
      return GLR_EARG;
    }
    GLR_CUDA(cudaMemsetAsync(d_out, 0, sizeof(double), glr::as_stream(stream)));
    return GLR_OK;
  }
  if (d_list == nullptr) {
    glr::set_error("glr_occlusion_count_list: null list");
    return GLR_EARG;
  }
  return glr::occlusion_run(d_xy, n, thr, reinterpret_cast<const int2 *>(d_list), list_len,
                            unit_begin, unit_end, d_out, glr::as_stream(stream),
                            "glr_occlusion_count_list");
}

}  // extern "C"
