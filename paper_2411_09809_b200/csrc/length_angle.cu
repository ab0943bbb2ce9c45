// Edge length variation M_l and minimum angle M_a: the O(|E|) and per-vertex
// passes.
//
// M_l replaces exact.py:127-142: lengths sqrt(dx*dx + dy*dy), d = b - a;
// mean; sum of (l - mean)^2; sqrt(S / (m*mean*mean)) / sqrt(m - 1).  Two
// grid-stride reduction passes with fixed grids (deterministic), partials
// combined with a Kahan sum.
//
// M_a replaces exact.py:88-124 and geometry.py:82-85: the 2m directed
// incident angles atan2(uy - vy, ux - vx) (+2pi when negative) are bucketed
// by vertex (degree histogram, exclusive scan, scatter), each vertex's
// segment is sorted by a hand-written segmented sort in three size classes
// (below), which also takes the minimum consecutive gap and the wrap gap
// (2pi - last) + first, d_v = (phi - gap)/phi with phi = 2pi/deg, and
// M_a = 1 - mean(d_v) over vertices of degree >= 1.

#include "common.cuh"

namespace glr {
namespace {

constexpr int kRedThreads = 256;
constexpr double kTwoPi = 6.283185307179586;  // 2.0 * math.pi

__global__ void set_value_kernel(double *out, double a, double b, double c) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    out[0] = a;
    out[1] = b;
    out[2] = c;
  }
}

__global__ void __launch_bounds__(kRedThreads)
lengths_kernel(const double2 *__restrict__ xy, const longlong2 *__restrict__ edges, int64_t m,
               double *__restrict__ len, double *__restrict__ part) {
  __shared__ double sh[kRedThreads / 32];
  double acc = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    longlong2 uv = edges[e];
    double2 a = xy[uv.x], b = xy[uv.y];
    double dx = __dsub_rn(b.x, a.x), dy = __dsub_rn(b.y, a.y);
    double l = __dsqrt_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)));
    len[e] = l;
    acc = __dadd_rn(acc, l);
  }
  double s = block_sum<kRedThreads>(acc, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void mean_kernel(const double *part, int nb, int64_t m, double *mean) {
  if (threadIdx.x == 0 && blockIdx.x == 0) mean[0] = kahan_sum(part, nb) / (double)m;
}

__global__ void __launch_bounds__(kRedThreads)
sqdev_kernel(const double *__restrict__ len, int64_t m, const double *__restrict__ mean,
             double *__restrict__ part) {
  __shared__ double sh[kRedThreads / 32];
  const double mu = mean[0];
  double acc = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    double d = __dsub_rn(len[e], mu);
    acc = __dadd_rn(acc, __dmul_rn(d, d));
  }
  double s = block_sum<kRedThreads>(acc, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void ml_finalize_kernel(const double *part, int nb, int64_t m, const double *mean,
                                   double *out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    const double S = kahan_sum(part, nb);
    const double mu = mean[0];
    // exact.py:141-142: sqrt(S / (m*mean*mean)) / sqrt(m - 1)
    const double la = sqrt(S / ((double)m * mu * mu));
    out[0] = mu;
    out[1] = S;
    out[2] = la / sqrt((double)(m - 1));
  }
}

// ---- minimum angle --------------------------------------------------------
//
// Per-vertex sort of the incident angles, hand-written in three size classes
// (the degree decides, warp-uniformly / block-uniformly):
//   W  deg <= 32:          one warp per vertex, bitonic network in registers
//                          (one angle per lane, width = next power of 2);
//   B  32 < deg <= 4096:   one 256-thread CTA per vertex, bitonic sort of the
//                          segment padded to a power of 2 in shared memory;
//   L  deg > 4096:         one 1024-thread CTA per vertex (hubs: C5-shaped
//                          graphs reach degree ~55k): 4096-angle runs sorted
//                          as in B and written to global memory, then rounds
//                          of pairwise rank merges (each element's output
//                          slot = its index + its lower/upper bound in the
//                          partner run, one binary search per element).
// Every class ends with the same gap step as the reference (exact.py:100-120):
// min over consecutive fl(a[k+1] - a[k]), the wrap fl(fl(2pi - last) + first),
// d_v = fl(fl(phi - gap) / phi), phi = fl(2pi / deg), written to dv[v].  The
// sort only permutes values (compare-and-select, no fmin/fmax), so the
// sorted sequence -- and with it every gap -- is the reference's exactly.

constexpr int kBlockSortMax = 4096;   // class B capacity = class L run length
constexpr int kSortThreadsB = 256;
constexpr int kSortThreadsL = 1024;
constexpr int kScanTile = 2048;       // degree scan: 256 threads x 8
constexpr double kPosInf = __builtin_huge_val();

__global__ void degree_kernel(const longlong2 *__restrict__ edges, int64_t m, int *deg) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    longlong2 uv = edges[e];
    atomicAdd(&deg[uv.x], 1);
    atomicAdd(&deg[uv.y], 1);
  }
}

// Exclusive scan of deg[0..cnt) into offs (three passes: tile totals, one-CTA
// scan of the totals, tile rescans with the tile's offset).
__device__ inline int block_exclusive_scan_256(int v, int *sh, int *total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[w] = x;
  __syncthreads();
  if (w == 0) {
    int s = lane < 8 ? sh[lane] : 0;
    for (int o = 1; o < 8; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < 8) sh[lane] = s;  // inclusive warp totals
  }
  __syncthreads();
  const int excl = x - v + (w > 0 ? sh[w - 1] : 0);
  *total = sh[7];
  __syncthreads();
  return excl;
}

__global__ void __launch_bounds__(256)
scan_tiles_kernel(const int *__restrict__ in, int64_t cnt, int *__restrict__ tile_sum) {
  __shared__ int sh[8];
  const int64_t base = (int64_t)blockIdx.x * kScanTile + threadIdx.x * 8;
  int s = 0;
  for (int k = 0; k < 8; ++k) s += base + k < cnt ? in[base + k] : 0;
  int tot;
  block_exclusive_scan_256(s, sh, &tot);
  if (threadIdx.x == 0) tile_sum[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(256)
scan_totals_kernel(int *__restrict__ tile_sum, int ntiles) {
  __shared__ int sh[8];
  int carry = 0;
  for (int b = 0; b < ntiles; b += 256) {
    const int i = b + threadIdx.x;
    const int v = i < ntiles ? tile_sum[i] : 0;
    int tot;
    const int e = block_exclusive_scan_256(v, sh, &tot);
    if (i < ntiles) tile_sum[i] = carry + e;
    carry += tot;
  }
}

__global__ void __launch_bounds__(256)
scan_apply_kernel(const int *__restrict__ in, int64_t cnt, const int *__restrict__ tile_off,
                  int *__restrict__ out) {
  __shared__ int sh[8];
  const int64_t base = (int64_t)blockIdx.x * kScanTile + threadIdx.x * 8;
  int v[8], s = 0;
  for (int k = 0; k < 8; ++k) {
    v[k] = base + k < cnt ? in[base + k] : 0;
    s += v[k];
  }
  int tot;
  int run = block_exclusive_scan_256(s, sh, &tot) + tile_off[blockIdx.x];
  for (int k = 0; k < 8; ++k) {
    if (base + k < cnt) out[base + k] = run;
    run += v[k];
  }
}

__global__ void scatter_angles_kernel(const double2 *__restrict__ xy,
                                      const longlong2 *__restrict__ edges, int64_t m,
                                      const int *__restrict__ offs, int *cursor,
                                      double *__restrict__ ang) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < 2 * m;
       k += (int64_t)gridDim.x * blockDim.x) {
    longlong2 uv = edges[k < m ? k : k - m];
    const long long v = k < m ? uv.x : uv.y;  // the vertex
    const long long u = k < m ? uv.y : uv.x;  // its neighbour
    double2 pv = xy[v], pu = xy[u];
    // geometry.py:82-85: arctan2(uy - vy, ux - vx), + 2pi where negative
    double a = atan2(__dsub_rn(pu.y, pv.y), __dsub_rn(pu.x, pv.x));
    if (a < 0.0) a = __dadd_rn(a, kTwoPi);
    int slot = offs[v] + atomicAdd(&cursor[v], 1);
    ang[slot] = a;
  }
}

// d_v from the sorted segment's min inner gap, first and last (exact.py:111-120)
__device__ inline double vertex_dev(double inner, double first, double last, int d) {
  const double wrap = __dadd_rn(__dsub_rn(kTwoPi, last), first);
  const double gap = inner < wrap ? inner : wrap;
  const double phi = __ddiv_rn(kTwoPi, (double)d);
  return __ddiv_rn(__dsub_rn(phi, gap), phi);
}

// compare-and-select keeping both values (a permutation: -0.0/+0.0 and
// duplicates survive as they are)
__device__ inline void cas(double &lo, double &hi) {
  const double a = lo, b = hi;
  const bool sw = b < a;
  lo = sw ? b : a;
  hi = sw ? a : b;
}

// Class W: one warp per vertex of degree 1..32; larger vertices are
// appended to the B / L work lists.
__global__ void __launch_bounds__(256)
sort_small_kernel(const double *__restrict__ ang, const int *__restrict__ offs, int64_t n,
                  double *__restrict__ dv, int *__restrict__ listB, int *__restrict__ listL,
                  int *__restrict__ counts) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = warp; v < n; v += nwarps) {
    const int s = offs[v], d = offs[v + 1] - s;
    if (d == 0) continue;
    if (d > 32) {
      if (lane == 0) {
        if (d <= kBlockSortMax) listB[atomicAdd(&counts[0], 1)] = (int)v;
        else listL[atomicAdd(&counts[1], 1)] = (int)v;
      }
      continue;
    }
    int w = 1;
    while (w < d) w <<= 1;
    double x = lane < d ? ang[s + lane] : kPosInf;
    for (int k = 2; k <= w; k <<= 1) {
      for (int j = k >> 1; j > 0; j >>= 1) {
        const double o = __shfl_xor_sync(0xffffffffu, x, j);
        const bool lower = (lane & j) == 0, up = (lane & k) == 0;
        // the lower lane of an ascending pair keeps the smaller value
        const bool take_o = (lower == up) ? (o < x) : (x < o);
        x = take_o ? o : x;
      }
    }
    const double nx = __shfl_down_sync(0xffffffffu, x, 1);
    double g = lane + 1 < d ? __dsub_rn(nx, x) : kPosInf;
    for (int o = 16; o > 0; o >>= 1) {
      const double y = __shfl_xor_sync(0xffffffffu, g, o);
      g = y < g ? y : g;
    }
    const double first = __shfl_sync(0xffffffffu, x, 0);
    const double last = __shfl_sync(0xffffffffu, x, d - 1);
    if (lane == 0) dv[v] = vertex_dev(g, first, last, d);
  }
}

// Bitonic sort of sh[0..P) (P a power of 2, padded with +inf) by the CTA.
template <int NT>
__device__ inline void block_bitonic(double *sh, int P) {
  for (int k = 2; k <= P; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int t = threadIdx.x; t < (P >> 1); t += NT) {
        const int i = 2 * t - (t & (j - 1));  // lower index of the pair
        double a = sh[i], b = sh[i + j];
        if ((i & k) == 0) cas(a, b); else cas(b, a);
        sh[i] = a;
        sh[i + j] = b;
      }
      __syncthreads();
    }
  }
}

// CTA-wide min of the consecutive gaps of a sorted array in `src` (shared or
// global), result in every thread.
template <int NT>
__device__ inline double block_min_gap(const double *src, int d, double *red) {
  double g = kPosInf;
  for (int k = threadIdx.x; k + 1 < d; k += NT) {
    const double y = __dsub_rn(src[k + 1], src[k]);
    g = y < g ? y : g;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double y = __shfl_xor_sync(0xffffffffu, g, o);
    g = y < g ? y : g;
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = g;
  __syncthreads();
  double r = kPosInf;
  for (int w = 0; w < NT / 32; ++w) r = red[w] < r ? red[w] : r;
  __syncthreads();
  return r;
}

__device__ inline int pow2_ceil(int d) {
  int p = 1;
  while (p < d) p <<= 1;
  return p;
}

// Class B: one CTA per listed vertex (32 < deg <= 4096).
__global__ void __launch_bounds__(kSortThreadsB)
sort_block_kernel(const double *__restrict__ ang, const int *__restrict__ offs,
                  const int *__restrict__ list, const int *__restrict__ counts,
                  double *__restrict__ dv) {
  __shared__ double sh[kBlockSortMax];
  __shared__ double red[kSortThreadsB / 32];
  const int cnt = counts[0];
  for (int q = blockIdx.x; q < cnt; q += gridDim.x) {
    const int v = list[q];
    const int s = offs[v], d = offs[v + 1] - s;
    const int P = pow2_ceil(d);
    for (int k = threadIdx.x; k < P; k += kSortThreadsB) sh[k] = k < d ? ang[s + k] : kPosInf;
    __syncthreads();
    block_bitonic<kSortThreadsB>(sh, P);
    const double g = block_min_gap<kSortThreadsB>(sh, d, red);
    if (threadIdx.x == 0) dv[v] = vertex_dev(g, sh[0], sh[d - 1], d);
    __syncthreads();
  }
}

// Number of elements of sorted run r[0..len) that are < x (strict) or <= x.
template <bool STRICT>
__device__ inline int rank_in(const double *r, int len, double x) {
  int lo = 0, hi = len;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    const bool before = STRICT ? (r[mid] < x) : !(x < r[mid]);
    if (before) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Class L: one CTA per listed hub (deg > 4096).  `buf` is a second array
// with the same segment offsets as `ang`; both are overwritten.
__global__ void __launch_bounds__(kSortThreadsL)
sort_large_kernel(double *__restrict__ ang, double *__restrict__ buf,
                  const int *__restrict__ offs, const int *__restrict__ list,
                  const int *__restrict__ counts, double *__restrict__ dv) {
  __shared__ double sh[kBlockSortMax];
  __shared__ double red[kSortThreadsL / 32];
  const int cnt = counts[1];
  for (int q = blockIdx.x; q < cnt; q += gridDim.x) {
    const int v = list[q];
    const int s = offs[v], d = offs[v + 1] - s;
    double *src = ang + s, *dst = buf + s;
    // runs of kBlockSortMax sorted in shared memory, written back in place
    for (int r0 = 0; r0 < d; r0 += kBlockSortMax) {
      const int len = d - r0 < kBlockSortMax ? d - r0 : kBlockSortMax;
      const int P = pow2_ceil(len);
      for (int k = threadIdx.x; k < P; k += kSortThreadsL)
        sh[k] = k < len ? src[r0 + k] : kPosInf;
      __syncthreads();
      block_bitonic<kSortThreadsL>(sh, P);
      for (int k = threadIdx.x; k < len; k += kSortThreadsL) src[r0 + k] = sh[k];
      __syncthreads();
    }
    // merge rounds: runs of `run` -> runs of 2*run, src -> dst, swap
    for (int run = kBlockSortMax; run < d; run <<= 1) {
      for (int k = threadIdx.x; k < d; k += kSortThreadsL) {
        const int a0 = (k / (2 * run)) * (2 * run);
        const int b0 = a0 + run;
        const double x = src[k];
        int out;
        if (k < b0) {  // left run: partner is the right run (if any)
          const int lb = b0 < d ? (d - b0 < run ? d - b0 : run) : 0;
          out = k + rank_in<true>(src + b0, lb, x);
        } else {       // right run: ties go after the left run's equals
          out = a0 + (k - b0) + rank_in<false>(src + a0, run, x);
        }
        dst[out] = x;
      }
      __syncthreads();
      double *t = src;
      src = dst;
      dst = t;
    }
    const double g = block_min_gap<kSortThreadsL>(src, d, red);
    if (threadIdx.x == 0) dv[v] = vertex_dev(g, src[0], src[d - 1], d);
    __syncthreads();
  }
}

// Sum of d_v and count over vertices of degree >= 1 (fixed grid: deterministic).
__global__ void __launch_bounds__(kRedThreads)
dv_sum_kernel(const double *__restrict__ dv, const int *__restrict__ offs, int64_t n,
              double *__restrict__ part_sum, unsigned long long *__restrict__ part_cnt) {
  __shared__ double sh[kRedThreads / 32];
  __shared__ unsigned long long shc[kRedThreads / 32];
  double acc = 0.0;
  unsigned long long cnt = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    if (offs[v + 1] > offs[v]) {
      acc = __dadd_rn(acc, dv[v]);
      cnt += 1;
    }
  }
  double bs = block_sum<kRedThreads>(acc, sh);
  unsigned long long bc = block_sum_u64<kRedThreads>(cnt, shc);
  if (threadIdx.x == 0) {
    part_sum[blockIdx.x] = bs;
    part_cnt[blockIdx.x] = bc;
  }
}

__global__ void ma_finalize_kernel(const double *part_sum, const unsigned long long *part_cnt,
                                   int nb, double *out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    unsigned long long c = 0;
    for (int i = 0; i < nb; ++i) c += part_cnt[i];
    const double s = kahan_sum(part_sum, nb);
    out[0] = s;
    out[1] = (double)c;
    out[2] = 1.0 - s / (double)c;
  }
}

int reduce_grid(int64_t work) {
  int64_t g = (work + kRedThreads - 1) / kRedThreads;
  const int64_t cap = (int64_t)sm_count() * 4;
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace
}  // namespace glr

extern "C" {

int glr_edge_length_variation(const double *d_xy, int64_t n, const int64_t *d_edges, int64_t m,
                              double *d_out, void *stream) {
  using namespace glr;
  cudaStream_t st = as_stream(stream);
  if (d_out == nullptr || m < 0 || n < 0 || (m > 0 && (d_xy == nullptr || d_edges == nullptr))) {
    set_error("glr_edge_length_variation: invalid arguments");
    return GLR_EARG;
  }
  if (m <= 1) {
    set_value_kernel<<<1, 1, 0, st>>>(d_out, 0.0, 0.0, 0.0);
    GLR_LAUNCHED("set_value_kernel");
    return GLR_OK;
  }
  const int nb = reduce_grid(m);
  Scratch scr((size_t)m * sizeof(double) + (size_t)(2 * nb + 1) * sizeof(double), st);
  GLR_CUDA(scr.err);
  double *len = scr.as<double>();
  double *part = len + m;
  double *part2 = part + nb;
  double *mean = part2 + nb;
  lengths_kernel<<<nb, kRedThreads, 0, st>>>(reinterpret_cast<const double2 *>(d_xy),
                                             reinterpret_cast<const longlong2 *>(d_edges), m, len,
                                             part);
  GLR_LAUNCHED("lengths_kernel");
  mean_kernel<<<1, 32, 0, st>>>(part, nb, m, mean);
  GLR_LAUNCHED("mean_kernel");
  sqdev_kernel<<<nb, kRedThreads, 0, st>>>(len, m, mean, part2);
  GLR_LAUNCHED("sqdev_kernel");
  ml_finalize_kernel<<<1, 32, 0, st>>>(part2, nb, m, mean, d_out);
  GLR_LAUNCHED("ml_finalize_kernel");
  return GLR_OK;
}

int glr_minimum_angle(const double *d_xy, int64_t n, const int64_t *d_edges, int64_t m,
                      double *d_out, void *stream) {
  using namespace glr;
  cudaStream_t st = as_stream(stream);
  if (d_out == nullptr || m < 0 || n < 0 || (m > 0 && (d_xy == nullptr || d_edges == nullptr))) {
    set_error("glr_minimum_angle: invalid arguments");
    return GLR_EARG;
  }
  if (m == 0) {
    set_value_kernel<<<1, 1, 0, st>>>(d_out, 0.0, 0.0, 1.0);
    GLR_LAUNCHED("set_value_kernel");
    return GLR_OK;
  }
  if (2 * m >= (int64_t)1 << 31 || n >= (int64_t)1 << 31) {
    set_error("glr_minimum_angle: graph too large for 32-bit offsets");
    return GLR_EARG;
  }
  const int64_t na = 2 * m;
  const int64_t ntiles = (n + 1 + kScanTile - 1) / kScanTile;
  const int nb = reduce_grid(n);
  auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
  const size_t b_deg = al((size_t)(n + 1) * sizeof(int));
  const size_t b_ang = al((size_t)na * sizeof(double));
  const size_t b_dv = al((size_t)n * sizeof(double));
  const size_t b_part = al((size_t)nb * (sizeof(double) + sizeof(unsigned long long)));
  const size_t b_tile = al((size_t)ntiles * sizeof(int));
  // deg | offs | cursor | listB | listL | counts | ang | buf | dv | partials | tile sums
  Scratch scr(5 * b_deg + 256 + 2 * b_ang + b_dv + b_part + b_tile, st);
  GLR_CUDA(scr.err);
  char *p = scr.as<char>();
  int *deg = reinterpret_cast<int *>(p);
  int *offs = reinterpret_cast<int *>(p + b_deg);
  int *cursor = reinterpret_cast<int *>(p + 2 * b_deg);
  int *listB = reinterpret_cast<int *>(p + 3 * b_deg);
  int *listL = reinterpret_cast<int *>(p + 4 * b_deg);
  int *counts = reinterpret_cast<int *>(p + 5 * b_deg);
  p += 5 * b_deg + 256;
  double *ang = reinterpret_cast<double *>(p);
  double *buf = reinterpret_cast<double *>(p + b_ang);
  double *dv = reinterpret_cast<double *>(p + 2 * b_ang);
  double *part_sum = reinterpret_cast<double *>(p + 2 * b_ang + b_dv);
  unsigned long long *part_cnt = reinterpret_cast<unsigned long long *>(part_sum + nb);
  int *tile_sum = reinterpret_cast<int *>(p + 2 * b_ang + b_dv + b_part);

  GLR_CUDA(cudaMemsetAsync(deg, 0, (size_t)(n + 1) * sizeof(int), st));
  GLR_CUDA(cudaMemsetAsync(cursor, 0, (size_t)(n + 1) * sizeof(int), st));
  GLR_CUDA(cudaMemsetAsync(counts, 0, 2 * sizeof(int), st));
  const longlong2 *E = reinterpret_cast<const longlong2 *>(d_edges);
  const double2 *XY = reinterpret_cast<const double2 *>(d_xy);
  degree_kernel<<<reduce_grid(m), kRedThreads, 0, st>>>(E, m, deg);
  GLR_LAUNCHED("degree_kernel");
  scan_tiles_kernel<<<(unsigned)ntiles, 256, 0, st>>>(deg, n + 1, tile_sum);
  GLR_LAUNCHED("scan_tiles_kernel");
  scan_totals_kernel<<<1, 256, 0, st>>>(tile_sum, (int)ntiles);
  GLR_LAUNCHED("scan_totals_kernel");
  scan_apply_kernel<<<(unsigned)ntiles, 256, 0, st>>>(deg, n + 1, tile_sum, offs);
  GLR_LAUNCHED("scan_apply_kernel");
  scatter_angles_kernel<<<reduce_grid(na), kRedThreads, 0, st>>>(XY, E, m, offs, cursor, ang);
  GLR_LAUNCHED("scatter_angles_kernel");
  sort_small_kernel<<<reduce_grid(n * 32), 256, 0, st>>>(ang, offs, n, dv, listB, listL, counts);
  GLR_LAUNCHED("sort_small_kernel");
  sort_block_kernel<<<sm_count() * 4, kSortThreadsB, 0, st>>>(ang, offs, listB, counts, dv);
  GLR_LAUNCHED("sort_block_kernel");
  sort_large_kernel<<<sm_count(), kSortThreadsL, 0, st>>>(ang, buf, offs, listL, counts, dv);
  GLR_LAUNCHED("sort_large_kernel");
  dv_sum_kernel<<<nb, kRedThreads, 0, st>>>(dv, offs, n, part_sum, part_cnt);
  GLR_LAUNCHED("dv_sum_kernel");
  ma_finalize_kernel<<<1, 32, 0, st>>>(part_sum, part_cnt, nb, d_out);
  GLR_LAUNCHED("ma_finalize_kernel");
  return GLR_OK;
}

}  // extern "C"
