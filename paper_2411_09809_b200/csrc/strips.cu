// Strip-sweep approximations of E_c and E_ca:
// the reference's edge_crossing_enhanced / crossing_angle_stats
// (metrics/enhanced.py:133-300) and their per-strip sweeps
// (metrics/sweep.py:60-402), for one strip orientation.
//
// Strips (enhanced.py:133-215): the host builds the boundaries exactly as
// build_strips does and passes them in; here each edge, oriented so its
// sweep-axis coordinate increases, contributes one segment to every strip it
// spans (kf = searchsorted(bounds, sx0, 'left'), kl = searchsorted(bounds,
// sx1, 'right') - 1), with l / r its ordinates at the strip's boundaries
// (sy0 + slope * (bound - sx0), slope = (sy1 - sy0) / (sx1 - sx0)) and theta
// its axis angle in the sweep frame.
//
// Count (sweep.py:60-108): inside a strip two segments cross when their l-
// and r-orders disagree.  The reference sweeps by (l, r) and counts earlier
// segments with strictly greater r; the same number is computed here as the
// inversions of the r sequence of the (strip, l, r)-sorted segments by
// bottom-up merge passes (every element finds its rank in the sibling run by
// binary search: O(S log^2 S) work, fully parallel, exact integers).
//
// Deviation (sweep.py:110-402): the reference totals |ideal - a_c| over the
// same pairs through eight angle categories and a 2-D range structure; here
// the inverted pairs of each strip are enumerated on the device (tile pairs
// of the sorted strip, a pair (a < b) is inverted iff r_a > r_b) and
// |ideal - min(d, pi - d)| is accumulated per pair (equal to the category
// algebra up to rounding: reals are compared at 1e-9).
#include <cub/cub.cuh>

#include <vector>

#include "common.cuh"

namespace glr {
namespace {

constexpr int kSegTile = 256;
constexpr int kSegThreads = 256;

__device__ inline double mod_pi_dev(double x) {
  const double PI = 3.141592653589793;
  double r = fmod(x, PI);
  if (r != 0.0) {
    if (r < 0.0) r = __dadd_rn(r, PI);
  } else {
    r = 0.0;
  }
  return r;
}

// number of bounds < v (searchsorted 'left') / <= v ('right')
__device__ inline int64_t ss_left(const double *b, int64_t len, double v) {
  int64_t lo = 0, hi = len;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (b[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}
__device__ inline int64_t ss_right(const double *b, int64_t len, double v) {
  int64_t lo = 0, hi = len;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (b[mid] <= v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

struct EdgeFrame {
  double sx0, sy0, sx1, sy1;
  int64_t kf, kl;
};

__device__ inline EdgeFrame edge_frame(const double2 *xy, longlong2 uv, int axis,
                                       const double *bounds, int64_t nb) {
  const double2 p = xy[uv.x], q = xy[uv.y];
  const double x0 = axis ? p.y : p.x, y0 = axis ? p.x : p.y;
  const double x1 = axis ? q.y : q.x, y1 = axis ? q.x : q.y;
  const bool swap = x1 < x0;
  EdgeFrame f;
  f.sx0 = swap ? x1 : x0;
  f.sy0 = swap ? y1 : y0;
  f.sx1 = swap ? x0 : x1;
  f.sy1 = swap ? y0 : y1;
  f.kf = ss_left(bounds, nb, f.sx0);
  f.kl = ss_right(bounds, nb, f.sx1) - 1;
  return f;
}

__global__ void seg_count_kernel(const double2 *__restrict__ xy,
                                 const longlong2 *__restrict__ edges, int64_t m,
                                 const double *__restrict__ bounds, int64_t nb, int axis,
                                 long long *__restrict__ cnt) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    const EdgeFrame f = edge_frame(xy, edges[e], axis, bounds, nb);
    cnt[e] = f.kl > f.kf ? f.kl - f.kf : 0;
  }
}

// keys are made sign-canonical (x + 0.0 turns -0.0 into +0.0) so the radix
// sort orders equal values as ties, like numpy's lexsort
__global__ void seg_fill_kernel(const double2 *__restrict__ xy,
                                const longlong2 *__restrict__ edges, int64_t m,
                                const double *__restrict__ bounds, int64_t nb, int axis,
                                const long long *__restrict__ offs, int *__restrict__ strip,
                                double *__restrict__ lv, double *__restrict__ rv,
                                double *__restrict__ th, int with_angle) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    const EdgeFrame f = edge_frame(xy, edges[e], axis, bounds, nb);
    if (f.kl <= f.kf) continue;
    const double slope = __ddiv_rn(__dsub_rn(f.sy1, f.sy0), __dsub_rn(f.sx1, f.sx0));
    const double theta =
        with_angle ? mod_pi_dev(atan2(__dsub_rn(f.sy1, f.sy0), __dsub_rn(f.sx1, f.sx0))) : 0.0;
    int64_t q = offs[e];
    for (int64_t k = f.kf; k < f.kl; ++k, ++q) {
      strip[q] = (int)k;
      lv[q] = __dadd_rn(__dadd_rn(f.sy0, __dmul_rn(slope, __dsub_rn(bounds[k], f.sx0))), 0.0);
      rv[q] =
          __dadd_rn(__dadd_rn(f.sy0, __dmul_rn(slope, __dsub_rn(bounds[k + 1], f.sx0))), 0.0);
      th[q] = theta;
    }
  }
}

__global__ void gather_d_kernel(const int *__restrict__ idx, const double *__restrict__ src,
                                double *__restrict__ dst, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[idx[i]];
}
__global__ void gather_i_kernel(const int *__restrict__ idx, const int *__restrict__ src,
                                int *__restrict__ dst, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[idx[i]];
}
__global__ void iota_kernel(int *__restrict__ v, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    v[i] = (int)i;
}

// soffs[k] = first sorted position of strip k (lower_bound), k = 0..ns
__global__ void strip_offsets_kernel(const int *__restrict__ strip, int64_t S, int64_t ns,
                                     long long *__restrict__ soffs) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k <= ns;
       k += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = S;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (strip[mid] < k) lo = mid + 1; else hi = mid;
    }
    soffs[k] = lo;
  }
}

__device__ inline int64_t upper_bound_d(const double *a, int64_t lo, int64_t hi, double v) {
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] <= v) lo = mid + 1; else hi = mid;
  }
  return lo;
}
__device__ inline int64_t lower_bound_d(const double *a, int64_t lo, int64_t hi, double v) {
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// One bottom-up merge pass over runs of width w inside each strip: every
// right-run element counts the left-run elements strictly greater than it
// (the inversions between the two runs), and every element moves to its
// place in the merged run (stable: left before right on ties).
__global__ void __launch_bounds__(kSegThreads)
merge_pass_kernel(const double *__restrict__ a, double *__restrict__ b,
                  const int *__restrict__ strip, const long long *__restrict__ soffs,
                  int64_t S, int64_t w, unsigned long long *__restrict__ inv) {
  unsigned long long local = 0;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < S;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int k = strip[q];
    const int64_t s0 = soffs[k], N = soffs[k + 1] - s0, t = q - s0;
    const int64_t p0 = (t / (2 * w)) * (2 * w);  // pair start (local)
    const int64_t l0 = s0 + p0, l1 = s0 + (p0 + w < N ? p0 + w : N);
    const int64_t r0 = l1, r1 = s0 + (p0 + 2 * w < N ? p0 + 2 * w : N);
    const double v = a[q];
    int64_t out;
    if (q < l1) {  // left run
      out = l0 + (q - l0) + (lower_bound_d(a, r0, r1, v) - r0);
    } else {  // right run
      const int64_t le = upper_bound_d(a, l0, l1, v) - l0;  // left elements <= v
      local += (unsigned long long)((l1 - l0) - le);
      out = l0 + (q - r0) + le;
    }
    b[out] = v;
  }
  for (int o = 16; o > 0; o >>= 1) local += __shfl_down_sync(0xffffffffu, local, o);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(inv, local);
}

// Deviation over the inverted pairs: units are (strip, ti <= tj) tile pairs
// of the sorted strips, enumerated through the per-strip unit prefix uoffs.
__device__ inline double dev_term(double t1, double t2, double kappa) {
  const double HALF_PI = 1.5707963267948966;
  const double d = __dsub_rn(t1, t2);
  const double e = __dsub_rn(HALF_PI, fabs(d));
  return fabs(__dsub_rn(fabs(e), kappa));
}

__global__ void __launch_bounds__(kSegTile)
strip_dev_kernel(const double *__restrict__ rs, const double *__restrict__ ths,
                 const long long *__restrict__ soffs, const long long *__restrict__ uoffs,
                 int64_t ns, double kappa, unsigned long long *__restrict__ cta_cnt,
                 double *__restrict__ cta_dev) {
  __shared__ double sr[kSegTile], st[kSegTile];
  __shared__ unsigned long long red_u[kSegTile / 32];
  __shared__ double red_d[kSegTile / 32];
  const uint64_t U = (uint64_t)uoffs[ns];
  unsigned long long cnt = 0;
  double dsum = 0.0, dcomp = 0.0;
  for (uint64_t u = blockIdx.x; u < U; u += gridDim.x) {
    int64_t lo = 0, hi = ns;  // strip k: uoffs[k] <= u < uoffs[k+1]
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if ((uint64_t)uoffs[mid] <= u) lo = mid; else hi = mid - 1;
    }
    const int64_t k = lo, s0 = soffs[k], N = soffs[k + 1] - s0;
    const uint64_t T = (uint64_t)((N + kSegTile - 1) / kSegTile);
    uint64_t ti, tj;
    tri_unit_coords(u - (uint64_t)uoffs[k], T, &ti, &tj);
    __syncthreads();
    const int64_t jb = (int64_t)tj * kSegTile;
    const int jn = (int)(N - jb < kSegTile ? N - jb : kSegTile);
    if ((int)threadIdx.x < jn) {
      sr[threadIdx.x] = rs[s0 + jb + threadIdx.x];
      st[threadIdx.x] = ths[s0 + jb + threadIdx.x];
    }
    __syncthreads();
    const int64_t i = (int64_t)ti * kSegTile + threadIdx.x;
    double s = 0.0;
    if (i < N) {
      const double ri = rs[s0 + i], thi = ths[s0 + i];
      const int j0 = ti == tj ? (int)threadIdx.x + 1 : 0;
      for (int jj = j0; jj < jn; ++jj) {
        if (ri > sr[jj]) {  // i before j in (l, r) order, r_i > r_j
          ++cnt;
          s = __dadd_rn(s, dev_term(thi, st[jj], kappa));
        }
      }
    }
    const double y = __dsub_rn(s, dcomp);
    const double t = __dadd_rn(dsum, y);
    dcomp = __dsub_rn(__dsub_rn(t, dsum), y);
    dsum = t;
  }
  const unsigned long long bc = block_sum_u64<kSegTile>(cnt, red_u);
  const double bd = block_sum<kSegTile>(dsum, red_d);
  if (threadIdx.x == 0) {
    cta_cnt[blockIdx.x] = bc;
    cta_dev[blockIdx.x] = bd;
  }
}

__global__ void strip_finalize_kernel(const unsigned long long *__restrict__ inv,
                                      const unsigned long long *__restrict__ cta_cnt,
                                      const double *__restrict__ cta_dev, int ncta,
                                      int with_angle, double *__restrict__ out,
                                      int *__restrict__ mismatch) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    out[0] = (double)inv[0];
    if (with_angle) {
      unsigned long long c = 0;
      for (int i = 0; i < ncta; ++i) c += cta_cnt[i];
      out[1] = kahan_sum(cta_dev, ncta);
      *mismatch = c != inv[0];
    } else {
      out[1] = 0.0;
      *mismatch = 0;
    }
  }
}

int blocks_s(int64_t work, int nt, int per_sm) {
  int64_t b = (work + nt - 1) / nt;
  const int64_t cap = (int64_t)sm_count() * per_sm;
  if (b > cap) b = cap;
  return (int)(b < 1 ? 1 : b);
}

}  // namespace

int strip_crossings(const double *d_xy, int64_t n, const int64_t *d_edges, int64_t m,
                    const double *d_bounds, int64_t nstrips, int axis, int with_angle,
                    double ideal, double *d_out, cudaStream_t st) {
  if (d_xy == nullptr || d_edges == nullptr || d_bounds == nullptr || d_out == nullptr ||
      n < 0 || m < 0 || nstrips < 1 || (axis != 0 && axis != 1)) {
    set_error("glr_strip_crossings: invalid arguments");
    return GLR_EARG;
  }
  if (with_angle && !(ideal > 0.0 && ideal <= 1.5707963267948966)) {
    set_error("glr_strip_crossings: ideal angle must lie in (0, pi/2], got %g", ideal);
    return GLR_EARG;
  }
  if (m >= ((int64_t)1 << 31) || nstrips >= ((int64_t)1 << 31)) {
    set_error("glr_strip_crossings: m or nstrips exceeds the 32-bit range");
    return GLR_EARG;
  }
  const int nt = 256;
  const int64_t nb = nstrips + 1;
  const double2 *xy = reinterpret_cast<const double2 *>(d_xy);
  const longlong2 *ed = reinterpret_cast<const longlong2 *>(d_edges);
  // 1. segments per edge, prefix
  size_t t_scan = 0;
  GLR_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t_scan, (long long *)nullptr,
                                         (long long *)nullptr, (int)(m + 1), st));
  Scratch s1((size_t)(m + 1) * 2 * sizeof(long long) + t_scan + 256, st);
  GLR_CUDA(s1.err);
  long long *cnt = s1.as<long long>();
  long long *offs = cnt + (m + 1);
  void *tmp1 = offs + (m + 1);
  GLR_CUDA(cudaMemsetAsync(cnt + m, 0, sizeof(long long), st));
  if (m > 0) {
    seg_count_kernel<<<blocks_s(m, nt, 8), nt, 0, st>>>(xy, ed, m, d_bounds, nb, axis, cnt);
    GLR_LAUNCHED("seg_count_kernel");
  }
  size_t tb = t_scan;
  GLR_CUDA(cub::DeviceScan::ExclusiveSum(tmp1, tb, cnt, offs, (int)(m + 1), st));
  count_launch(2);
  long long S = 0;
  GLR_CUDA(cudaMemcpyAsync(&S, offs + m, sizeof(S), cudaMemcpyDeviceToHost, st));
  GLR_CUDA(cudaStreamSynchronize(st));
  if (S >= ((long long)1 << 31)) {
    set_error("glr_strip_crossings: %lld strip segments exceed the 32-bit range", S);
    return GLR_EARG;
  }
  if (S < 2) {
    GLR_CUDA(cudaMemsetAsync(d_out, 0, 2 * sizeof(double), st));
    return GLR_OK;
  }
  // 2. segments, sorted by (strip, l, r): stable radix sorts by r, l, strip
  size_t t_d = 0, t_i = 0;
  GLR_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, t_d, (const double *)nullptr,
                                           (double *)nullptr, (const int *)nullptr,
                                           (int *)nullptr, (int)S, 0, 64, st));
  GLR_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, t_i, (const int *)nullptr, (int *)nullptr,
                                           (const int *)nullptr, (int *)nullptr, (int)S, 0, 32,
                                           st));
  const size_t t_sort = t_d > t_i ? t_d : t_i;
  const size_t aS8 = ((size_t)S * 8 + 255) & ~(size_t)255, aS4 = ((size_t)S * 4 + 255) & ~(size_t)255;
  const size_t a_soffs = (((size_t)nb + 1) * 8 + 255) & ~(size_t)255;
  Scratch s2(6 * aS8 + 4 * aS4 + 2 * a_soffs + t_sort + 256, st);
  GLR_CUDA(s2.err);
  char *p = s2.as<char>();
  double *lv = reinterpret_cast<double *>(p); p += aS8;
  double *rv = reinterpret_cast<double *>(p); p += aS8;
  double *th = reinterpret_cast<double *>(p); p += aS8;
  double *kd0 = reinterpret_cast<double *>(p); p += aS8;
  double *kd1 = reinterpret_cast<double *>(p); p += aS8;
  double *kd2 = reinterpret_cast<double *>(p); p += aS8;
  int *strip = reinterpret_cast<int *>(p); p += aS4;
  int *perm0 = reinterpret_cast<int *>(p); p += aS4;
  int *perm1 = reinterpret_cast<int *>(p); p += aS4;
  int *ki = reinterpret_cast<int *>(p); p += aS4;
  long long *soffs = reinterpret_cast<long long *>(p); p += a_soffs;
  long long *uoffs = reinterpret_cast<long long *>(p); p += a_soffs;
  unsigned long long *inv = reinterpret_cast<unsigned long long *>(p); p += 256;
  void *tmp2 = p;
  seg_fill_kernel<<<blocks_s(m, nt, 8), nt, 0, st>>>(xy, ed, m, d_bounds, nb, axis, offs, strip,
                                                     lv, rv, th, with_angle);
  GLR_LAUNCHED("seg_fill_kernel");
  const int gS = blocks_s(S, nt, 16);
  iota_kernel<<<gS, nt, 0, st>>>(perm0, S);
  GLR_LAUNCHED("iota_kernel");
  // by r
  tb = t_sort;
  GLR_CUDA(cub::DeviceRadixSort::SortPairs(tmp2, tb, rv, kd0, perm0, perm1, (int)S, 0, 64, st));
  count_launch(4);
  // by l (stable), keys gathered through the current permutation
  gather_d_kernel<<<gS, nt, 0, st>>>(perm1, lv, kd1, S);
  GLR_LAUNCHED("gather_d_kernel");
  tb = t_sort;
  GLR_CUDA(cub::DeviceRadixSort::SortPairs(tmp2, tb, kd1, kd2, perm1, perm0, (int)S, 0, 64, st));
  count_launch(4);
  // by strip (stable)
  gather_i_kernel<<<gS, nt, 0, st>>>(perm0, strip, ki, S);
  GLR_LAUNCHED("gather_i_kernel");
  tb = t_sort;
  GLR_CUDA(cub::DeviceRadixSort::SortPairs(tmp2, tb, ki, perm1 /* sorted strip ids */, perm0,
                                           reinterpret_cast<int *>(kd1) /* final perm */, (int)S,
                                           0, 32, st));
  count_launch(4);
  int *sstrip = perm1;
  int *perm = reinterpret_cast<int *>(kd1);
  double *rs = kd0, *ths = kd2;
  gather_d_kernel<<<gS, nt, 0, st>>>(perm, rv, rs, S);
  GLR_LAUNCHED("gather_d_kernel");
  gather_d_kernel<<<gS, nt, 0, st>>>(perm, th, ths, S);
  GLR_LAUNCHED("gather_d_kernel");
  strip_offsets_kernel<<<blocks_s(nb + 1, nt, 4), nt, 0, st>>>(sstrip, S, nstrips, soffs);
  GLR_LAUNCHED("strip_offsets_kernel");
  // host copy of strip offsets: sizes the passes and the deviation units
  std::vector<long long> h_soffs((size_t)nb);
  GLR_CUDA(cudaMemcpyAsync(h_soffs.data(), soffs, sizeof(long long) * nb,
                           cudaMemcpyDeviceToHost, st));
  GLR_CUDA(cudaStreamSynchronize(st));
  long long maxN = 0;
  std::vector<long long> h_uoffs((size_t)nb);
  h_uoffs[0] = 0;
  for (int64_t k = 0; k < nstrips; ++k) {
    const long long N = h_soffs[k + 1] - h_soffs[k];
    if (N > maxN) maxN = N;
    const long long T = (N + kSegTile - 1) / kSegTile;
    h_uoffs[k + 1] = h_uoffs[k] + T * (T + 1) / 2;
  }
  // 3. deviation over inverted pairs (before the merge passes reorder r)
  const int dgrid = sm_count() * 8;
  Scratch s3((size_t)dgrid * (sizeof(unsigned long long) + sizeof(double)) + 256, st);
  GLR_CUDA(s3.err);
  unsigned long long *cc = s3.as<unsigned long long>();
  double *cd = reinterpret_cast<double *>(cc + dgrid);
  int *mismatch = reinterpret_cast<int *>(cd + dgrid);
  if (with_angle) {
    GLR_CUDA(cudaMemcpyAsync(uoffs, h_uoffs.data(), sizeof(long long) * nb,
                             cudaMemcpyHostToDevice, st));
    strip_dev_kernel<<<dgrid, kSegTile, 0, st>>>(rs, ths, soffs, uoffs, nstrips,
                                                 1.5707963267948966 - ideal, cc, cd);
    GLR_LAUNCHED("strip_dev_kernel");
  }
  // 4. inversion count: merge passes of the r sequence (ping-pong rs / lv)
  GLR_CUDA(cudaMemsetAsync(inv, 0, sizeof(unsigned long long), st));
  double *a = rs, *b = lv;
  for (int64_t w = 1; w < maxN; w *= 2) {
    merge_pass_kernel<<<gS, kSegThreads, 0, st>>>(a, b, sstrip, soffs, S, w, inv);
    GLR_LAUNCHED("merge_pass_kernel");
    double *t = a;
    a = b;
    b = t;
  }
  strip_finalize_kernel<<<1, 32, 0, st>>>(inv, cc, cd, dgrid, with_angle, d_out, mismatch);
  GLR_LAUNCHED("strip_finalize_kernel");
  int h_mis = 0;
  GLR_CUDA(cudaMemcpyAsync(&h_mis, mismatch, sizeof(int), cudaMemcpyDeviceToHost, st));
  GLR_CUDA(cudaStreamSynchronize(st));
  if (h_mis) {  // sweep.py:396-399 cross-checks its two counts the same way
    set_error("glr_strip_crossings: pair enumeration and inversion count disagree");
    return GLR_EINVARIANT;
  }
  return GLR_OK;
}

}  // namespace glr

extern "C" int glr_strip_crossings(const double *d_xy, int64_t n, const int64_t *d_edges,
                                   int64_t m, const double *d_bounds, int64_t nstrips, int axis,
                                   int with_angle, double ideal, double *d_out, void *stream) {
  return glr::strip_crossings(d_xy, n, d_edges, m, d_bounds, nstrips, axis, with_angle, ideal,
                              d_out, glr::as_stream(stream));
}
