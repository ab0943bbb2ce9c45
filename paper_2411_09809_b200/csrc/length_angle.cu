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
// segment is sorted (CUB segmented radix sort; library primitive, this is not
// the all-pairs hot path), then one warp per vertex takes the minimum
// consecutive gap and the wrap gap (2pi - last) + first, d_v = (phi - gap)/phi
// with phi = 2pi/deg, and M_a = 1 - mean(d_v) over vertices of degree >= 1.
#include <cub/cub.cuh>

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

__global__ void degree_kernel(const longlong2 *__restrict__ edges, int64_t m, int *deg) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    longlong2 uv = edges[e];
    atomicAdd(&deg[uv.x], 1);
    atomicAdd(&deg[uv.y], 1);
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
    double a = atan2(__dsub_rn(pu.y, pv.y), __dsub_rn(pu.x, pv.x));
    if (a < 0.0) a = __dadd_rn(a, kTwoPi);
    int slot = offs[v] + atomicAdd(&cursor[v], 1);
    ang[slot] = a;
  }
}

// One warp per vertex: min consecutive gap of the sorted segment and the
// wrap gap; per-block partial sums of d_v and of the vertex count.
__global__ void __launch_bounds__(kRedThreads)
vertex_gap_kernel(const double *__restrict__ ang, const int *__restrict__ offs, int64_t n,
                  double *__restrict__ part_sum, unsigned long long *__restrict__ part_cnt) {
  __shared__ double sh[kRedThreads / 32];
  __shared__ unsigned long long shc[kRedThreads / 32];
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double acc = 0.0;
  unsigned long long cnt = 0;
  for (int64_t v = warp; v < n; v += nwarps) {
    const int s = offs[v], e = offs[v + 1];
    const int d = e - s;
    if (d == 0) continue;
    double g = __longlong_as_double(0x7ff0000000000000ll);  // +inf
    for (int p = s + lane; p + 1 < e; p += 32) g = fmin(g, __dsub_rn(ang[p + 1], ang[p]));
    for (int o = 16; o > 0; o >>= 1) g = fmin(g, __shfl_xor_sync(0xffffffffu, g, o));
    if (lane == 0) {
      const double wrap = __dadd_rn(__dsub_rn(kTwoPi, ang[e - 1]), ang[s]);
      const double gap = fmin(g, wrap);
      const double phi = kTwoPi / (double)d;
      acc = __dadd_rn(acc, __ddiv_rn(__dsub_rn(phi, gap), phi));
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
  size_t scan_bytes = 0, sort_bytes = 0;
  GLR_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (int *)nullptr, (int *)nullptr,
                                         (int)(n + 1), st));
  GLR_CUDA(cub::DeviceSegmentedSort::SortKeys(nullptr, sort_bytes, (const double *)nullptr,
                                              (double *)nullptr, (int)na, (int)n,
                                              (const int *)nullptr, (const int *)nullptr, st));
  const int nb = reduce_grid(n * 32);
  auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
  const size_t b_deg = al((size_t)(n + 1) * sizeof(int));
  const size_t b_ang = al((size_t)na * sizeof(double));
  const size_t b_part = al((size_t)nb * (sizeof(double) + sizeof(unsigned long long)));
  const size_t b_tmp = al(scan_bytes > sort_bytes ? scan_bytes : sort_bytes);
  Scratch scr(3 * b_deg + 2 * b_ang + b_part + b_tmp, st);
  GLR_CUDA(scr.err);
  char *p = scr.as<char>();
  int *deg = reinterpret_cast<int *>(p);
  int *offs = reinterpret_cast<int *>(p + b_deg);
  int *cursor = reinterpret_cast<int *>(p + 2 * b_deg);
  double *ang = reinterpret_cast<double *>(p + 3 * b_deg);
  double *sorted = reinterpret_cast<double *>(p + 3 * b_deg + b_ang);
  double *part_sum = reinterpret_cast<double *>(p + 3 * b_deg + 2 * b_ang);
  unsigned long long *part_cnt = reinterpret_cast<unsigned long long *>(part_sum + nb);
  void *tmp = p + 3 * b_deg + 2 * b_ang + b_part;

  GLR_CUDA(cudaMemsetAsync(deg, 0, (size_t)(n + 1) * sizeof(int), st));
  GLR_CUDA(cudaMemsetAsync(cursor, 0, (size_t)(n + 1) * sizeof(int), st));
  const longlong2 *E = reinterpret_cast<const longlong2 *>(d_edges);
  const double2 *XY = reinterpret_cast<const double2 *>(d_xy);
  degree_kernel<<<reduce_grid(m), kRedThreads, 0, st>>>(E, m, deg);
  GLR_LAUNCHED("degree_kernel");
  size_t tb = scan_bytes;
  GLR_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, deg, offs, (int)(n + 1), st));
  count_launch(2);
  scatter_angles_kernel<<<reduce_grid(na), kRedThreads, 0, st>>>(XY, E, m, offs, cursor, ang);
  GLR_LAUNCHED("scatter_angles_kernel");
  tb = sort_bytes;
  GLR_CUDA(cub::DeviceSegmentedSort::SortKeys(tmp, tb, ang, sorted, (int)na, (int)n, offs,
                                              offs + 1, st));
  count_launch(3);
  vertex_gap_kernel<<<nb, kRedThreads, 0, st>>>(sorted, offs, n, part_sum, part_cnt);
  GLR_LAUNCHED("vertex_gap_kernel");
  ma_finalize_kernel<<<1, 32, 0, st>>>(part_sum, part_cnt, nb, d_out);
  GLR_LAUNCHED("ma_finalize_kernel");
  return GLR_OK;
}

}  // extern "C"
