// Spatial (Morton / Z-order) reordering of edges and vertices, the first
// step of the culled variants.
//
// The exact metrics do not depend on the order of edges or vertices (the pair
// predicate is symmetric and every unordered pair is visited once, the
// adjacency correction uses the same indexing), so a permutation is free to
// choose.  Sorting vertices by the Morton code of the position, and edges by
// the 4-D Morton code of their bbox sides, makes each 1024- or 256-element
// tile spatially compact, so most tile pairs have disjoint tile bounding
// boxes and are skipped by the candidate lists built in occlusion.cu and
// crossing.cu.  The direction order (glr_theta_sort_edges) serves the dense
// crossing pass instead.  The permutation only affects speed, never results.
#include <cub/cub.cuh>

#include "common.cuh"

namespace glr {
namespace {

// order-preserving 64-bit key of a double (total order, -0 < +0)
__device__ inline unsigned long long dkey(double v) {
  unsigned long long b = (unsigned long long)__double_as_longlong(v);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ inline double dunkey(unsigned long long k) {
  unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)b);
}

// global [xmin, xmax] x [ymin, ymax] of the coordinates as order-preserving keys
__global__ void bounds_kernel(const double2 *__restrict__ xy, int64_t n, unsigned long long *b) {
  unsigned long long x0 = ~0ull, x1 = 0, y0 = ~0ull, y1 = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double2 p = xy[i];
    const unsigned long long kx = dkey(p.x), ky = dkey(p.y);
    x0 = kx < x0 ? kx : x0;
    x1 = kx > x1 ? kx : x1;
    y0 = ky < y0 ? ky : y0;
    y1 = ky > y1 ? ky : y1;
  }
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long a;
    a = __shfl_down_sync(0xffffffffu, x0, o); x0 = a < x0 ? a : x0;
    a = __shfl_down_sync(0xffffffffu, x1, o); x1 = a > x1 ? a : x1;
    a = __shfl_down_sync(0xffffffffu, y0, o); y0 = a < y0 ? a : y0;
    a = __shfl_down_sync(0xffffffffu, y1, o); y1 = a > y1 ? a : y1;
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&b[0], x0);
    atomicMax(&b[1], x1);
    atomicMin(&b[2], y0);
    atomicMax(&b[3], y1);
  }
}

__device__ inline unsigned spread16(unsigned v) {
  v &= 0xffffu;
  v = (v | (v << 8)) & 0x00ff00ffu;
  v = (v | (v << 4)) & 0x0f0f0f0fu;
  v = (v | (v << 2)) & 0x33333333u;
  v = (v | (v << 1)) & 0x55555555u;
  return v;
}

__device__ inline unsigned quant16(double v, double lo, double scale) {
  double q = (v - lo) * scale;  // scale = 65535 / (hi - lo), or 0 for a flat axis
  if (!(q >= 0.0)) q = 0.0;     // also catches NaN from inf - inf
  if (q > 65535.0) q = 65535.0;
  return (unsigned)q;
}

__device__ inline unsigned morton(double x, double y, const unsigned long long *b) {
  const double x0 = dunkey(b[0]), x1 = dunkey(b[1]), y0 = dunkey(b[2]), y1 = dunkey(b[3]);
  const double sx = (x1 > x0 && isfinite(x1 - x0)) ? 65535.0 / (x1 - x0) : 0.0;
  const double sy = (y1 > y0 && isfinite(y1 - y0)) ? 65535.0 / (y1 - y0) : 0.0;
  return spread16(quant16(x, x0, sx)) | (spread16(quant16(y, y0, sy)) << 1);
}

__global__ void degree_kernel(const longlong2 *__restrict__ e, int64_t m, int *deg) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const longlong2 uv = e[i];
    atomicAdd(&deg[uv.x], 1);
    atomicAdd(&deg[uv.y], 1);
  }
}

__global__ void edge_theta_keys_kernel(const double2 *__restrict__ xy,
                                       const longlong2 *__restrict__ e, int64_t m,
                                       const int *__restrict__ deg, int64_t hub_degree,
                                       unsigned long long *keys, int *idx) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const longlong2 uv = e[i];
    const double2 p = xy[uv.x], q = xy[uv.y];
    double t = atan2(q.y - p.y, q.x - p.x);
    if (t < 0.0) t += 3.141592653589793;
    double k = t * (4294967296.0 / 3.141592653589793);
    if (!(k >= 0.0)) k = 0.0;  // also NaN
    if (k > 4294967295.0) k = 4294967295.0;
    const int du = deg[uv.x], dv = deg[uv.y];
    const long long hub = (du >= dv) ? uv.x : uv.y;  // ties: the smaller index
    const unsigned long long grp =
        ((du > dv ? du : dv) >= hub_degree) ? (unsigned long long)hub + 1ull : 0ull;
    keys[i] = (grp << 32) | (unsigned long long)(unsigned)k;
    idx[i] = (int)i;
  }
}

// Crossing-cull order (glr_spatial_sort_edges): key = (hub group, 4-D
// Morton code of the bbox (xmin, xmax, ymin, ymax), 8 bits per axis,
// diagonal orientation).  Tiles of edges with similar extents on all four sides have
// tight tile boxes even for long edges (a 2-D centre key leaves long random
// edges' tiles spanning the domain), so glr_crossing_candidates can drop
// tile pairs whose boxes are disjoint -- on random long edges about half of
// them (C5: 60% of the tile pairs remain).  Hub groups keep shared-vertex
// pairs in star tiles.
__device__ inline unsigned long long spread8x4(unsigned v) {
  unsigned long long r = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) r |= (unsigned long long)((v >> i) & 1u) << (4 * i);
  return r;
}
__device__ inline unsigned quant8(double v, double lo, double scale) {
  double q = (v - lo) * scale;  // scale = 255 / (hi - lo), or 0 for a flat axis
  if (!(q >= 0.0)) q = 0.0;
  if (q > 255.0) q = 255.0;
  return (unsigned)q;
}
// Sum over edges of the quantised bbox half-perimeter (|dx| + |dy| on the
// 8-bit grid of the Morton code): integer atomics, so the order decision
// below is deterministic.
__global__ void edge_extent_kernel(const double2 *__restrict__ xy,
                                   const longlong2 *__restrict__ e, int64_t m,
                                   const unsigned long long *b, unsigned long long *lsum) {
  const double x0 = dunkey(b[0]), x1 = dunkey(b[1]), y0 = dunkey(b[2]), y1 = dunkey(b[3]);
  const double sx = (x1 > x0 && isfinite(x1 - x0)) ? 255.0 / (x1 - x0) : 0.0;
  const double sy = (y1 > y0 && isfinite(y1 - y0)) ? 255.0 / (y1 - y0) : 0.0;
  unsigned long long s = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const longlong2 uv = e[i];
    const double2 p = xy[uv.x], q = xy[uv.y];
    s += (unsigned long long)(quant8(fmax(p.x, q.x), x0, sx) - quant8(fmin(p.x, q.x), x0, sx)) +
         (unsigned long long)(quant8(fmax(p.y, q.y), y0, sy) - quant8(fmin(p.y, q.y), y0, sy));
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(lsum, s);
}

// mean quantised half-perimeter (of 510) from which edges count as long
#ifndef GLR_LONG_EDGE_EXTENT
#define GLR_LONG_EDGE_EXTENT 16
#endif

__global__ void edge_box_keys_kernel(const double2 *__restrict__ xy,
                                     const longlong2 *__restrict__ e, int64_t m,
                                     const unsigned long long *b, const int *__restrict__ deg,
                                     int64_t hub_degree, const unsigned long long *lsum,
                                     unsigned long long *keys, int *idx) {
  const double x0 = dunkey(b[0]), x1 = dunkey(b[1]), y0 = dunkey(b[2]), y1 = dunkey(b[3]);
  const double sx = (x1 > x0 && isfinite(x1 - x0)) ? 255.0 / (x1 - x0) : 0.0;
  const double sy = (y1 > y0 && isfinite(y1 - y0)) ? 255.0 / (y1 - y0) : 0.0;
  const bool long_edges = *lsum >= (unsigned long long)GLR_LONG_EDGE_EXTENT * (unsigned long long)m;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const longlong2 uv = e[i];
    const double2 p = xy[uv.x], q = xy[uv.y];
    const unsigned long long mk =
        spread8x4(quant8(fmin(p.x, q.x), x0, sx)) |
        (spread8x4(quant8(fmax(p.x, q.x), x0, sx)) << 1) |
        (spread8x4(quant8(fmin(p.y, q.y), y0, sy)) << 2) |
        (spread8x4(quant8(fmax(p.y, q.y), y0, sy)) << 3);
    const unsigned long long up = ((q.x - p.x) * (q.y - p.y) >= 0.0) ? 1ull : 0ull;
    const int du = deg[uv.x], dv = deg[uv.y];
    const long long hub = (du >= dv) ? uv.x : uv.y;
    const unsigned long long grp =
        ((du > dv ? du : dv) >= hub_degree) ? (unsigned long long)hub + 1ull : 0ull;
    // Long edges (mean bbox half-perimeter >= 1/32 of the grid's): the
    // orientation goes ABOVE the Morton code, so a tile holds one diagonal
    // orientation, its P (smaller-x) and Q endpoints form two compact boxes
    // and its theta range is narrow -- what tile_class_kernel needs to
    // certify whole units as crossing everywhere or nowhere, and what lets
    // the angle pass use the signed form (unit_shift).  It costs a little
    // bbox culling (C5: 55.7% vs 54.2% of the tile pairs remain), which the
    // certified classes repay (C5: ~15% of the remaining units certified
    // empty, ~10% full).  Short edges keep it below the Morton code: there a
    // top-level split gives every region tiles of both orientations (C3
    // culled units 22,229 vs 11,688).
    keys[i] = long_edges ? ((grp << 33) | (up << 32) | mk) : ((grp << 33) | (mk << 1) | up);
    idx[i] = (int)i;
  }
}

int theta_sort(const double *d_xy, int64_t n, const int64_t *d_edges, int64_t m,
               int64_t hub_degree, int64_t *d_out, cudaStream_t st);
// Hub degree of the culled (4-D bbox) order: a hub group's tiles have boxes
// anchored at the hub, so only hubs whose shared-vertex pairs would cost more
// fallbacks than their boxes cost candidate units get a group (C5 culled:
// 3.70 s at 256, 3.19 s at 1024, 2.98 s at 4096, 2.92 s at 16384, 3.05 s
// with none; tools/cull_probe.py).
#ifndef GLR_BOX_HUB_DEGREE
#define GLR_BOX_HUB_DEGREE 16384
#endif
int box_sort(const double *d_xy, int64_t n, const int64_t *d_edges, int64_t m,
             int64_t hub_degree, int64_t *d_out, cudaStream_t st);

__global__ void vertex_keys_kernel(const double2 *__restrict__ xy, int64_t n,
                                   const unsigned long long *b, unsigned *keys, int *idx) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double2 p = xy[i];
    keys[i] = morton(p.x, p.y, b);
    idx[i] = (int)i;
  }
}

__global__ void gather_edges_kernel(const longlong2 *__restrict__ e, const int *__restrict__ perm,
                                    int64_t m, longlong2 *out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = e[perm[i]];
}

__global__ void gather_xy_kernel(const double2 *__restrict__ xy, const int *__restrict__ perm,
                                 int64_t n, double2 *out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = xy[perm[i]];
}

int grid_of(int64_t work) {
  int64_t b = (work + 255) / 256;
  const int64_t cap = (int64_t)sm_count() * 16;
  if (b > cap) b = cap;
  return (int)(b < 1 ? 1 : b);
}

// Vertex order: bounds, Morton keys of the positions, stable radix sort of
// (key, index), gather.
int vertex_sort(const double *d_xy, int64_t n, double *d_out, cudaStream_t st) {
  if (n <= 1) {
    if (n == 1) GLR_CUDA(cudaMemcpyAsync(d_out, d_xy, 16, cudaMemcpyDeviceToDevice, st));
    return GLR_OK;
  }
  size_t t_sort = 0;
  GLR_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, t_sort, (const unsigned *)nullptr,
                                           (unsigned *)nullptr, (const int *)nullptr,
                                           (int *)nullptr, (int)n, 0, 32, st));
  const size_t a4 = ((size_t)n * 4 + 255) & ~(size_t)255;
  Scratch scr(4 * a4 + 256 + t_sort, st);
  GLR_CUDA(scr.err);
  char *p = scr.as<char>();
  unsigned *keys = reinterpret_cast<unsigned *>(p);
  unsigned *keys_out = reinterpret_cast<unsigned *>(p + a4);
  int *idx = reinterpret_cast<int *>(p + 2 * a4);
  int *perm = reinterpret_cast<int *>(p + 3 * a4);
  unsigned long long *b = reinterpret_cast<unsigned long long *>(p + 4 * a4);
  void *tmp = p + 4 * a4 + 256;
  // bound words: min keys start at ~0, max keys at 0 (memsets, no host staging)
  GLR_CUDA(cudaMemsetAsync(b, 0xff, 8, st));
  GLR_CUDA(cudaMemsetAsync(b + 1, 0x00, 8, st));
  GLR_CUDA(cudaMemsetAsync(b + 2, 0xff, 8, st));
  GLR_CUDA(cudaMemsetAsync(b + 3, 0x00, 8, st));
  bounds_kernel<<<grid_of(n), 256, 0, st>>>(reinterpret_cast<const double2 *>(d_xy), n, b);
  GLR_LAUNCHED("bounds_kernel");
  vertex_keys_kernel<<<grid_of(n), 256, 0, st>>>(reinterpret_cast<const double2 *>(d_xy), n, b,
                                                 keys, idx);
  GLR_LAUNCHED("vertex_keys_kernel");
  size_t tb = t_sort;
  GLR_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, keys, keys_out, idx, perm, (int)n, 0, 32, st));
  count_launch(4);
  gather_xy_kernel<<<grid_of(n), 256, 0, st>>>(reinterpret_cast<const double2 *>(d_xy), perm, n,
                                               reinterpret_cast<double2 *>(d_out));
  GLR_LAUNCHED("gather_xy_kernel");
  return GLR_OK;
}

template <bool BOX>
int keyed_sort(const double *d_xy, int64_t n, const int64_t *d_edges, int64_t m,
               int64_t hub_degree, int64_t *d_out, cudaStream_t st) {
  if (m <= 1) {
    if (m == 1) GLR_CUDA(cudaMemcpyAsync(d_out, d_edges, 16, cudaMemcpyDeviceToDevice, st));
    return GLR_OK;
  }
  const int low = BOX ? 33 : 32;  // key bits below the group
  int end_bit = low;
  while (end_bit < 64 && ((unsigned long long)(n + 1) >> (end_bit - low)) != 0) ++end_bit;
  size_t t_sort = 0;
  GLR_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, t_sort, (const unsigned long long *)nullptr,
                                           (unsigned long long *)nullptr, (const int *)nullptr,
                                           (int *)nullptr, (int)m, 0, end_bit, st));
  const size_t a8 = ((size_t)m * 8 + 255) & ~(size_t)255;
  const size_t a4 = ((size_t)m * 4 + 255) & ~(size_t)255;
  const size_t an = ((size_t)n * 4 + 255) & ~(size_t)255;
  Scratch scr(2 * a8 + 2 * a4 + an + 256 + t_sort, st);
  GLR_CUDA(scr.err);
  char *p = scr.as<char>();
  auto *keys = reinterpret_cast<unsigned long long *>(p);
  auto *keys_out = reinterpret_cast<unsigned long long *>(p + a8);
  int *idx = reinterpret_cast<int *>(p + 2 * a8);
  int *perm = reinterpret_cast<int *>(p + 2 * a8 + a4);
  int *deg = reinterpret_cast<int *>(p + 2 * a8 + 2 * a4);
  unsigned long long *b = reinterpret_cast<unsigned long long *>(p + 2 * a8 + 2 * a4 + an);
  void *tmp = p + 2 * a8 + 2 * a4 + an + 256;
  const auto *e2 = reinterpret_cast<const longlong2 *>(d_edges);
  GLR_CUDA(cudaMemsetAsync(deg, 0, (size_t)n * 4, st));
  degree_kernel<<<grid_of(m), 256, 0, st>>>(e2, m, deg);
  GLR_LAUNCHED("degree_kernel");
  if (BOX) {
    GLR_CUDA(cudaMemsetAsync(b, 0xff, 8, st));
    GLR_CUDA(cudaMemsetAsync(b + 1, 0x00, 8, st));
    GLR_CUDA(cudaMemsetAsync(b + 2, 0xff, 8, st));
    GLR_CUDA(cudaMemsetAsync(b + 3, 0x00, 8, st));
    bounds_kernel<<<grid_of(n), 256, 0, st>>>(reinterpret_cast<const double2 *>(d_xy), n, b);
    GLR_LAUNCHED("bounds_kernel");
    GLR_CUDA(cudaMemsetAsync(b + 4, 0x00, 8, st));
    edge_extent_kernel<<<grid_of(m), 256, 0, st>>>(reinterpret_cast<const double2 *>(d_xy), e2, m,
                                                   b, b + 4);
    GLR_LAUNCHED("edge_extent_kernel");
    edge_box_keys_kernel<<<grid_of(m), 256, 0, st>>>(reinterpret_cast<const double2 *>(d_xy), e2,
                                                     m, b, deg, hub_degree, b + 4, keys, idx);
    GLR_LAUNCHED("edge_box_keys_kernel");
  } else {
    edge_theta_keys_kernel<<<grid_of(m), 256, 0, st>>>(reinterpret_cast<const double2 *>(d_xy),
                                                       e2, m, deg, hub_degree, keys, idx);
    GLR_LAUNCHED("edge_theta_keys_kernel");
  }
  size_t tb = t_sort;
  GLR_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, keys, keys_out, idx, perm, (int)m, 0, end_bit,
                                           st));
  count_launch(4);
  gather_edges_kernel<<<grid_of(m), 256, 0, st>>>(e2, perm, m, reinterpret_cast<longlong2 *>(d_out));
  GLR_LAUNCHED("gather_edges_kernel");
  return GLR_OK;
}

int theta_sort(const double *d_xy, int64_t n, const int64_t *d_edges, int64_t m,
               int64_t hub_degree, int64_t *d_out, cudaStream_t st) {
  return keyed_sort<false>(d_xy, n, d_edges, m, hub_degree, d_out, st);
}
int box_sort(const double *d_xy, int64_t n, const int64_t *d_edges, int64_t m,
             int64_t hub_degree, int64_t *d_out, cudaStream_t st) {
  return keyed_sort<true>(d_xy, n, d_edges, m, hub_degree, d_out, st);
}

}  // namespace
}  // namespace glr

extern "C" {

int glr_spatial_sort_edges(const double *d_xy, int64_t n, const int64_t *d_edges, int64_t m,
                           int64_t *d_edges_out, void *stream) {
  if (n < 0 || m < 0 || (m > 0 && (d_xy == nullptr || d_edges == nullptr || d_edges_out == nullptr)) ||
      m >= ((int64_t)1 << 31)) {
    glr::set_error("glr_spatial_sort_edges: invalid arguments");
    return GLR_EARG;
  }
  if (n >= ((int64_t)1 << 31)) {
    glr::set_error("glr_spatial_sort_edges: invalid arguments");
    return GLR_EARG;
  }
  return glr::box_sort(d_xy, n, d_edges, m, GLR_BOX_HUB_DEGREE, d_edges_out,
                       glr::as_stream(stream));
}

int glr_theta_sort_edges(const double *d_xy, int64_t n, const int64_t *d_edges, int64_t m,
                         int64_t hub_degree, int64_t *d_edges_out, void *stream) {
  if (n < 0 || m < 0 || (m > 0 && (d_xy == nullptr || d_edges == nullptr || d_edges_out == nullptr)) ||
      m >= ((int64_t)1 << 31) || n >= ((int64_t)1 << 31)) {
    glr::set_error("glr_theta_sort_edges: invalid arguments");
    return GLR_EARG;
  }
  if (hub_degree <= 0) hub_degree = GLR_HUB_DEGREE_DEFAULT;
  return glr::theta_sort(d_xy, n, d_edges, m, hub_degree, d_edges_out, glr::as_stream(stream));
}

int glr_spatial_sort_vertices(const double *d_xy, int64_t n, double *d_xy_out, void *stream) {
  if (n < 0 || (n > 0 && (d_xy == nullptr || d_xy_out == nullptr)) || n >= ((int64_t)1 << 31)) {
    glr::set_error("glr_spatial_sort_vertices: invalid arguments");
    return GLR_EARG;
  }
  return glr::vertex_sort(d_xy, n, d_xy_out, glr::as_stream(stream));
}

}  // extern "C"
