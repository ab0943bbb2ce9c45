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


// ---- k-d order for long edges ----------------------------------------------
//
// Long edges (see GLR_LONG_EDGE_EXTENT) are ordered by a balanced k-d tree
// over the 4-D point (P.x, P.y, Q.x, Q.y) -- P the endpoint of smaller x, Q
// the other -- below the top-level key (hub group, diagonal orientation).
// Every range of positions is split at the aligned position nearest its
// middle (a tile boundary while the range spans one, then 128, then 64: the
// warp slices and j-quarters of the sub-unit masks), along the coordinate of
// largest extent, by a stable radix sort on (range, coordinate) that keeps
// each range in place.  Every 256-edge tile, 128-edge slice and 64-edge
// quarter is then exactly one k-d cell: P box and Q box as tight as a
// balanced partition allows, where a Morton curve's runs of 256 straddle
// cell boundaries (C5: mean tile box side 0.079 of the domain vs 0.089-0.138,
// mixed units 42.7M vs 50.5M, fused pass 2.07 -> 1.77 s).  Level-synchronous,
// no host round trips: the range table lives on the device.
#ifndef GLR_XTHREADS
#define GLR_XTHREADS 128
#endif
#ifndef GLR_XK
#define GLR_XK 2
#endif
constexpr int kKdTile = GLR_XTHREADS * GLR_XK;  // crossing.cu's kTile
#ifndef GLR_XSUBQ
#define GLR_XSUBQ 4
#endif
constexpr int kKdLeaf = kKdTile / GLR_XSUBQ;    // crossing.cu's kSubJ (j-quarter)
// tuning / cross-check knob (glr_spatial_set_kd): 0 keeps the Morton order,
// 1 (default) builds the tree from kKdMinEdges edges on -- below that the
// dense pass costs a millisecond or two and the tree's ~1 ms of small
// launches is not repaid (C2, 40k edges: auto 2.5 ms with it, 1.4 without)
// -- 2 builds it for any size (tests)
constexpr int64_t kKdMinEdges = (int64_t)1 << 17;
int &kd_flag() {
  static int f = 1;
  return f;
}
inline bool kd_long_edges(int64_t m) {
  return kd_flag() == 2 || (kd_flag() == 1 && m >= kKdMinEdges);
}

__device__ inline unsigned quant32(double v, double lo, double scale) {
  double q = (v - lo) * scale;  // scale = (2^32 - 1) / (hi - lo), or 0 for a flat axis
  if (!(q >= 0.0)) q = 0.0;     // also NaN
  if (q > 4294967295.0) q = 4294967295.0;
  return (unsigned)q;
}

// per edge: quantised (P.x, P.y, Q.x, Q.y) (field-major), top key, identity index
__global__ void kd_prep_kernel(const double2 *__restrict__ xy, const longlong2 *__restrict__ e,
                               int64_t m, const unsigned long long *b,
                               const int *__restrict__ deg, int64_t hub_degree,
                               unsigned *__restrict__ qc, unsigned long long *__restrict__ top,
                               int *__restrict__ idx) {
  const double x0 = dunkey(b[0]), x1 = dunkey(b[1]), y0 = dunkey(b[2]), y1 = dunkey(b[3]);
  const double sx = (x1 > x0 && isfinite(x1 - x0)) ? 4294967295.0 / (x1 - x0) : 0.0;
  const double sy = (y1 > y0 && isfinite(y1 - y0)) ? 4294967295.0 / (y1 - y0) : 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const longlong2 uv = e[i];
    const double2 u = xy[uv.x], v = xy[uv.y];
    const bool pu = u.x < v.x || (u.x == v.x && u.y <= v.y);
    const double2 p = pu ? u : v, q = pu ? v : u;
    qc[i] = quant32(p.x, x0, sx);
    qc[m + i] = quant32(p.y, y0, sy);
    qc[2 * m + i] = quant32(q.x, x0, sx);
    qc[3 * m + i] = quant32(q.y, y0, sy);
    const unsigned long long up = ((q.x - p.x) * (q.y - p.y) >= 0.0) ? 1ull : 0ull;
    const int du = deg[uv.x], dv = deg[uv.y];
    const long long hub = (du >= dv) ? uv.x : uv.y;
    const unsigned long long grp =
        ((du > dv ? du : dv) >= hub_degree) ? (unsigned long long)hub + 1ull : 0ull;
    top[i] = (grp << 1) | up;
    idx[i] = (int)i;
  }
}

// head flags of the runs of equal top keys (1 at the first position of a run)
__global__ void kd_heads_kernel(const unsigned long long *__restrict__ top, int64_t m,
                                int *__restrict__ head) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < m;
       p += (int64_t)gridDim.x * blockDim.x)
    head[p] = (p == 0 || top[p] != top[p - 1]) ? 1 : 0;
}

// rid = inclusive scan of the heads - 1; the runs become the initial ranges
// (more runs than the table holds: the tail runs share the last range, which
// only costs tightness)
__global__ void kd_ranges_init_kernel(int *__restrict__ rid, int64_t m, int rmax,
                                      int2 *__restrict__ rng, int *__restrict__ nr) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < m;
       p += (int64_t)gridDim.x * blockDim.x) {
    int r = rid[p] - 1;
    const int prev = p > 0 ? rid[p - 1] - 1 : -1;
    if (r > rmax - 1) r = rmax - 1;
    const int rp = prev > rmax - 1 ? rmax - 1 : prev;
    if (r != rp) {
      rng[r].x = (int)p;
      if (rp >= 0) rng[rp].y = (int)p;
    }
    if (p == m - 1) {
      rng[r].y = (int)m;
      *nr = r + 1;
    }
  }
}
__global__ void kd_rid_clamp_kernel(int *__restrict__ rid, int64_t m, int rmax) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < m;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int r = rid[p] - 1;
    rid[p] = r > rmax - 1 ? rmax - 1 : r;
  }
}

// per range: min / max of the four quantised coordinates of its edges
__global__ void __launch_bounds__(256)
kd_extent_kernel(const int *__restrict__ rid, const int *__restrict__ perm,
                 const unsigned *__restrict__ qc, int64_t m, unsigned *__restrict__ emin,
                 unsigned *__restrict__ emax) {
  __shared__ int wr[8];
  __shared__ unsigned wmn[8][4], wmx[8][4];
  const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t span = (int64_t)gridDim.x * blockDim.x;
  const int64_t rounds = (m + span - 1) / span;
  for (int64_t it = 0; it < rounds; ++it) {
    const int64_t p = it * span + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const bool valid = p < m;
    int r = -1;
    unsigned v[4] = {0, 0, 0, 0};
    if (valid) {
      r = rid[p];
      const int e = perm[p];
#pragma unroll
      for (int d = 0; d < 4; ++d) v[d] = qc[(int64_t)d * m + e];
    }
    const int r0 = __shfl_sync(0xffffffffu, r, 0);
    const bool uni = __all_sync(0xffffffffu, valid && r == r0);
    if (uni) {
#pragma unroll
      for (int d = 0; d < 4; ++d) {
        const unsigned mn = __reduce_min_sync(0xffffffffu, v[d]);
        const unsigned mx = __reduce_max_sync(0xffffffffu, v[d]);
        if (lane == 0) { wmn[warp][d] = mn; wmx[warp][d] = mx; }
      }
    } else if (valid) {
#pragma unroll
      for (int d = 0; d < 4; ++d) {
        atomicMin(&emin[(int64_t)r * 4 + d], v[d]);
        atomicMax(&emax[(int64_t)r * 4 + d], v[d]);
      }
    }
    if (lane == 0) wr[warp] = uni ? r0 : -1;
    __syncthreads();
    if (threadIdx.x < 8) {
      const int d = threadIdx.x & 3;
      const bool mx = threadIdx.x >= 4;
      // one atomic per run of warps with the same range
      int w = 0;
      while (w < 8) {
        const int rr = wr[w];
        unsigned a = mx ? wmx[w][d] : wmn[w][d];
        int w2 = w + 1;
        while (rr >= 0 && w2 < 8 && wr[w2] == rr) {
          const unsigned c = mx ? wmx[w2][d] : wmn[w2][d];
          a = mx ? (c > a ? c : a) : (c < a ? c : a);
          ++w2;
        }
        if (rr >= 0) {
          if (mx) atomicMax(&emax[(int64_t)rr * 4 + d], a);
          else atomicMin(&emin[(int64_t)rr * 4 + d], a);
        }
        w = w2;
      }
    }
    __syncthreads();
  }
}

// One CTA: every range picks its split position and coordinate; the ranges
// of the next level are numbered in position order (block scan), their
// extent slots reset.  sp[r] = {split position or -1, coordinate, first new
// index}.  Every split takes a distinct multiple of kKdLeaf inside (0, m), so
// a table of (initial ranges + m / kKdLeaf + 1) entries never fills.
constexpr int kKdSplitThreads = 1024;
__global__ void __launch_bounds__(kKdSplitThreads)
kd_split_kernel(const int2 *__restrict__ rng, const int *__restrict__ nr,
                const unsigned *__restrict__ emin, const unsigned *__restrict__ emax,
                int4 *__restrict__ sp, int2 *__restrict__ rng_next, int *__restrict__ nr_next,
                unsigned *__restrict__ emin_next, unsigned *__restrict__ emax_next) {
  __shared__ int wsum[kKdSplitThreads / 32];
  __shared__ int carry;
  const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int R = *nr;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < R; base += kKdSplitThreads) {
    const int r = base + (int)threadIdx.x;
    int split = -1, dim = 0, kids = 0;
    int2 se = make_int2(0, 0);
    if (r < R) {
      se = rng[r];
      kids = 1;
      unsigned best = 0;
#pragma unroll
      for (int d = 0; d < 4; ++d) {
        const unsigned lo = emin[(int64_t)r * 4 + d], hi = emax[(int64_t)r * 4 + d];
        const unsigned ext = hi > lo ? hi - lo : 0u;
        if (ext > best) { best = ext; dim = d; }
      }
      if (best > 0) {
        for (int al = kKdTile; al >= kKdLeaf; al >>= 1) {
          const int lo = se.x / al + 1, hi = (se.y - 1) / al;
          if (lo <= hi) {
            long long bi = ((long long)se.x + se.y + al) / (2ll * al);
            if (bi < lo) bi = lo;
            if (bi > hi) bi = hi;
            split = (int)bi * al;
            break;
          }
        }
      }
      if (split >= 0) kids = 2;
    }
    // exclusive block scan of kids
    int inc = kids;
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, inc, o);
      if ((int)lane >= o) inc += t;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    int woff = 0, tot = 0;
    for (int w = 0; w < kKdSplitThreads / 32; ++w) {
      if (w < (int)warp) woff += wsum[w];
      tot += wsum[w];
    }
    const int f = carry + woff + inc - kids;
    if (r < R) {
      sp[r] = make_int4(split, dim, f, 0);
      if (split >= 0) {
        rng_next[f] = make_int2(se.x, split);
        rng_next[f + 1] = make_int2(split, se.y);
      } else {
        rng_next[f] = se;
      }
      for (int k = 0; k < kids; ++k)
#pragma unroll
        for (int d = 0; d < 4; ++d) {
          emin_next[(int64_t)(f + k) * 4 + d] = 0xffffffffu;
          emax_next[(int64_t)(f + k) * 4 + d] = 0u;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) *nr_next = carry;
}

// sort keys (range, coordinate along the range's split axis) and the range
// index each position has after the split
__global__ void kd_keys_kernel(int *__restrict__ rid, const int *__restrict__ perm,
                               const unsigned *__restrict__ qc, int64_t m,
                               const int4 *__restrict__ sp, unsigned long long *__restrict__ keys) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < m;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int r = rid[p];
    const int4 s = sp[r];
    unsigned c = 0;
    if (s.x >= 0) c = qc[(int64_t)s.y * m + perm[p]];
    keys[p] = ((unsigned long long)(unsigned)r << 32) | c;
    rid[p] = s.z + ((s.x >= 0 && p >= s.x) ? 1 : 0);
  }
}

int theta_sort(const double *d_xy, int64_t n, const int64_t *d_edges, int64_t m,
               int64_t hub_degree, int64_t *d_out, cudaStream_t st);
// Hub degree of the culled (4-D bbox) order: a hub group's tiles have boxes
// anchored at the hub, so only hubs whose shared-vertex pairs would cost more
// fallbacks than their boxes cost candidate units get a group (C5 culled:
// 3.70 s at 256, 3.19 s at 1024, 2.98 s at 4096, 2.92 s at 16384, 3.05 s
// with none; tools/cull_probe.py; with the k-d order and the final kernels:
// 1447 ms at 8192, 1439 at 16384, 1444 at 32768, 1457 with none).
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



// k-d order of long edges (kernels above): deg and the bound words b come
// from the caller.
int kd_sort(const double *d_xy, int64_t n, const int64_t *d_edges, int64_t m,
            int64_t hub_degree, const int *deg, const unsigned long long *b, int64_t *d_out,
            cudaStream_t st) {
  const int64_t T = (m + kKdTile - 1) / kKdTile;
  int levels = 2;  // the 128 and 64 alignments below the tile
  while (levels < 40 && ((int64_t)1 << (levels - 2)) < T + 1) ++levels;
  // initial ranges: the runs of (hub group, orientation); at most two per
  // vertex of degree >= hub_degree, plus group 0's
  int64_t r0 = 2 * (2 * m / (hub_degree > 0 ? hub_degree : 1) + 2);
  if (r0 > m / kKdLeaf + 1024) r0 = m / kKdLeaf + 1024;
  const int rmax = (int)(r0 + m / kKdLeaf + 2);
  int rbits = 1;
  while (rbits < 31 && ((int64_t)1 << rbits) < rmax) ++rbits;
  int top_bits = 2;
  while (top_bits < 64 && ((unsigned long long)(n + 1) >> (top_bits - 1)) != 0) ++top_bits;
  size_t t_top = 0, t_lvl = 0, t_scan = 0;
  GLR_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, t_top, (const unsigned long long *)nullptr,
                                           (unsigned long long *)nullptr, (const int *)nullptr,
                                           (int *)nullptr, (int)m, 0, top_bits, st));
  GLR_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, t_lvl, (const unsigned long long *)nullptr,
                                           (unsigned long long *)nullptr, (const int *)nullptr,
                                           (int *)nullptr, (int)m, 0, 32 + rbits, st));
  GLR_CUDA(cub::DeviceScan::InclusiveSum(nullptr, t_scan, (const int *)nullptr, (int *)nullptr,
                                         (int)m, st));
  size_t t_cub = t_top > t_lvl ? t_top : t_lvl;
  if (t_scan > t_cub) t_cub = t_scan;
  auto al = [](size_t v) { return (v + 255) & ~(size_t)255; };
  const size_t a8 = al((size_t)m * 8), a4 = al((size_t)m * 4);
  const size_t a_rng = al((size_t)rmax * sizeof(int2)), a_ext = al((size_t)rmax * 16);
  const size_t a_sp = al((size_t)rmax * sizeof(int4));
  Scratch scr(2 * a8 + 4 * a4 + 4 * a4 + 2 * a_rng + 4 * a_ext + a_sp + 256 + t_cub, st);
  GLR_CUDA(scr.err);
  char *p = scr.as<char>();
  auto take = [&p](size_t bytes) { char *q = p; p += bytes; return q; };
  auto *keys = reinterpret_cast<unsigned long long *>(take(a8));
  auto *keys_out = reinterpret_cast<unsigned long long *>(take(a8));
  int *perm = reinterpret_cast<int *>(take(a4));
  int *perm_out = reinterpret_cast<int *>(take(a4));
  int *rid = reinterpret_cast<int *>(take(a4));
  int *head = reinterpret_cast<int *>(take(a4));
  unsigned *qc = reinterpret_cast<unsigned *>(take(4 * a4));
  int2 *rng[2] = {reinterpret_cast<int2 *>(take(a_rng)), reinterpret_cast<int2 *>(take(a_rng))};
  unsigned *emin[2], *emax[2];
  for (int k = 0; k < 2; ++k) {
    emin[k] = reinterpret_cast<unsigned *>(take(a_ext));
    emax[k] = reinterpret_cast<unsigned *>(take(a_ext));
  }
  int4 *sp = reinterpret_cast<int4 *>(take(a_sp));
  int *nr = reinterpret_cast<int *>(take(256));  // nr[0], nr[1]: range counts (ping-pong)
  void *tmp = p;
  const auto *e2 = reinterpret_cast<const longlong2 *>(d_edges);
  const int g = grid_of(m);
  // field-major qc rows are m apart (not a4 / 4): allocate by m exactly
  kd_prep_kernel<<<g, 256, 0, st>>>(reinterpret_cast<const double2 *>(d_xy), e2, m, b, deg,
                                    hub_degree, qc, keys, perm);
  GLR_LAUNCHED("kd_prep_kernel");
  size_t tb = t_cub;
  GLR_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, keys, keys_out, perm, perm_out, (int)m, 0,
                                           top_bits, st));
  count_launch(4);
  { int *t = perm; perm = perm_out; perm_out = t; }
  kd_heads_kernel<<<g, 256, 0, st>>>(keys_out, m, head);
  GLR_LAUNCHED("kd_heads_kernel");
  tb = t_cub;
  GLR_CUDA(cub::DeviceScan::InclusiveSum(tmp, tb, head, rid, (int)m, st));
  count_launch(2);
  kd_ranges_init_kernel<<<g, 256, 0, st>>>(rid, m, (int)r0, rng[0], nr);
  GLR_LAUNCHED("kd_ranges_init_kernel");
  kd_rid_clamp_kernel<<<g, 256, 0, st>>>(rid, m, (int)r0);
  GLR_LAUNCHED("kd_rid_clamp_kernel");
  GLR_CUDA(cudaMemsetAsync(emin[0], 0xff, a_ext, st));
  GLR_CUDA(cudaMemsetAsync(emax[0], 0x00, a_ext, st));
  for (int lv = 0; lv < levels; ++lv) {
    const int c = lv & 1, x = c ^ 1;
    kd_extent_kernel<<<g, 256, 0, st>>>(rid, perm, qc, m, emin[c], emax[c]);
    GLR_LAUNCHED("kd_extent_kernel");
    kd_split_kernel<<<1, kKdSplitThreads, 0, st>>>(rng[c], nr + c, emin[c], emax[c], sp, rng[x],
                                                   nr + x, emin[x], emax[x]);
    GLR_LAUNCHED("kd_split_kernel");
    kd_keys_kernel<<<g, 256, 0, st>>>(rid, perm, qc, m, sp, keys);
    GLR_LAUNCHED("kd_keys_kernel");
    tb = t_cub;
    GLR_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, keys, keys_out, perm, perm_out, (int)m, 0,
                                             32 + rbits, st));
    count_launch(4);
    int *t = perm; perm = perm_out; perm_out = t;
  }
  gather_edges_kernel<<<g, 256, 0, st>>>(e2, perm, m, reinterpret_cast<longlong2 *>(d_out));
  GLR_LAUNCHED("gather_edges_kernel");
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
    // long edges take the k-d order (one 8-byte read back decides; the culled
    // plan synchronises for its candidate count anyway)
    unsigned long long lsum = 0;
    if (kd_long_edges(m)) {
      GLR_CUDA(cudaMemcpyAsync(&lsum, b + 4, 8, cudaMemcpyDeviceToHost, st));
      GLR_CUDA(cudaStreamSynchronize(st));
    }
    if (kd_long_edges(m) && lsum >= (unsigned long long)GLR_LONG_EDGE_EXTENT * (unsigned long long)m)
      return kd_sort(d_xy, n, d_edges, m, hub_degree, deg, b, d_out, st);
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

int glr_spatial_set_kd(int on) {
  const int was = glr::kd_flag();
  if (on >= 0) glr::kd_flag() = on > 2 ? 1 : on;
  return was;
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
