// Edge crossing E_c and crossing angle E_ca: the O(|E|^2) all-pairs pass.
//
// Replaces the numpy body of the reference's _crossing_scan
// (/root/reference/pkg/src/glare/metrics/exact.py:145-222) and the vectorised
// predicate proper_intersection_mask (geometry.py:62-79).  A pair (i < j)
// counts when (exact.py:187-217)
//   closed bbox overlap in x and y  AND  no shared vertex index  AND
//   straddle(c1, c2) AND straddle(c3, c4)
// with c1..c4 the reference's four cross products evaluated with the same
// IEEE operations and operand order (no FMA), each compared against zero
// separately.  dev_sum accumulates |ideal - min(d, pi - d)| over hits
// (exact.py:219-221, geometry.py:107-110).
//
// Work decomposition: edges are cut into tiles of kTile = kThreads*K; a
// "unit" is an upper-triangular tile pair (ti <= tj).  Persistent CTAs take a
// contiguous unit range; each thread keeps K i-edges in registers and streams
// the j-tile from shared memory (broadcast LDS, no bank conflicts).
//
// FP64 budget per pair: 6 DADD coordinate differences, 8 DMUL, 4 DADD for
// c1..c4 = 18 FP64 instructions (c3 reuses the c1 differences:
// fl(ay-cy) = -fl(cy-ay) exactly).  Everything else runs on the ALU/FMA pipes:
//  - bbox: exact 32-bit ranks of xmin/xmax/ymin/ymax (rank order == double
//    order, built by glr_crossing_prepare), 4 ISETP;
//  - signs (fast path): the high word of each c, viewed as a float f, has the
//    sign of c, is zero iff c == 0 and lies in [2^-53, 2^127) whenever every
//    nonzero |coordinate| lies in [2^-160, 2^500] (DESIGN.md "fast sign
//    path"), so straddle(c1,c2) == (f1*f2 <= 0) with an FP32 FMUL that cannot
//    underflow: 2 FMUL (FMA pipe) + 2 FSETP;
//  - shared vertices (fast path): NOT tested per pair.  Two distinct edges
//    that share a vertex index always pass the fast predicate (their bboxes
//    share the point, and one of c1/c2 and one of c3/c4 is exactly 0 --
//    DESIGN.md), so the kernel counts them and adj_kernel subtracts them:
//    sum over vertices of C(deg, 2) pairs, each assigned to its tile-pair
//    unit so unit-range partials stay exact.
// Inputs outside the fast window use the general instantiation, which
// compares the doubles themselves (numpy's NaN-is-false semantics) and tests
// vertex ids per pair.
#include <cub/cub.cuh>

#include "common.cuh"

namespace glr {
namespace {

// Tunables (overridable at build time for the tuning sweeps in tools/;
// defaults chosen by tools/variant_bench.py on a C5-shaped graph, see
// profiles/r01_variants.txt: K=2 i-edges/thread, 4 CTAs/SM (16 warps), j-loop
// unrolled 4x, PTX predicate tail).
#ifndef GLR_XTHREADS
#define GLR_XTHREADS 128
#endif
#ifndef GLR_XK
#define GLR_XK 2
#endif
#ifndef GLR_XMINB
#define GLR_XMINB 4
#endif
#ifndef GLR_XUNROLL
#define GLR_XUNROLL 4
#endif
#ifndef GLR_XNOPTXTAIL
#define GLR_XPTXTAIL 1
#endif
constexpr int kThreads = GLR_XTHREADS;  // threads per CTA
constexpr int kK = GLR_XK;              // i-edges per thread
constexpr int kTile = kThreads * kK;
constexpr int kMinBlocks = GLR_XMINB;   // CTAs per SM
constexpr int kUnroll = GLR_XUNROLL;    // j-loop unroll of the off-diagonal tiles
constexpr int kAdjTile = 128;           // incidence-list tile of adj_kernel
// j-tiles per band of the unit order (common.cuh band_unit_coords): 2048
// tiles x 256 edges x ~76 B of records/theta/flags = 40 MB, so the j-tiles
// the CTAs are sweeping at any moment stay in the 126 MB L2.
#ifndef GLR_XBAND
#define GLR_XBAND 2048
#endif
constexpr int kBandTiles = GLR_XBAND;
#ifndef GLR_XCHUNK
#define GLR_XCHUNK 256
#endif
constexpr int kMaxChunk = GLR_XCHUNK;  // units per round-robin chunk (upper bound)
#ifndef GLR_XFBLOCK
#define GLR_XFBLOCK 4
#endif
constexpr int kFilterBlock = GLR_XFBLOCK;  // j-edges per filter block (one warp vote each)
#ifndef GLR_XFBLOCK_C
#define GLR_XFBLOCK_C 2
#endif
constexpr int kFilterBlockCount = GLR_XFBLOCK_C;  // same for the count-only kernel
#ifndef GLR_XFBLOCK_S
#define GLR_XFBLOCK_S 4
#endif
constexpr int kFilterBlockSigned = GLR_XFBLOCK_S;  // same for signed units
// unroll of the j-block loops over a tile (signed units / count-only, t = 1)
#ifndef GLR_XJUNROLL_S
#define GLR_XJUNROLL_S 1
#endif
#ifndef GLR_XJUNROLL_C
#define GLR_XJUNROLL_C 1
#endif
constexpr int kJUnrollS = GLR_XJUNROLL_S;
constexpr int kJUnrollC = GLR_XJUNROLL_C;
// CTAs per SM of the filter kernel (fused 4 -> <= 128 registers, count-only
// 5 -> <= 102, with kFK = 4):
// tools/c5_time.py and tools/config_bench.py, profiles/r01_variants_filter.txt
#ifndef GLR_XFMINB_A
#define GLR_XFMINB_A 4
#endif
#ifndef GLR_XFMINB_C
#define GLR_XFMINB_C 5
#endif
constexpr int kFilterMinBlocksAngle = GLR_XFMINB_A;
#ifndef GLR_XFSTAGES
#define GLR_XFSTAGES 4
#endif
constexpr int kStages = GLR_XFSTAGES;  // j-tile ring depth of the filter kernel
constexpr int kFilterMinBlocksCount = GLR_XFMINB_C;


// Largest edge count whose pair count m(m-1)/2 stays below 2^53, where the
// float64 count slot of d_out is exact.
constexpr int64_t kMaxExactEdges = (int64_t)1 << 27;
// units per launch segment of the angle pass (fixup bitmap <= 1 GB)
constexpr uint64_t kMaxSegUnits = (uint64_t)1 << 32;

// Fast sign path admissibility bounds on nonzero |coordinate|.
constexpr double kMaxAbsFast = 0x1p500;
constexpr double kMinAbsFast = 0x1p-160;

struct __align__(16) EdgeRec {
  double ax, ay, bx, by;           // a = xy[edges[:,0]], b = xy[edges[:,1]]
  double abx, aby;                 // b - a  (geometry.py:69-70)
  int rxmin, rxmax, rymin, rymax;  // exact order-preserving bbox ranks
};
static_assert(sizeof(EdgeRec) == 64, "EdgeRec must be 64 bytes");

struct __align__(16) RecHeader {
  int fast;        // pair-kernel mode: kModeGeneral / kModeSign / kModeFilter
  int admissible;  // 1: every nonzero |coordinate| in [2^-160, 2^500]
  long long n;
  long long m;
  long long m_pad;
  unsigned long long maxabs_bits;  // max |coord| (bit pattern)
  unsigned long long minabs_bits;  // min nonzero |coord| (bit pattern)
  char pad[208];
};
static_assert(sizeof(RecHeader) == 256, "RecHeader must be 256 bytes");

// Pair-kernel modes (RecHeader::fast).  General: doubles compared directly,
// ids tested per pair (any input).  Sign: float view of the FP64 cross
// products + adjacency correction (fast window only).  Filter: certified
// packed-FP32 filter with exact FP64 fallback (fast window only, default).
constexpr int kModeGeneral = 0;
constexpr int kModeSign = 1;
constexpr int kModeFilter = 2;
#ifdef GLR_XNOFILTER
constexpr int kModeFastDefault = kModeSign;
#else
constexpr int kModeFastDefault = kModeFilter;
#endif

// Filter record of an edge: endpoint coordinates translated to the
// lower-left corner of the edges' bounding box and scaled by a power of two
// into [0, 1/2], rounded to FP32 (ax, ay, bx, by); the FP32 direction
// (abx, aby) = (bx - ax, by - ay) and the line constant ka = ab x a =
// abx*ay - aby*ax (FP64 from the FP32 values, rounded once), all three
// scaled by a per-edge power of two 2^k and stored as (sabx, nsaby =
// -saby, nska = -ska); theta.  Then the scaled cross product of a point p
// with the line is one FFMA pair: ab x (p - a) = sabx*py + (nsaby*px + nska),
// and 2^k is chosen so that a product of two such values exceeding 1 in
// magnitude certifies both factors' signs.
enum FField { kFAx, kFAy, kFBx, kFBy, kFSabx, kFNsaby, kFNska, kFFields };

// Filter kernel work split: a unit's i-tile is cut into slices of 32 lanes
// x kFK i-edges (a warp's work item); lane l, i-edge k of slice s is tile
// slot s*32*kFK + 32k + l, and i-edges (2g, 2g+1) share packed registers.
#ifndef GLR_XFK
#define GLR_XFK 4
#endif
constexpr int kFK = GLR_XFK;             // i-edges per lane in the filter kernel
constexpr int kFGroups = kFK / 2;        // packed i-edge pairs per lane
constexpr int kFSlices = kTile / (32 * kFK);  // warp slices per unit
// Sub-unit masks of the classified candidate list (sub_mask_kernel): per
// mixed unit, block s * kSubQuarters + q is warp-slice s x j-quarter q (kSubJ
// consecutive j-edges).  Bit b of the mask: the block is certified empty;
// bit kSubBits + b: certified full (every pair crosses).  The filter kernel
// skips both kinds; cross_subfull_kernel counts the full ones.
#ifndef GLR_XSUBQ
#define GLR_XSUBQ 4
#endif
// unroll of orient_ranges' corner loop (a multiple of 4 keeps the hoisted
// differences in registers)
#ifndef GLR_XCORNERUNROLL
#define GLR_XCORNERUNROLL 16
#endif
constexpr int kCornerUnroll = GLR_XCORNERUNROLL;
// CTAs per SM of the classification kernels (register cap: 1 -> 255, 2 -> 128
// with ~200 B of spills, 3 -> 80): C5 classes + masks 53.3 / 43.7 ms at 1 / 2
// (tools/classtime.sh); corner-loop unroll 4 / 8 / 16: 60.1 / 53.2 / 53.3 ms
#ifndef GLR_XCLASSMINB
#define GLR_XCLASSMINB 2
#endif
// one-kink angle form in the fused filter kernel (range_kink)
#ifndef GLR_XKINK
#define GLR_XKINK 1
#endif
constexpr int kSubQuarters = GLR_XSUBQ;
constexpr int kSubJ = kTile / kSubQuarters;
constexpr unsigned kSubQuarterMask = (kSubQuarters >= 32) ? 0xffffffffu : (1u << kSubQuarters) - 1u;
constexpr int kSubBits = kFSlices * kSubQuarters;  // blocks per unit
static_assert(2 * kSubBits <= 64 && 32 % kSubBits == 0, "sub-masks: none + full bits in <= 64");
static_assert((32 * kFK) % kSubJ == 0, "a warp slice is a whole number of sub-blocks");
static_assert(kSubJ % 4 == 0 && kSubJ >= 8, "j-quarters are whole filter blocks");
template <int BITS> struct SubMaskOf { typedef uint64_t type; };
template <> struct SubMaskOf<16> { typedef unsigned short type; };
template <> struct SubMaskOf<8> { typedef unsigned short type; };
template <> struct SubMaskOf<32> { typedef unsigned type; };
typedef SubMaskOf<2 * kSubBits>::type SubMask;
// independent hit counters / angle accumulators per lane (ILP vs registers;
// one counter makes the count-only kernel 3% faster, profiles/r01_variants_filter.txt;
// in the fused kernel's general units 1 counter + 2 angle accumulators free
// the registers ptxas otherwise shuffles with moves: C5 culled 2.96 -> 2.81 s,
// dense 4.48 -> 4.45 s, profiles/r02_variants_acc.txt)
#ifndef GLR_XFCNT_A
#define GLR_XFCNT_A 1
#endif
#ifndef GLR_XFCNT_C
#define GLR_XFCNT_C 1
#endif
#ifndef GLR_XFDEV
#define GLR_XFDEV 2
#endif
constexpr int kCntAccAngle = GLR_XFCNT_A;
constexpr int kCntAccCount = GLR_XFCNT_C;
constexpr int kDevAcc = GLR_XFDEV;
#ifndef GLR_XA2
#define GLR_XA2 2
#endif
constexpr int kA2 = GLR_XA2;  // signed units: alternating sum_j h_j theta_j accumulators (1 or 2)
static_assert(kA2 == 1 || kA2 == 2, "kA2");
static_assert(kFK % 2 == 0 && kFK <= 4 && kTile % (32 * kFK) == 0, "filter slice shape");

__host__ __device__ inline int fslot(int slice, int k, int lane) {
  return slice * 32 * kFK + 32 * k + lane;
}

// In HBM the filter records of a tile are stored field-major and paired the
// way the kernel packs its i-edges: v[f][P], P = (s*kFGroups + g)*32 + l,
// holds (field f of slot fslot(s, 2g, l), of slot fslot(s, 2g+1, l)), so
// each packed i-register pair is one 64-bit load.
struct __align__(16) FTile {
  float2 v[kFFields][kTile / 2];
  double theta[kTile];
};
static_assert(sizeof(FTile) == (size_t)kTile * 36, "FTile must be 36 B per edge");

// The same record in the j role, 32 B per edge, stored by PAIRS of
// consecutive edges (2p, 2p+1) so that the j-endpoint coordinates of the two
// are adjacent floats (one packed register pair each, see filter_m2):
//   [cx0 cx1 cy0 cy1] [dx0 dx1 dy0 dy1] [scdx0 -scdy0 -skc0 scdx1]
//   [-scdy1 -skc1 0 0]
// read by all lanes of a warp at once (broadcast).
struct __align__(16) JRec {
  float4 c;
  float4 k;
};
struct __align__(16) JPair {
  float4 cxy, dxy, k0, k1;
};
static_assert(sizeof(JPair) == 2 * sizeof(JRec), "a j pair is two records");
__device__ inline void jrec_store(JRec *jrec, int64_t e, float ax, float ay, float bx, float by,
                                  float sabx, float nsaby, float nska) {
  float *w = reinterpret_cast<float *>(jrec + (e & ~1ll));
  const int h = (int)(e & 1);
  w[0 + h] = ax; w[2 + h] = ay; w[4 + h] = bx; w[6 + h] = by;
  if (h == 0) {
    w[8] = sabx; w[9] = nsaby; w[10] = nska;
  } else {
    w[11] = sabx; w[12] = nsaby; w[13] = nska; w[14] = 0.0f; w[15] = 0.0f;
  }
}
__device__ inline float4 jrec_points(const JRec *jrec, int64_t e) {  // (ax, ay, bx, by)
  const float *w = reinterpret_cast<const float *>(jrec + (e & ~1ll));
  const int h = (int)(e & 1);
  return make_float4(w[0 + h], w[2 + h], w[4 + h], w[6 + h]);
}

// Per tile: box of its edges' scaled FP32 endpoints and the largest L =
// |abx| + |aby|; a unit's two boxes bound |p - a| for all its pairs, which
// tightens the filter's certification threshold for spatially local units.
struct __align__(16) TileBox {
  float xlo, xhi, ylo, yhi;
  float lmax;
  float thlo, thhi;  // bounds of the tile's theta, rounded outward (empty: inf, -inf)
  int star;          // v if every real edge of the tile is incident to vertex v, else -1
};

// Records buffer: header | rec[m_pad] | theta[m_pad] | ids[m_pad] |
// newc[m_pad] | frec[m_pad] | inc[2m] (incident edge ids grouped by vertex) |
// offs[n+1] | wofs[n+1].
struct RecView {
  RecHeader *hdr;
  EdgeRec *rec;
  FTile *ftile;
  JRec *jrec;
  TileBox *tbox;
  double *theta;
  int2 *ids;
  int *newc;  // 1 if edge e starts a run of edges sharing endpoint a (or a tile)
  int *inc;
  int *offs;
  long long *wofs;
};

inline int64_t pad_edges(int64_t m) { return ((m + kTile - 1) / kTile) * kTile; }
inline size_t al256(size_t b) { return (b + 255) & ~(size_t)255; }

struct Layout {
  size_t rec, theta, ids, newc, frec, jrec, tbox, inc, offs, wofs, total;
};

inline Layout layout(int64_t n, int64_t m) {
  const int64_t mp = pad_edges(m < 1 ? 1 : m);
  const int64_t nn = n < 0 ? 0 : n;
  Layout L;
  L.rec = sizeof(RecHeader);
  L.theta = L.rec + al256((size_t)mp * sizeof(EdgeRec));
  L.ids = L.theta + al256((size_t)mp * sizeof(double));
  L.newc = L.ids + al256((size_t)mp * sizeof(int2));
  L.frec = L.newc + al256((size_t)mp * sizeof(int));
  L.jrec = L.frec + al256((size_t)(mp / kTile) * sizeof(FTile));
  L.tbox = L.jrec + al256((size_t)mp * sizeof(JRec));
  L.inc = L.tbox + al256((size_t)(mp / kTile) * sizeof(TileBox));
  L.offs = L.inc + al256((size_t)(2 * (m < 0 ? 0 : m)) * sizeof(int));
  L.wofs = L.offs + al256((size_t)(nn + 1) * sizeof(int));
  L.total = L.wofs + al256((size_t)(nn + 1) * sizeof(long long));
  return L;
}

inline RecView view(void *base, int64_t n, int64_t m) {
  const Layout L = layout(n, m);
  char *p = reinterpret_cast<char *>(base);
  RecView v;
  v.hdr = reinterpret_cast<RecHeader *>(p);
  v.rec = reinterpret_cast<EdgeRec *>(p + L.rec);
  v.theta = reinterpret_cast<double *>(p + L.theta);
  v.ids = reinterpret_cast<int2 *>(p + L.ids);
  v.newc = reinterpret_cast<int *>(p + L.newc);
  v.ftile = reinterpret_cast<FTile *>(p + L.frec);
  v.jrec = reinterpret_cast<JRec *>(p + L.jrec);
  v.tbox = reinterpret_cast<TileBox *>(p + L.tbox);
  v.inc = reinterpret_cast<int *>(p + L.inc);
  v.offs = reinterpret_cast<int *>(p + L.offs);
  v.wofs = reinterpret_cast<long long *>(p + L.wofs);
  return v;
}

// np.mod(x, pi) for b = pi > 0 (numpy npy_divmod): fmod, shift negatives
// into range, +0.0 for a zero remainder.
__device__ inline double mod_pi(double x) {
  const double PI = 3.141592653589793;
  double r = fmod(x, PI);
  if (r != 0.0) {
    if (r < 0.0) r = __dadd_rn(r, PI);
  } else {
    r = 0.0;
  }
  return r;
}

// ---------------------------------------------------------------- prepare --

__global__ void gather_kernel(const double2 *__restrict__ xy, const longlong2 *__restrict__ edges,
                              int64_t m, int64_t m_pad, RecView rv, double *xs, double *ys,
                              int *deg, int *keys, int *vals) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m_pad;
       e += (int64_t)gridDim.x * blockDim.x) {
    EdgeRec r;
    if (e < m) {
      longlong2 uv = edges[e];
      double2 a = xy[uv.x], b = xy[uv.y];
      r.ax = a.x; r.ay = a.y; r.bx = b.x; r.by = b.y;
      r.abx = __dsub_rn(b.x, a.x);
      r.aby = __dsub_rn(b.y, a.y);
      r.rxmin = r.rxmax = r.rymin = r.rymax = 0;
      // axis angle of a->b, geometry.py:94-97
      rv.theta[e] = mod_pi(atan2(r.aby, r.abx));
      rv.ids[e] = make_int2((int)uv.x, (int)uv.y);
      // edges are sorted by their first endpoint: runs share a = xy[u]
      rv.newc[e] = (e % kTile == 0 || edges[e - 1].x != uv.x) ? 1 : 0;
      xs[e] = fmin(a.x, b.x);
      xs[m + e] = fmax(a.x, b.x);
      ys[e] = fmin(a.y, b.y);
      ys[m + e] = fmax(a.y, b.y);
      atomicAdd(&deg[uv.x], 1);
      atomicAdd(&deg[uv.y], 1);
      keys[e] = (int)uv.x;
      keys[m + e] = (int)uv.y;
      vals[e] = (int)e;
      vals[m + e] = (int)e;
    } else {
      // padding: zero coordinates, empty bbox (never overlaps), unique ids
      r.ax = r.ay = r.bx = r.by = r.abx = r.aby = 0.0;
      r.rxmin = r.rymin = 0x7fffffff;
      r.rxmax = r.rymax = -1;
      rv.theta[e] = 0.0;
      rv.ids[e] = make_int2(-1 - (int)(e - m), -1 - (int)(e - m));
      rv.newc[e] = 1;
    }
    rv.rec[e] = r;
  }
}

// lower_bound with double comparisons: equal values (and -0.0/+0.0) share a
// rank and rank order equals double order.
__device__ inline int lower_rank(const double *sorted, int64_t len, double v) {
  int64_t lo = 0, hi = len;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (sorted[mid] < v) lo = mid + 1; else hi = mid;
  }
  return (int)lo;
}

__global__ void rank_kernel(int64_t m, RecView rv, const double *xs, const double *ys,
                            const double *sx, const double *sy) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    EdgeRec *r = &rv.rec[e];
    r->rxmin = lower_rank(sx, 2 * m, xs[e]);
    r->rxmax = lower_rank(sx, 2 * m, xs[m + e]);
    r->rymin = lower_rank(sy, 2 * m, ys[e]);
    r->rymax = lower_rank(sy, 2 * m, ys[m + e]);
  }
}

// Adjacent-pair work units per vertex: the C(deg,2) pairs of its incidence
// list, tiled kAdjTile x kAdjTile over the upper triangle.
__global__ void adj_units_kernel(const int *__restrict__ deg, int64_t n, long long *wunits) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v <= n;
       v += (int64_t)gridDim.x * blockDim.x) {
    long long d = v < n ? deg[v] : 0;
    long long T = (d + kAdjTile - 1) / kAdjTile;
    wunits[v] = d >= 2 ? T * (T + 1) / 2 : 0;
  }
}

// max |c| and min nonzero |c| over all coordinates, as ordered bit patterns.
__global__ void magnitude_kernel(const double *__restrict__ xy, int64_t count,
                                 unsigned long long *maxb, unsigned long long *minb) {
  unsigned long long mx = 0, mn = ~0ull;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long b = (unsigned long long)__double_as_longlong(fabs(xy[i]));
    mx = b > mx ? b : mx;
    if (b != 0) mn = b < mn ? b : mn;
  }
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long a = __shfl_down_sync(0xffffffffu, mx, o);
    unsigned long long c = __shfl_down_sync(0xffffffffu, mn, o);
    mx = a > mx ? a : mx;
    mn = c < mn ? c : mn;
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(maxb, mx);
    atomicMin(minb, mn);
  }
}

__global__ void header_kernel(RecHeader *hdr, int64_t n, int64_t m, int64_t m_pad,
                              const unsigned long long *maxb, const unsigned long long *minb) {
  unsigned long long mx = *maxb, mn = *minb;
  double dmx = __longlong_as_double((long long)mx);
  double dmn = mn == ~0ull ? 1.0 : __longlong_as_double((long long)mn);
  hdr->n = n;
  hdr->m = m;
  hdr->m_pad = m_pad;
  hdr->maxabs_bits = mx;
  hdr->minabs_bits = mn;
  const int ok = (dmx <= kMaxAbsFast && dmn >= kMinAbsFast) ? 1 : 0;
  hdr->admissible = ok;
  hdr->fast = ok ? kModeFastDefault : kModeGeneral;
}

// Filter records (FTile).  x0/y0 = smallest endpoint coordinate, W = largest
// extent rounded up, s = 2^-(ilogb(W)+2) so that (x - x0) * s lies in
// [0, 1/2] after the (monotone) roundings.  Per edge, with L = |abx| + |aby|
// of the FP32 direction: every cross product c of a point with the edge's
// line, evaluated in FP32 from these records, is within E = 2^-23 (1 + 3L)
// of the exact one (2x the bound derived in DESIGN.md, which also covers the
// reference's own FP64 rounding) and |c| <= C = L/2 (1 + 2^-20) + E.  The
// direction and line constant are scaled by sigma <= 1/sqrt(E C (1 + 2^-20))
// (FP32, rounded down; the scaling rounding is part of E), so a product of
// two scaled cross products above 1 in magnitude certifies both signs.
// Degenerate FP32 directions (L == 0) get zeros: products 0, never certain.
__global__ void frec_kernel(int64_t m, int64_t m_pad, RecView rv, const double *sx,
                            const double *sy) {
  const double x0 = sx[0], y0 = sy[0];
  const double W = fmax(__dsub_ru(sx[2 * m - 1], x0), __dsub_ru(sy[2 * m - 1], y0));
  const double s = (W > 0.0 && W <= 0x1p1000) ? ldexp(1.0, -(ilogb(W) + 2)) : 1.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m_pad;
       e += (int64_t)gridDim.x * blockDim.x) {
    float f[kFFields] = {0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
    double theta = 0.0;
    if (e < m) {
      const EdgeRec r = rv.rec[e];
      const float ax = __double2float_rn(__dmul_rn(__dsub_rn(r.ax, x0), s));
      const float ay = __double2float_rn(__dmul_rn(__dsub_rn(r.ay, y0), s));
      const float bx = __double2float_rn(__dmul_rn(__dsub_rn(r.bx, x0), s));
      const float by = __double2float_rn(__dmul_rn(__dsub_rn(r.by, y0), s));
      const float abx = __fsub_rn(bx, ax), aby = __fsub_rn(by, ay);
      // ka = ab x a: products of FP32 values are exact in FP64, one rounding
      const double ka = __dsub_rn(__dmul_rn((double)abx, (double)ay),
                                  __dmul_rn((double)aby, (double)ax));
      const double L = fabs((double)abx) + fabs((double)aby);
      f[kFAx] = ax; f[kFAy] = ay; f[kFBx] = bx; f[kFBy] = by;
      if (L > 0.0) {
        // E: error bound of a scaled cross product (relative to the scale),
        // C: its magnitude bound; scale sigma <= 1/sqrt(E C (1+u)) so that
        // |product of two| > 1 certifies both signs
        const double E = 0x1p-23 * (1.0 + 3.0 * L);
        const double C = 0.5 * L * (1.0 + 0x1p-20) + E;
        const double tau = E * C * (1.0 + 0x1p-20);
        const float sig = __double2float_rd((1.0 / sqrt(tau)) * (1.0 - 0x1p-40));
        f[kFSabx] = __double2float_rn((double)abx * (double)sig);
        f[kFNsaby] = -__double2float_rn((double)aby * (double)sig);
        f[kFNska] = -__double2float_rn(ka * (double)sig);
      }
      theta = rv.theta[e];
    }
    FTile &t = rv.ftile[e / kTile];
    const int slot = (int)(e % kTile);
    const int sl = slot / (32 * kFK), kk = (slot % (32 * kFK)) / 32, ln = slot % 32;
    const int P = (sl * kFGroups + kk / 2) * 32 + ln, h = kk & 1;
#pragma unroll
    for (int k = 0; k < kFFields; ++k) reinterpret_cast<float *>(&t.v[k][P])[h] = f[k];
    t.theta[slot] = theta;
    jrec_store(rv.jrec, e, f[kFAx], f[kFAy], f[kFBx], f[kFBy], f[kFSabx], f[kFNsaby],
               f[kFNska]);
  }
}

// One CTA (kTile threads) per tile: box of the real edges' scaled endpoints
// and max L (pad edges are skipped; an all-pad tile gets an empty box).
__global__ void __launch_bounds__(kTile) tile_fbox_kernel(int64_t m, RecView rv) {
  __shared__ float red[7][kTile / 32];
  __shared__ int2 first;
  __shared__ int star_ok[2];
  const int64_t e = (int64_t)blockIdx.x * kTile + threadIdx.x;
  if (threadIdx.x == 0) {
    first = rv.ids[(int64_t)blockIdx.x * kTile];  // a real edge unless the tile is all pad
    star_ok[0] = star_ok[1] = 1;
  }
  __syncthreads();
  float xlo = INFINITY, xhi = -INFINITY, ylo = INFINITY, yhi = -INFINITY, l = 0.0f;
  float tlo = INFINITY, thi = -INFINITY;
  if (e < m) {
    const float4 j = jrec_points(rv.jrec, e);
    xlo = fminf(j.x, j.z); xhi = fmaxf(j.x, j.z);
    ylo = fminf(j.y, j.w); yhi = fmaxf(j.y, j.w);
    // L of the FP32 direction (exact float differences, rounded up)
    l = __fadd_ru(fabsf(__fsub_rn(j.z, j.x)), fabsf(__fsub_rn(j.w, j.y)));
    const double th = rv.theta[e];
    tlo = __double2float_rd(th);
    thi = __double2float_ru(th);
    const int2 id = rv.ids[e];
    if (id.x != first.x && id.y != first.x) star_ok[0] = 0;
    if (id.x != first.y && id.y != first.y) star_ok[1] = 0;
  }
  for (int o = 16; o > 0; o >>= 1) {
    xlo = fminf(xlo, __shfl_down_sync(0xffffffffu, xlo, o));
    xhi = fmaxf(xhi, __shfl_down_sync(0xffffffffu, xhi, o));
    ylo = fminf(ylo, __shfl_down_sync(0xffffffffu, ylo, o));
    yhi = fmaxf(yhi, __shfl_down_sync(0xffffffffu, yhi, o));
    l = fmaxf(l, __shfl_down_sync(0xffffffffu, l, o));
    tlo = fminf(tlo, __shfl_down_sync(0xffffffffu, tlo, o));
    thi = fmaxf(thi, __shfl_down_sync(0xffffffffu, thi, o));
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    red[0][w] = xlo; red[1][w] = xhi; red[2][w] = ylo; red[3][w] = yhi; red[4][w] = l;
    red[5][w] = tlo; red[6][w] = thi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < kTile / 32; ++i) {
      xlo = fminf(xlo, red[0][i]); xhi = fmaxf(xhi, red[1][i]);
      ylo = fminf(ylo, red[2][i]); yhi = fmaxf(yhi, red[3][i]);
      l = fmaxf(l, red[4][i]);
      tlo = fminf(tlo, red[5][i]); thi = fmaxf(thi, red[6][i]);
    }
    TileBox b;
    b.xlo = xlo; b.xhi = xhi; b.ylo = ylo; b.yhi = yhi; b.lmax = l;
    b.thlo = tlo; b.thhi = thi;
    // all-pad tile (first id negative): no star
    b.star = first.x < 0 ? -1 : star_ok[0] ? first.x : star_ok[1] ? first.y : -1;
    rv.tbox[blockIdx.x] = b;
  }
}

// Certification threshold of a unit (tiles ti, tj).  With D = the larger
// side of the union of the two tile boxes (so |p - a| <= D per axis for
// every pair of the unit) and Lm = the larger tile lmax, the cross-product
// error and magnitude bounds become E_u = 2^-23 (1.5 D + 3 L) and C_u = L D +
// E_u, and a product above t = (1.5 D + 3 Lm)(3.5 D + 3 Lm)
// (1 + 2^-18) >= sigma^2 E_u C_u (1 + 2^-20) certifies both signs; t is
// capped at 1 (the unit-independent bound) and rounded up to FP32.
__device__ inline float unit_threshold(const TileBox &a, const TileBox &b) {
  const double D = fmax((double)fmaxf(a.xhi, b.xhi) - (double)fminf(a.xlo, b.xlo),
                        (double)fmaxf(a.yhi, b.yhi) - (double)fminf(a.ylo, b.ylo));
  const double Lm = (double)fmaxf(a.lmax, b.lmax);
  if (!(D >= 0.0)) return 1.0f;  // an empty box (all-pad tile): keep the global bound
  const double t = (1.5 * D + 3.0 * Lm) * (3.5 * D + 3.0 * Lm) * (1.0 + 0x1p-18);
  return t >= 1.0 ? 1.0f : __double2float_ru(t);
}

__global__ void set_mode_kernel(RecHeader *hdr, int mode) {
  hdr->fast = (mode != kModeGeneral && hdr->admissible) ? mode : kModeGeneral;
}

// ------------------------------------------------------------ pair kernels --

template <bool IDS>
struct IRegs {
  double ax[kK], ay[kK], bx[kK], by[kK], abx[kK], aby[kK], th[kK];
  int rx0[kK], rx1[kK], ry0[kK], ry1[kK];
  int u[IDS ? kK : 1], v[IDS ? kK : 1];
};

template <bool IDS, bool ANGLE>
__device__ inline void load_i(IRegs<IDS> &R, const EdgeRec *__restrict__ rec,
                              const double *__restrict__ theta, const int2 *__restrict__ ids,
                              uint64_t ti) {
#pragma unroll
  for (int k = 0; k < kK; ++k) {
    const int64_t e = (int64_t)ti * kTile + threadIdx.x + k * kThreads;
    const double4 *p = reinterpret_cast<const double4 *>(rec + e);
    double4 q0 = p[0];
    double2 q1 = reinterpret_cast<const double2 *>(rec + e)[2];
    int4 rk = reinterpret_cast<const int4 *>(rec + e)[3];
    R.ax[k] = q0.x; R.ay[k] = q0.y; R.bx[k] = q0.z; R.by[k] = q0.w;
    R.abx[k] = q1.x; R.aby[k] = q1.y;
    R.rx0[k] = rk.x; R.rx1[k] = rk.y; R.ry0[k] = rk.z; R.ry1[k] = rk.w;
    if (IDS) {
      int2 id = ids[e];
      R.u[k] = id.x; R.v[k] = id.y;
    }
    R.th[k] = ANGLE ? theta[e] : 0.0;
  }
}

__device__ inline float hi_view(double c) { return __int_as_float(__double2hiint(c)); }

// ideal - min(d, pi - d) with d = |t1 - t2| (its absolute value is the
// pair's deviation): the reference's own operation sequence
// (geometry.py:107-110, exact.py:219-221), so every pair's deviation is
// bit-identical to numpy's for the same axis angles.  For d in [0, pi]
// (pi = 2 fl(pi/2) exactly), min(d, fl(pi - d)) == (d <= fl(pi/2) ? d :
// fl(pi - d)) by monotone rounding: one compare instead of a NaN-aware min.
// Symmetric in (t1, t2) bit for bit.
__device__ inline double angle_dev_signed(double t1, double t2, double ideal) {
  const double HALF_PI = 1.5707963267948966, PI = 3.141592653589793;
  const double d = fabs(__dsub_rn(t1, t2));
  const double a = d <= HALF_PI ? d : __dsub_rn(PI, d);
  return __dsub_rn(ideal, a);
}
__device__ inline double angle_dev(double t1, double t2, double ideal) {
  return fabs(angle_dev_signed(t1, t2, ideal));
}
// The same deviation as ||pi/2 - d| - kappa|, kappa = fl(pi/2 - ideal):
// 3 DADD and no select, within 2^-50 of angle_dev (each of the two
// formulas is within 2^-51 of the exact function of the rounded d).  The
// filter kernel's general units use it; a warp-slice whose mean deviation
// per hit is below 2^-16 -- where 2^-50 per pair could exceed 1e-9 of the
// sum -- is re-evaluated with angle_dev by cross_fixup_kernel.
__device__ inline double angle_dev_fast_signed(double t1, double t2, double kappa) {
  const double HALF_PI = 1.5707963267948966;
  const double d = __dsub_rn(t1, t2);
  const double e = __dsub_rn(HALF_PI, fabs(d));
  return __dsub_rn(fabs(e), kappa);
}

// One j-edge against the thread's K i-edges.  FAST selects the float-view
// sign test and skips the vertex-id test (corrected by adj_kernel); otherwise
// the doubles are compared directly (NaN -> false, as numpy) and ids are
// tested.  DIAG masks pairs with j <= i inside a diagonal tile.
template <bool FAST, bool ANGLE, bool DIAG>
__device__ inline void pair_row(const IRegs<!FAST> &R, const EdgeRec *sj, const double *sth,
                                const int2 *sid, int jj, unsigned (&cnt)[kK],
                                double (&dev)[kK], double ideal) {
  const double4 cq = reinterpret_cast<const double4 *>(sj + jj)[0];
  const double2 cdq = reinterpret_cast<const double2 *>(sj + jj)[2];
  const int4 rk = reinterpret_cast<const int4 *>(sj + jj)[3];
  const double cx = cq.x, cy = cq.y, dx = cq.z, dy = cq.w;
  const double cdx = cdq.x, cdy = cdq.y;
  const double thj = ANGLE ? sth[jj] : 0.0;
  int2 idj = make_int2(0, 0);
  if (!FAST) idj = sid[jj];
#pragma unroll
  for (int k = 0; k < kK; ++k) {
    // closed bbox overlap via exact ranks (exact.py:191-194)
    bool ok = (rk.y >= R.rx0[k]) & (R.rx1[k] >= rk.x) & (rk.w >= R.ry0[k]) & (R.ry1[k] >= rk.z);
    if (!FAST)  // no shared vertex index (exact.py:205-210)
      ok &= (R.u[k] != idj.x) & (R.u[k] != idj.y) & (R.v[k] != idj.x) & (R.v[k] != idj.y);
    if (DIAG) ok &= jj > (int)threadIdx.x + k * kThreads;
    // coordinate differences: (cx-ax), (cy-ay), (dx-ax), (dy-ay), (bx-cx), (by-cy)
    const double dcx = __dsub_rn(cx, R.ax[k]);
    const double dcy = __dsub_rn(cy, R.ay[k]);
    const double ddx = __dsub_rn(dx, R.ax[k]);
    const double ddy = __dsub_rn(dy, R.ay[k]);
    const double ebx = __dsub_rn(R.bx[k], cx);
    const double eby = __dsub_rn(R.by[k], cy);
    // geometry.py:71-76, same roundings:
    const double c1 = __dsub_rn(__dmul_rn(R.abx[k], dcy), __dmul_rn(R.aby[k], dcx));
    const double c2 = __dsub_rn(__dmul_rn(R.abx[k], ddy), __dmul_rn(R.aby[k], ddx));
    const double c3 = __dsub_rn(__dmul_rn(cdy, dcx), __dmul_rn(cdx, dcy));
    const double c4 = __dsub_rn(__dmul_rn(cdx, eby), __dmul_rn(cdy, ebx));
    bool hit;
    if (FAST) {
      // sign(f1*f2) = sign(c1)*sign(c2), zero iff c1 or c2 is zero; the
      // product never underflows or turns NaN inside the fast window
      const float p12 = __fmul_rn(hi_view(c1), hi_view(c2));
      const float p34 = __fmul_rn(hi_view(c3), hi_view(c4));
      hit = ok & (p12 <= 0.0f) & (p34 <= 0.0f);
    } else {
      const bool s_cd = ((c1 <= 0.0) & (c2 >= 0.0)) | ((c1 >= 0.0) & (c2 <= 0.0));
      const bool s_ab = ((c3 <= 0.0) & (c4 >= 0.0)) | ((c3 >= 0.0) & (c4 <= 0.0));
      hit = ok & s_cd & s_ab;
    }
    cnt[k] += hit ? 1u : 0u;
    if (ANGLE) {
      const double t = angle_dev(R.th[k], thj, ideal);
      if (hit) dev[k] = __dadd_rn(dev[k], t);
    }
  }
}

// Terms of a pair that depend on the i-edge and only the FIRST endpoint c of
// the j-edge: (a,c) and (b,c) differences and c1 (as its float view).  The
// j-tile is sorted by first endpoint, so consecutive j-edges sharing c reuse
// them -- the `snew` flag is the same for every lane (j is broadcast), so the
// branch never diverges.  Per pair this leaves 2 DADD (d - a) + 3 x (2 DMUL +
// 1 DADD) for c2, c3, c4 = 11 FP64 instead of 18, bit-identical values.
struct SRegs {
  double dcx[kK], dcy[kK], ebx[kK], eby[kK];
  float f1[kK];
};

// Hit test tail in PTX so it maps 1:1 onto ISETP/FSETP predicate chains and
// predicated adds: bbox ranks (4 compares) AND p12 <= 0 AND p34 <= 0 AND the
// diagonal mask, then @hit cnt += 1 (and dev += t).
__device__ inline void tail_count(unsigned &cnt, int jx1, int ix0, int ix1, int jx0, int jy1,
                                  int iy0, int iy1, int jy0, float p12, float p34, int diag_ok) {
  asm("{\n\t.reg .pred p;\n\t"
      "setp.ge.s32 p, %1, %2;\n\t"
      "setp.ge.and.s32 p, %3, %4, p;\n\t"
      "setp.ge.and.s32 p, %5, %6, p;\n\t"
      "setp.ge.and.s32 p, %7, %8, p;\n\t"
      "setp.le.and.f32 p, %9, 0f00000000, p;\n\t"
      "setp.le.and.f32 p, %10, 0f00000000, p;\n\t"
      "setp.ne.and.s32 p, %11, 0, p;\n\t"
      "@p add.u32 %0, %0, 1;\n\t}"
      : "+r"(cnt)
      : "r"(jx1), "r"(ix0), "r"(ix1), "r"(jx0), "r"(jy1), "r"(iy0), "r"(iy1), "r"(jy0),
        "f"(p12), "f"(p34), "r"(diag_ok));
}

__device__ inline void tail_count_dev(unsigned &cnt, double &dev, double t, int jx1, int ix0,
                                      int ix1, int jx0, int jy1, int iy0, int iy1, int jy0,
                                      float p12, float p34, int diag_ok) {
  asm("{\n\t.reg .pred p;\n\t"
      "setp.ge.s32 p, %2, %3;\n\t"
      "setp.ge.and.s32 p, %4, %5, p;\n\t"
      "setp.ge.and.s32 p, %6, %7, p;\n\t"
      "setp.ge.and.s32 p, %8, %9, p;\n\t"
      "setp.le.and.f32 p, %10, 0f00000000, p;\n\t"
      "setp.le.and.f32 p, %11, 0f00000000, p;\n\t"
      "setp.ne.and.s32 p, %12, 0, p;\n\t"
      "@p add.u32 %0, %0, 1;\n\t"
      "@p add.rn.f64 %1, %1, %13;\n\t}"
      : "+r"(cnt), "+d"(dev)
      : "r"(jx1), "r"(ix0), "r"(ix1), "r"(jx0), "r"(jy1), "r"(iy0), "r"(iy1), "r"(jy0),
        "f"(p12), "f"(p34), "r"(diag_ok), "d"(t));
}

template <bool ANGLE, bool DIAG>
__device__ inline void pair_row_fast(const IRegs<false> &R, SRegs &S, const EdgeRec *sj,
                                     const double *sth, const int *snew, int jj,
                                     unsigned (&cnt)[kK], double (&dev)[kK], double ideal) {
  const double4 cq = reinterpret_cast<const double4 *>(sj + jj)[0];
  const double2 cdq = reinterpret_cast<const double2 *>(sj + jj)[2];
  const int4 rk = reinterpret_cast<const int4 *>(sj + jj)[3];
  const double cx = cq.x, cy = cq.y, dx = cq.z, dy = cq.w;
  const double cdx = cdq.x, cdy = cdq.y;
  const double thj = ANGLE ? sth[jj] : 0.0;
  if (snew[jj]) {
#pragma unroll
    for (int k = 0; k < kK; ++k) {
      S.dcx[k] = __dsub_rn(cx, R.ax[k]);
      S.dcy[k] = __dsub_rn(cy, R.ay[k]);
      S.ebx[k] = __dsub_rn(R.bx[k], cx);
      S.eby[k] = __dsub_rn(R.by[k], cy);
      S.f1[k] = hi_view(__dsub_rn(__dmul_rn(R.abx[k], S.dcy[k]), __dmul_rn(R.aby[k], S.dcx[k])));
    }
  }
#pragma unroll
  for (int k = 0; k < kK; ++k) {
    bool ok = (rk.y >= R.rx0[k]) & (R.rx1[k] >= rk.x) & (rk.w >= R.ry0[k]) & (R.ry1[k] >= rk.z);
    if (DIAG) ok &= jj > (int)threadIdx.x + k * kThreads;
    const double ddx = __dsub_rn(dx, R.ax[k]);
    const double ddy = __dsub_rn(dy, R.ay[k]);
    const double c2 = __dsub_rn(__dmul_rn(R.abx[k], ddy), __dmul_rn(R.aby[k], ddx));
    const double c3 = __dsub_rn(__dmul_rn(cdy, S.dcx[k]), __dmul_rn(cdx, S.dcy[k]));
    const double c4 = __dsub_rn(__dmul_rn(cdx, S.eby[k]), __dmul_rn(cdy, S.ebx[k]));
    const float p12 = __fmul_rn(S.f1[k], hi_view(c2));
    const float p34 = __fmul_rn(hi_view(c3), hi_view(c4));
#ifdef GLR_XPTXTAIL
    (void)ok;
    const int diag_ok = DIAG ? (jj > (int)threadIdx.x + k * kThreads) : 1;
    if (ANGLE)
      tail_count_dev(cnt[k], dev[k], angle_dev(R.th[k], thj, ideal), rk.y, R.rx0[k], R.rx1[k],
                     rk.x, rk.w, R.ry0[k], R.ry1[k], rk.z, p12, p34, diag_ok);
    else
      tail_count(cnt[k], rk.y, R.rx0[k], R.rx1[k], rk.x, rk.w, R.ry0[k], R.ry1[k], rk.z, p12,
                 p34, diag_ok);
#else
    const bool hit = ok & (p12 <= 0.0f) & (p34 <= 0.0f);
    cnt[k] += hit ? 1u : 0u;
    if (ANGLE) {
      const double t = angle_dev(R.th[k], thj, ideal);
      if (hit) dev[k] = __dadd_rn(dev[k], t);
    }
#endif
  }
}

// ------------------------------------------------ certified FP32 filter --
//
// Packed-FP32 (FFMA2/FMUL2/FADD2) evaluation of the four cross products of
// two i-edges against one j-edge per instruction.  With the FTile scaling,
// c1^ = 2^ki c1~, c2^ = 2^ki c2~ (ki from edge i), c3^, c4^ with kj, where
// |c~ - c_exact| <= E = 2^-21 for every c (error analysis in DESIGN.md,
// including the FP64 rounding of the reference's own c), and |c~| <= C.
// P12 = fl(c1^ c2^) > 1 in magnitude therefore implies |c1~|, |c2~| > E, so
// sign(c1_fp64) = sign(c1~) != 0 (same for c2), and likewise P34.  With
// M = max(P12, P34):
//   M < -1  : both pairs strictly straddle in exact arithmetic, so the
//             segments cross properly -> bboxes overlap, no shared vertex
//             (a shared vertex makes one exact c zero): the reference counts
//             the pair;
//   M > 1   : one pair certainly does not straddle: not counted;
//   |M| <= 1: uncertain -> exact FP64 evaluation (exact_pair) of the
//             reference predicate for that pair.
// The fast window (hdr->admissible) guarantees the reference's FP64
// products c1*c2 never underflow, so its test equals the sign test.

__device__ __forceinline__ uint64_t f2_pack(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ uint64_t f2_bcast(float a) { return f2_pack(a, a); }
__device__ __forceinline__ float f2_lo(uint64_t v) {
  float lo;
  asm("mov.b64 {%0, _}, %1;" : "=f"(lo) : "l"(v));
  return lo;
}
__device__ __forceinline__ float f2_hi(uint64_t v) {
  float hi;
  asm("mov.b64 {_, %0}, %1;" : "=f"(hi) : "l"(v));
  return hi;
}
__device__ __forceinline__ uint64_t f2_mul(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t f2_fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}

constexpr int kGroups = kFGroups;  // packed i-edge pairs per lane

struct FIRegs {
  uint64_t ax[kGroups], ay[kGroups], bx[kGroups], by[kGroups];
  uint64_t sabx[kGroups], nsaby[kGroups], nska[kGroups];
};

// Lane `lane` of slice `slice`: i-edge k is tile slot fslot(slice, k, lane);
// group g holds k = 2g (low half) and 2g + 1 (high half), one 64-bit load.
template <bool ANGLE>
__device__ inline void load_fi(FIRegs &R, const FTile *__restrict__ ftile, uint64_t ti,
                               int slice, int lane) {
  const FTile &t = ftile[ti];
#pragma unroll
  for (int g = 0; g < kGroups; ++g) {
    const int P = (slice * kFGroups + g) * 32 + lane;
    const uint64_t *v = reinterpret_cast<const uint64_t *>(&t.v[0][P]);
    constexpr int kField = kTile / 2;  // uint64 stride between fields
    R.ax[g] = v[kFAx * kField];
    R.ay[g] = v[kFAy * kField];
    R.bx[g] = v[kFBx * kField];
    R.by[g] = v[kFBy * kField];
    R.sabx[g] = v[kFSabx * kField];
    R.nsaby[g] = v[kFNsaby * kField];
    R.nska[g] = v[kFNska * kField];
  }
}

// Signed units.  If a unit's theta difference dt = theta_j - theta_i keeps
// one side of 0 and of +-pi/2 for every pair (tile theta bounds, e.g. after
// glr_theta_sort_edges), a = min(|dt|, pi - |dt|) is one affine branch and
// |ideal - a| = |theta_j - (theta_i + s)| with
//   dt in [0, pi/2]: s = ideal          dt in [pi/2, pi): s = pi - ideal
//   dt in [-pi/2, 0]: s = -ideal        dt in (-pi, -pi/2]: s = ideal - pi.
// If the dt range also keeps kSignMargin away from s (return 1), every
// pair's v = theta_j - (theta_i + s) has the sign *sigma, and the lane's
// deviation sum over hits is
//   sigma * (sum_j h_j theta_j - sum_k C_k x_k),  x_k = theta_i_k + s,
// with h_j the lane's hits on j-edge j and C_k those of i-edge k: one DFMA
// per j-edge (4 pairs) instead of the per-pair formula.  Rounding: the sum
// of at most kTile terms of at most kFK pi each loses <= kTile kFK pi 2^-53
// per hit, against a deviation of >= kSignMargin per hit: relative error
// <= 256 * 4 pi 2^-53 / 2^-8 < 1e-10 (tests/test_filter_bound.py).  Every
// other unit (0: within the margin of s; -1: straddles a branch point)
// evaluates the reference's per-pair formula (angle_dev), so small
// deviations are bit-identical to numpy's.
constexpr double kSignMargin = 0x1p-8;
__device__ inline int range_shift(float athlo, float athhi, float bthlo, float bthhi,
                                  double ideal, double *s, double *sigma) {
  const double HALF_PI = 1.5707963267948966, PI = 3.141592653589793;
  // float bounds are outward-rounded; their double differences are exact
  // or off by far less than kSignMargin
  const double lo = (double)bthlo - (double)athhi, hi = (double)bthhi - (double)athlo;
  if (!(lo <= hi)) return -1;  // empty tile
  double sh;
  if (lo >= 0.0 && hi <= HALF_PI) sh = ideal;
  else if (lo >= HALF_PI) sh = __dsub_rn(PI, ideal);
  else if (hi <= 0.0 && lo >= -HALF_PI) sh = -ideal;
  else if (hi <= -HALF_PI) sh = __dsub_rn(ideal, PI);
  else return -1;
  *s = sh;
  if (hi <= sh - kSignMargin) { *sigma = -1.0; return 1; }
  if (lo >= sh + kSignMargin) { *sigma = 1.0; return 1; }
  return 0;
}
__device__ inline int unit_shift(const TileBox &a, const TileBox &b, double ideal, double *s,
                                 double *sigma) {
  return range_shift(a.thlo, a.thhi, b.thlo, b.thhi, ideal, s, sigma);
}

// One-kink units.  The deviation f(dt) = |ideal - min(|dt|, pi - |dt|)| is
// piecewise linear on (-pi, pi) with kinks at 0, +-ideal, +-pi/2, +-(pi -
// ideal).  A unit whose dt range holds at most ONE kink beta and keeps
// kSignMargin away from beta's two neighbours has, for every pair,
//   f = |dt - beta|                    beta = +-ideal, +-(pi - ideal)
//   f = f(beta) - |dt - beta|          beta = 0 (f(beta) = ideal), +-pi/2
//                                      (f(beta) = pi/2 - ideal),
// so with x_k = theta_i_k + beta a pair costs v = theta_j - x_k and |v| in
// the accumulate (2 DADD instead of the general formula's 4), and the
// second kind finishes as hits * f(beta) - sum |v| (every term f(beta) - |v|
// >= kSignMargin: the cancellation costs < 2^-44 relative).  Rounding
// differs from exact.py's by a few ulps of pi per pair; a slice whose mean
// deviation per hit is below kFixupMeanDev is re-evaluated with the
// reference formula like every fast-formula slice (cross_fixup_kernel).
// Returns 1 and (*beta, *fbeta, *minus) or 0.
__device__ inline int range_kink(float athlo, float athhi, float bthlo, float bthhi,
                                 double ideal, double *beta, double *fbeta, int *minus) {
  const double HALF_PI = 1.5707963267948966, PI = 3.141592653589793;
  const double lo = (double)bthlo - (double)athhi, hi = (double)bthhi - (double)athlo;
  if (!(lo <= hi)) return 0;
  const double pmi = __dsub_rn(PI, ideal), hmi = __dsub_rn(HALF_PI, ideal);
  // kinks in ascending order, -pi and pi as outer neighbours (not kinks of f
  // on (-pi, pi): no margin there); written out so that nothing is indexed
  const double mg = kSignMargin;
#define GLR_KINK(LEFT, B, RIGHT, MINUS, FB)                      \
  if (lo >= (LEFT) && hi <= (RIGHT)) {                           \
    *beta = (B); *minus = (MINUS); *fbeta = (FB);                \
    return 1;                                                    \
  }
  GLR_KINK(-PI, -pmi, -HALF_PI - mg, 0, hmi)
  GLR_KINK(-pmi + mg, -HALF_PI, -ideal - mg, 1, hmi)
  GLR_KINK(-HALF_PI + mg, -ideal, -mg, 0, hmi)
  GLR_KINK(-ideal + mg, 0.0, ideal - mg, 1, ideal)
  GLR_KINK(mg, ideal, HALF_PI - mg, 0, hmi)
  GLR_KINK(ideal + mg, HALF_PI, pmi - mg, 1, hmi)
  GLR_KINK(HALF_PI + mg, pmi, PI, 0, hmi)
#undef GLR_KINK
  return 0;
}

// Exact reference predicate for one pair (general semantics: doubles
// compared directly, ids tested), used for the filter's uncertain pairs.
// Returns -1 for no hit, else the pair's angle deviation (0 without ANGLE).
template <bool ANGLE>
__device__ __forceinline__ double exact_pair(const EdgeRec *__restrict__ rec,
                                             const int2 *__restrict__ ids,
                                             const double *__restrict__ theta, int64_t ei,
                                             int64_t ej, double ideal) {
  const EdgeRec a = rec[ei], c = rec[ej];
  const int2 ia = ids[ei], ic = ids[ej];
  bool ok = (c.rxmax >= a.rxmin) & (a.rxmax >= c.rxmin) & (c.rymax >= a.rymin) &
            (a.rymax >= c.rymin);
  ok &= (ia.x != ic.x) & (ia.x != ic.y) & (ia.y != ic.x) & (ia.y != ic.y);
  const double dcx = __dsub_rn(c.ax, a.ax);
  const double dcy = __dsub_rn(c.ay, a.ay);
  const double ddx = __dsub_rn(c.bx, a.ax);
  const double ddy = __dsub_rn(c.by, a.ay);
  const double ebx = __dsub_rn(a.bx, c.ax);
  const double eby = __dsub_rn(a.by, c.ay);
  const double c1 = __dsub_rn(__dmul_rn(a.abx, dcy), __dmul_rn(a.aby, dcx));
  const double c2 = __dsub_rn(__dmul_rn(a.abx, ddy), __dmul_rn(a.aby, ddx));
  const double c3 = __dsub_rn(__dmul_rn(c.aby, dcx), __dmul_rn(c.abx, dcy));
  const double c4 = __dsub_rn(__dmul_rn(c.abx, eby), __dmul_rn(c.aby, ebx));
  const bool s_cd = ((c1 <= 0.0) & (c2 >= 0.0)) | ((c1 >= 0.0) & (c2 <= 0.0));
  const bool s_ab = ((c3 <= 0.0) & (c4 >= 0.0)) | ((c3 >= 0.0) & (c4 <= 0.0));
  if (!(ok & s_cd & s_ab)) return -1.0;
  return ANGLE ? angle_dev(theta[ei], theta[ej], ideal) : 0.0;
}

// M_k = max(P12, P34) of a j-edge (shared memory) against the thread's K
// i-edges; masked pairs of a diagonal tile get M = 2 (certain miss).
// Per pair: 8 FFMA + 2 FMUL/FFMA, issued as packed pairs (filter_m2).
// Shared-memory loads by 32-bit shared address (the stage base is computed
// once per unit, so the block loop carries no generic-to-shared conversions).
// volatile: never hoisted above the stage's mbarrier wait.
#ifndef GLR_LDS_ASM
#define GLR_LDS_ASM asm volatile
#endif
__device__ __forceinline__ float4 lds_f4(unsigned addr) {
  float4 v;
  GLR_LDS_ASM("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr));
  return v;
}
__device__ __forceinline__ double lds_f64(unsigned addr) {
  double v;
  GLR_LDS_ASM("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}

// FOLD (count-only kernel): M_k = max(RN(c1 c2 + t), RN(c3 c4 + t)) with
// the unit threshold t folded into the products' FFMA (RN keeps the sign of
// the exact value and is monotone; t and 2t are floats): M < 0 <=> both
// exact products < -t (certain hit), M > 2t => one exact product > t
// (certain miss), M in [0, 2t] uncertain -- the partition of
// max(RN(c1 c2), RN(c3 c4)) against -t and t, but the hit is M's sign bit
// (one LEA.HI) and the vote an unsigned minimum.  Masked pairs of a
// diagonal tile get M = 4 (t <= 1).  The fused kernel keeps FMUL2 products
// (its SEL needs a predicate anyway, and the third FFMA2 operand cost it
// 5%: 5.34 vs 5.08 s on C5).
// M of a PAIR of j-edges (jj, jj+1; jj even) against the lane's kFK i-edges,
// M2[h][k] for j-edge jj + h.  Mixed packing (the kernel is bound by
// register-file reads, tools/rf_model.py): c1, c2 (the i-edge's line at the
// two j-endpoints) are packed over the two j-edges -- the j coordinates are
// a register pair of the JPair layout and the i-line constants scalars (4
// reads instead of 5 in the inner FFMA2) -- while c3, c4 (the j-edge's line
// at the i-endpoints) stay packed over the lane's i-edge pair with the
// j-line constants as scalars.  The max of P12 and P34 is taken per 32-bit
// half, so the two packings meet there.  Identical roundings to filter_m.
template <bool DIAG, bool FOLD>
__device__ __forceinline__ void filter_m2(const FIRegs &R, unsigned jaddr, int jj, int islot,
                                          uint64_t T2, float (&M2)[2][kFK]) {
  const unsigned pa = jaddr + (unsigned)jj * (unsigned)sizeof(JRec);
  const float4 a0 = lds_f4(pa);       // cx0 cx1 cy0 cy1
  const float4 a1 = lds_f4(pa + 16);  // dx0 dx1 dy0 dy1
  const float4 a2 = lds_f4(pa + 32);  // scdx0 -scdy0 -skc0 scdx1
  const float4 a3 = lds_f4(pa + 48);  // -scdy1 -skc1 0 0
  const uint64_t CX = f2_pack(a0.x, a0.y), CY = f2_pack(a0.z, a0.w);
  const uint64_t DX = f2_pack(a1.x, a1.y), DY = f2_pack(a1.z, a1.w);
  const float scdx[2] = {a2.x, a2.w}, nscdy[2] = {a2.y, a3.x}, nskc[2] = {a2.z, a3.y};
#pragma unroll
  for (int g = 0; g < kGroups; ++g) {
    uint64_t p12[2], p34[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {  // i-edge 2g + h: its line over (j0, j1)
      const float sx = h ? f2_hi(R.sabx[g]) : f2_lo(R.sabx[g]);
      const float ny = h ? f2_hi(R.nsaby[g]) : f2_lo(R.nsaby[g]);
      const float nk = h ? f2_hi(R.nska[g]) : f2_lo(R.nska[g]);
      // c1 = ab x (c - a), c2 = ab x (d - a): fma(sabx, y, fma(-saby, x, -ska))
      const uint64_t c1 = f2_fma(f2_bcast(sx), CY, f2_fma(f2_bcast(ny), CX, f2_bcast(nk)));
      const uint64_t c2 = f2_fma(f2_bcast(sx), DY, f2_fma(f2_bcast(ny), DX, f2_bcast(nk)));
      p12[h] = FOLD ? f2_fma(c1, c2, T2) : f2_mul(c1, c2);
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {  // j-edge q: its line over the i-pair
      // c3 = cd x (a - c), c4 = cd x (b - c)
      const uint64_t c3 =
          f2_fma(f2_bcast(scdx[q]), R.ay[g], f2_fma(f2_bcast(nscdy[q]), R.ax[g], f2_bcast(nskc[q])));
      const uint64_t c4 =
          f2_fma(f2_bcast(scdx[q]), R.by[g], f2_fma(f2_bcast(nscdy[q]), R.bx[g], f2_bcast(nskc[q])));
      p34[q] = FOLD ? f2_fma(c3, c4, T2) : f2_mul(c3, c4);
    }
    // (i_h, j_q): p12[h] half q, p34[q] half h
#pragma unroll
    for (int q = 0; q < 2; ++q) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const float a = q ? f2_hi(p12[h]) : f2_lo(p12[h]);
        const float b = h ? f2_hi(p34[q]) : f2_lo(p34[q]);
        M2[q][2 * g + h] = FOLD ? __int_as_float(max(__float_as_int(a), __float_as_int(b)))
                                : fmaxf(a, b);
      }
    }
  }
  if (DIAG) {
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
      for (int k = 0; k < kFK; ++k)
        if (!(jj + q > islot + 32 * k)) M2[q][k] = FOLD ? 4.0f : 2.0f;
  }
}

// Uncertain pairs are not evaluated where they are found: each warp queues
// them in shared memory (16-bit entry = tile slot of the i-edge << 8 | j slot) and
// evaluates the queue with all 32 lanes at once (exact_pair's FP64 records
// come from L2: one round-trip per 32 pairs instead of per pair) at the end
// of the slice, or when the queue is full.  Results go to the lane's
// cnt[0]/dev[0]: the queue order and the drain points depend only on the
// slice, so sums stay deterministic.
constexpr unsigned kQCap = GLR_XFBLOCK_S > 4 ? 32 * GLR_XFBLOCK_S * 4 : 512;  // per warp (>= 32 lanes x NJ x kFK)
static_assert(kTile <= 256, "queue entries hold 8-bit tile slots");
template <bool ANGLE>
__device__ __forceinline__ void drain_queue(const unsigned short *wq, unsigned qn, unsigned lane,
                                         const EdgeRec *__restrict__ rec,
                                         const int2 *__restrict__ ids,
                                         const double *__restrict__ theta, int64_t ibase,
                                         int64_t jbase, double ideal, unsigned &cnt,
                                         double &dev) {
  __syncwarp();
  for (unsigned b = 0; b < qn; b += 32) {
    if (b + lane < qn) {
      const unsigned ent = wq[b + lane];  // i slot << 8 | j slot
      const int64_t ei = ibase + (ent >> 8), ej = jbase + (ent & 255u);
#ifndef GLR_XNOIDCHECK
      // a shared vertex index: never counted (exact.py:205-210), and most
      // uncertain pairs are such pairs (an exact cross product is 0) -- skip
      // exact_pair's random record loads for them
      const int2 ia = ids[ei], ic = ids[ej];
      if (ia.x == ic.x || ia.x == ic.y || ia.y == ic.x || ia.y == ic.y) continue;
#endif
      const double t = exact_pair<ANGLE>(rec, ids, theta, ei, ej, ideal);
      if (t >= 0.0) {
        cnt += 1u;
        if (ANGLE) dev = __dadd_rn(dev, t);
      }
    }
  }
  __syncwarp();
}

// NJ consecutive j-edges against the thread's K i-edges.  Certain hits are
// counted (and their angle deviations summed) with predicated adds; one
// warp vote per block decides whether any lane met an uncertain pair, and
// only then is the block re-filtered to queue those pairs, so the hot path
// has no branch inside the block and the compiler can interleave its NJ
// independent j-steps.
#ifdef GLR_XFSTATS
// debug build only: [vote blocks that fell back, uncertain pairs evaluated]
__device__ unsigned long long g_fstats[2];
#endif
// AM (angle mode of the unit): 0 the fast per-pair formula
// (angle_dev_fast_signed), 2 the signed form (unit_shift), 3 the reference's
// per-pair formula (angle_dev: cross_fixup_kernel); the count-only kernel
// uses 0.
template <bool ANGLE, bool DIAG, int NJ, int AM, bool T1 = false>
__device__ __forceinline__ void filter_block(const FIRegs &R, const double (&th)[kFK],
                                             unsigned jaddr,
                                             unsigned thaddr, int jj0, int islot, float thr_u,
                                             unsigned (&cnt)[kFK], double (&dev)[kFK],
                                             double (&A2)[2], double ideal, double kappa,
                                             const EdgeRec *__restrict__ rec,
                                             const int2 *__restrict__ ids,
                                             const double *__restrict__ theta, int64_t ibase,
                                             int64_t jbase, unsigned short *wq, unsigned &qn,
                                             unsigned &qc) {
  constexpr bool SIGNED = ANGLE && AM == 2;
#ifdef GLR_XGENNOFOLD
  constexpr bool FOLD = !ANGLE || SIGNED;
#else
  constexpr bool FOLD = true;  // every mode: the hit is M's sign bit
#endif
  // T1: the unit's threshold is the global bound 1 (every unit of a
  // domain-spanning tile order): a compile-time constant, so the FOLD
  // products take it as an immediate (one register read less per FFMA2)
  const float thr = T1 ? 1.0f : thr_u;
  const uint64_t T2 = f2_bcast(thr);
  // FOLD: uncertain <=> M in [+0, 2t] <=> M's bits <= 2t's bits (unsigned: a
  // negative M, a certain hit, lies above every non-negative float), so the
  // block vote is one unsigned minimum (VIMNMX3 per two pairs)
  const unsigned vbits = __float_as_uint(2.0f * thr);
  unsigned mmin = 0xffffffffu;
  bool any = false;
  static_assert(NJ % 2 == 0, "j-edges come in pairs (filter_m2)");
  float MB[NJ][kFK];
#pragma unroll
  for (int q = 0; q < NJ; q += 2)
    filter_m2<DIAG, FOLD>(R, jaddr, jj0 + q, islot, T2,
                          *reinterpret_cast<float (*)[2][kFK]>(&MB[q][0]));
#pragma unroll
  for (int q = 0; q < NJ; ++q) {
    float (&M)[kFK] = MB[q];
    const double thj = ANGLE ? lds_f64(thaddr + (jj0 + q) * 8u) : 0.0;
    if constexpr (SIGNED) {
      // hits are M's sign bits: C_k += hit (LEA.HI), h = hits on this j-edge,
      // A += h * theta_j (one DFMA per j-edge; unit_shift).  Short dependency
      // chains: pairwise hit sums, two alternating A accumulators, and the
      // vote minimum as a tree over the block (one chain per j-edge here).
      unsigned b[kFK];
#pragma unroll
      for (int k = 0; k < kFK; ++k) {
        b[k] = __float_as_uint(M[k]);
        cnt[k] += b[k] >> 31;
      }
      unsigned h = b[0] >> 31;
#pragma unroll
      for (int k = 1; k < kFK; ++k) h += b[k] >> 31;
      A2[q & (kA2 - 1)] = fma((double)h, thj, A2[q & (kA2 - 1)]);
      unsigned mq = b[0];
#pragma unroll
      for (int k = 1; k < kFK; ++k) mq = min(mq, b[k]);
      mmin = q == 0 ? mq : min(mmin, mq);
    } else {
#pragma unroll
    for (int k = 0; k < kFK; ++k) {
      if (FOLD) {
        mmin = min(mmin, __float_as_uint(M[k]));
      } else {
        any |= fabsf(M[k]) <= thr;
      }
      // hit: cnt += 1 (and dev += t)
      if (ANGLE) {
        // dev += hit ? t : 0 with t = |v|: a miss clears v's HIGH word only
        // (one SEL, in place), leaving {lo, 0}, a subnormal below 2^-1042.
        // A genuine deviation is 0 or at least 2^-766, so the
        // slice's sum is cleared when below 2^-900 and otherwise differs
        // from the masked sum by a relative 2^-265 at most (DADD, no zeroing
        // MOV or {0,1} multiplier per pair).
        double v = AM == 3 ? angle_dev_signed(th[k], thj, ideal)
                   : AM == 1 ? __dsub_rn(thj, th[k])  // one-kink units (range_kink)
                             : angle_dev_fast_signed(th[k], thj, kappa);
        if (FOLD) {  // hit <=> M's sign bit (an integer test: -0 is a hit)
          asm("{\n\t.reg .pred p;\n\t.reg .b32 lo, hi;\n\t"
              "setp.lt.s32 p, %2, 0;\n\t"
              "@p add.u32 %0, %0, 1;\n\t"
              "mov.b64 {lo, hi}, %1;\n\t"
              "selp.b32 hi, hi, 0, p;\n\t"
              "mov.b64 %1, {lo, hi};\n\t}"
              : "+r"(cnt[k % kCntAccAngle]), "+d"(v)
              : "r"(__float_as_int(M[k])));
        } else {
          asm("{\n\t.reg .pred p;\n\t.reg .b32 lo, hi;\n\t"
              "setp.lt.f32 p, %2, %3;\n\t"
              "@p add.u32 %0, %0, 1;\n\t"
              "mov.b64 {lo, hi}, %1;\n\t"
              "selp.b32 hi, hi, 0, p;\n\t"
              "mov.b64 %1, {lo, hi};\n\t}"
              : "+r"(cnt[k % kCntAccAngle]), "+d"(v)
              : "f"(M[k]), "f"(-thr));
        }
        dev[k % kDevAcc] = __dadd_rn(dev[k % kDevAcc], fabs(v));
      } else {
        // the sign bit of M is the hit (LEA.HI: one instruction)
        cnt[k % kCntAccCount] += __float_as_uint(M[k]) >> 31;
      }
    }
    }  // not SIGNED
  }
  if (__any_sync(0xffffffffu, FOLD ? mmin <= vbits : any)) {
    // the block's M values (still live) into a per-lane mask of its
    // uncertain pairs (bit q*kFK + k); a warp prefix sum places the lanes'
    // entries: positions depend only on lane and bit order (deterministic),
    // and the queue is drained by all 32 lanes at once
    unsigned U = 0;
#pragma unroll
    for (int q = 0; q < NJ; ++q)
#pragma unroll
      for (int k = 0; k < kFK; ++k) {
        const bool u = FOLD ? __float_as_uint(MB[q][k]) <= vbits : fabsf(MB[q][k]) <= thr;
        U |= (u ? 1u : 0u) << (q * kFK + k);
      }
    const unsigned lane = (unsigned)islot & 31u;
    const unsigned n = __popc(U);
    unsigned incl = n;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= (unsigned)o) incl += v;
    }
    const unsigned total = __shfl_sync(0xffffffffu, incl, 31);
#ifdef GLR_XFSTATS
    if (lane == 0) {
      atomicAdd(&g_fstats[0], 1ull);
      atomicAdd(&g_fstats[1], (unsigned long long)total);
    }
#endif
    if (qn + total > kQCap) {  // total <= 32 * NJ * kFK <= kQCap
      // queued hits: the signed form's C_k multiply x_k, so they count
      // apart (qc); their deviations go to dev[0], unused by that form
      // (one-kink units, AM 1: their filter hits multiply f(beta), so the
      // queued ones count apart too, deviations in A2[0], unused there)
      drain_queue<ANGLE>(wq, qn, lane, rec, ids, theta, ibase, jbase, ideal,
                         (SIGNED || AM == 1) ? qc : cnt[0], AM == 1 ? A2[0] : dev[0]);
      qn = 0;
    }
    unsigned pos = qn + incl - n;
    while (U != 0u) {
      const int b = __ffs(U) - 1;
      U &= U - 1u;
      wq[pos++] = (unsigned short)(((unsigned)(islot + 32 * (b % kFK)) << 8) |
                                   (unsigned)(jj0 + b / kFK));
    }
    qn += total;
  }
}

template <bool FAST, bool ANGLE>
__global__ void __launch_bounds__(kThreads, kMinBlocks)
cross_pairs_kernel(const RecHeader *__restrict__ hdr, const EdgeRec *__restrict__ rec,
                   const double *__restrict__ theta, const int2 *__restrict__ ids,
                   const int *__restrict__ newc, const int2 *__restrict__ ulist, uint64_t T,
                   uint64_t W, uint64_t ubeg, uint64_t uend, uint64_t chunk,
                   unsigned srank, unsigned sworld, double ideal, int filter_ok,
                   unsigned long long *__restrict__ cta_cnt, double *__restrict__ cta_dev) {
  // ulist == nullptr: units are the implicit upper triangle of tile pairs;
  // otherwise unit u is the explicit tile pair ulist[u] (culled candidates).
  // The sign kernel also stands in for the filter when !filter_ok.
  const int mode = (hdr->fast == kModeFilter && !filter_ok) ? kModeSign : hdr->fast;
  if (mode != (FAST ? kModeSign : kModeGeneral)) return;
  constexpr bool IDS = !FAST;
  __shared__ __align__(16) EdgeRec sj[kTile];
  __shared__ double sth[ANGLE ? kTile : 1];
  __shared__ int2 sid[IDS ? kTile : 1];
  __shared__ int snew[FAST ? kTile : 1];
  SRegs S;
  __shared__ unsigned long long red_u[kThreads / 32];
  __shared__ double red_d[kThreads / 32];

  // Chunks of `chunk` consecutive units are dealt round-robin to the CTAs:
  // unit cost varies along the triangle (run structure of the j-tile), and
  // interleaving gives every CTA the same mix (a contiguous split left the
  // slowest CTA ~15% behind).  Consecutive units inside a chunk mostly share
  // ti, so the i-edges stay in registers.
  // Interleaved sharding: this call owns the chunks whose index is
  // srank (mod sworld) -- every rank sees the same mix of unit costs.
  const uint64_t nchunks = (uend - ubeg + chunk - 1) / chunk;

  unsigned long long total = 0;
  double dsum = 0.0, dcomp = 0.0;  // Kahan over per-unit partials
  IRegs<IDS> R;
  uint64_t ti = 0, tj = 0, cur_ti = ~0ull;
  for (uint64_t ch = srank + (uint64_t)sworld * blockIdx.x; ch < nchunks;
       ch += (uint64_t)sworld * gridDim.x) {
  const uint64_t b = ubeg + ch * chunk;
  const uint64_t e = b + chunk < uend ? b + chunk : uend;
  if (ulist == nullptr) band_unit_coords(b, T, W, &ti, &tj);
  for (uint64_t u = b; u < e; ++u) {
    if (ulist != nullptr) {
      const int2 p = ulist[u];
      ti = (uint64_t)p.x;
      tj = (uint64_t)p.y;
    }
    if (ti != cur_ti) {
      load_i<IDS, ANGLE>(R, rec, theta, ids, ti);
      cur_ti = ti;
    }
    __syncthreads();  // previous tile fully consumed
    {
      const int4 *src = reinterpret_cast<const int4 *>(rec + (int64_t)tj * kTile);
      int4 *dst = reinterpret_cast<int4 *>(sj);
#pragma unroll 4
      for (int q = threadIdx.x; q < kTile * 4; q += kThreads) dst[q] = src[q];
      for (int q = threadIdx.x; q < kTile; q += kThreads) {
        if (IDS) sid[q] = ids[(int64_t)tj * kTile + q];
        if (FAST) snew[q] = newc[(int64_t)tj * kTile + q];
        if (ANGLE) sth[q] = theta[(int64_t)tj * kTile + q];
      }
    }
    __syncthreads();
    unsigned cnt[kK];
    double dev[kK];
#pragma unroll
    for (int k = 0; k < kK; ++k) { cnt[k] = 0; dev[k] = 0.0; }
    if constexpr (FAST) {
      if (ti == tj) {
        for (int jj = 0; jj < kTile; ++jj)
          pair_row_fast<ANGLE, true>(R, S, sj, sth, snew, jj, cnt, dev, ideal);
      } else {
#pragma unroll kUnroll
        for (int jj = 0; jj < kTile; ++jj)
          pair_row_fast<ANGLE, false>(R, S, sj, sth, snew, jj, cnt, dev, ideal);
      }
    } else {
      if (ti == tj) {
        for (int jj = 0; jj < kTile; ++jj)
          pair_row<FAST, ANGLE, true>(R, sj, sth, sid, jj, cnt, dev, ideal);
      } else {
#pragma unroll kUnroll
        for (int jj = 0; jj < kTile; ++jj)
          pair_row<FAST, ANGLE, false>(R, sj, sth, sid, jj, cnt, dev, ideal);
      }
    }
    unsigned c = 0;
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < kK; ++k) { c += cnt[k]; s = __dadd_rn(s, dev[k]); }
    total += c;
    if (ANGLE) {
      double y = __dsub_rn(s, dcomp);
      double t = __dadd_rn(dsum, y);
      dcomp = __dsub_rn(__dsub_rn(t, dsum), y);
      dsum = t;
    }
    if (ulist == nullptr) band_advance(T, W, &ti, &tj);
  }
  }  // chunks
  unsigned long long bc = block_sum_u64<kThreads>(total, red_u);
  double bd = block_sum<kThreads>(dsum, red_d);
  if (threadIdx.x == 0) {
    cta_cnt[blockIdx.x] = bc;
    cta_dev[blockIdx.x] = bd;
  }
}

__device__ __forceinline__ unsigned smem_u32(const void *p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
#ifdef GLR_XWATCHDOG
  for (long long spin = 0;; ++spin) {
    unsigned ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (ok) return;
    if (spin == 2000000) {
      printf("mbar_wait stuck: block %d thread %d bar %p parity %u\n", blockIdx.x, threadIdx.x,
             bar, parity);
      __trap();
    }
  }
#else
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
#endif
}
// TMA bulk copy global -> shared, completion signalled on `bar`.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes,
                                         uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Filter-mode pair kernel (hdr->fast == kModeFilter): same unit space and
// chunk ownership as cross_pairs_kernel.  The j-tile records (8 KB, + 2 KB
// of theta) of the CTA's next kStages units sit in a ring of shared-memory
// stages filled by TMA bulk copies.  Work is handed out in SLICES: a unit's
// i-tile is cut into kFSlices slices of 32 lanes x kFK i-edges, and each warp
// takes the CTA's next slice from a shared counter, so fast warps simply do
// more slices -- warps never wait for each other (a per-unit CTA barrier,
// or a ring where the slowest warp gates the refills, cost 10-19%: warps of
// a CTA progress at persistently different rates).  The warp that finishes
// a unit's last slice refills its stage with the unit kStages ahead.
// Sums are made order-independent so results stay deterministic: counts are
// integers, and each lane's per-slice angle sum is added as a 2^-50
// fixed-point integer into a 128-bit accumulator.
// Shared-vertex pairs are never certain (an exact c is 0), so they reach
// exact_pair, which tests ids: no adjacency correction in this mode.
//
// Exact accumulator of the angle sums.  Every warp-slice's deviation sum S
// (a non-negative double below 2^16: 32 lanes x kFK x kTile deviations of at
// most pi/2) is added EXACTLY to a per-warp fixed-point number in units of
// 2^-1074 (the smallest subnormal), stored as kAccWords 64-bit words of
// 32-bit digits (w[i] weighs 2^(32 i - 1074)) with 32 bits of carry room:
// the final sum is the exact sum of the S rounded once, whatever order the
// slices ran in -- deterministic AND relatively accurate at any magnitude
// (a fixed 2^-50 quantum is not: 1e-12 deviations would lose 4 digits).
constexpr int kAccWords = 36;  // 36 x 32 bits above 2^-1074: values < 2^78
// mean deviation per hit below which a fast-formula slice is re-evaluated
#ifndef GLR_XFIXUPDEV
#define GLR_XFIXUPDEV 0x1p-16
#endif
constexpr double kFixupMeanDev = GLR_XFIXUPDEV;

// w += v for a finite v >= 0 (no carries propagated: each digit word takes
// < 2^32 additions, see the launch bound in crossing_pairs)
__device__ __forceinline__ void xacc_add(unsigned long long *w, double v) {
  // (-0.0 adds nothing: the sign bit is dropped)
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  const int ex = (int)((b >> 52) & 0x7ff);
  unsigned long long mant = b & 0xfffffffffffffull;
  int p = 0;  // weight of mant's LSB: 2^(p - 1074)
  if (ex != 0) {
    mant |= 1ull << 52;
    p = ex - 1;
  }
  const int k = p >> 5, o = p & 31;
  const unsigned long long lo = mant << o;                // bits 0..63 of mant * 2^o
  const unsigned long long hi = o ? mant >> (64 - o) : 0;  // bits 64..84
  w[k] += lo & 0xffffffffull;
  w[k + 1] += lo >> 32;
  w[k + 2] += hi;
}

// carries out of every digit word (in place); afterwards w[i] < 2^32 for
// i < kAccWords - 1
__device__ __forceinline__ void xacc_normalize(unsigned long long *w) {
  for (int i = 0; i + 1 < kAccWords; ++i) {
    w[i + 1] += w[i] >> 32;
    w[i] &= 0xffffffffull;
  }
}

// the normalised accumulator as the correctly rounded double
__device__ inline double xacc_value(const unsigned long long *w) {
  int t = kAccWords - 1;
  while (t > 0 && w[t] == 0) --t;
  if (t <= 1 && (w[1] >> 21) == 0) {  // integer < 2^53 units: exact as a double
    return ldexp((double)((w[1] << 32) | w[0]), -1074);
  }
  // 64 bits from the top digit down, the rest folded into a sticky bit
  // (>= 54 significant bits, so __ull2double_rn rounds it correctly)
  const unsigned long long w1 = t >= 1 ? w[t - 1] : 0, w2 = t >= 2 ? w[t - 2] : 0;
  const int lz = __clzll(w[t]) - 32;  // w[t] < 2^32 (t < kAccWords - 1)
  unsigned long long top = (w[t] << (32 + lz)) | (w1 << lz) | (lz ? w2 >> (32 - lz) : 0ull);
  bool sticky = lz ? (w2 & ((1ull << (32 - lz)) - 1)) != 0 : w2 != 0;
  for (int i = t - 3; i >= 0 && !sticky; --i) sticky = w[i] != 0;
  top |= sticky ? 1ull : 0ull;
  return ldexp(__ull2double_rn(top), 32 * t + 31 - lz - 63 - 1074);
}

struct CtaUnits {  // the CTA's units as a flat sequence (see cross_pairs_kernel)
  const int2 *ulist;
  uint64_t T, W, ubeg, uend, chunk, nchunks, step, ch0;
  __device__ bool at(uint64_t uq, uint64_t *ti, uint64_t *tj, uint64_t *unit = nullptr) const {
    const uint64_t ch = ch0 + (uq / chunk) * step;
    if (ch >= nchunks) return false;
    const uint64_t u = ubeg + ch * chunk + uq % chunk;
    if (u >= uend) return false;
    if (unit != nullptr) *unit = u;
    if (ulist != nullptr) {
      const int2 p = ulist[u];
      *ti = (uint64_t)p.x;
      *tj = (uint64_t)p.y;
    } else {
      band_unit_coords(u, T, W, ti, tj);
    }
    return true;
  }
};

template <bool ANGLE>
__global__ void __launch_bounds__(kThreads,
                                  ANGLE ? kFilterMinBlocksAngle : kFilterMinBlocksCount)
cross_filter_kernel(const RecHeader *__restrict__ hdr, const EdgeRec *__restrict__ rec,
                    const FTile *__restrict__ ftile, const JRec *__restrict__ jrec,
                    const TileBox *__restrict__ tbox, const double *__restrict__ theta,
                    const int2 *__restrict__ ids, const int2 *__restrict__ ulist,
                    const SubMask *__restrict__ usub, uint64_t T,
                    uint64_t W, uint64_t ubeg,
                    uint64_t uend, uint64_t chunk, unsigned srank, unsigned sworld, double ideal,
                    double kappa, int filter_ok,
                    unsigned long long *__restrict__ cta_cnt,
                    unsigned long long *__restrict__ cta_acc, unsigned *__restrict__ fixup) {
  if (hdr->fast != kModeFilter || !filter_ok) return;
  constexpr int kWarps = kThreads / 32;
  constexpr int kNJ = ANGLE ? kFilterBlock : kFilterBlockCount;
  static_assert(kFSlices >= 1, "at least one slice per unit");
  static_assert(kQCap >= 32u * kNJ * kFK, "a block's uncertain pairs must fit the queue");
  __shared__ __align__(128) JRec sj[kStages][kTile];
  __shared__ __align__(128) double sth[kStages][ANGLE ? kTile : 2];
  __shared__ __align__(8) uint64_t full[kStages];
  __shared__ unsigned done[kStages];  // slices finished with the stage, cumulative
  __shared__ unsigned next_slice;
  __shared__ unsigned long long acc_cnt;
  // per-warp exact accumulators of the slices' angle sums (xacc_add)
  __shared__ unsigned long long wacc[ANGLE ? kWarps : 1][ANGLE ? kAccWords : 1];
  __shared__ unsigned short wqueue[kWarps][kQCap];  // uncertain pairs (filter_block)
  constexpr unsigned kJBytes = kTile * sizeof(JRec);
  constexpr unsigned kThBytes = ANGLE ? kTile * sizeof(double) : 0;
  const unsigned lane = threadIdx.x & 31;
  const int warp = (int)(threadIdx.x >> 5);

  CtaUnits cu;
  cu.ulist = ulist; cu.T = T; cu.W = W; cu.ubeg = ubeg; cu.uend = uend; cu.chunk = chunk;
  cu.nchunks = (uend - ubeg + chunk - 1) / chunk;
  cu.step = (uint64_t)sworld * gridDim.x;
  cu.ch0 = srank + (uint64_t)sworld * blockIdx.x;

  auto issue = [&](int st, uint64_t tj_) {
    mbar_expect_tx(&full[st], kJBytes + kThBytes);
    bulk_g2s(sj[st], jrec + (int64_t)tj_ * kTile, kJBytes, &full[st]);
    if (ANGLE) bulk_g2s(sth[st], theta + (int64_t)tj_ * kTile, kThBytes, &full[st]);
  };
  if (ANGLE)
    for (int i = threadIdx.x; i < kWarps * kAccWords; i += kThreads) (&wacc[0][0])[i] = 0;
  if (threadIdx.x == 0) {
    for (int st = 0; st < kStages; ++st) {
      mbar_init(&full[st], 1);
      done[st] = 0;
    }
    next_slice = 0;
    acc_cnt = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int st = 0; st < kStages; ++st) {
      uint64_t a, b;
      if (cu.at((uint64_t)st, &a, &b)) issue(st, b);
    }
  }
  __syncthreads();

  unsigned long long total = 0;
  FIRegs R;
  uint64_t cur_ti = ~0ull;
  int cur_slice = -1;
  // shift / signed forms need ideal >= 2^-100 (genuine deviations then are
  // 0 or >= 2^-766, see filter_block)
  const bool shift_ok = ANGLE && ideal >= 0x1p-100;
  for (;;) {
    unsigned q = 0;
    if (lane == 0) q = atomicAdd(&next_slice, 1u);
    q = __shfl_sync(0xffffffffu, q, 0);
    const uint64_t uq = q / kFSlices;
    const int slice = (int)(q % kFSlices);
    uint64_t ti, tj, unit;
    if (!cu.at(uq, &ti, &tj, &unit)) break;
    const int islot = fslot(slice, 0, (int)lane);  // slot of i-edge k: islot + 32 k
    if (ti != cur_ti || slice != cur_slice) {
      load_fi<ANGLE>(R, ftile, ti, slice, (int)lane);
      cur_ti = ti;
      cur_slice = slice;
    }
    const int stage = (int)(uq % kStages);
    const unsigned use = (unsigned)(uq / kStages);
    // this unit's theta_i (+ shift s, see unit_shift), loaded before the waits
    const TileBox bi = tbox[ti], bj = tbox[tj];
    // both tiles are stars of one vertex: every pair shares it, and
    // exact.py:205 never counts such a pair -- the unit contributes nothing
    const bool star = bi.star >= 0 && bi.star == bj.star;
    // j-quarters certified empty or full for this slice (sub_mask_kernel)
    unsigned skip = 0u;
    if (usub != nullptr) {
      const uint64_t sm = (uint64_t)usub[unit];
      skip = (unsigned)((sm | (sm >> kSubBits)) >> (kSubQuarters * slice)) & kSubQuarterMask;
    }
    double th[kFK];
    int am = 0;  // angle mode: 0 general formula, 1 one kink, 2 signed
    double sigma = 1.0, fbeta = 0.0;
    int kminus = 0;
    if (ANGLE) {
      double sh = 0.0;
      if (ti != tj && shift_ok && unit_shift(bi, bj, ideal, &sh, &sigma) == 1) am = 2;
#if GLR_XKINK
      else if (ti != tj && shift_ok &&
               range_kink(bi.thlo, bi.thhi, bj.thlo, bj.thhi, ideal, &sh, &fbeta, &kminus) == 1)
        am = 1;
#endif
      const double *tt = ftile[ti].theta;
#pragma unroll
      for (int k = 0; k < kFK; ++k) th[k] = tt[islot + 32 * k];
      if (am != 0) {
#pragma unroll
        for (int k = 0; k < kFK; ++k) th[k] = __dadd_rn(th[k], sh);
      }
    }
    // the stage's previous unit must be fully released (its refill issued)
    // before its mbarrier phase parity identifies this use unambiguously
    while (*(volatile unsigned *)&done[stage] < use * kFSlices) {
    }
    mbar_wait(&full[stage], use & 1u);  // this unit's j-tile has landed
    const unsigned jr = smem_u32(sj[stage]);
    const unsigned jth = smem_u32(sth[stage]);
    unsigned cnt[kFK];
    double dev[kFK];
#pragma unroll
    for (int k = 0; k < kFK; ++k) { cnt[k] = 0; dev[k] = 0.0; }
    double A2[2] = {0.0, 0.0};  // signed form: sum_j h_j theta_j (even / odd j)
    unsigned qc = 0;  // signed form: queued (uncertain) pairs that hit
    const int64_t ibase = (int64_t)ti * kTile, jbase = (int64_t)tj * kTile;
    const float thr = unit_threshold(bi, bj);
    unsigned short *wq = wqueue[warp];
    unsigned qn = 0;  // warp-uniform queue length
    if (star) {
#ifdef GLR_XONLYSIGNED  // measurement only: registers / speed of the signed path alone
    } else if (!(ANGLE && am == 2)) {
#endif
    } else if (ti == tj) {
      for (int jj = 0; jj < kTile; jj += kNJ)
        filter_block<ANGLE, true, kNJ, 0>(R, th, jr, jth, jj, islot, thr, cnt, dev, A2, ideal, kappa,
                                          rec, ids, theta, ibase, jbase, wq, qn, qc);
    } else if (ANGLE && am == 2) {
      // runs of consecutive j-quarters that are not skipped (the whole tile
      // without masks: one loop, as in a dense pass)
      for (unsigned act = ~skip & kSubQuarterMask; act != 0u;) {
        const int q0 = __ffs(act) - 1;
        const int len = __ffs(~(act >> q0)) - 1;
        act &= ~(((1u << len) - 1u) << q0);
        const int j0 = q0 * kSubJ, j1 = j0 + len * kSubJ;
        if (thr == 1.0f) {
#pragma unroll kJUnrollS
          for (int jj = j0; jj < j1; jj += kFilterBlockSigned)
            filter_block<ANGLE, false, kFilterBlockSigned, 2, true>(
                R, th, jr, jth, jj, islot, thr, cnt, dev, A2, ideal, kappa, rec, ids, theta, ibase,
                jbase, wq, qn, qc);
        } else {
#pragma unroll 1
          for (int jj = j0; jj < j1; jj += kFilterBlockSigned)
            filter_block<ANGLE, false, kFilterBlockSigned, 2>(R, th, jr, jth, jj, islot, thr, cnt,
                                                              dev, A2, ideal, kappa, rec, ids,
                                                              theta, ibase, jbase, wq, qn, qc);
        }
      }
    } else if (ANGLE && am == 1) {
      // runs of consecutive j-quarters that are not skipped (the whole tile
      // without masks: one loop, as in a dense pass)
      for (unsigned act = ~skip & kSubQuarterMask; act != 0u;) {
        const int q0 = __ffs(act) - 1;
        const int len = __ffs(~(act >> q0)) - 1;
        act &= ~(((1u << len) - 1u) << q0);
        const int j0 = q0 * kSubJ, j1 = j0 + len * kSubJ;
        if (thr == 1.0f) {
#pragma unroll kJUnrollC
          for (int jj = j0; jj < j1; jj += kNJ)
            filter_block<ANGLE, false, kNJ, 1, true>(R, th, jr, jth, jj, islot, thr, cnt, dev, A2,
                                                     ideal, kappa, rec, ids, theta, ibase, jbase,
                                                     wq, qn, qc);
        } else {
#pragma unroll 1
          for (int jj = j0; jj < j1; jj += kNJ)
            filter_block<ANGLE, false, kNJ, 1>(R, th, jr, jth, jj, islot, thr, cnt, dev, A2,
                                               ideal, kappa, rec, ids, theta, ibase, jbase, wq,
                                               qn, qc);
        }
      }
    } else {
      // runs of consecutive j-quarters that are not skipped (the whole tile
      // without masks: one loop, as in a dense pass)
      for (unsigned act = ~skip & kSubQuarterMask; act != 0u;) {
        const int q0 = __ffs(act) - 1;
        const int len = __ffs(~(act >> q0)) - 1;
        act &= ~(((1u << len) - 1u) << q0);
        const int j0 = q0 * kSubJ, j1 = j0 + len * kSubJ;
        if (thr == 1.0f) {  // general units too: FOLD products with an immediate t
#pragma unroll kJUnrollC
          for (int jj = j0; jj < j1; jj += kNJ)
            filter_block<ANGLE, false, kNJ, 0, true>(R, th, jr, jth, jj, islot, thr, cnt, dev, A2,
                                                     ideal, kappa, rec, ids, theta, ibase, jbase,
                                                     wq, qn, qc);
        } else {
#pragma unroll 1
          for (int jj = j0; jj < j1; jj += kNJ)
            filter_block<ANGLE, false, kNJ, 0>(R, th, jr, jth, jj, islot, thr, cnt, dev, A2,
                                               ideal, kappa, rec, ids, theta, ibase, jbase, wq,
                                               qn, qc);
        }
      }
    }
    // release the slice; the warp finishing the unit refills its stage
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      const unsigned old = atomicAdd(&done[stage], 1u);
      if (old + 1 == (use + 1) * kFSlices) {
        uint64_t a, b;
        if (cu.at(uq + kStages, &a, &b)) {
          __threadfence_block();
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          issue(stage, b);
        }
      }
    }
    // the slice's queued uncertain pairs (global records only, so after the
    // stage is released)
    if (qn != 0) {
      if (ANGLE && am == 2)
        drain_queue<ANGLE>(wq, qn, lane, rec, ids, theta, ibase, jbase, ideal, qc, dev[0]);
      else if (ANGLE && am == 1)
        drain_queue<ANGLE>(wq, qn, lane, rec, ids, theta, ibase, jbase, ideal, qc, A2[0]);
      else
        drain_queue<ANGLE>(wq, qn, lane, rec, ids, theta, ibase, jbase, ideal, cnt[0], dev[0]);
    }
    unsigned c = qc;
#pragma unroll
    for (int k = 0; k < kFK; ++k) c += cnt[k];
    total += c;
    if (ANGLE) {
      double s = 0.0;
      if (am == 2) {
        // sigma * (sum_j h_j theta_j - sum_k C_k x_k): every term has sign
        // sigma by the unit's margin, so this is the sum of |v| over hits
        double cx = 0.0;
#pragma unroll
        for (int k = 0; k < kFK; ++k) cx = fma((double)cnt[k], th[k], cx);
        // + the queued hits' deviations (dev[0])
        s = __dadd_rn(sigma * __dsub_rn(__dadd_rn(A2[0], A2[1]), cx), dev[0]);
      } else {
#pragma unroll
        for (int k = 0; k < kFK; ++k) s = __dadd_rn(s, dev[k]);
        s = s < 0x1p-900 ? 0.0 : s;  // only cleared-miss leftovers (< 2^-1031)
        if (am == 1) {
          // one-kink units: the filter's hits (c - qc) give hits * f(beta) -
          // sum |v| or sum |v|; + the queued hits' deviations (A2[0])
          if (kminus) {
            const double t = __dsub_rn(__dmul_rn((double)(c - qc), fbeta), s);
            s = t > 0.0 ? t : 0.0;
          }
          s = __dadd_rn(s, A2[0]);
        }
      }
      // warp sums in a fixed shuffle tree; lane 0 adds the deviation sum
      // exactly, unless the slice's mean deviation per hit is below 2^-16
      // in a unit of the fast formula: then the slice is marked for
      // cross_fixup_kernel, which re-evaluates it with the reference formula
      unsigned cw = c;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        s = __dadd_rn(s, __shfl_down_sync(0xffffffffu, s, o));
        cw += __shfl_down_sync(0xffffffffu, cw, o);
      }
      if (lane == 0) {
        if (am != 2 && s < (double)cw * kFixupMeanDev) {
          const uint64_t bit = (unit - ubeg) * kFSlices + (uint64_t)slice;
          atomicOr(&fixup[bit >> 5], 1u << (bit & 31));
        } else {
          xacc_add(wacc[warp], s);
        }
      }
    }
  }
  // order-independent CTA reduction (integer atomics commute)
  for (int o = 16; o > 0; o >>= 1) total += __shfl_down_sync(0xffffffffu, total, o);
  if (lane == 0) {
    atomicAdd(&acc_cnt, total);
    if (ANGLE) xacc_normalize(wacc[warp]);
  }
  __syncthreads();
  // += : crossing_pairs may launch several unit segments into the same slots
  if (threadIdx.x == 0) cta_cnt[blockIdx.x] += acc_cnt;
  if (ANGLE) {
    for (int i = threadIdx.x; i < kAccWords; i += kThreads) {
      unsigned long long v = 0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) v += wacc[w][i];
      cta_acc[(size_t)blockIdx.x * kAccWords + i] += v;
    }
  }
}

// Re-evaluates the warp-slices cross_filter_kernel marked in `fixup` (a
// fast-formula unit whose slice has a mean deviation per hit below
// kFixupMeanDev) with the reference's per-pair formula (AM 3): one warp per
// marked slice, its j-tile staged into the warp's own shared memory, the
// same filter, queue and exact fallback.  Only the deviation sums are taken
// (the filter kernel counted the slice's hits); they go to this kernel's own
// CTA accumulators.  Marked slices are rare (all hits of a slice within
// ~1.5e-5 rad of the ideal angle on average), so the kernel mostly scans an
// all-zero bitmap.
constexpr int kFixThreads = 64;  // 2 warps: a staged j-tile (10 KB) per warp
__global__ void __launch_bounds__(kFixThreads)
cross_fixup_kernel(const RecHeader *__restrict__ hdr, const EdgeRec *__restrict__ rec,
                   const FTile *__restrict__ ftile, const JRec *__restrict__ jrec,
                   const TileBox *__restrict__ tbox, const double *__restrict__ theta,
                   const int2 *__restrict__ ids, const int2 *__restrict__ ulist,
                   const SubMask *__restrict__ usub, uint64_t T,
                   uint64_t W, uint64_t ubeg, uint64_t nbits, double ideal, double kappa,
                   int filter_ok, const unsigned *__restrict__ fixup,
                   unsigned long long *__restrict__ cta_acc) {
  if (hdr->fast != kModeFilter || !filter_ok) return;
  constexpr int kWarps = kFixThreads / 32;
  __shared__ __align__(128) JRec sj[kWarps][kTile];
  __shared__ __align__(16) double sth[kWarps][kTile];
  __shared__ unsigned short wqueue[kWarps][kQCap];
  __shared__ unsigned long long wacc[kWarps][kAccWords];
  const unsigned lane = threadIdx.x & 31;
  const int warp = (int)(threadIdx.x >> 5);
  for (int i = threadIdx.x; i < kWarps * kAccWords; i += kFixThreads) (&wacc[0][0])[i] = 0;
  __syncthreads();
  const uint64_t nwords = (nbits + 31) / 32;
  for (uint64_t wd = (uint64_t)blockIdx.x * kWarps + warp; wd < nwords;
       wd += (uint64_t)gridDim.x * kWarps) {
    unsigned bits = fixup[wd];
    while (bits != 0u) {
      const uint64_t bit = wd * 32 + (uint64_t)(__ffs(bits) - 1);
      bits &= bits - 1u;
      const uint64_t u = ubeg + bit / kFSlices;
      const int slice = (int)(bit % kFSlices);
      uint64_t ti, tj;
      if (ulist != nullptr) {
        ti = (uint64_t)ulist[u].x;
        tj = (uint64_t)ulist[u].y;
      } else {
        band_unit_coords(u, T, W, &ti, &tj);
      }
      __syncwarp();
      for (int q = (int)lane; q < kTile; q += 32) {
        sj[warp][q] = jrec[(int64_t)tj * kTile + q];
        sth[warp][q] = theta[(int64_t)tj * kTile + q];
      }
      __syncwarp();
      FIRegs R;
      load_fi<true>(R, ftile, ti, slice, (int)lane);
      const int islot = fslot(slice, 0, (int)lane);
      double th[kFK];
#pragma unroll
      for (int k = 0; k < kFK; ++k) th[k] = ftile[ti].theta[islot + 32 * k];
      const TileBox bi = tbox[ti], bj = tbox[tj];
      const float thr = unit_threshold(bi, bj);
      unsigned cnt[kFK];
      double dev[kFK];
#pragma unroll
      for (int k = 0; k < kFK; ++k) { cnt[k] = 0; dev[k] = 0.0; }
      double A2[2] = {0.0, 0.0};
      unsigned qc = 0, qn = 0;
      const unsigned jr = smem_u32(sj[warp]), jth = smem_u32(sth[warp]);
      const int64_t ibase = (int64_t)ti * kTile, jbase = (int64_t)tj * kTile;
      unsigned short *wq = wqueue[warp];
      if (ti == tj) {
        for (int jj = 0; jj < kTile; jj += kFilterBlock)
          filter_block<true, true, kFilterBlock, 3>(R, th, jr, jth, jj, islot, thr, cnt, dev, A2,
                                                    ideal, kappa, rec, ids, theta, ibase, jbase,
                                                    wq, qn, qc);
      } else {
        // the j-quarters the filter kernel skipped for this slice (certified
        // empty, or full: cross_subfull_kernel owns those deviations)
        unsigned skip = 0u;
        if (usub != nullptr) {
          const uint64_t sm = (uint64_t)usub[u];
          skip = (unsigned)((sm | (sm >> kSubBits)) >> (kSubQuarters * slice)) & kSubQuarterMask;
        }
        for (int q = 0; q < kSubQuarters; ++q) {
          if (skip & (1u << q)) continue;
#pragma unroll 1
          for (int jj = q * kSubJ; jj < (q + 1) * kSubJ; jj += kFilterBlock)
            filter_block<true, false, kFilterBlock, 3>(R, th, jr, jth, jj, islot, thr, cnt, dev,
                                                       A2, ideal, kappa, rec, ids, theta, ibase,
                                                       jbase, wq, qn, qc);
        }
      }
      if (qn != 0)
        drain_queue<true>(wq, qn, lane, rec, ids, theta, ibase, jbase, ideal, cnt[0], dev[0]);
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < kFK; ++k) s = __dadd_rn(s, dev[k]);
      s = s < 0x1p-900 ? 0.0 : s;  // only cleared-miss leftovers (< 2^-1031)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s = __dadd_rn(s, __shfl_down_sync(0xffffffffu, s, o));
      if (lane == 0) xacc_add(wacc[warp], s);
    }
  }
  if (lane == 0) xacc_normalize(wacc[warp]);
  __syncthreads();
  for (int i = threadIdx.x; i < kAccWords; i += kFixThreads) {
    unsigned long long v = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) v += wacc[w][i];
    cta_acc[(size_t)blockIdx.x * kAccWords + i] += v;
  }
}

// Adjacent edge pairs (sharing a vertex index) whose tile-pair unit lies in
// [ubeg, uend): count and angle-deviation sum, subtracted from the fast
// kernel's totals.  One CTA per (vertex, incidence tile pair) work item,
// grid-stride; fixed grid and order, so results are deterministic.
template <bool ANGLE>
__global__ void __launch_bounds__(kAdjTile)
adj_kernel(const RecHeader *__restrict__ hdr, const double *__restrict__ theta,
           const int *__restrict__ inc, const int *__restrict__ offs,
           const long long *__restrict__ wofs, const int2 *__restrict__ ulist, uint64_t ulen,
           uint64_t T, uint64_t W, uint64_t ubeg, uint64_t uend, uint64_t chunk,
           unsigned srank, unsigned sworld, double ideal, int filter_ok,
           unsigned long long *__restrict__ part_cnt, double *__restrict__ part_dev) {
  // Each adjacent pair belongs to the unit of its tile pair (tl, th): for the
  // implicit space its index is band_unit_index(tl, th); a culled candidate
  // list is sorted row-major and contains every tile pair whose tile bboxes
  // overlap (hence every adjacent pair's), so its index is found by binary
  // search on key(ti, tj) = ti*T + tj.  The pair is removed here iff the
  // pair kernel evaluated that unit: u in [ubeg, uend) and its chunk is one
  // of this call's (interleaved sharding, see cross_pairs_kernel).
  __shared__ int s_e[kAdjTile];
  __shared__ double s_t[kAdjTile];
  __shared__ long long s_v;
  __shared__ unsigned long long red_u[kAdjTile / 32];
  __shared__ double red_d[kAdjTile / 32];
  const int mode = (hdr->fast == kModeFilter && !filter_ok) ? kModeSign : hdr->fast;
  if (mode != kModeSign) {  // the other kernels test ids per pair: nothing to remove
    if (threadIdx.x == 0) {
      part_cnt[blockIdx.x] = 0;
      part_dev[blockIdx.x] = 0.0;
    }
    return;
  }
  const long long n = hdr->n;
  const long long nwork = wofs[n];
  unsigned long long cnt = 0;
  double dsum = 0.0, dcomp = 0.0;
  for (long long w = blockIdx.x; w < nwork; w += gridDim.x) {
    if (threadIdx.x == 0) {  // vertex owning work item w: last v with wofs[v] <= w
      long long lo = 0, hi = n;
      while (lo < hi) {
        long long mid = (lo + hi + 1) >> 1;
        if (wofs[mid] <= w) lo = mid; else hi = mid - 1;
      }
      s_v = lo;
    }
    __syncthreads();
    const long long v = s_v;
    const int base = offs[v];
    const int d = offs[v + 1] - base;
    const uint64_t Tv = (uint64_t)(d + kAdjTile - 1) / kAdjTile;
    uint64_t ti, tj;
    tri_unit_coords((uint64_t)(w - wofs[v]), Tv, &ti, &tj);
    const int q0 = (int)tj * kAdjTile;
    if (q0 + (int)threadIdx.x < d) {
      const int ej = inc[base + q0 + threadIdx.x];
      s_e[threadIdx.x] = ej;
      s_t[threadIdx.x] = ANGLE ? theta[ej] : 0.0;
    }
    __syncthreads();
    const int p = (int)ti * kAdjTile + threadIdx.x;
    double s = 0.0;
    if (p < d) {
      const int e1 = inc[base + p];
      const double t1 = ANGLE ? theta[e1] : 0.0;
      const int qn = min(kAdjTile, d - q0);
      for (int qq = (ti == tj) ? (int)threadIdx.x + 1 : 0; qq < qn; ++qq) {
        const int e2 = s_e[qq];
        const uint64_t lo = (uint64_t)min(e1, e2) / kTile, hi = (uint64_t)max(e1, e2) / kTile;
        uint64_t unit;
        if (ulist == nullptr) {
          unit = band_unit_index(lo, hi, T, W);
        } else {
          const uint64_t key = lo * T + hi;
          uint64_t a = 0, z = ulen;
          while (a < z) {
            const uint64_t mid = (a + z) >> 1;
            const uint64_t k = (uint64_t)ulist[mid].x * T + (uint64_t)ulist[mid].y;
            if (k < key) a = mid + 1; else z = mid;
          }
          unit = a;
        }
        const bool in = unit >= ubeg && unit < uend &&
                        ((unit - ubeg) / chunk) % sworld == srank;
        if (in) {
          ++cnt;
          if (ANGLE) s = __dadd_rn(s, angle_dev(t1, s_t[qq], ideal));
        }
      }
    }
    if (ANGLE) {
      double y = __dsub_rn(s, dcomp);
      double t = __dadd_rn(dsum, y);
      dcomp = __dsub_rn(__dsub_rn(t, dsum), y);
      dsum = t;
    }
    __syncthreads();
  }
  unsigned long long bc = block_sum_u64<kAdjTile>(cnt, red_u);
  double bd = block_sum<kAdjTile>(dsum, red_d);
  if (threadIdx.x == 0) {
    part_cnt[blockIdx.x] = bc;
    part_dev[blockIdx.x] = bd;
  }
}

// Totals: count = sum of the CTA counts minus the adjacency correction
// (mode 1); dev = the pair kernels' CTA sums (modes 0/1, Kahan) minus the
// correction, or the exact sum of the filter kernel's per-CTA accumulators
// (mode 2: zero words otherwise).  One warp per accumulator word.
__global__ void __launch_bounds__(1024)
cross_finalize_kernel(const unsigned long long *cta_cnt, const double *cta_dev,
                      const unsigned long long *cta_acc, int ncta, int nacc,
                      const unsigned long long *adj_cnt, const double *adj_dev, int nadj,
                      double *out) {
  __shared__ unsigned long long w[kAccWords];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = warp; i < kAccWords; i += 32) {
    unsigned long long v = 0;  // < nacc * segments * 2^34: no overflow
    for (int c = lane; c < nacc; c += 32) v += cta_acc[(size_t)c * kAccWords + i];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) w[i] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long c = 0, a = 0;
    for (int i = 0; i < ncta; ++i) c += cta_cnt[i];
    for (int i = 0; i < nadj; ++i) a += adj_cnt[i];
    out[0] = (double)(c - a);
    xacc_normalize(w);
    const double fsum = xacc_value(w);
    out[1] = __dadd_rn(__dsub_rn(kahan_sum(cta_dev, ncta), kahan_sum(adj_dev, nadj)), fsum);
  }
}

// ---- culled candidate list: tile pairs whose tile rank boxes overlap ------

// per tile: (min rxmin, max rxmax, min rymin, max rymax); pad edges hold
// (INT_MAX, -1, INT_MAX, -1), so an all-pad tile's box is empty
__global__ void __launch_bounds__(kTile)
tile_box_kernel(const EdgeRec *__restrict__ rec, int4 *__restrict__ box) {
  __shared__ int4 red[kTile / 32];
  const EdgeRec &r = rec[(int64_t)blockIdx.x * kTile + threadIdx.x];
  int x0 = r.rxmin, x1 = r.rxmax, y0 = r.rymin, y1 = r.rymax;
  for (int o = 16; o > 0; o >>= 1) {
    x0 = min(x0, __shfl_down_sync(0xffffffffu, x0, o));
    x1 = max(x1, __shfl_down_sync(0xffffffffu, x1, o));
    y0 = min(y0, __shfl_down_sync(0xffffffffu, y0, o));
    y1 = max(y1, __shfl_down_sync(0xffffffffu, y1, o));
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = make_int4(x0, x1, y0, y1);
  __syncthreads();
  if (threadIdx.x == 0) {
    int4 b = red[0];
    for (int w = 1; w < kTile / 32; ++w) {
      b.x = min(b.x, red[w].x); b.y = max(b.y, red[w].y);
      b.z = min(b.z, red[w].z); b.w = max(b.w, red[w].w);
    }
    box[blockIdx.x] = b;
  }
}

__device__ inline bool boxes_overlap(int4 a, int4 b) {
  return b.y >= a.x && a.y >= b.x && b.w >= a.z && a.w >= b.z;
}

// FILL == false: count candidates of row ti; FILL == true: write them at
// offs[ti] (row-major, so the list is sorted by (ti, tj)).
template <bool FILL>
__global__ void tile_pairs_kernel(const int4 *__restrict__ box, int64_t T,
                                  unsigned long long *__restrict__ counts,
                                  const unsigned long long *__restrict__ offs, int2 *list) {
  for (int64_t ti = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; ti < T;
       ti += (int64_t)gridDim.x * blockDim.x) {
    const int4 a = box[ti];
    unsigned long long c = 0, o = FILL ? offs[ti] : 0;
    for (int64_t tj = ti; tj < T; ++tj) {
      if (boxes_overlap(a, box[tj])) {
        if (FILL) list[o + c] = make_int2((int)ti, (int)tj);
        ++c;
      }
    }
    if (!FILL) counts[ti] = c;
  }
}

// Per j-tile cost weight for balanced sharding: a continuing j-edge of a run
// costs 1, a run start 1 + beta (it also recomputes the (a,c)/(b,c) terms).
__global__ void __launch_bounds__(kTile)
tile_weight_kernel(const int *__restrict__ newc, double beta, double *__restrict__ w) {
  __shared__ int red[kTile / 32];
  int s = newc[(int64_t)blockIdx.x * kTile + threadIdx.x] != 0 ? 1 : 0;
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int i = 0; i < kTile / 32; ++i) t += red[i];
    w[blockIdx.x] = (double)kTile + beta * (double)t;
  }
}

// ---- classified candidate list: tile pairs certified to cross everywhere --
//
// The reference's predicate for a pair (a, b) x (c, d) needs c1, c2 (c and d
// against line ab) to straddle zero and c3, c4 (a and b against line cd) to
// straddle zero (geometry.py:62-79).  Name each edge's endpoints P (smaller
// x, ties smaller y) and Q; the straddle tests do not depend on which
// endpoint the reference calls a.  Per tile, PQBox bounds the P's and the
// Q's of its real edges.  The exact orientation (Q - P) x (r - P) is affine
// in each of the six coordinates separately, so over P-box x Q-box x r-box it
// takes its extremes at box corners: evaluating the 16 (P, Q) corner lines
// against the r-box (monotone in rx and ry) gives the exact range up to the
// evaluation error.  Both the corner evaluation and the reference's own
// fl(c) differ from the exact value by at most 2^-49 Ux Uy (four roundings
// of u = 2^-53 on |dx dy| + |dy dx| <= 2 Ux Uy, Ux / Uy the extents of the
// union of the four boxes), so a computed corner range beyond kClassMargin
// Ux Uy = 2^-47 Ux Uy certifies the sign the reference computes for EVERY
// pair of the unit:
//   * "none": c and d strictly on one side of every line ab (or a and b of
//     every line cd) -- no pair straddles, the unit is dropped;
//   * "full": both straddles strictly certified for every pair -- every pair
//     properly crosses, so the bboxes overlap and no vertex is shared (a
//     shared vertex would make an exact orientation 0): the unit contributes
//     na * nb crossings and the pairs' deviations (cross_full_kernel), with
//     no per-pair predicate at all.
// Only admissible inputs (finite, |coords| in [2^-160, 2^500], no overflow
// or underflow in these products) are classified; otherwise every
// overlapping unit stays "mixed".
struct __align__(16) PQBox {
  double px0, px1, py0, py1;  // P (smaller-x endpoint) box
  double qx0, qx1, qy0, qy1;  // Q box
};
constexpr double kClassMargin = 0x1p-47;
enum UnitClass { kUnitNone = 0, kUnitMixed = 1, kUnitFull = 2 };

// one CTA of NB threads per block of NB consecutive edges (NB = kTile:
// tiles; NB = kSubJ: the sub-blocks of the sub-unit masks)
template <int NB>
__global__ void __launch_bounds__(NB < 32 ? 32 : NB)
tile_pq_kernel(const EdgeRec *__restrict__ rec, int64_t m, PQBox *__restrict__ out) {
  constexpr int kNT = NB < 32 ? 32 : NB;  // a warp holds 32 / NB blocks when NB < 32
  constexpr int kW = NB < 32 ? NB : 32;   // lanes combined by shuffles
  __shared__ double red[8][kNT / 32];
  const int64_t e = (int64_t)blockIdx.x * kNT + threadIdx.x;
  // v[0..3]: -P.x, P.x, -P.y, P.y maxima; v[4..7] the same for Q
  double v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = -INFINITY;
  if (e < m) {
    const EdgeRec &r = rec[e];
    const bool pa = r.ax < r.bx || (r.ax == r.bx && r.ay <= r.by);
    const double px = pa ? r.ax : r.bx, py = pa ? r.ay : r.by;
    const double qx = pa ? r.bx : r.ax, qy = pa ? r.by : r.ay;
    v[0] = -px; v[1] = px; v[2] = -py; v[3] = py;
    v[4] = -qx; v[5] = qx; v[6] = -qy; v[7] = qy;
  }
#pragma unroll
  for (int i = 0; i < 8; ++i)
    for (int o = kW / 2; o > 0; o >>= 1)
      v[i] = fmax(v[i], __shfl_down_sync(0xffffffffu, v[i], o, kW));
  if (NB < 32) {
    // even slots hold -min: negate back (an empty block gets lo = +inf, hi = -inf)
    if (threadIdx.x % kW == 0) {
      double *o = reinterpret_cast<double *>(out + (int64_t)blockIdx.x * (kNT / NB) +
                                             threadIdx.x / kW);
#pragma unroll
      for (int i = 0; i < 8; ++i) o[i] = (i & 1) ? v[i] : -v[i];
    }
    return;
  }
  if ((threadIdx.x & 31) == 0)
#pragma unroll
    for (int i = 0; i < 8; ++i) red[i][threadIdx.x >> 5] = v[i];
  __syncthreads();
  if (threadIdx.x < 8) {
    double x = red[threadIdx.x][0];
    for (int w = 1; w < kNT / 32; ++w) x = fmax(x, red[threadIdx.x][w]);
    reinterpret_cast<double *>(out + blockIdx.x)[threadIdx.x] = (threadIdx.x & 1) ? x : -x;
  }
}

// Computed ranges of (Q - P) x (r - P) over the lines of L's edges, for r in
// R's P-box (lo[0], hi[0]) and Q-box (lo[1], hi[1]).
__device__ inline void orient_ranges(const PQBox &L, const PQBox &R, double (&lo)[2],
                                     double (&hi)[2]) {
  lo[0] = lo[1] = INFINITY;
  hi[0] = hi[1] = -INFINITY;
  // Differences r - P for the two values of each P coordinate, hoisted out
  // of the corner loop: u[k][y][0..1] = (ry0, ry1) - py, w[k][x][0..1] =
  // (rx0, rx1) - px; u0 <= u1 and w0 <= w1 by monotone rounding.
  const double rb[2][4] = {{R.px0, R.px1, R.py0, R.py1}, {R.qx0, R.qx1, R.qy0, R.qy1}};
  double u[2][2][2], w[2][2][2];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    u[k][0][0] = __dsub_rn(rb[k][2], L.py0); u[k][0][1] = __dsub_rn(rb[k][3], L.py0);
    u[k][1][0] = __dsub_rn(rb[k][2], L.py1); u[k][1][1] = __dsub_rn(rb[k][3], L.py1);
    w[k][0][0] = __dsub_rn(rb[k][0], L.px0); w[k][0][1] = __dsub_rn(rb[k][1], L.px0);
    w[k][1][0] = __dsub_rn(rb[k][0], L.px1); w[k][1][1] = __dsub_rn(rb[k][1], L.px1);
  }
#pragma unroll kCornerUnroll
  for (int c = 0; c < 16; ++c) {
    const int xs = c & 1, ys = (c >> 1) & 1;
    const double px = xs ? L.px1 : L.px0, py = ys ? L.py1 : L.py0;
    const double qx = (c & 4) ? L.qx1 : L.qx0, qy = (c & 8) ? L.qy1 : L.qy0;
    const double a = __dsub_rn(qx, px), b = __dsub_rn(qy, py);
    // min / max of a product with an ordered pair is picked by the factor's
    // sign (multiplication by a fixed factor is monotone under rounding):
    // the same values as min(a u0, a u1) etc.
    const bool an = a < 0.0, bn = b < 0.0;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const double u0 = u[k][ys][0], u1 = u[k][ys][1], w0 = w[k][xs][0], w1 = w[k][xs][1];
      const double t1lo = __dmul_rn(a, an ? u1 : u0), t1hi = __dmul_rn(a, an ? u0 : u1);
      const double t2lo = __dmul_rn(b, bn ? w1 : w0), t2hi = __dmul_rn(b, bn ? w0 : w1);
      lo[k] = fmin(lo[k], __dsub_rn(t1lo, t2hi));
      hi[k] = fmax(hi[k], __dsub_rn(t1hi, t2lo));
    }
  }
}

__device__ inline PQBox pq_union(const PQBox &a, const PQBox &b) {
  PQBox u;
  u.px0 = fmin(a.px0, b.px0); u.px1 = fmax(a.px1, b.px1);
  u.py0 = fmin(a.py0, b.py0); u.py1 = fmax(a.py1, b.py1);
  u.qx0 = fmin(a.qx0, b.qx0); u.qx1 = fmax(a.qx1, b.qx1);
  u.qy0 = fmin(a.qy0, b.qy0); u.qy1 = fmax(a.qy1, b.qy1);
  return u;
}

// The closed bboxes of A's edges and of B's edges are disjoint (P has the
// smaller x, so the x-range is [px0, qx1]): every pair fails the reference's
// closed-bbox test (exact.py:191-194) -- exact, plain double comparisons.
__device__ inline bool pq_disjoint(const PQBox &A, const PQBox &B) {
  return A.qx1 < B.px0 || B.qx1 < A.px0 || fmax(A.py1, A.qy1) < fmin(B.py0, B.qy0) ||
         fmax(B.py1, B.qy1) < fmin(A.py0, A.qy0);
}

__device__ inline int unit_class(const PQBox &A, const PQBox &B) {
  const double x0 = fmin(fmin(A.px0, A.qx0), fmin(B.px0, B.qx0));
  const double x1 = fmax(fmax(A.px1, A.qx1), fmax(B.px1, B.qx1));
  const double y0 = fmin(fmin(A.py0, A.qy0), fmin(B.py0, B.qy0));
  const double y1 = fmax(fmax(A.py1, A.qy1), fmax(B.py1, B.qy1));
  // kClassMargin Ux Uy, rounded up by far more than the few ulps of the
  // extents' own rounding; + 2^-1000 keeps it positive for flat boxes
  const double thr = __dadd_ru(__dmul_ru(__dmul_ru(__dsub_ru(x1, x0), __dsub_ru(y1, y0)),
                                         kClassMargin * (1.0 + 0x1p-20)),
                               0x1p-1000);
  double la[2], ha[2], lb[2], hb[2];
  orient_ranges(A, B, la, ha);  // c, d against lines ab
  orient_ranges(B, A, lb, hb);  // a, b against lines cd
  const bool pa0 = la[0] > thr, na0 = ha[0] < -thr, pa1 = la[1] > thr, na1 = ha[1] < -thr;
  const bool pb0 = lb[0] > thr, nb0 = hb[0] < -thr, pb1 = lb[1] > thr, nb1 = hb[1] < -thr;
  if ((pa0 && pa1) || (na0 && na1) || (pb0 && pb1) || (nb0 && nb1)) return kUnitNone;
  if (((pa0 && na1) || (na0 && pa1)) && ((pb0 && nb1) || (nb0 && pb1))) return kUnitFull;
  return kUnitMixed;
}

// Sub-unit masks of the mixed part of a classified list: thread (u, b)
// classifies block b of unit u -- warp-slice b / kSubQuarters of tile ti
// against j-quarter b % kSubQuarters of tile tj -- with unit_class on the
// blocks' own endpoint boxes (a block without real edges, or with disjoint
// closed bboxes, is empty too); the unit's bits are gathered with two
// ballots.  Diagonal units and inadmissible inputs keep 0.
static_assert(32 % kSubBits == 0, "a warp covers whole units");
__global__ void __launch_bounds__(256, GLR_XCLASSMINB)
sub_mask_kernel(const RecHeader *__restrict__ hdr, const int2 *__restrict__ list,
                uint64_t mixed, const PQBox *__restrict__ pqs, SubMask *__restrict__ sub) {
  constexpr int kPer = kTile / kSubJ;             // sub-blocks per tile
  constexpr int kSliceBlocks = 32 * kFK / kSubJ;  // sub-blocks per warp slice
  const bool classify = hdr->admissible != 0;
  const unsigned lane = threadIdx.x & 31;
  const uint64_t total = mixed * kSubBits;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < total;
       base += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t idx = base + threadIdx.x;
    bool none = false, full = false;
    uint64_t u = idx / kSubBits;
    if (idx < total) {
      const int2 p = list[u];
      const int bit = (int)(idx % kSubBits);
      if (classify && p.x != p.y) {
        const int sl = bit / kSubQuarters, q = bit % kSubQuarters;
        PQBox a = pqs[(int64_t)p.x * kPer + sl * kSliceBlocks];
        for (int k = 1; k < kSliceBlocks; ++k)
          a = pq_union(a, pqs[(int64_t)p.x * kPer + sl * kSliceBlocks + k]);
        const PQBox b = pqs[(int64_t)p.y * kPer + q];
        none = !(a.px0 <= a.px1) || !(b.px0 <= b.px1) || pq_disjoint(a, b);
        if (!none) {
          const int c = unit_class(a, b);
          none = c == kUnitNone;
          full = c == kUnitFull;
        }
      }
    }
    const unsigned bn = __ballot_sync(0xffffffffu, none);
    const unsigned bf = __ballot_sync(0xffffffffu, full);
    if (idx < total && lane % kSubBits == 0) {
      const uint64_t mask = (1ull << kSubBits) - 1ull;
      sub[u] = (SubMask)((((uint64_t)bn >> lane) & mask) | ((((uint64_t)bf >> lane) & mask) << kSubBits));
    }
  }
}

// Row ti of the classified list: one CTA per row, tj = ti..T-1 in blocks of
// kClassThreads, order-preserving compaction (warp ballots).  FILL == false
// counts mixed / full units per row; FILL == true writes mixed units at
// off_m[ti] and full units at off_m[T] + off_f[ti] (both parts row-major).
constexpr int kClassThreads = 256;
template <bool FILL>
__global__ void __launch_bounds__(kClassThreads, GLR_XCLASSMINB)
tile_class_kernel(const RecHeader *__restrict__ hdr, const int4 *__restrict__ box,
                  const PQBox *__restrict__ pq, int64_t T, int row_rank, int row_world,
                  unsigned long long *__restrict__ cnt_m, unsigned long long *__restrict__ cnt_f,
                  const unsigned long long *__restrict__ off_m,
                  const unsigned long long *__restrict__ off_f, int2 *__restrict__ list) {
  constexpr int kWarps = kClassThreads / 32;
  __shared__ unsigned wm[kWarps], wf[kWarps];
  const int64_t ti = blockIdx.x;
  if (ti % row_world != row_rank) {  // another rank's row (glr_crossing_candidates_rows)
    if (!FILL && threadIdx.x == 0) {
      cnt_m[ti] = 0;
      cnt_f[ti] = 0;
    }
    return;
  }
  const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool classify = hdr->admissible != 0;
  const int4 a = box[ti];
  const PQBox pa = pq[ti];
  unsigned long long om = FILL ? off_m[ti] : 0ull, of = FILL ? off_m[T] + off_f[ti] : 0ull;
  unsigned long long nm = 0, nf = 0;
  for (int64_t base = ti; base < T; base += kClassThreads) {
    const int64_t tj = base + threadIdx.x;
    int c = kUnitNone;
    if (tj < T && boxes_overlap(a, box[tj]))
      c = (classify && tj != ti) ? unit_class(pa, pq[tj]) : kUnitMixed;
    const unsigned bm = __ballot_sync(0xffffffffu, c == kUnitMixed);
    const unsigned bf = __ballot_sync(0xffffffffu, c == kUnitFull);
    if (lane == 0) {
      wm[warp] = __popc(bm);
      wf[warp] = __popc(bf);
    }
    __syncthreads();
    unsigned pm = 0, pf = 0, tm = 0, tf = 0;
#pragma unroll
    for (unsigned w = 0; w < (unsigned)kWarps; ++w) {
      if (w < warp) { pm += wm[w]; pf += wf[w]; }
      tm += wm[w];
      tf += wf[w];
    }
    if (FILL) {
      const unsigned below = (1u << lane) - 1u;
      if (c == kUnitMixed) list[om + pm + __popc(bm & below)] = make_int2((int)ti, (int)tj);
      if (c == kUnitFull) list[of + pf + __popc(bf & below)] = make_int2((int)ti, (int)tj);
    }
    om += tm; of += tf; nm += tm; nf += tf;
    __syncthreads();
  }
  if (!FILL && threadIdx.x == 0) {
    cnt_m[ti] = nm;
    cnt_f[ti] = nf;
  }
}

// per tile: sum of theta over its real edges (fixed reduction tree)
__global__ void __launch_bounds__(kTile) tile_theta_sum_kernel(const double *__restrict__ theta,
                                                               int64_t m, double *__restrict__ ts) {
  __shared__ double sh[kTile / 32];
  const int64_t e = (int64_t)blockIdx.x * kTile + threadIdx.x;
  const double s = block_sum<kTile>(e < m ? theta[e] : 0.0, sh);
  if (threadIdx.x == 0) ts[blockIdx.x] = s;
}

// Per NB-block of edges: theta of the real edges sorted ascending (pads
// +inf, at the end) and the exclusive prefix sums of the sorted values --
// what piecewise_dev needs.  One CTA of NB threads per block, bitonic network
// in shared memory (comparisons and moves only), Hillis-Steele scan.
template <int NB>
__global__ void __launch_bounds__(NB)
theta_sort_kernel(const double *__restrict__ theta, int64_t m, double *__restrict__ ts,
                  double *__restrict__ tp) {
  __shared__ double v[NB];
  __shared__ double sc[2][NB];
  const int t = (int)threadIdx.x;
  const int64_t e = (int64_t)blockIdx.x * NB + t;
  v[t] = e < m ? theta[e] : INFINITY;
  __syncthreads();
  for (int k = 2; k <= NB; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      const int p = t ^ j;
      if (p > t) {
        const double a = v[t], b = v[p];
        const bool up = (t & k) == 0;
        if ((a > b) == up) { v[t] = b; v[p] = a; }
      }
      __syncthreads();
    }
  }
  const double x = v[t];
  int cur = 0;
  sc[0][t] = isfinite(x) ? x : 0.0;  // theta is finite in [0, pi]
  __syncthreads();
  for (int o = 1; o < NB; o <<= 1) {
    const double a = sc[cur][t], b = t >= o ? sc[cur][t - o] : 0.0;
    sc[cur ^ 1][t] = t >= o ? __dadd_rn(b, a) : a;
    cur ^= 1;
    __syncthreads();
  }
  ts[e] = x;
  tp[e] = t > 0 ? sc[cur][t - 1] : 0.0;  // exclusive
}

// sum over j of |ideal - min(|d|, pi - |d|)|, d = s[j] - ti, for the n sorted
// angles s[0..n) with exclusive prefix sums pre[] and total tot: the
// deviation (geometry.py:107-110, exact.py:219-221) is piecewise linear in d
// on (-pi, pi) with kinks at 0, +-ideal, +-pi/2, +-(pi - ideal), so seven
// binary searches cut the sorted angles into eight runs on which it is c +
// sg * d, and each run contributes cnt * c + sg * (sum of its angles - cnt *
// ti).  The value is continuous at the kinks, so an angle within an ulp of
// one may fall on either side.  Absolute error <= ~1e-12 per call (sums of
// <= 256 angles); callers re-evaluate per pair when the mean deviation is
// small (kPiecewiseMeanDev).
constexpr double kPiecewiseMeanDev = 0x1p-12;
// NB: the block size (a power of two); s[n..NB) hold +inf, so a branchless
// search never passes n.  A block's angles span a fraction of a radian, so
// most kinks fall outside [s[0], s[n-1]] and are placed by two comparisons;
// only the one or two inside are searched, and only non-empty runs are
// evaluated (the lanes of a warp mostly agree on which: their theta_i lie in
// one tile's narrow range).
template <int NB>
__device__ inline double piecewise_dev(double ti, const double *s, const double *pre, int n,
                                       double tot, double ideal) {
  const double HALF_PI = 1.5707963267948966, PI = 3.141592653589793;
  const double pmi = __dsub_rn(PI, ideal);
  const double bp[7] = {-pmi, -HALF_PI, -ideal, 0.0, ideal, HALF_PI, pmi};
  const double c[8] = {-pmi, pmi, -ideal, ideal, ideal, -ideal, pmi, -pmi};
  const double s0 = s[0], sl = s[n - 1];
  int a = 0;
  double pa = 0.0, acc = 0.0;
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    int b = n;
    if (p < 7) {
      const double x = __dadd_rn(ti, bp[p]);
      if (!(s0 < x)) {
        b = 0;  // no angle below x
      } else if (!(sl < x)) {
        int pos = 0;  // number of angles below x
#pragma unroll
        for (int step = NB / 2; step >= 1; step >>= 1) pos += s[pos + step - 1] < x ? step : 0;
        pos += s[pos] < x ? 1 : 0;
        b = pos > n ? n : pos;
      }
    }
    if (b > a) {
      const double pb = b < n ? pre[b] : tot;
      const double cnt = (double)(b - a);
      const double lin = __dsub_rn(__dsub_rn(pb, pa), __dmul_rn(cnt, ti));
      const double v = __dadd_rn(__dmul_rn(cnt, c[p]), (p & 1) ? lin : -lin);
      acc = __dadd_rn(acc, v > 0.0 ? v : 0.0);
      a = b;
      pa = pb;
    }
  }
  return acc;
}

// Full units (every pair crosses, tile_class_kernel): na * nb crossings and
// the deviation sum.  Units whose theta ranges give unit_shift's signed form
// take it in closed form from the tiles' theta sums,
//   sum_ij |theta_j - theta_i - s| = sigma (na sum_j theta_j - nb sum_i
//   theta_i - na nb s),
// (each term at least kSignMargin, so the cancellation costs < 1e-12
// relative); the others sum the piecewise-linear deviation over the j-tile's
// sorted angles (piecewise_dev: seven binary searches per i-edge instead of
// nb per-pair evaluations), falling back to the reference's per-pair formula
// (angle_dev) when the unit's mean deviation is below kPiecewiseMeanDev.
// FP64 only, no predicate.  Same chunk ownership as the pair kernels; the
// sums go to exact accumulators.
constexpr int kFullThreads = kTile;  // thread t: i-edge t of the unit
template <bool ANGLE>
__global__ void __launch_bounds__(kFullThreads)
cross_full_kernel(const TileBox *__restrict__ tbox, const double *__restrict__ theta,
                  const double *__restrict__ tsum, const double *__restrict__ tsorted,
                  const double *__restrict__ tprefix, const int2 *__restrict__ flist,
                  uint64_t fbeg, uint64_t fend, uint64_t chunk, unsigned srank, unsigned sworld,
                  int64_t m, double ideal, unsigned long long *__restrict__ cta_cnt,
                  unsigned long long *__restrict__ cta_acc) {
  constexpr int kWarps = kFullThreads / 32;
  __shared__ double sth[ANGLE ? kTile : 1], spre[ANGLE ? kTile : 1];
  __shared__ double red[kWarps];
  __shared__ int per_pair;
  __shared__ int wneed[kWarps];
  __shared__ int2 todo[ANGLE ? kFullThreads : 1];
  __shared__ unsigned long long wacc[ANGLE ? kWarps : 1][ANGLE ? kAccWords : 1];
  const unsigned lane = threadIdx.x & 31;
  const int warp = (int)(threadIdx.x >> 5);
  CtaUnits cu;
  cu.ulist = flist; cu.T = 0; cu.W = 0; cu.ubeg = fbeg; cu.uend = fend; cu.chunk = chunk;
  cu.nchunks = (fend - fbeg + chunk - 1) / chunk;
  cu.step = (uint64_t)sworld * gridDim.x;
  cu.ch0 = srank + (uint64_t)sworld * blockIdx.x;
  if (ANGLE)
    for (int i = threadIdx.x; i < kWarps * kAccWords; i += kFullThreads) (&wacc[0][0])[i] = 0;
  __syncthreads();
  const bool shift_ok = ANGLE && ideal >= 0x1p-100;
  unsigned long long total = 0;
  // Batches of kFullThreads units.  Phase 1: thread t looks at unit uq0 + t
  // -- its pair count, and its deviation sum if the closed form applies
  // (warp sums go to the exact accumulators).  Phase 2: the other units are
  // compacted into shared memory and taken one at a time by the whole CTA.
  for (uint64_t uq0 = 0;; uq0 += kFullThreads) {
    uint64_t ti = 0, tj = 0;
    const bool valid = cu.at(uq0 + threadIdx.x, &ti, &tj);
    if (!__syncthreads_or(valid ? 1 : 0)) break;  // also orders the reuse of todo[]
    bool need = false;
    double cf = 0.0;
    if (valid) {
      const int64_t ra = m - (int64_t)ti * kTile, rb = m - (int64_t)tj * kTile;
      const int na = (int)(ra < kTile ? ra : kTile), nb = (int)(rb < kTile ? rb : kTile);
      total += (unsigned long long)na * (unsigned long long)nb;
      if (ANGLE) {
        const TileBox bi = tbox[ti], bj = tbox[tj];
        double sh = 0.0, sigma = 1.0;
        if (shift_ok && unit_shift(bi, bj, ideal, &sh, &sigma) == 1) {
          const double v = sigma * __dsub_rn(__dsub_rn(__dmul_rn((double)na, tsum[tj]),
                                                       __dmul_rn((double)nb, tsum[ti])),
                                             __dmul_rn((double)na * (double)nb, sh));
          cf = v > 0.0 ? v : 0.0;
        } else {
          need = true;
        }
      }
    }
    if (!ANGLE) continue;
    for (int o = 16; o > 0; o >>= 1) cf = __dadd_rn(cf, __shfl_down_sync(0xffffffffu, cf, o));
    if (lane == 0 && cf > 0.0) xacc_add(wacc[warp], cf);
    const unsigned bal = __ballot_sync(0xffffffffu, need);
    if (lane == 0) wneed[warp] = __popc(bal);
    __syncthreads();
    int off = 0, ntodo = 0;
    for (int w = 0; w < kWarps; ++w) {
      if (w < warp) off += wneed[w];
      ntodo += wneed[w];
    }
    if (need) todo[off + __popc(bal & ((1u << lane) - 1u))] = make_int2((int)ti, (int)tj);
    __syncthreads();
    for (int k = 0; k < ntodo; ++k) {
      const int2 unit = todo[k];
      const int64_t ra = m - (int64_t)unit.x * kTile, rb = m - (int64_t)unit.y * kTile;
      const int na = (int)(ra < kTile ? ra : kTile), nb = (int)(rb < kTile ? rb : kTile);
      // piecewise-linear sums over the j-tile's sorted angles (piecewise_dev)
      __syncthreads();  // the previous unit's angles are consumed
      sth[threadIdx.x] = tsorted[(int64_t)unit.y * kTile + threadIdx.x];
      spre[threadIdx.x] = tprefix[(int64_t)unit.y * kTile + threadIdx.x];
      __syncthreads();
      const double t =
          (int)threadIdx.x < na ? theta[(int64_t)unit.x * kTile + threadIdx.x] : 0.0;
      {
        const double tot = __dadd_rn(sth[nb - 1], spre[nb - 1]);
        double d = (int)threadIdx.x < na ? piecewise_dev<kTile>(t, sth, spre, nb, tot, ideal) : 0.0;
        for (int o = 16; o > 0; o >>= 1) d = __dadd_rn(d, __shfl_down_sync(0xffffffffu, d, o));
        if (lane == 0) red[warp] = d;
        __syncthreads();
        if (threadIdx.x == 0) {
          double v = 0.0;
          for (int w = 0; w < kWarps; ++w) v = __dadd_rn(v, red[w]);
          // small mean deviation: the per-pair formula below (bit-identical
          // to numpy's for each pair) instead
          per_pair = v < (double)na * (double)nb * kPiecewiseMeanDev ? 1 : 0;
          if (!per_pair) xacc_add(wacc[0], v);
        }
        __syncthreads();
      }
      if (!per_pair) continue;
      double d = 0.0;
      if ((int)threadIdx.x < na) {
        double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
        int j = 0;
        for (; j + 4 <= nb; j += 4) {
          d0 = __dadd_rn(d0, angle_dev(t, sth[j], ideal));
          d1 = __dadd_rn(d1, angle_dev(t, sth[j + 1], ideal));
          d2 = __dadd_rn(d2, angle_dev(t, sth[j + 2], ideal));
          d3 = __dadd_rn(d3, angle_dev(t, sth[j + 3], ideal));
        }
        for (; j < nb; ++j) d0 = __dadd_rn(d0, angle_dev(t, sth[j], ideal));
        d = __dadd_rn(__dadd_rn(d0, d1), __dadd_rn(d2, d3));
      }
      for (int o = 16; o > 0; o >>= 1) d = __dadd_rn(d, __shfl_down_sync(0xffffffffu, d, o));
      if (lane == 0) xacc_add(wacc[warp], d);
    }
  }
  for (int o = 16; o > 0; o >>= 1) total += __shfl_down_sync(0xffffffffu, total, o);
  __shared__ unsigned long long acc_cnt;
  if (threadIdx.x == 0) acc_cnt = 0;
  __syncthreads();
  if (lane == 0) atomicAdd(&acc_cnt, total);
  if (ANGLE && lane == 0) xacc_normalize(wacc[warp]);
  __syncthreads();
  if (threadIdx.x == 0) cta_cnt[blockIdx.x] += acc_cnt;
  if (ANGLE) {
    for (int i = threadIdx.x; i < kAccWords; i += kFullThreads) {
      unsigned long long v = 0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) v += wacc[w][i];
      cta_acc[(size_t)blockIdx.x * kAccWords + i] += v;
    }
  }
}

// Per kSubJ-block of edges: theta sum (fixed tree) and outward-rounded float
// theta bounds of its real edges -- what cross_subfull_kernel needs for the
// closed form of a certified-full block.
struct SubStat {
  double tsum;
  float thlo, thhi;
};
__global__ void __launch_bounds__(kSubJ < 32 ? 32 : kSubJ)
sub_stat_kernel(const double *__restrict__ theta, int64_t m, SubStat *__restrict__ out) {
  // one warp per block when kSubJ < 32 would waste lanes: a CTA of
  // max(kSubJ, 32) threads handles max(1, 32 / kSubJ) blocks
  constexpr int kNT = kSubJ < 32 ? 32 : kSubJ;
  constexpr int kPerCta = kNT / kSubJ;
  __shared__ double sh[kNT / 32];
  __shared__ float slo[kNT / 32], shi[kNT / 32];
  const int64_t e = (int64_t)blockIdx.x * kNT + threadIdx.x;
  double t = 0.0;
  float lo = INFINITY, hi = -INFINITY;
  if (e < m) {
    t = theta[e];
    lo = __double2float_rd(t);
    hi = __double2float_ru(t);
  }
  constexpr int kW = kSubJ < 32 ? kSubJ : 32;  // lanes combined by shuffles
  for (int o = kW / 2; o > 0; o >>= 1) {
    t += __shfl_down_sync(0xffffffffu, t, o, kW);
    lo = fminf(lo, __shfl_down_sync(0xffffffffu, lo, o, kW));
    hi = fmaxf(hi, __shfl_down_sync(0xffffffffu, hi, o, kW));
  }
  if (kSubJ <= 32) {
    if (threadIdx.x % kSubJ == 0) {
      SubStat r; r.tsum = t; r.thlo = lo; r.thhi = hi;
      out[(int64_t)blockIdx.x * kPerCta + threadIdx.x / kSubJ] = r;
    }
  } else {
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) { sh[w] = t; slo[w] = lo; shi[w] = hi; }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int i = 1; i < kNT / 32; ++i) {
        t += sh[i];
        lo = fminf(lo, slo[i]);
        hi = fmaxf(hi, shi[i]);
      }
      SubStat r; r.tsum = t; r.thlo = lo; r.thhi = hi;
      out[blockIdx.x] = r;
    }
  }
}

// Certified-full blocks of the mixed units (sub_mask_kernel's upper mask
// bits): every pair of warp-slice s of tile ti and j-quarter q of tile tj
// crosses properly, so the block contributes n_i * n_j crossings and its
// pairs' deviations -- in closed form when the block's theta ranges give
// range_shift's signed form (as cross_full_kernel does per unit), else by
// the reference's per-pair formula (angle_dev), FP64 only.  One warp per
// unit; lanes first scan 32 units' masks.  Units are owned by ranks in the
// chunks of the pair kernels ((u - ubeg) / chunk mod world); runs only in
// filter mode, like the kernel that skips these blocks.
constexpr int kSubfullThreads = 256;
template <bool ANGLE>
__global__ void __launch_bounds__(kSubfullThreads)
cross_subfull_kernel(const RecHeader *__restrict__ hdr, int filter_ok,
                     const int2 *__restrict__ ulist, const SubMask *__restrict__ usub,
                     uint64_t ubeg, uint64_t uend, uint64_t chunk, unsigned srank, unsigned sworld,
                     int64_t m, const double *__restrict__ theta,
                     const SubStat *__restrict__ sstat, const double *__restrict__ qsorted,
                     const double *__restrict__ qprefix, double ideal,
                     unsigned long long *__restrict__ cta_cnt,
                     unsigned long long *__restrict__ cta_acc) {
  if (hdr->fast != kModeFilter || !filter_ok) return;
  constexpr int kWarps = kSubfullThreads / 32;
  constexpr int kSliceEdges = 32 * kFK;
  constexpr int kSliceBlocks = kSliceEdges / kSubJ;
  constexpr int kPer = kTile / kSubJ;
  __shared__ unsigned long long wacc[ANGLE ? kWarps : 1][ANGLE ? kAccWords : 1];
  __shared__ double wsrt[ANGLE ? kWarps : 1][ANGLE ? kSubJ : 1], wpre[ANGLE ? kWarps : 1][ANGLE ? kSubJ : 1];
  __shared__ unsigned long long acc_cnt;
  const unsigned lane = threadIdx.x & 31;
  const int warp = (int)(threadIdx.x >> 5);
  if (ANGLE)
    for (int i = threadIdx.x; i < kWarps * kAccWords; i += kSubfullThreads) (&wacc[0][0])[i] = 0;
  if (threadIdx.x == 0) acc_cnt = 0;
  __syncthreads();
  const bool shift_ok = ANGLE && ideal >= 0x1p-100;
  const uint64_t fullmask = (1ull << kSubBits) - 1ull;
  unsigned long long total = 0;
  const uint64_t nwarps = (uint64_t)gridDim.x * kWarps;
  for (uint64_t base = ubeg + ((uint64_t)blockIdx.x * kWarps + warp) * 32; base < uend;
       base += nwarps * 32) {
    const uint64_t mine = base + lane;
    uint64_t fm = 0;
    if (mine < uend && ((mine - ubeg) / chunk) % sworld == srank)
      fm = ((uint64_t)usub[mine] >> kSubBits) & fullmask;
    // Phase 1, one lane per unit: pair counts of its full blocks, and their
    // deviation sums where the closed form applies (pm: the other blocks)
    uint64_t pm = 0;
    double cf = 0.0;
    if (fm != 0) {
      const int2 p = ulist[mine];
      uint64_t bits = fm;
      while (bits) {
        const int b = __ffsll((long long)bits) - 1;
        bits &= bits - 1;
        const int sl = b / kSubQuarters, q = b % kSubQuarters;
        const int64_t ri = m - ((int64_t)p.x * kTile + (int64_t)sl * kSliceEdges);
        const int64_t rj = m - ((int64_t)p.y * kTile + (int64_t)q * kSubJ);
        const int ni = (int)(ri < 0 ? 0 : ri < kSliceEdges ? ri : kSliceEdges);
        const int nj = (int)(rj < 0 ? 0 : rj < kSubJ ? rj : kSubJ);
        total += (unsigned long long)ni * (unsigned long long)nj;
        if (!ANGLE || ni == 0 || nj == 0) continue;
        const SubStat sj = sstat[(int64_t)p.y * kPer + q];
        float ilo = INFINITY, ihi = -INFINITY;
        double isum = 0.0;
#pragma unroll
        for (int k = 0; k < kSliceBlocks; ++k) {
          const SubStat si = sstat[(int64_t)p.x * kPer + sl * kSliceBlocks + k];
          ilo = fminf(ilo, si.thlo);
          ihi = fmaxf(ihi, si.thhi);
          isum = __dadd_rn(isum, si.tsum);
        }
        double sh = 0.0, sigma = 1.0;
        if (shift_ok && range_shift(ilo, ihi, sj.thlo, sj.thhi, ideal, &sh, &sigma) == 1) {
          const double v = sigma * __dsub_rn(__dsub_rn(__dmul_rn((double)ni, sj.tsum),
                                                       __dmul_rn((double)nj, isum)),
                                             __dmul_rn((double)ni * (double)nj, sh));
          cf = __dadd_rn(cf, v > 0.0 ? v : 0.0);
        } else {
          pm |= 1ull << b;
        }
      }
    }
    if (!ANGLE) continue;
    for (int o = 16; o > 0; o >>= 1) cf = __dadd_rn(cf, __shfl_down_sync(0xffffffffu, cf, o));
    if (lane == 0 && cf > 0.0) xacc_add(wacc[warp], cf);
    // Phase 2, the warp per remaining block
    unsigned have = __ballot_sync(0xffffffffu, pm != 0);
    while (have) {
      const int src = __ffs(have) - 1;
      have &= have - 1;
      const uint64_t u = base + src;
      uint64_t bits = __shfl_sync(0xffffffffu, pm, src);
      const int2 p = ulist[u];
      const int64_t ib = (int64_t)p.x * kTile, jb = (int64_t)p.y * kTile;
      while (bits) {
        const int b = __ffsll((long long)bits) - 1;
        bits &= bits - 1;
        const int sl = b / kSubQuarters, q = b % kSubQuarters;
        const int64_t i0 = ib + (int64_t)sl * kSliceEdges, j0 = jb + (int64_t)q * kSubJ;
        const int64_t ri = m - i0, rj = m - j0;
        const int ni = (int)(ri < kSliceEdges ? ri : kSliceEdges);
        const int nj = (int)(rj < kSubJ ? rj : kSubJ);
        // lane l takes i-edges l, l + 32, ... of the slice: piecewise-linear
        // sums over the j-quarter's sorted angles (piecewise_dev), or the
        // per-pair formula when the block's mean deviation is small
        double ti[kFK];
#pragma unroll
        for (int k = 0; k < kFK; ++k)
          ti[k] = (int)lane + 32 * k < ni ? theta[i0 + lane + 32 * k] : 0.0;
        __syncwarp();
        for (int j = (int)lane; j < kSubJ; j += 32) {
          wsrt[warp][j] = qsorted[j0 + j];
          wpre[warp][j] = qprefix[j0 + j];
        }
        __syncwarp();
        const double tot = __dadd_rn(wsrt[warp][nj - 1], wpre[warp][nj - 1]);
        double ds = 0.0;
#pragma unroll
        for (int k = 0; k < kFK; ++k)
          if ((int)lane + 32 * k < ni)
            ds = __dadd_rn(ds, piecewise_dev<kSubJ>(ti[k], wsrt[warp], wpre[warp], nj, tot, ideal));
        for (int o = 16; o > 0; o >>= 1) ds = __dadd_rn(ds, __shfl_down_sync(0xffffffffu, ds, o));
        ds = __shfl_sync(0xffffffffu, ds, 0);
        if (ds < (double)ni * (double)nj * kPiecewiseMeanDev) {
          double d[kFK];
#pragma unroll
          for (int k = 0; k < kFK; ++k) d[k] = 0.0;
          for (int j = 0; j < nj; ++j) {
            const double tj = wsrt[warp][j];
#pragma unroll
            for (int k = 0; k < kFK; ++k) d[k] = __dadd_rn(d[k], angle_dev(ti[k], tj, ideal));
          }
          ds = 0.0;
#pragma unroll
          for (int k = 0; k < kFK; ++k)
            if ((int)lane + 32 * k < ni) ds = __dadd_rn(ds, d[k]);
          for (int o = 16; o > 0; o >>= 1)
            ds = __dadd_rn(ds, __shfl_down_sync(0xffffffffu, ds, o));
        }
        if (lane == 0) xacc_add(wacc[warp], ds);
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) total += __shfl_down_sync(0xffffffffu, total, o);
  if (lane == 0) {
    atomicAdd(&acc_cnt, total);
    if (ANGLE) xacc_normalize(wacc[warp]);
  }
  __syncthreads();
  if (threadIdx.x == 0) cta_cnt[blockIdx.x] += acc_cnt;
  if (ANGLE) {
    for (int i = threadIdx.x; i < kAccWords; i += kSubfullThreads) {
      unsigned long long v = 0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) v += wacc[w][i];
      cta_acc[(size_t)blockIdx.x * kAccWords + i] += v;
    }
  }
}

int grid_for(uint64_t units, int per_sm = kMinBlocks) {
  uint64_t g = (uint64_t)sm_count() * per_sm;
  if (units < g) g = units;
  return (int)(g < 1 ? 1 : g);
}

int blocks_for(int64_t work, int nt, int per_sm) {
  int64_t b = (work + nt - 1) / nt;
  const int64_t cap = (int64_t)sm_count() * per_sm;
  if (b > cap) b = cap;
  return (int)(b < 1 ? 1 : b);
}

int bits_for(int64_t n) {
  int b = 1;
  while (b < 31 && ((int64_t)1 << b) <= n) ++b;
  return b;
}

}  // namespace

int crossing_prepare(const double *d_xy, int64_t n, const int64_t *d_edges, int64_t m,
                     void *d_records, cudaStream_t st) {
  if (m < 0 || n < 0 || d_records == nullptr || (m > 0 && (d_xy == nullptr || d_edges == nullptr))) {
    set_error("glr_crossing_prepare: invalid arguments (n=%lld, m=%lld)", (long long)n,
              (long long)m);
    return GLR_EARG;
  }
  if (m >= (int64_t)1 << 29 || n >= (int64_t)1 << 31) {
    set_error("glr_crossing_prepare: n=%lld, m=%lld exceed the 32-bit index range",
              (long long)n, (long long)m);
    return GLR_EARG;
  }
  if (reinterpret_cast<uintptr_t>(d_records) % 256 != 0) {
    set_error("glr_crossing_prepare: records buffer must be 256-byte aligned");
    return GLR_EARG;
  }
  const int64_t m_pad = pad_edges(m < 1 ? 1 : m);
  RecView rv = view(d_records, n, m);
  const int64_t mm = m;
  // scratch: xs, ys, sorted xs, sorted ys (2m f64 each); deg (n+1), sort keys
  // in/out (2m i32 each), sort values in (2m), work units (n+1 i64); two
  // magnitude words; CUB temp
  size_t t_sort = 0, t_pairs = 0, t_scan = 0, t_scan64 = 0;
  if (mm > 0) {
    GLR_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, t_sort, (const double *)nullptr,
                                            (double *)nullptr, (int)(2 * mm), 0, 64, st));
    GLR_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, t_pairs, (const int *)nullptr, (int *)nullptr,
                                             (const int *)nullptr, (int *)nullptr, (int)(2 * mm), 0,
                                             bits_for(n), st));
  }
  GLR_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t_scan, (int *)nullptr, (int *)nullptr,
                                         (int)(n + 1), st));
  GLR_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t_scan64, (long long *)nullptr,
                                         (long long *)nullptr, (int)(n + 1), st));
  size_t t_cub = t_sort;
  if (t_pairs > t_cub) t_cub = t_pairs;
  if (t_scan > t_cub) t_cub = t_scan;
  if (t_scan64 > t_cub) t_cub = t_scan64;
  const size_t a_f64 = al256((size_t)(2 * mm) * sizeof(double));
  const size_t a_i32 = al256((size_t)(2 * mm) * sizeof(int));
  const size_t a_deg = al256((size_t)(n + 1) * sizeof(int));
  const size_t a_wu = al256((size_t)(n + 1) * sizeof(long long));
  Scratch scr(4 * a_f64 + 3 * a_i32 + a_deg + a_wu + 256 + t_cub, st);
  GLR_CUDA(scr.err);
  char *base = scr.as<char>();
  double *xs = reinterpret_cast<double *>(base);
  double *ys = reinterpret_cast<double *>(base + a_f64);
  double *sx = reinterpret_cast<double *>(base + 2 * a_f64);
  double *sy = reinterpret_cast<double *>(base + 3 * a_f64);
  char *p = base + 4 * a_f64;
  int *keys = reinterpret_cast<int *>(p);
  int *keys_out = reinterpret_cast<int *>(p + a_i32);
  int *vals = reinterpret_cast<int *>(p + 2 * a_i32);
  p += 3 * a_i32;
  int *deg = reinterpret_cast<int *>(p);
  long long *wunits = reinterpret_cast<long long *>(p + a_deg);
  unsigned long long *mag = reinterpret_cast<unsigned long long *>(p + a_deg + a_wu);
  void *cub_tmp = p + a_deg + a_wu + 256;

  const int nt = 256;
  GLR_CUDA(cudaMemsetAsync(deg, 0, (size_t)(n + 1) * sizeof(int), st));
  gather_kernel<<<blocks_for(m_pad, nt, 16), nt, 0, st>>>(
      reinterpret_cast<const double2 *>(d_xy), reinterpret_cast<const longlong2 *>(d_edges), mm,
      m_pad, rv, xs, ys, deg, keys, vals);
  GLR_LAUNCHED("gather_kernel");
  size_t tb;
  if (mm > 0) {
    tb = t_cub;
    GLR_CUDA(cub::DeviceRadixSort::SortKeys(cub_tmp, tb, xs, sx, (int)(2 * mm), 0, 64, st));
    count_launch(4);
    tb = t_cub;
    GLR_CUDA(cub::DeviceRadixSort::SortKeys(cub_tmp, tb, ys, sy, (int)(2 * mm), 0, 64, st));
    count_launch(4);
    rank_kernel<<<blocks_for(mm, nt, 16), nt, 0, st>>>(mm, rv, xs, ys, sx, sy);
    GLR_LAUNCHED("rank_kernel");
    frec_kernel<<<blocks_for(m_pad, nt, 16), nt, 0, st>>>(mm, m_pad, rv, sx, sy);
    GLR_LAUNCHED("frec_kernel");
    tile_fbox_kernel<<<(unsigned)(m_pad / kTile), kTile, 0, st>>>(mm, rv);
    GLR_LAUNCHED("tile_fbox_kernel");
    // incidence lists grouped by vertex; stable, so each list is ordered
    // (edges where the vertex is first, then where it is second, by edge id)
    tb = t_cub;
    GLR_CUDA(cub::DeviceRadixSort::SortPairs(cub_tmp, tb, keys, keys_out, vals, rv.inc,
                                             (int)(2 * mm), 0, bits_for(n), st));
    count_launch(4);
  }
  tb = t_cub;
  GLR_CUDA(cub::DeviceScan::ExclusiveSum(cub_tmp, tb, deg, rv.offs, (int)(n + 1), st));
  count_launch(2);
  adj_units_kernel<<<blocks_for(n + 1, nt, 8), nt, 0, st>>>(deg, n, wunits);
  GLR_LAUNCHED("adj_units_kernel");
  tb = t_cub;
  GLR_CUDA(cub::DeviceScan::ExclusiveSum(cub_tmp, tb, wunits, rv.wofs, (int)(n + 1), st));
  count_launch(2);
  GLR_CUDA(cudaMemsetAsync(mag, 0x00, sizeof(unsigned long long), st));
  GLR_CUDA(cudaMemsetAsync(mag + 1, 0xff, sizeof(unsigned long long), st));
  if (n > 0) {
    magnitude_kernel<<<blocks_for(2 * n, nt, 8), nt, 0, st>>>(d_xy, 2 * n, mag, mag + 1);
    GLR_LAUNCHED("magnitude_kernel");
  }
  header_kernel<<<1, 1, 0, st>>>(rv.hdr, n, mm, m_pad, mag, mag + 1);
  GLR_LAUNCHED("header_kernel");
  return GLR_OK;
}

// Chunk of interleaved ownership: >= 8 chunks per CTA of every rank, <=
// kMaxChunk units per chunk (each chunk reloads its i-tile, so longer chunks
// mean less L2/DRAM traffic).  A function of the whole range, the rank count
// and constants only (not of this device's SM count), so all ranks cut the
// same chunks (glr_crossing_chunk).
uint64_t chunk_for(uint64_t span, int sworld) {
  const uint64_t cta_ref = (uint64_t)kNumSmB200 * kMinBlocks;
  if (span == 0 || sworld < 1) return 1;
  uint64_t chunk = span / ((span < cta_ref ? span : cta_ref) * 8 * (uint64_t)sworld);
  if (chunk > (uint64_t)kMaxChunk) chunk = (uint64_t)kMaxChunk;
  if (chunk < 1) chunk = 1;
  return chunk;
}

int crossing_pairs(const void *d_records, int64_t n, int64_t m, int with_angle, double ideal,
                   const int2 *d_list, uint64_t list_len, uint64_t ubeg, uint64_t uend,
                   int srank, int sworld, double *d_out, cudaStream_t st,
                   const int2 *d_full = nullptr, uint64_t fbeg = 0, uint64_t fend = 0,
                   const SubMask *d_sub = nullptr) {
  if (d_records == nullptr || d_out == nullptr || m < 0 || n < 0 || sworld < 1 || srank < 0 ||
      srank >= sworld) {
    set_error("glr_crossing_pairs: invalid arguments");
    return GLR_EARG;
  }
  if (m > kMaxExactEdges) {  // the float64 count slot is exact below 2^53
    set_error("glr_crossing_pairs: m=%lld edges: m(m-1)/2 reaches 2^53, counts would round",
              (long long)m);
    return GLR_EARG;
  }
  const int64_t m_pad = pad_edges(m < 1 ? 1 : m);
  const uint64_t T = (uint64_t)(m_pad / kTile);
  const uint64_t U = d_list != nullptr ? list_len : tri_units(T);
  if (ubeg > uend || uend > U) {
    set_error("glr_crossing_pairs: unit range [%llu, %llu) outside [0, %llu)",
              (unsigned long long)ubeg, (unsigned long long)uend, (unsigned long long)U);
    return GLR_EARG;
  }
  if (with_angle && !(ideal > 0.0 && ideal <= 1.5707963267948966)) {
    set_error("glr_crossing_pairs: ideal angle must lie in (0, pi/2], got %g", ideal);
    return GLR_EARG;
  }
  if (fbeg > fend || (fend > fbeg && d_full == nullptr)) {
    set_error("glr_crossing_pairs: invalid full-unit range");
    return GLR_EARG;
  }
  if (m < 2 || (ubeg == uend && fbeg == fend)) {
    GLR_CUDA(cudaMemsetAsync(d_out, 0, 2 * sizeof(double), st));
    return GLR_OK;
  }
  RecView rv = view(const_cast<void *>(d_records), n, m);
  const uint64_t span = uend - ubeg;
  const uint64_t fspan = fend - fbeg;
  // full units (cross_full_kernel): their own CTA slots after the pair kernels'
  const int ggrid = fspan > 0 ? grid_for((fspan + sworld - 1) / sworld, 8) : 0;
  const uint64_t fchunk = chunk_for(fspan, sworld);
  const int grid = grid_for((span + sworld - 1) / sworld);
  const int fgrid = grid_for((span + sworld - 1) / sworld,
                             with_angle ? kFilterMinBlocksAngle : kFilterMinBlocksCount);
  const int cgrid = grid > fgrid ? grid : fgrid;  // CTA partial slots
  const int agrid = sm_count() * 8;
  const int xgrid = with_angle ? sm_count() * 4 : 0;  // cross_fixup_kernel CTAs
  const uint64_t chunk = chunk_for(span, sworld);
  // The angle pass runs in unit segments of at most kMaxSegUnits whose
  // offsets are multiples of chunk * world (so chunk ownership is the one of
  // the whole range); each segment's warp-slices have one bit in the fixup
  // bitmap (cross_fixup_kernel).
  const uint64_t seg_align = chunk * (uint64_t)sworld;
  uint64_t seg_len = (kMaxSegUnits / seg_align) * seg_align;
  if (seg_len < seg_align) seg_len = seg_align;
  const uint64_t seg_max = span < seg_len ? span : seg_len;
  const size_t a_fix = with_angle ? al256((size_t)((seg_max * kFSlices + 31) / 32) * 4) : 0;
  // certified-full blocks of the mixed units (cross_subfull_kernel)
  const int sgrid = (d_sub != nullptr && span > 0)
                        ? blocks_for((int64_t)((span + sworld - 1) / sworld), kSubfullThreads, 8)
                        : 0;
  const int ncta = cgrid + ggrid + sgrid;          // count / FP64 slots: pair, full, sub-full
  const int nacc = cgrid + xgrid + ggrid + sgrid;  // exact accumulators: filter, fixup, full, sub-full
  const size_t a_acc = (size_t)nacc * kAccWords * sizeof(unsigned long long);
  const size_t a_ts = (with_angle && fspan > 0) ? al256((size_t)(m_pad / kTile) * sizeof(double)) : 0;
  const size_t a_ss = (with_angle && sgrid > 0) ? al256((size_t)(m_pad / kSubJ) * sizeof(SubStat)) : 0;
  // sorted angles + prefix sums per tile (full units) and per j-quarter (full blocks)
  const size_t a_srt = al256((size_t)m_pad * sizeof(double));
  const int n_srt = with_angle ? (fspan > 0 ? 2 : 0) + (sgrid > 0 ? 2 : 0) : 0;
  Scratch scr((size_t)(ncta + agrid) * (sizeof(unsigned long long) + sizeof(double)) + a_acc +
                  a_fix + a_ts + a_ss + n_srt * a_srt + 1024,
              st);
  GLR_CUDA(scr.err);
  unsigned long long *cc = scr.as<unsigned long long>();
  unsigned long long *ac = cc + ncta;
  double *cd = reinterpret_cast<double *>(ac + agrid);
  double *ad = cd + ncta;
  unsigned long long *xa = reinterpret_cast<unsigned long long *>(ad + agrid);
  unsigned *fix = reinterpret_cast<unsigned *>(
      (reinterpret_cast<uintptr_t>(xa + (size_t)nacc * kAccWords) + 255) & ~(uintptr_t)255);
  double *tsum = reinterpret_cast<double *>(
      (reinterpret_cast<uintptr_t>(fix) + a_fix + 255) & ~(uintptr_t)255);
  SubStat *sstat = reinterpret_cast<SubStat *>(
      (reinterpret_cast<uintptr_t>(tsum) + a_ts + 255) & ~(uintptr_t)255);
  char *srt = reinterpret_cast<char *>(
      (reinterpret_cast<uintptr_t>(sstat) + a_ss + 255) & ~(uintptr_t)255);
  double *tsort = reinterpret_cast<double *>(srt);
  double *tpre = reinterpret_cast<double *>(srt + a_srt);
  double *qsort = reinterpret_cast<double *>(srt + (fspan > 0 ? 2 : 0) * a_srt);
  double *qpre = reinterpret_cast<double *>(srt + (fspan > 0 ? 3 : 1) * a_srt);
  // only the kernel of the records' mode writes its CTA slots
  GLR_CUDA(cudaMemsetAsync(cc, 0, (size_t)ncta * sizeof(unsigned long long), st));
  GLR_CUDA(cudaMemsetAsync(cd, 0, (size_t)ncta * sizeof(double), st));
  GLR_CUDA(cudaMemsetAsync(xa, 0, a_acc, st));
  if (fspan > 0) {
    if (with_angle) {
      tile_theta_sum_kernel<<<(unsigned)(m_pad / kTile), kTile, 0, st>>>(rv.theta, m, tsum);
      GLR_LAUNCHED("tile_theta_sum_kernel");
      theta_sort_kernel<kTile><<<(unsigned)(m_pad / kTile), kTile, 0, st>>>(rv.theta, m, tsort,
                                                                            tpre);
      GLR_LAUNCHED("theta_sort_kernel");
      cross_full_kernel<true><<<ggrid, kFullThreads, 0, st>>>(
          rv.tbox, rv.theta, tsum, tsort, tpre, d_full, fbeg, fend, fchunk, (unsigned)srank,
          (unsigned)sworld, m, ideal, cc + cgrid, xa + (size_t)(cgrid + xgrid) * kAccWords);
      GLR_LAUNCHED("cross_full_kernel<angle>");
    } else {
      cross_full_kernel<false><<<ggrid, kFullThreads, 0, st>>>(
          rv.tbox, rv.theta, nullptr, nullptr, nullptr, d_full, fbeg, fend, fchunk,
          (unsigned)srank, (unsigned)sworld, m, 0.0, cc + cgrid,
          xa + (size_t)(cgrid + xgrid) * kAccWords);
      GLR_LAUNCHED("cross_full_kernel");
    }
  }
  if (sgrid > 0) {
    const uint64_t chunk_s = chunk_for(span, sworld);
    const int filter_ok_s = (!with_angle || ideal >= 0x1p-100) ? 1 : 0;
    unsigned long long *scc = cc + cgrid + ggrid;
    unsigned long long *sxa = xa + (size_t)(cgrid + xgrid + ggrid) * kAccWords;
    if (with_angle) {
      constexpr int kNT = kSubJ < 32 ? 32 : kSubJ;
      sub_stat_kernel<<<(unsigned)(m_pad / kNT), kNT, 0, st>>>(rv.theta, m, sstat);
      GLR_LAUNCHED("sub_stat_kernel");
      theta_sort_kernel<kSubJ><<<(unsigned)(m_pad / kSubJ), kSubJ, 0, st>>>(rv.theta, m, qsort,
                                                                            qpre);
      GLR_LAUNCHED("theta_sort_kernel<sub>");
      cross_subfull_kernel<true><<<sgrid, kSubfullThreads, 0, st>>>(
          rv.hdr, filter_ok_s, d_list, d_sub, ubeg, uend, chunk_s, (unsigned)srank,
          (unsigned)sworld, m, rv.theta, sstat, qsort, qpre, ideal, scc, sxa);
      GLR_LAUNCHED("cross_subfull_kernel<angle>");
    } else {
      cross_subfull_kernel<false><<<sgrid, kSubfullThreads, 0, st>>>(
          rv.hdr, filter_ok_s, d_list, d_sub, ubeg, uend, chunk_s, (unsigned)srank,
          (unsigned)sworld, m, rv.theta, nullptr, nullptr, nullptr, 0.0, scc, sxa);
      GLR_LAUNCHED("cross_subfull_kernel");
    }
  }
  if (span > 0) {
    const uint64_t W = (uint64_t)kBandTiles;
    const unsigned r = (unsigned)srank, g = (unsigned)sworld;
    // the filter's shift/signed forms and cleared-miss leftovers assume an
    // ideal angle >= 2^-100; below it the FP64 sign kernel (mode 1) runs
    const int filter_ok = (!with_angle || ideal >= 0x1p-100) ? 1 : 0;
    const double kappa = 1.5707963267948966 - ideal;  // host IEEE double
    if (with_angle) {
      cross_pairs_kernel<true, true><<<grid, kThreads, 0, st>>>(
          rv.hdr, rv.rec, rv.theta, rv.ids, rv.newc, d_list, T, W, ubeg, uend, chunk, r, g, ideal,
          filter_ok, cc, cd);
      GLR_LAUNCHED("cross_pairs_kernel<fast,angle>");
      cross_pairs_kernel<false, true><<<grid, kThreads, 0, st>>>(
          rv.hdr, rv.rec, rv.theta, rv.ids, rv.newc, d_list, T, W, ubeg, uend, chunk, r, g, ideal,
          filter_ok, cc, cd);
      GLR_LAUNCHED("cross_pairs_kernel<general,angle>");
      for (uint64_t sb = ubeg; sb < uend; sb += seg_len) {
        const uint64_t se = uend - sb < seg_len ? uend : sb + seg_len;
        const uint64_t nbits = (se - sb) * kFSlices;
        GLR_CUDA(cudaMemsetAsync(fix, 0, (size_t)((nbits + 31) / 32) * 4, st));
        cross_filter_kernel<true><<<fgrid, kThreads, 0, st>>>(
            rv.hdr, rv.rec, rv.ftile, rv.jrec, rv.tbox, rv.theta, rv.ids, d_list, d_sub, T, W,
            sb, se, chunk, r, g, ideal, kappa, filter_ok, cc, xa, fix);
        GLR_LAUNCHED("cross_filter_kernel<angle>");
        cross_fixup_kernel<<<xgrid, kFixThreads, 0, st>>>(
            rv.hdr, rv.rec, rv.ftile, rv.jrec, rv.tbox, rv.theta, rv.ids, d_list, d_sub, T, W, sb,
            nbits, ideal, kappa, filter_ok, fix, xa + (size_t)cgrid * kAccWords);
        GLR_LAUNCHED("cross_fixup_kernel");
      }
      adj_kernel<true><<<agrid, kAdjTile, 0, st>>>(rv.hdr, rv.theta, rv.inc, rv.offs, rv.wofs,
                                                   d_list, U, T, W, ubeg, uend, chunk, r, g, ideal,
                                                   filter_ok, ac, ad);
      GLR_LAUNCHED("adj_kernel<angle>");
    } else {
      cross_pairs_kernel<true, false><<<grid, kThreads, 0, st>>>(
          rv.hdr, rv.rec, rv.theta, rv.ids, rv.newc, d_list, T, W, ubeg, uend, chunk, r, g, 0.0,
          filter_ok, cc, cd);
      GLR_LAUNCHED("cross_pairs_kernel<fast>");
      cross_pairs_kernel<false, false><<<grid, kThreads, 0, st>>>(
          rv.hdr, rv.rec, rv.theta, rv.ids, rv.newc, d_list, T, W, ubeg, uend, chunk, r, g, 0.0,
          filter_ok, cc, cd);
      GLR_LAUNCHED("cross_pairs_kernel<general>");
      cross_filter_kernel<false><<<fgrid, kThreads, 0, st>>>(
          rv.hdr, rv.rec, rv.ftile, rv.jrec, rv.tbox, rv.theta, rv.ids, d_list, d_sub, T, W, ubeg,
          uend, chunk, r, g, 0.0, 0.0, filter_ok, cc, xa, nullptr);
      GLR_LAUNCHED("cross_filter_kernel");
      adj_kernel<false><<<agrid, kAdjTile, 0, st>>>(rv.hdr, rv.theta, rv.inc, rv.offs, rv.wofs,
                                                    d_list, U, T, W, ubeg, uend, chunk, r, g, 0.0,
                                                    filter_ok, ac, ad);
      GLR_LAUNCHED("adj_kernel");
    }
  } else {
    GLR_CUDA(cudaMemsetAsync(ac, 0, (size_t)agrid * sizeof(unsigned long long), st));
    GLR_CUDA(cudaMemsetAsync(ad, 0, (size_t)agrid * sizeof(double), st));
  }
  cross_finalize_kernel<<<1, 1024, 0, st>>>(cc, cd, xa, ncta, nacc, ac, ad, agrid, d_out);
  GLR_LAUNCHED("cross_finalize_kernel");
  return GLR_OK;
}

int crossing_candidates(const void *d_records, int64_t n, int64_t m, int2 *d_list,
                        uint64_t capacity, uint64_t *h_count, cudaStream_t st) {
  if (d_records == nullptr || h_count == nullptr || m < 0 || n < 0) {
    set_error("glr_crossing_candidates: invalid arguments");
    return GLR_EARG;
  }
  const int64_t m_pad = pad_edges(m < 1 ? 1 : m);
  const int64_t T = m_pad / kTile;
  RecView rv = view(const_cast<void *>(d_records), n, m);
  size_t t_scan = 0;
  GLR_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t_scan, (unsigned long long *)nullptr,
                                         (unsigned long long *)nullptr, (int)(T + 1), st));
  const size_t a_box = al256((size_t)T * sizeof(int4));
  const size_t a_cnt = al256((size_t)(T + 1) * sizeof(unsigned long long));
  Scratch scr(a_box + 2 * a_cnt + t_scan, st);
  GLR_CUDA(scr.err);
  char *p = scr.as<char>();
  int4 *box = reinterpret_cast<int4 *>(p);
  unsigned long long *counts = reinterpret_cast<unsigned long long *>(p + a_box);
  unsigned long long *offs = reinterpret_cast<unsigned long long *>(p + a_box + a_cnt);
  void *tmp = p + a_box + 2 * a_cnt;
  tile_box_kernel<<<(unsigned)T, kTile, 0, st>>>(rv.rec, box);
  GLR_LAUNCHED("tile_box_kernel");
  GLR_CUDA(cudaMemsetAsync(counts + T, 0, sizeof(unsigned long long), st));
  const int rb = blocks_for(T, 128, 16);
  tile_pairs_kernel<false><<<rb, 128, 0, st>>>(box, T, counts, nullptr, nullptr);
  GLR_LAUNCHED("tile_pairs_kernel<count>");
  size_t tb = t_scan;
  GLR_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, counts, offs, (int)(T + 1), st));
  count_launch(2);
  unsigned long long total = 0;
  GLR_CUDA(cudaMemcpyAsync(&total, offs + T, sizeof(total), cudaMemcpyDeviceToHost, st));
  GLR_CUDA(cudaStreamSynchronize(st));
  *h_count = total;
  if (d_list != nullptr && capacity >= total && total > 0) {
    tile_pairs_kernel<true><<<rb, 128, 0, st>>>(box, T, nullptr, offs, d_list);
    GLR_LAUNCHED("tile_pairs_kernel<fill>");
  }
  return GLR_OK;
}

// Classified candidate list (tile_class_kernel): [mixed units | full units],
// each part row-major; none-certified units are dropped.
int crossing_candidates_classified(const void *d_records, int64_t n, int64_t m, int2 *d_list,
                                   SubMask *d_sub, uint64_t capacity, uint64_t *h_counts,
                                   cudaStream_t st, int row_rank = 0, int row_world = 1) {
  if (d_records == nullptr || h_counts == nullptr || m < 0 || n < 0 || row_world < 1 ||
      row_rank < 0 || row_rank >= row_world) {
    set_error("glr_crossing_candidates_classified: invalid arguments");
    return GLR_EARG;
  }
  const int64_t m_pad = pad_edges(m < 1 ? 1 : m);
  const int64_t T = m_pad / kTile;
  RecView rv = view(const_cast<void *>(d_records), n, m);
  size_t t_scan = 0;
  GLR_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t_scan, (unsigned long long *)nullptr,
                                         (unsigned long long *)nullptr, (int)(T + 1), st));
  const size_t a_box = al256((size_t)T * sizeof(int4));
  const size_t a_pq = al256((size_t)T * sizeof(PQBox));
  const size_t a_pqs = al256((size_t)(m_pad / kSubJ) * sizeof(PQBox));
  const size_t a_cnt = al256((size_t)(T + 1) * sizeof(unsigned long long));
  Scratch scr(a_box + a_pq + a_pqs + 4 * a_cnt + t_scan, st);
  GLR_CUDA(scr.err);
  char *p = scr.as<char>();
  int4 *box = reinterpret_cast<int4 *>(p);
  PQBox *pq = reinterpret_cast<PQBox *>(p + a_box);
  PQBox *pqs = reinterpret_cast<PQBox *>(p + a_box + a_pq);
  p += a_box + a_pq + a_pqs;
  unsigned long long *cnt_m = reinterpret_cast<unsigned long long *>(p);
  unsigned long long *cnt_f = reinterpret_cast<unsigned long long *>(p + a_cnt);
  unsigned long long *off_m = reinterpret_cast<unsigned long long *>(p + 2 * a_cnt);
  unsigned long long *off_f = reinterpret_cast<unsigned long long *>(p + 3 * a_cnt);
  void *tmp = p + 4 * a_cnt;
  tile_box_kernel<<<(unsigned)T, kTile, 0, st>>>(rv.rec, box);
  GLR_LAUNCHED("tile_box_kernel");
  tile_pq_kernel<kTile><<<(unsigned)T, kTile, 0, st>>>(rv.rec, m, pq);
  GLR_LAUNCHED("tile_pq_kernel");
  GLR_CUDA(cudaMemsetAsync(cnt_m + T, 0, sizeof(unsigned long long), st));
  GLR_CUDA(cudaMemsetAsync(cnt_f + T, 0, sizeof(unsigned long long), st));
  tile_class_kernel<false><<<(unsigned)T, kClassThreads, 0, st>>>(
      rv.hdr, box, pq, T, row_rank, row_world, cnt_m, cnt_f, nullptr, nullptr, nullptr);
  GLR_LAUNCHED("tile_class_kernel<count>");
  size_t tb = t_scan;
  GLR_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, cnt_m, off_m, (int)(T + 1), st));
  count_launch(2);
  tb = t_scan;
  GLR_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, cnt_f, off_f, (int)(T + 1), st));
  count_launch(2);
  unsigned long long tot[2] = {0, 0};
  GLR_CUDA(cudaMemcpyAsync(&tot[0], off_m + T, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                           st));
  GLR_CUDA(cudaMemcpyAsync(&tot[1], off_f + T, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                           st));
  GLR_CUDA(cudaStreamSynchronize(st));
  h_counts[0] = tot[0];
  h_counts[1] = tot[1];
  if (d_list != nullptr && capacity >= tot[0] + tot[1] && tot[0] + tot[1] > 0) {
    tile_class_kernel<true><<<(unsigned)T, kClassThreads, 0, st>>>(
        rv.hdr, box, pq, T, row_rank, row_world, nullptr, nullptr, off_m, off_f, d_list);
    GLR_LAUNCHED("tile_class_kernel<fill>");
    if (d_sub != nullptr) {
      GLR_CUDA(cudaMemsetAsync(d_sub, 0, (size_t)(tot[0] + tot[1]) * sizeof(SubMask), st));
      if (tot[0] > 0) {
        constexpr int kPqThreads = kSubJ < 32 ? 32 : kSubJ;
        tile_pq_kernel<kSubJ><<<(unsigned)(m_pad / kPqThreads), kPqThreads, 0, st>>>(rv.rec, m,
                                                                                     pqs);
        GLR_LAUNCHED("tile_pq_kernel<sub>");
        sub_mask_kernel<<<blocks_for((int64_t)(tot[0] * kSubBits), 256, 16), 256, 0, st>>>(
            rv.hdr, d_list, tot[0], pqs, d_sub);
        GLR_LAUNCHED("sub_mask_kernel");
      }
    }
  }
  return GLR_OK;
}

}  // namespace glr

#ifdef GLR_XFSTATS
extern "C" int glr_debug_fstats(unsigned long long *h, int reset) {
  if (cudaDeviceSynchronize() != cudaSuccess) return GLR_ECUDA;
  if (cudaMemcpyFromSymbol(h, glr::g_fstats, sizeof(unsigned long long) * 2) != cudaSuccess)
    return GLR_ECUDA;
  if (reset) {
    const unsigned long long z[2] = {0, 0};
    if (cudaMemcpyToSymbol(glr::g_fstats, z, sizeof(z)) != cudaSuccess) return GLR_ECUDA;
  }
  return GLR_OK;
}
#endif

extern "C" {

int glr_crossing_tile(void) { return glr::kTile; }

int glr_crossing_sub_mask_bytes(void) { return (int)sizeof(glr::SubMask); }

int glr_crossing_sub_quarters(void) { return glr::kSubQuarters; }

int glr_crossing_band(void) { return glr::kBandTiles; }

uint64_t glr_crossing_chunk(uint64_t span, int world) { return glr::chunk_for(span, world); }

int glr_crossing_tile_weights(const void *d_records, int64_t n, int64_t m, double beta,
                              double *d_w, void *stream) {
  if (d_records == nullptr || d_w == nullptr || m < 0 || n < 0) {
    glr::set_error("glr_crossing_tile_weights: invalid arguments");
    return GLR_EARG;
  }
  const int64_t m_pad = glr::pad_edges(m < 1 ? 1 : m);
  glr::RecView rv = glr::view(const_cast<void *>(d_records), n, m);
  glr::tile_weight_kernel<<<(unsigned)(m_pad / glr::kTile), glr::kTile, 0,
                            glr::as_stream(stream)>>>(rv.newc, beta, d_w);
  GLR_LAUNCHED("tile_weight_kernel");
  return GLR_OK;
}

int glr_crossing_pairs_interleaved(const void *d_records, int64_t n, int64_t m, int with_angle,
                                   double ideal, const void *d_list, uint64_t list_len, int rank,
                                   int world, double *d_out, void *stream) {
  const uint64_t U = d_list != nullptr ? list_len : glr_crossing_units(m);
  return glr::crossing_pairs(d_records, n, m, with_angle, ideal,
                             reinterpret_cast<const int2 *>(d_list), list_len, 0, U, rank, world,
                             d_out, glr::as_stream(stream));
}

int glr_crossing_candidates(const void *d_records, int64_t n, int64_t m, void *d_list,
                            uint64_t capacity, uint64_t *h_count, void *stream) {
  return glr::crossing_candidates(d_records, n, m, reinterpret_cast<int2 *>(d_list), capacity,
                                  h_count, glr::as_stream(stream));
}

int glr_crossing_pairs_list(const void *d_records, int64_t n, int64_t m, int with_angle,
                            double ideal, const void *d_list, uint64_t list_len,
                            uint64_t unit_begin, uint64_t unit_end, double *d_out, void *stream) {
  if (d_list == nullptr && list_len > 0) {
    glr::set_error("glr_crossing_pairs_list: null list");
    return GLR_EARG;
  }
  if (list_len == 0) {
    if (unit_begin != 0 || unit_end != 0) {
      glr::set_error("glr_crossing_pairs_list: unit range outside an empty list");
      return GLR_EARG;
    }
    cudaStream_t st = glr::as_stream(stream);
    GLR_CUDA(cudaMemsetAsync(d_out, 0, 2 * sizeof(double), st));
    return GLR_OK;
  }
  return glr::crossing_pairs(d_records, n, m, with_angle, ideal,
                             reinterpret_cast<const int2 *>(d_list), list_len, unit_begin,
                             unit_end, 0, 1, d_out, glr::as_stream(stream));
}

int glr_crossing_candidates_classified(const void *d_records, int64_t n, int64_t m,
                                       void *d_list, void *d_sub, uint64_t capacity,
                                       uint64_t *h_counts, void *stream) {
  return glr::crossing_candidates_classified(d_records, n, m, reinterpret_cast<int2 *>(d_list),
                                             reinterpret_cast<glr::SubMask *>(d_sub), capacity,
                                             h_counts, glr::as_stream(stream));
}

int glr_crossing_candidates_rows(const void *d_records, int64_t n, int64_t m, void *d_list,
                                 void *d_sub, uint64_t capacity, uint64_t *h_counts, int rank,
                                 int world, void *stream) {
  return glr::crossing_candidates_classified(d_records, n, m, reinterpret_cast<int2 *>(d_list),
                                             reinterpret_cast<glr::SubMask *>(d_sub), capacity,
                                             h_counts, glr::as_stream(stream), rank, world);
}

int glr_crossing_pairs_classified(const void *d_records, int64_t n, int64_t m, int with_angle,
                                  double ideal, const void *d_list, const void *d_sub,
                                  uint64_t mixed_len, uint64_t full_len, uint64_t unit_begin,
                                  uint64_t unit_end, int rank, int world, double *d_out,
                                  void *stream) {
  const uint64_t U = mixed_len + full_len;
  if ((d_list == nullptr && U > 0) || unit_begin > unit_end || unit_end > U || U < mixed_len) {
    glr::set_error("glr_crossing_pairs_classified: unit range [%llu, %llu) outside [0, %llu)",
                   (unsigned long long)unit_begin, (unsigned long long)unit_end,
                   (unsigned long long)U);
    return GLR_EARG;
  }
  const int2 *lst = reinterpret_cast<const int2 *>(d_list);
  const uint64_t mb = unit_begin < mixed_len ? unit_begin : mixed_len;
  const uint64_t me = unit_end < mixed_len ? unit_end : mixed_len;
  const uint64_t fb = (unit_begin > mixed_len ? unit_begin : mixed_len) - mixed_len;
  const uint64_t fe = (unit_end > mixed_len ? unit_end : mixed_len) - mixed_len;
  return glr::crossing_pairs(d_records, n, m, with_angle, ideal, mixed_len ? lst : nullptr,
                             mixed_len, mb, me, rank, world, d_out, glr::as_stream(stream),
                             full_len ? lst + mixed_len : nullptr, fb, fe,
                             reinterpret_cast<const glr::SubMask *>(d_sub));
}

uint64_t glr_crossing_units(int64_t m) {
  const int64_t m_pad = glr::pad_edges(m < 1 ? 1 : m);
  return glr::tri_units((uint64_t)(m_pad / glr::kTile));
}

size_t glr_crossing_records_bytes(int64_t n, int64_t m) { return glr::layout(n, m).total; }

int glr_crossing_prepare(const double *d_xy, int64_t n, const int64_t *d_edges, int64_t m,
                         void *d_records, void *stream) {
  return glr::crossing_prepare(d_xy, n, d_edges, m, d_records, glr::as_stream(stream));
}

int glr_crossing_pairs(const void *d_records, int64_t n, int64_t m, int with_angle, double ideal,
                       uint64_t unit_begin, uint64_t unit_end, double *d_out, void *stream) {
  return glr::crossing_pairs(d_records, n, m, with_angle, ideal, nullptr, 0, unit_begin,
                             unit_end, 0, 1, d_out, glr::as_stream(stream));
}

int glr_crossing_scan(const double *d_xy, int64_t n, const int64_t *d_edges, int64_t m,
                      int with_angle, double ideal, uint64_t unit_begin, uint64_t unit_end,
                      double *d_out, void *stream) {
  cudaStream_t st = glr::as_stream(stream);
  glr::Scratch rec(glr::layout(n, m).total, st);
  GLR_CUDA(rec.err);
  int rc = glr::crossing_prepare(d_xy, n, d_edges, m, rec.ptr, st);
  if (rc != GLR_OK) return rc;
  return glr::crossing_pairs(rec.ptr, n, m, with_angle, ideal, nullptr, 0, unit_begin, unit_end,
                             0, 1, d_out, st);
}

int glr_crossing_set_mode(void *d_records, int mode, void *stream) {
  if (d_records == nullptr || mode < glr::kModeGeneral || mode > glr::kModeFilter) {
    glr::set_error("glr_crossing_set_mode: invalid arguments (mode %d)", mode);
    return GLR_EARG;
  }
  glr::set_mode_kernel<<<1, 1, 0, glr::as_stream(stream)>>>(
      reinterpret_cast<glr::RecHeader *>(d_records), mode);
  GLR_LAUNCHED("set_mode_kernel");
  return GLR_OK;
}

int glr_crossing_fast_path(const void *d_records, void *stream) {
  int fast = -1;
  cudaStream_t st = glr::as_stream(stream);
  if (cudaMemcpyAsync(&fast, d_records, sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess) {
    glr::set_error("glr_crossing_fast_path: copy failed");
    return -1;
  }
  return fast;
}

}  // extern "C"
