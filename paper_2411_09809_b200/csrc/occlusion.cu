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
#ifndef GLR_OMINB
#define GLR_OMINB 4
#endif
constexpr int kMinBlocks = GLR_OMINB;  // CTAs per SM

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

struct OccHeader;
__device__ inline int occ_header_use(const void *h) { return *reinterpret_cast<const int *>(h); }

__global__ void __launch_bounds__(kThreads, kMinBlocks)
occlusion_pairs_kernel(const double2 *__restrict__ xy, int64_t n, const int2 *__restrict__ ulist,
                       uint64_t T, uint64_t ubeg, uint64_t uend, unsigned long long thr_bits,
                       const void *__restrict__ hdr, unsigned long long *__restrict__ cta_cnt) {
  if (hdr != nullptr && occ_header_use(hdr)) return;  // the FP32 filter kernel runs instead
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

// ---- certified FP32 filter (the default when the input admits it) --------
//
// Coordinates translated to their bounding-box corner and scaled by a power
// of two into [0, 1/2] (X = RN32((x - x0) sc)); per pair S = RN(RN(dX dX) +
// dY dY) with dX = RN32(Xi - Xj) (FADD2/FMUL2/FFMA2 over two i-vertices).
// |S - sc^2 d^2| <= E(S) = 3 2^-25 sqrt(2.01 S) + 2^-21 S + 2^-48 (quantisation
// 2^-26 per coordinate, the subtraction, the two roundings, the reference's
// own FP64 rounding), so with T = sc^2 thr:
//   S < T_lo = RD32(T - E(T))       certainly occluding (s_fp64 < thr),
//   S > T_hi = RU32(T + E(4T))      certainly not,
// and pairs in [T_lo, T_hi] -- exact ties included -- are re-tested in FP64.
// Admissible when every coordinate is finite with magnitude <= 2^500, the
// extent W in [2^-400, 2^500] and T in [1e-14, 1e30]; otherwise the FP64
// kernel runs (both are launched; the header decides on the device).
struct OccHeader {
  int use;
  int pad;
  double x0, y0, sc;
  float tlo, thi, tmid, thw;
};

__global__ void __launch_bounds__(1024)
occ_header_kernel(const double2 *__restrict__ xy, int64_t n, double thr, OccHeader *h) {
  __shared__ double red[5][32];
  __shared__ int bad_any;
  if (threadIdx.x == 0) bad_any = 0;
  __syncthreads();
  double x0 = INFINITY, x1 = -INFINITY, y0 = INFINITY, y1 = -INFINITY, amax = 0.0;
  int bad = 0;
  for (int64_t v = threadIdx.x; v < n; v += blockDim.x) {
    const double2 p = xy[v];
    if (!isfinite(p.x) || !isfinite(p.y)) bad = 1;
    x0 = fmin(x0, p.x); x1 = fmax(x1, p.x);
    y0 = fmin(y0, p.y); y1 = fmax(y1, p.y);
    amax = fmax(amax, fmax(fabs(p.x), fabs(p.y)));
  }
  if (bad) bad_any = 1;
  for (int o = 16; o > 0; o >>= 1) {
    x0 = fmin(x0, __shfl_down_sync(0xffffffffu, x0, o));
    x1 = fmax(x1, __shfl_down_sync(0xffffffffu, x1, o));
    y0 = fmin(y0, __shfl_down_sync(0xffffffffu, y0, o));
    y1 = fmax(y1, __shfl_down_sync(0xffffffffu, y1, o));
    amax = fmax(amax, __shfl_down_sync(0xffffffffu, amax, o));
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    red[0][w] = x0; red[1][w] = x1; red[2][w] = y0; red[3][w] = y1; red[4][w] = amax;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  for (int i = 1; i < (int)(blockDim.x >> 5); ++i) {
    x0 = fmin(x0, red[0][i]); x1 = fmax(x1, red[1][i]);
    y0 = fmin(y0, red[2][i]); y1 = fmax(y1, red[3][i]);
    amax = fmax(amax, red[4][i]);
  }
  OccHeader H;
  H.use = 0;
  H.pad = 0;
  H.x0 = x0;
  H.y0 = y0;
  H.sc = 1.0;
  H.tlo = H.thi = H.tmid = H.thw = 0.0f;
  const double W = fmax(__dsub_ru(x1, x0), __dsub_ru(y1, y0));
  if (!bad_any && amax <= 0x1p500 && W >= 0x1p-400 && W <= 0x1p500 && thr >= 0x1p-600) {
    const double sc = ldexp(1.0, -(ilogb(W) + 2));
    const double T = thr * sc * sc;  // exact: sc is a power of two, no over/underflow here
    if (T >= 1e-14 && T <= 1e30) {
      auto E = [](double S) { return 3.0 * 0x1p-25 * sqrt(2.01 * S) + 0x1p-21 * S + 0x1p-48; };
      const float tlo = __double2float_rd(T - E(T));
      const float thi = __double2float_ru(T + E(4.0 * T));
      H.use = 1;
      H.sc = sc;
      H.tlo = tlo;
      H.thi = thi;
      // uncertain band [tlo, thi] as |S - tmid| <= thw, widened by rounding
      H.tmid = __double2float_rn(0.5 * ((double)tlo + (double)thi));
      H.thw = __double2float_ru(0.5 * ((double)thi - (double)tlo) * (1.0 + 0x1p-20) +
                                0x1p-100);
    }
  }
  *h = H;
}

// Scaled FP32 coordinates twice: sxy[v] (the j role, staged per unit in
// shared memory) and, for the i role, NEGATED and packed per thread so that
// one 128-bit load gives a thread's i-vertex pair (v0, v1 = v0 + kThreads)
// as two register pairs (-x0, -x1 | -y0, -y1): nip[(tile*kK/2 + g)*kThreads
// + t] for tile slot t + 2g kThreads.  Pads (v >= n, up to the tile end):
// i side -3e38 (negated +3e38), so every difference with a pad overflows to
// infinity.
constexpr float kOccPad = 3.0e38f;
__global__ void occ_scale_kernel(const double2 *__restrict__ xy, int64_t n, int64_t n_pad,
                                 const OccHeader *__restrict__ h, float2 *__restrict__ sxy,
                                 float *__restrict__ nip) {
  if (!h->use) return;
  const double x0 = h->x0, y0 = h->y0, sc = h->sc;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n_pad;
       v += (int64_t)gridDim.x * blockDim.x) {
    float x = kOccPad, y = kOccPad;
    if (v < n) {
      const double2 p = xy[v];
      x = __double2float_rn(__dmul_rn(__dsub_rn(p.x, x0), sc));
      y = __double2float_rn(__dmul_rn(__dsub_rn(p.y, y0), sc));
      sxy[v] = make_float2(x, y);
    }
    const int64_t tile = v / kTile;
    const int slot = (int)(v % kTile), t = slot % kThreads, k = slot / kThreads;
    float *q = nip + 4 * ((tile * (kK / 2) + k / 2) * kThreads + t);
    q[k & 1] = -x;
    q[2 + (k & 1)] = -y;
  }
}

__device__ __forceinline__ uint64_t o2_pack(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float o2_lo(uint64_t v) {
  float lo;
  asm("mov.b64 {%0, _}, %1;" : "=f"(lo) : "l"(v));
  return lo;
}
__device__ __forceinline__ float o2_hi(uint64_t v) {
  float hi;
  asm("mov.b64 {_, %0}, %1;" : "=f"(hi) : "l"(v));
  return hi;
}
__device__ __forceinline__ uint64_t o2_add(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t o2_fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}

constexpr int kOccFBlock = 4;  // j-vertices per filter block (one warp vote)

// The threshold folded into the products (default): per pair
//   d = RN(dY dY + RN(dX dX - t_lo))
// (two FFMA2 per two pairs instead of FMUL2 + FFMA2 + FADD2: the filter is
// bound by register-file reads, tools/rf_model.py).  The sign bit of d is
// the exact pre-rounding value's sign, so d < 0 certifies occlusion and
// d > RU(t_hi - t_lo) certifies non-occlusion with the same t_lo / t_hi as
// the unfolded test (K3: the two roundings stay within 2^-23
// max(S, t_lo), the budget the band already allots them;
// tests/test_filter_bound.py checks it with exact rationals).  Masked
// diagonal pairs -> +inf.
template <bool DIAG>
__device__ __forceinline__ void occ_d(const uint64_t (&X)[kK / 2], const uint64_t (&Y)[kK / 2],
                                      float2 pj, int jj, uint64_t NEGTLO2, float (&D)[kK]) {
  const uint64_t XJ = o2_pack(pj.x, pj.x), YJ = o2_pack(pj.y, pj.y);
#pragma unroll
  for (int g = 0; g < kK / 2; ++g) {
    // X, Y hold the NEGATED i coordinates: dx = xj + (-xi) = RN(xj - xi)
    const uint64_t dx = o2_add(XJ, X[g]), dy = o2_add(YJ, Y[g]);
    const uint64_t d = o2_fma(dy, dy, o2_fma(dx, dx, NEGTLO2));
    D[2 * g] = o2_lo(d);
    D[2 * g + 1] = o2_hi(d);
  }
  if (DIAG) {
#pragma unroll
    for (int k = 0; k < kK; ++k)
      if (!(jj > (int)threadIdx.x + k * kThreads)) D[k] = INFINITY;
  }
}

template <bool DIAG>
__device__ __forceinline__ void occ_filter_block(const uint64_t (&X)[kK / 2],
                                                 const uint64_t (&Y)[kK / 2], const float2 *sj,
                                                 int jj0, const OccHeader &H,
                                                 unsigned vote_bits,
                                                 const double2 *__restrict__ xy, int64_t ibase,
                                                 int64_t jbase, int64_t n,
                                                 unsigned long long thr_bits,
                                                 unsigned (&cnt)[kK]) {
  // min over the block of d viewed as unsigned: a non-negative float orders
  // like its bit pattern and a negative one (certain hit) is above every
  // non-negative, so one VIMNMX3 per two pairs finds whether any d lies in
  // [+0, RU(thi - tlo)], the uncertain band
  unsigned m = 0xffffffffu;
  const uint64_t NEGTLO2 = o2_pack(-H.tlo, -H.tlo);
#pragma unroll
  for (int q = 0; q < kOccFBlock; ++q) {
    float D[kK];
    occ_d<DIAG>(X, Y, sj[jj0 + q], jj0 + q, NEGTLO2, D);
#pragma unroll
    for (int k = 0; k < kK; ++k) {
      const unsigned b = __float_as_uint(D[k]);
      cnt[k] += b >> 31;  // certain hit: the sign bit
      m = min(m, b);      // uncertain: bits in [+0, RU(thi - tlo)]
    }
  }
  if (__any_sync(0xffffffffu, m <= vote_bits)) {
#pragma unroll 1
    for (int q = 0; q < kOccFBlock; ++q) {
      float D[kK];
      occ_d<DIAG>(X, Y, sj[jj0 + q], jj0 + q, NEGTLO2, D);
      const int64_t vj = jbase + jj0 + q;
#pragma unroll
      for (int k = 0; k < kK; ++k) {
        if (__float_as_uint(D[k]) <= vote_bits) {  // uncertain: the reference's FP64 test
          const int64_t vi = ibase + threadIdx.x + k * kThreads;
          if (vi < n && vj < n) {
            const double2 a = xy[vi], b = xy[vj];
            const double dx = __dsub_rn(a.x, b.x), dy = __dsub_rn(a.y, b.y);
            const double s = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
            if ((unsigned long long)__double_as_longlong(s) < thr_bits) cnt[k] += 1u;
          }
        }
      }
    }
  }

}

__global__ void __launch_bounds__(kThreads, kMinBlocks)
occlusion_filter_kernel(const double2 *__restrict__ xy, const float2 *__restrict__ sxy,
                        const float4 *__restrict__ nip,
                        const OccHeader *__restrict__ hdr, int64_t n,
                        const int2 *__restrict__ ulist, uint64_t T, uint64_t ubeg, uint64_t uend,
                        unsigned long long thr_bits, unsigned long long *__restrict__ cta_cnt) {
  if (!hdr->use) return;
  const OccHeader H = *hdr;
  // packed constant tlo; vote bound = the band width rounded up, as bits
  const unsigned vote_bits = __float_as_uint(__fsub_ru(H.thi, H.tlo));
  __shared__ __align__(16) float2 sj[kTile];
  __shared__ unsigned long long red[kThreads / 32];
  const uint64_t span = uend - ubeg;
  const uint64_t b = ubeg + span * blockIdx.x / gridDim.x;
  const uint64_t e = ubeg + span * (blockIdx.x + 1) / gridDim.x;
  // pads: i side +3e38 (nip), j side -3e38: differences overflow, d = inf
  const float PADF = kOccPad;
  unsigned long long total = 0;
  uint64_t X[kK / 2], Y[kK / 2];
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
      for (int g = 0; g < kK / 2; ++g) {
        // the negated i coordinates (exact), so the pair loop adds with no
        // per-iteration negation
        const float4 q = nip[((int64_t)ti * (kK / 2) + g) * kThreads + threadIdx.x];
        X[g] = o2_pack(q.x, q.y);
        Y[g] = o2_pack(q.z, q.w);
      }
      cur = ti;
    }
    __syncthreads();
    for (int q = threadIdx.x; q < kTile; q += kThreads) {
      const int64_t v = (int64_t)tj * kTile + q;
      sj[q] = v < n ? sxy[v] : make_float2(-PADF, -PADF);
    }
    __syncthreads();
    unsigned cnt[kK];
#pragma unroll
    for (int k = 0; k < kK; ++k) cnt[k] = 0;
    const int64_t ibase = (int64_t)ti * kTile, jbase = (int64_t)tj * kTile;
    if (ti == tj) {
      for (int jj = 0; jj < kTile; jj += kOccFBlock)
        occ_filter_block<true>(X, Y, sj, jj, H, vote_bits, xy, ibase, jbase, n,
                               thr_bits, cnt);
    } else {
#pragma unroll 1
      for (int jj = 0; jj < kTile; jj += kOccFBlock)
        occ_filter_block<false>(X, Y, sj, jj, H, vote_bits, xy, ibase, jbase, n,
                                thr_bits, cnt);
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

// process-wide switch for cross-checks (glr_occlusion_set_filter)
int g_occ_filter = 1;

int occ_blocks(int64_t work) {
  int64_t b = (work + 127) / 128;
  const int64_t cap = (int64_t)sm_count() * 16;
  if (b > cap) b = cap;
  return (int)(b < 1 ? 1 : b);
}

int occlusion_run(const double *d_xy, int64_t n, double thr, const int2 *d_list,
                  uint64_t list_len, uint64_t ubeg, uint64_t uend, double *d_out,
                  cudaStream_t st, const char *who) {
  const bool use_filter = g_occ_filter != 0;
  if (d_out == nullptr || n < 0 || (n > 0 && d_xy == nullptr)) {
    set_error("%s: invalid arguments", who);
    return GLR_EARG;
  }
  if (n > ((int64_t)1 << 26) * 2) {  // the float64 count slot is exact below 2^53 pairs
    set_error("%s: n=%lld vertices: n(n-1)/2 reaches 2^53, counts would round", who,
              (long long)n);
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
  const size_t a_cta = ((size_t)grid * sizeof(unsigned long long) + 255) & ~(size_t)255;
  const size_t a_hdr = 256;
  const int64_t n_pad = (int64_t)T * kTile;
  const size_t a_sxy = ((size_t)n * sizeof(float2) + 255) & ~(size_t)255;
  const size_t a_nip = ((size_t)n_pad * sizeof(float2) + 255) & ~(size_t)255;
  Scratch scr(a_cta + a_hdr + (use_filter ? a_sxy + a_nip : 0), st);
  GLR_CUDA(scr.err);
  unsigned long long *cta = scr.as<unsigned long long>();
  OccHeader *hdr = reinterpret_cast<OccHeader *>(scr.as<char>() + a_cta);
  float2 *sxy = reinterpret_cast<float2 *>(scr.as<char>() + a_cta + a_hdr);
  float *nip = reinterpret_cast<float *>(scr.as<char>() + a_cta + a_hdr + a_sxy);
  unsigned long long thr_bits;
  memcpy(&thr_bits, &thr, sizeof(thr));
  const double2 *xy = reinterpret_cast<const double2 *>(d_xy);
  if (use_filter) {
    occ_header_kernel<<<1, 1024, 0, st>>>(xy, n, thr, hdr);
    GLR_LAUNCHED("occ_header_kernel");
    occ_scale_kernel<<<occ_blocks(n_pad), 128, 0, st>>>(xy, n, n_pad, hdr, sxy, nip);
    GLR_LAUNCHED("occ_scale_kernel");
    occlusion_filter_kernel<<<grid, kThreads, 0, st>>>(
        xy, sxy, reinterpret_cast<const float4 *>(nip), hdr, n, d_list, T, ubeg, uend, thr_bits,
        cta);
    GLR_LAUNCHED("occlusion_filter_kernel");
  }
  occlusion_pairs_kernel<<<grid, kThreads, 0, st>>>(xy, n, d_list, T, ubeg, uend, thr_bits,
                                                    use_filter ? hdr : nullptr, cta);
  GLR_LAUNCHED("occlusion_pairs_kernel");
  occ_finalize_kernel<<<1, 32, 0, st>>>(scr.as<unsigned long long>(), grid, d_out);
  GLR_LAUNCHED("occ_finalize_kernel");
  return GLR_OK;
}

}  // namespace
}  // namespace glr

extern "C" {

int glr_occlusion_set_filter(int enable) {
  const int prev = glr::g_occ_filter;
  glr::g_occ_filter = enable ? 1 : 0;
  return prev;
}

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
