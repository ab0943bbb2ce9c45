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
occlusion_pairs_kernel(const double2 *__restrict__ xy, int64_t n, uint64_t T, uint64_t ubeg,
                       uint64_t uend, unsigned long long thr_bits,
                       unsigned long long *__restrict__ cta_cnt) {
  __shared__ __align__(16) double2 sj[kTile];
  __shared__ unsigned long long red[kThreads / 32];
  const uint64_t span = uend - ubeg;
  const uint64_t b = ubeg + span * blockIdx.x / gridDim.x;
  const uint64_t e = ubeg + span * (blockIdx.x + 1) / gridDim.x;
  // padding vertices sit at +inf: every difference with them is inf or NaN,
  // and inf/NaN squared sums never compare below a finite threshold as bits
  // (NaN bit patterns exceed +inf's).
  const double PAD = __longlong_as_double(0x7ff0000000000000ll);
  unsigned long long total = 0;
  double xi[kK], yi[kK];
  uint64_t ti = 0, tj = 0, cur = ~0ull;
  if (b < e) tri_unit_coords(b, T, &ti, &tj);
  for (uint64_t u = b; u < e; ++u) {
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
    if (++tj == T) { ++ti; tj = ti; }
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
  using namespace glr;
  cudaStream_t st = as_stream(stream);
  if (d_out == nullptr || n < 0 || (n > 0 && d_xy == nullptr)) {
    set_error("glr_occlusion_count: invalid arguments");
    return GLR_EARG;
  }
  const uint64_t U = glr_occlusion_units(n);
  if (unit_begin > unit_end || unit_end > U) {
    set_error("glr_occlusion_count: unit range [%llu, %llu) outside [0, %llu)",
              (unsigned long long)unit_begin, (unsigned long long)unit_end,
              (unsigned long long)U);
    return GLR_EARG;
  }
  if (n < 2 || unit_begin == unit_end || !(thr > 0.0)) {
    GLR_CUDA(cudaMemsetAsync(d_out, 0, sizeof(double), st));
    return GLR_OK;
  }
  const uint64_t T = (uint64_t)(pad_vertices(n) / kTile);
  uint64_t g = (uint64_t)sm_count() * kMinBlocks;
  if (unit_end - unit_begin < g) g = unit_end - unit_begin;
  const int grid = (int)g;
  Scratch scr((size_t)grid * sizeof(unsigned long long), st);
  GLR_CUDA(scr.err);
  unsigned long long thr_bits;
  memcpy(&thr_bits, &thr, sizeof(thr));
  occlusion_pairs_kernel<<<grid, kThreads, 0, st>>>(reinterpret_cast<const double2 *>(d_xy), n, T,
                                                    unit_begin, unit_end, thr_bits,
                                                    scr.as<unsigned long long>());
  GLR_LAUNCHED("occlusion_pairs_kernel");
  occ_finalize_kernel<<<1, 32, 0, st>>>(scr.as<unsigned long long>(), grid, d_out);
  GLR_LAUNCHED("occ_finalize_kernel");
  return GLR_OK;
}

}  // extern "C"
