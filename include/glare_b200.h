/* glare_b200 -- C ABI of the B200-native exact readability-metric kernels.
 *
 * The reference (glare, /root/reference/pkg/src/glare) is pure Python and has
 * no FFI; its "operator API" for this path is the set of Python functions
 * re-exported by glare.metrics (metrics/__init__.py:11-25) and called by the
 * oracle mode of the engine (engine.py:74-94).  Each entry point below
 * replaces the numpy body of one of those functions; the Python package
 * paper_2411_09809_b200 binds them with ctypes and keeps the reference
 * signatures, validation and degenerate-case returns.
 *
 * Conventions
 *  - every pointer argument named d_* is a DEVICE pointer owned by the caller;
 *    the library never frees caller memory and allocates only stream-ordered
 *    scratch (cudaMallocAsync on `stream`) that it releases before returning;
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default);
 *    calls are asynchronous on it unless stated otherwise;
 *  - xy is float64 (n,2) row-major (interleaved double2), edges is int64
 *    (m,2) row-major index pairs normalised exactly as LayoutGraph does
 *    (model.py:56-132: small index first, lexicographically sorted, unique,
 *    no loops, no zero-length edges);
 *  - return value: GLR_OK (0) or an error code; glr_last_error() returns a
 *    thread-local message for the last failing call on this thread.
 *
 * Sharding: the O(m^2)/O(n^2) passes enumerate an upper-triangular space of
 * tile pairs ("units", glr_*_units).  A call processes units
 * [unit_begin, unit_end); partial results of disjoint ranges add up to the
 * full result, so ranks of a multi-GPU job each take one contiguous range and
 * sum their partials with one allreduce.
 */
#ifndef GLARE_B200_H
#define GLARE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  GLR_OK = 0,
  GLR_EARG = 1,       /* invalid argument (ParameterError / InputError side) */
  GLR_ECUDA = 2,      /* CUDA runtime error */
  GLR_ENCCL = 3,      /* NCCL unavailable or failed (collective entry points) */
  GLR_EINVARIANT = 4, /* internal consistency check failed (InvariantError) */
  GLR_EFALLBACK = 8,  /* reserved (earlier loaders deferred to Python with it) */
  GLR_EPARSE = 16     /* loaders: malformed input, see glr_parse_status() */
};

/* ABI version: (major << 16) | minor. */
int glr_version(void);

/* Thread-local message describing the last error on this thread. */
const char *glr_last_error(void);

/* ---- node occlusion: reference metrics/exact.py:55-74 -------------------- */

/* Vertices per tile of the occlusion unit space. */
int glr_occlusion_tile(void);

/* Number of vertex tile-pair units for n vertices: T(T+1)/2 with
 * T = ceil(n / glr_occlusion_tile()), unit u = (ti, tj), ti <= tj, row-major. */
uint64_t glr_occlusion_units(int64_t n);

/* Writes to d_out[0] (float64, exact below 2^53) the number of unordered
 * vertex pairs (i < j) whose tile pair lies in units [unit_begin, unit_end)
 * and satisfies
 *     fl(fl(dx*dx) + fl(dy*dy)) < thr,  dx = x_i - x_j, dy = y_i - y_j,
 * where thr = (2.0*r)**2 computed by the caller exactly as exact.py:63. */
int glr_occlusion_count(const double *d_xy, int64_t n, double thr,
                        uint64_t unit_begin, uint64_t unit_end,
                        double *d_out, void *stream);

/* ---- edge crossing / crossing angle: exact.py:145-238, geometry.py:62-110 */

/* Edges per tile of the crossing unit space. */
int glr_crossing_tile(void);

/* j-tiles per band of the crossing unit order.  Crossing units are the same
 * tile pairs (ti <= tj) as for occlusion, T = ceil(m / glr_crossing_tile()),
 * but ordered by (band of tj, ti, tj) with bands of glr_crossing_band()
 * consecutive j-tiles (within a band: rows ti below the band first, then the
 * band's own triangle), so concurrently running CTAs share j-tiles in L2. */
int glr_crossing_band(void);

/* Units per chunk of interleaved sharding for a unit range of `span` units
 * over `world` ranks (glr_crossing_pairs_interleaved): a function of span,
 * world and compile-time constants only -- never of the device -- so every
 * rank cuts the same chunks; rank r owns the chunks whose index is r mod
 * world, i.e. unit u of [b, e) belongs to rank ((u - b) / chunk) % world. */
uint64_t glr_crossing_chunk(uint64_t span, int world);

/* Number of edge tile-pair units for m edges: T(T+1)/2. */
uint64_t glr_crossing_units(int64_t m);

/* Bytes of the record buffer glr_crossing_prepare fills for n vertices and
 * m edges (caller allocates, 256-byte aligned). */
size_t glr_crossing_records_bytes(int64_t n, int64_t m);

/* Builds the per-edge records (endpoint coordinates a = xy[edges[:,0]],
 * b = xy[edges[:,1]], b - a, exact order-preserving 32-bit bbox ranks, axis
 * angle theta = mod(atan2(by-ay, bx-ax), pi), endpoint ids) and the
 * per-vertex incidence lists into d_records.  Also decides whether the input
 * admits the fast sign path (every nonzero |coordinate| in [2^-160, 2^500],
 * see DESIGN.md); the decision is stored in the records header. */
int glr_crossing_prepare(const double *d_xy, int64_t n, const int64_t *d_edges,
                         int64_t m, void *d_records, void *stream);

/* Writes to d_out[0..1] the partial (count, dev_sum) of the crossing scan
 * restricted to edge pairs (i < j) whose tile pair (i / tile, j / tile) lies
 * in units [unit_begin, unit_end): count of pairs with closed-bbox overlap,
 * no shared vertex index and the straddle predicate of geometry.py:62-79;
 * dev_sum = sum over those pairs of |ideal - min(d, pi - d)|,
 * d = |theta_i - theta_j| (0 when !with_angle).  Partials of a disjoint cover
 * of [0, glr_crossing_units(m)) sum exactly (counts) to exact.py's result. */
int glr_crossing_pairs(const void *d_records, int64_t n, int64_t m,
                       int with_angle, double ideal, uint64_t unit_begin,
                       uint64_t unit_end, double *d_out, void *stream);

/* prepare + pairs over [unit_begin, unit_end) with internal scratch. */
int glr_crossing_scan(const double *d_xy, int64_t n, const int64_t *d_edges,
                      int64_t m, int with_angle, double ideal,
                      uint64_t unit_begin, uint64_t unit_end, double *d_out,
                      void *stream);

/* Interleaved sharding of the whole unit space (dense triangle when d_list is
 * NULL, else the candidate list of length list_len): units are cut into
 * chunks (size derived from the unit count and `world` only) and this call
 * takes the chunks whose index is rank (mod world).  Every rank sees the same
 * mix of unit costs, and the partials of ranks 0..world-1 sum exactly to the
 * whole (the adjacency correction follows the same chunk ownership). */
int glr_crossing_pairs_interleaved(const void *d_records, int64_t n, int64_t m,
                                   int with_angle, double ideal,
                                   const void *d_list, uint64_t list_len,
                                   int rank, int world, double *d_out,
                                   void *stream);

/* Per-tile cost weights of prepared records for balanced sharding: d_w[t] =
 * tile + beta * (run starts in tile t), t < ceil(m / glr_crossing_tile()).
 * Unit (ti, tj) of the pair space costs about d_w[tj] (half on the
 * diagonal), because a j-edge that starts a run of edges sharing its first
 * endpoint recomputes the per-run terms. */
int glr_crossing_tile_weights(const void *d_records, int64_t n, int64_t m,
                              double beta, double *d_w, void *stream);

/* ---- culled variants (results identical) ---------- *
 * The GPU form of the reference oracle's own pruning: exact.py:170-199 sorts
 * edges by xmin and skips pairs whose x-ranges are disjoint (they fail the
 * closed-bbox test of exact.py:191-194); node_occlusion_grid
 * (metrics/enhanced.py:42-127) buckets vertices so only neighbouring cells
 * are compared.  Here whole tile pairs are skipped when their boxes are
 * disjoint (crossing) or farther apart than 2r (occlusion). */

/* Writes to d_edges_out the edge list in the culled plan's order -- rows
 * unchanged, only their order; hub groups as in glr_theta_sort_edges, for
 * vertices of degree >= 16384.  Short edges: (hub group, 4-D Morton code of
 * the edge's bbox sides xmin, xmax, ymin, ymax, diagonal orientation).  Long
 * edges (mean bbox half-perimeter >= 1/32 of the domain's): (hub group,
 * diagonal orientation), then a balanced k-d tree over the endpoints (P.x,
 * P.y, Q.x, Q.y) whose cells are the 256-edge tiles, 128-edge warp slices and
 * 64-edge quarters (spatial.cu), from 131,072 edges on; one 8-byte read back
 * decides between the two, so the call then synchronises the stream.  The metrics do not depend on
 * edge order (exact.py:145-222 visits every unordered pair once); compact
 * tiles let glr_crossing_candidates* skip or certify most tile pairs. */
int glr_spatial_sort_edges(const double *d_xy, int64_t n, const int64_t *d_edges,
                           int64_t m, int64_t *d_edges_out, void *stream);

/* Writes to d_edges_out the edge list reordered by (group, direction theta
 * = atan2(b - a) mod pi, exact.py:217-220's angle; rows unchanged).  Edges
 * incident to a vertex of degree >= hub_degree (0: GLR_HUB_DEGREE_DEFAULT)
 * form one group per such hub, the rest group 0.  Dense passes over this
 * order evaluate the crossing-angle deviation with one FP64 subtraction per
 * pair in units whose theta difference stays on one side of 0 and pi/2
 * (crossing.cu unit_shift), and skip units of two tiles of one hub's edges
 * (every pair shares the hub).  Results do not depend on the order. */
#ifndef GLR_HUB_DEGREE_DEFAULT
#define GLR_HUB_DEGREE_DEFAULT 4096  /* C5 sweep: 1024 4634 ms, 4096 4543, 8192 4570, none 4823 (profiles/r02_hub_sweep.txt) */
#endif
int glr_theta_sort_edges(const double *d_xy, int64_t n, const int64_t *d_edges,
                         int64_t m, int64_t hub_degree, int64_t *d_edges_out, void *stream);

/* Tuning / cross-check knob for glr_spatial_sort_edges: on = 0 keeps the
 * Morton order for long edges too, 1 (default) takes the k-d order from
 * 131,072 edges on (below that the tree's small launches cost more than the
 * pass), 2 takes it for any size, < 0 only queries.  Returns the previous
 * setting.  Results never depend on it. */
int glr_spatial_set_kd(int on);

/* Writes to d_xy_out the vertex positions reordered by Morton code (node
 * occlusion does not depend on vertex order). */
int glr_spatial_sort_vertices(const double *d_xy, int64_t n, double *d_xy_out,
                              void *stream);

/* Candidate tile pairs of prepared records: every (ti <= tj) whose tile rank
 * boxes overlap, row-major sorted, as int32 pairs (int2).  Synchronous:
 * *h_count receives the number of candidates; the list is written only when
 * d_list != NULL and capacity >= *h_count.  A pair with overlapping edge
 * bboxes always lies in a candidate tile pair, so scanning the candidates
 * gives exactly the dense result. */
int glr_crossing_candidates(const void *d_records, int64_t n, int64_t m,
                            void *d_list, uint64_t capacity, uint64_t *h_count,
                            void *stream);

/* glr_crossing_pairs over units [unit_begin, unit_end) of a candidate list
 * (unit u = tile pair d_list[u]); partials of a disjoint cover of
 * [0, list_len) sum to the dense result. */
int glr_crossing_pairs_list(const void *d_records, int64_t n, int64_t m,
                            int with_angle, double ideal, const void *d_list,
                            uint64_t list_len, uint64_t unit_begin,
                            uint64_t unit_end, double *d_out, void *stream);

/* Classified candidate tile pairs (the culled plan's list; replaces the
 * per-pair work of exact.py:170-217 for whole tile pairs).  Every (ti <= tj)
 * with overlapping tile rank boxes is certified, from per-tile boxes of the
 * edges' two endpoints and an error bound on the reference's own FP64 cross
 * products (admissible inputs only, see crossing.cu tile_class_kernel), as
 *   - none: no pair can pass proper_intersection_mask (dropped),
 *   - full: every pair passes it and shares no vertex, or
 *   - mixed: anything else.
 * d_list receives [mixed units | full units], each part row-major, as int2;
 * h_counts[0] = mixed units, h_counts[1] = full units.  Synchronous; the list
 * is written only when d_list != NULL and capacity >= both counts' sum.
 * d_sub (optional, one mask of glr_crossing_sub_mask_bytes() bytes per list
 * entry): for each mixed unit, block b = s * Q + q is warp-slice s (128
 * i-edges) x j-quarter q (256 / Q j-edges, Q = glr_crossing_sub_quarters());
 * bit b set: the block is certified empty, bit 2Q + b: certified full (the
 * same two certificates, on the blocks' own endpoint boxes).  The pair pass
 * skips both kinds and counts a full block as n_i * n_j crossings with the
 * pairs' deviations (closed form or exact.py:217-221 per pair). */
int glr_crossing_candidates_classified(const void *d_records, int64_t n, int64_t m,
                                       void *d_list, void *d_sub, uint64_t capacity,
                                       uint64_t *h_counts, void *stream);
/* The same list restricted to the tile rows ti = rank (mod world): rank's
 * share of the classified plan when the ROWS are dealt to the ranks, so that
 * each rank classifies only its own rows (the plan build shards with the
 * pass; no rank ever holds the whole list).  The world lists partition the
 * full list; each rank scans its own with glr_crossing_pairs_classified as
 * rank 0 of 1 and the partials sum to the dense result
 * (glr_allreduce_sum_f64 or any allreduce). */
int glr_crossing_candidates_rows(const void *d_records, int64_t n, int64_t m,
                                 void *d_list, void *d_sub, uint64_t capacity,
                                 uint64_t *h_counts, int rank, int world, void *stream);
/* Layout of d_sub: bytes per mask (2, 4 or 8) and j-quarters per tile. */
int glr_crossing_sub_mask_bytes(void);
int glr_crossing_sub_quarters(void);

/* Units [unit_begin, unit_end) of a classified list (unit u = d_list[u]; u <
 * mixed_len: the pair kernels, which skip the blocks d_sub marks -- the full
 * ones are counted whole like full units; otherwise a full unit: na * nb
 * crossings and the pairs' deviations (exact.py:217-221) from a closed form
 * where the unit's theta ranges fix the formula's branch, else from
 * piecewise-linear sums over the j-tile's sorted angles, else -- small mean
 * deviation -- pair by pair), under interleaved chunk ownership
 * for rank of world (0 of 1: the whole range).  Partials over a disjoint
 * cover of [0, mixed_len + full_len), or over all ranks, sum to the dense
 * result. */
int glr_crossing_pairs_classified(const void *d_records, int64_t n, int64_t m,
                                  int with_angle, double ideal, const void *d_list,
                                  const void *d_sub, uint64_t mixed_len, uint64_t full_len,
                                  uint64_t unit_begin, uint64_t unit_end, int rank,
                                  int world, double *d_out, void *stream);

/* Candidate vertex tile pairs: (ti <= tj) whose tile boxes are closer than
 * reach = 2r on both axes (fl(gap) < reach); same protocol as
 * glr_crossing_candidates.  Pairs in skipped tile pairs provably fail the
 * strict test fl(fl(dx*dx)+fl(dy*dy)) < (2r)^2. */
int glr_occlusion_candidates(const double *d_xy, int64_t n, double reach,
                             void *d_list, uint64_t capacity, uint64_t *h_count,
                             void *stream);

/* glr_occlusion_count over units [unit_begin, unit_end) of a candidate list. */
int glr_occlusion_count_list(const double *d_xy, int64_t n, double thr,
                             const void *d_list, uint64_t list_len,
                             uint64_t unit_begin, uint64_t unit_end,
                             double *d_out, void *stream);

/* ---- edge length variation: exact.py:127-142 ----------------------------- */

/* d_out[0..2] = (mean length, sum of (l - mean)^2, M_l); M_l = 0.0 and the
 * sums 0.0 when m <= 1.  Callers that need the reference's Python-level
 * exceptions (ZeroDivisionError when every length underflows to 0) apply
 * exact.py:141-142 to d_out[0..1] on the host. */
int glr_edge_length_variation(const double *d_xy, int64_t n,
                              const int64_t *d_edges, int64_t m, double *d_out,
                              void *stream);

/* ---- minimum angle: exact.py:88-124, geometry.py:82-85 -------------------- */

/* d_out[0..2] = (sum of d_v over vertices of degree >= 1, number of such
 * vertices, M_a); M_a = 1.0 when m == 0. */
int glr_minimum_angle(const double *d_xy, int64_t n, const int64_t *d_edges,
                      int64_t m, double *d_out, void *stream);

/* ---- strip-sweep approximations: enhanced.py:133-300, sweep.py:60-402 ---- */

/* One orientation of the reference's strip sweep.
 * d_bounds: the nstrips + 1 strip boundaries along the sweep axis, built as
 * build_strips does (enhanced.py:155-167); axis 0 = vertical strips (x is
 * the sweep axis), 1 = horizontal.  d_out[0] = the strip crossings (order
 * inversions, exact), d_out[1] = the deviation sum |ideal - a_c| over them
 * when with_angle (else 0).  Synchronous (the segment count sizes the
 * scratch).  GLR_EINVARIANT if the two counting routes disagree. */
int glr_strip_crossings(const double *d_xy, int64_t n, const int64_t *d_edges, int64_t m,
                        const double *d_bounds, int64_t nstrips, int axis, int with_angle,
                        double ideal, double *d_out, void *stream);

/* ---- force-directed layout: graphio.py:151-197 --- */

/* Runs `iterations` rounds of the reference's fr_layout on d_pos (n x 2
 * float64, row-major): in = the seeded start layout, out = the final layout
 * rescaled into [0, extent]^2.  d_ei/d_ej: the normalized edges as indices
 * into the sorted vertex ids (m int64 each).  Bit-identical to the
 * reference's numpy iteration (pairwise-summation order of the repulsion
 * sums, np.add.at order of the spring pulls). */
int glr_fr_layout(double *d_pos, int64_t n, const int64_t *d_ei, const int64_t *d_ej,
                  int64_t m, int iterations, double extent, void *stream);

/* ---- native loaders: graphio.py:46-117 ----------- */

/* Both loaders take the reference's whole input grammar: UTF-8 text, the
 * line boundaries of str.splitlines(), the whitespace of str.isspace(), and
 * int() / float() of a str (Unicode decimal digits, underscores between
 * digits, int()'s 4300-digit limit, inf/infinity/nan).  On a malformed
 * input they return GLR_EPARSE and glr_parse_status() describes it; the
 * caller formats the reference's message (graphio.py:46-117) from it. */
enum {
  GLR_PARSE_UTF8 = 1,         /* not valid UTF-8 (open(..., encoding="utf-8").read() fails) */
  GLR_PARSE_TOKENS = 2,       /* edge list: "expected two ids per line, got {line!r}" */
  GLR_PARSE_NOT_INT = 3,      /* edge list: "ids must be integers, got {line!r}" */
  GLR_PARSE_NEGATIVE = 4,     /* edge list: "ids must be nonnegative" */
  GLR_PARSE_NO_EDGES = 5,     /* edge list: "no edges found" */
  GLR_PARSE_OVERFLOW = 6,     /* an id beyond int64 (OverflowError of the int64 conversion) */
  GLR_PARSE_EMPTY_LAYOUT = 7, /* layout: "empty layout file" */
  GLR_PARSE_HEADER = 8,       /* layout: "expected header 'id,x,y', got {lines[0]!r}" */
  GLR_PARSE_FIELDS = 9,       /* layout: "expected 3 fields, got {line!r}" */
  GLR_PARSE_MALFORMED = 10,   /* layout: "malformed row {line!r}" */
  GLR_PARSE_NONFINITE = 11,   /* layout: "non-finite coordinate" */
  GLR_PARSE_DUPLICATE = 12,   /* layout: "duplicate vertex id {vid}" */
  GLR_PARSE_NO_ROWS = 13      /* layout: "layout file has no rows" */
};

/* Parses a SNAP-style edge list held in memory (graphio.parse_edgelist
 * before normalisation): *count = the number of id pairs; the first `cap`
 * are written to out (2 int64 each); call with out = NULL to size. */
int glr_parse_edgelist(const char *buf, size_t len, int64_t *out, int64_t cap,
                       int64_t *count);

/* Parses an "id,x,y" layout CSV held in memory (graphio.read_layout): ids
 * and row-major xy of the first `cap` rows in file order, *count = number of
 * rows. */
int glr_parse_layout(const char *buf, size_t len, int64_t *ids, double *xy, int64_t cap,
                     int64_t *count);

/* The last GLR_EPARSE on this thread: info[0] = GLR_PARSE_* kind, info[1] =
 * 1-based line number (0 if none), info[2..3] = byte span [begin, end) of
 * the line the message quotes (GLR_PARSE_DUPLICATE: info[2] = the id). */
int glr_parse_status(int64_t *info);

/* ---- introspection (tests / bench) --------------------------------------- */

/* Enables (1, the default) or disables (0) the certified FP32 occlusion
 * filter process-wide, for cross-checking it against the FP64 kernel; both
 * give identical counts.  Returns the previous setting. */
int glr_occlusion_set_filter(int enable);

/* Self-test of the repulsion kernel's branch-free division against
 * __ddiv_rn on `samples` pseudo-random positive operand pairs (2^-60..2^60,
 * plus near-midpoint quotients); *h_mismatches receives the number of
 * differing results (synchronous). */
int glr_selftest_division(uint64_t samples, uint64_t seed, uint64_t *h_mismatches,
                          void *stream);

/* Pair-kernel mode of the prepared records (synchronous: reads the records
 * header): 0 = general exact-comparison path (any input), 1 = FP64 float-view
 * sign path with adjacency correction, 2 = certified packed-FP32 filter with
 * exact FP64 fallback (the default whenever every nonzero |coordinate| lies
 * in [2^-160, 2^500]).  All modes give identical results; -1 on error. */
int glr_crossing_fast_path(const void *d_records, void *stream);

/* Overrides the pair-kernel mode (0, 1 or 2, see glr_crossing_fast_path) of
 * prepared records, for cross-checking the modes against each other; modes
 * 1 and 2 fall back to 0 when the input is outside the fast window.
 * Stream-ordered. */
int glr_crossing_set_mode(void *d_records, int mode, void *stream);

/* Number of kernel launches issued by this thread since the last call
 * (counter is reset by the call). */
uint64_t glr_take_launch_count(void);

/* ---- combining shards -------------------------------
 * The partials of disjoint unit ranges add up; these entry points sum them
 * across GPUs with NCCL (opened with dlopen on first use; GLR_ENCCL when it
 * is missing).  Replaces the torch.distributed all_reduce of
 * paper_2411_09809_b200/sharding.py for hosts without Python. */

/* One process, ndev GPUs: d_bufs[i] (count float64 on devices[i]) are summed
 * in place over all i.  Communicators are created once per device list and
 * cached; synchronous on return. */
int glr_allreduce_sum_f64(int ndev, const int *devices, double **d_bufs, int count);

/* One process per GPU: rank 0 creates the id (glr_nccl_id_bytes() bytes) and
 * the host hands it to every rank; each rank then creates its communicator on
 * its current device.  The allreduce is in place and asynchronous on
 * `stream`. */
int glr_nccl_id_bytes(void);
int glr_nccl_unique_id(void *id_out);
int glr_nccl_comm_init(const void *id, int rank, int world, void **comm_out);
int glr_allreduce_sum_f64_comm(void *comm, double *d_buf, int count, void *stream);
int glr_nccl_comm_destroy(void *comm);

#ifdef __cplusplus
}
#endif

#endif /* GLARE_B200_H */
