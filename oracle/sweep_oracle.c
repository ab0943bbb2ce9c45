/* Multi-threaded C restatement of the reference's serial oracle for the two
 * all-pairs metrics -- TEST INFRASTRUCTURE (checker + CPU baseline only).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs load this library.  The product path never does.
 *
 * Restates, per unordered pair:
 *   crossing  -- /root/reference/pkg/src/glare/metrics/exact.py:145-222 and
 *                geometry.py:62-79: the x-sorted sweep of the reference
 *                (exact.py:170-199) with the closed-bbox prefilter
 *                (exact.py:191-194), index-disjointness (exact.py:205-210)
 *                and the four cross products in the reference's operand
 *                order, each compared against zero separately.  The deviation
 *                sum |ideal - min(d, pi - d)| (geometry.py:107-110,
 *                exact.py:219-221) takes per-edge axis angles computed by the
 *                caller with numpy (geometry.py:94-97).
 *   occlusion -- exact.py:55-74: fl(fl(dx*dx)+fl(dy*dy)) < thr, strict.
 *                The x-sorted sweep stops once fl(x_j - x_i) >= 2r, which by
 *                monotone rounding implies fl(dx*dx) >= thr.
 *
 * Build with -ffp-contract=off (no FMA contraction: the reference evaluates
 * each numpy ufunc separately).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  const double *ax, *ay, *bx, *by, *xmin, *xmax, *ymin, *ymax, *theta;
  const int64_t *u, *v;
  int64_t m;
  double ideal;
  int with_angle;
  int nthreads, tid;
  uint64_t count;
  double dev;
} cross_job;

static int straddle(double ax, double ay, double bx, double by,
                    double cx, double cy, double dx, double dy) {
  double abx = bx - ax;
  double aby = by - ay;
  double c1 = abx * (cy - ay) - aby * (cx - ax);
  double c2 = abx * (dy - ay) - aby * (dx - ax);
  double cdx = dx - cx;
  double cdy = dy - cy;
  double c3 = cdx * (ay - cy) - cdy * (ax - cx);
  double c4 = cdx * (by - cy) - cdy * (bx - cx);
  int s_cd = ((c1 <= 0.0) && (c2 >= 0.0)) || ((c1 >= 0.0) && (c2 <= 0.0));
  int s_ab = ((c3 <= 0.0) && (c4 >= 0.0)) || ((c3 >= 0.0) && (c4 <= 0.0));
  return s_cd && s_ab;
}

static void *cross_worker(void *arg) {
  cross_job *J = (cross_job *)arg;
  uint64_t cnt = 0;
  double dev = 0.0, comp = 0.0; /* Kahan-compensated per-thread sum */
  const double PI = 3.141592653589793;
  /* rows are the x-sorted edges; interleave rows in chunks of 64 across
     threads so the triangular work is balanced */
  for (int64_t base = (int64_t)J->tid * 64; base < J->m; base += (int64_t)J->nthreads * 64) {
    int64_t end = base + 64 < J->m ? base + 64 : J->m;
    for (int64_t i = base; i < end; ++i) {
      const double xi1 = J->xmax[i], yi0 = J->ymin[i], yi1 = J->ymax[i];
      const int64_t ui = J->u[i], vi = J->v[i];
      for (int64_t j = i + 1; j < J->m; ++j) {
        /* sorted by xmin: once xmin_j > xmax_i no later j overlaps in x */
        if (J->xmin[j] > xi1) break;
        if (J->ymax[j] < yi0 || J->ymin[j] > yi1) continue;
        const int64_t uj = J->u[j], vj = J->v[j];
        if (ui == uj || ui == vj || vi == uj || vi == vj) continue;
        if (!straddle(J->ax[j], J->ay[j], J->bx[j], J->by[j],
                      J->ax[i], J->ay[i], J->bx[i], J->by[i]))
          continue;
        ++cnt;
        if (J->with_angle) {
          double d = fabs(J->theta[i] - J->theta[j]);
          double a = d < PI - d ? d : PI - d;
          double t = fabs(J->ideal - a) - comp;
          double s = dev + t;
          comp = (s - dev) - t;
          dev = s;
        }
      }
    }
  }
  J->count = cnt;
  J->dev = dev;
  return NULL;
}

static const double *g_sort_key;
static int cmp_by_key(const void *a, const void *b) {
  int64_t i = *(const int64_t *)a, j = *(const int64_t *)b;
  double ki = g_sort_key[i], kj = g_sort_key[j];
  if (ki < kj) return -1;
  if (ki > kj) return 1;
  return (i > j) - (i < j); /* stable */
}

/* xy: (n,2) row-major; edges: (m,2) int64 index pairs (small index first);
 * theta: per-edge axis angle (only read when with_angle).
 * Outputs the crossing count and the deviation sum.  Returns 0 on success. */
int oracle_crossing_scan(const double *xy, int64_t n, const int64_t *edges, int64_t m,
                         const double *theta, int with_angle, double ideal,
                         int nthreads, uint64_t *out_count, double *out_dev) {
  (void)n;
  *out_count = 0;
  *out_dev = 0.0;
  if (m < 2) return 0;
  int64_t *order = (int64_t *)malloc(sizeof(int64_t) * m);
  double *buf = (double *)malloc(sizeof(double) * m * 10);
  int64_t *ids = (int64_t *)malloc(sizeof(int64_t) * m * 2);
  if (!order || !buf || !ids) { free(order); free(buf); free(ids); return 1; }
  double *xmin0 = buf;
  for (int64_t k = 0; k < m; ++k) {
    double ax = xy[2 * edges[2 * k]], bx = xy[2 * edges[2 * k + 1]];
    xmin0[k] = ax < bx ? ax : bx;
    order[k] = k;
  }
  g_sort_key = xmin0;
  qsort(order, (size_t)m, sizeof(int64_t), cmp_by_key);
  double *ax = buf + m, *ay = buf + 2 * m, *bx = buf + 3 * m, *by = buf + 4 * m;
  double *xmin = buf + 5 * m, *xmax = buf + 6 * m, *ymin = buf + 7 * m, *ymax = buf + 8 * m;
  double *th = buf + 9 * m;
  int64_t *u = ids, *v = ids + m;
  for (int64_t k = 0; k < m; ++k) {
    int64_t e = order[k];
    int64_t a = edges[2 * e], b = edges[2 * e + 1];
    ax[k] = xy[2 * a]; ay[k] = xy[2 * a + 1];
    bx[k] = xy[2 * b]; by[k] = xy[2 * b + 1];
    xmin[k] = ax[k] < bx[k] ? ax[k] : bx[k];
    xmax[k] = ax[k] > bx[k] ? ax[k] : bx[k];
    ymin[k] = ay[k] < by[k] ? ay[k] : by[k];
    ymax[k] = ay[k] > by[k] ? ay[k] : by[k];
    th[k] = with_angle ? theta[e] : 0.0;
    u[k] = a; v[k] = b;
  }
  if (nthreads < 1) nthreads = 1;
  cross_job *jobs = (cross_job *)calloc((size_t)nthreads, sizeof(cross_job));
  pthread_t *tids = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
  for (int t = 0; t < nthreads; ++t) {
    cross_job *J = &jobs[t];
    J->ax = ax; J->ay = ay; J->bx = bx; J->by = by;
    J->xmin = xmin; J->xmax = xmax; J->ymin = ymin; J->ymax = ymax; J->theta = th;
    J->u = u; J->v = v; J->m = m; J->ideal = ideal; J->with_angle = with_angle;
    J->nthreads = nthreads; J->tid = t;
    pthread_create(&tids[t], NULL, cross_worker, J);
  }
  uint64_t cnt = 0;
  double dev = 0.0;
  for (int t = 0; t < nthreads; ++t) {
    pthread_join(tids[t], NULL);
    cnt += jobs[t].count;
    dev += jobs[t].dev;
  }
  *out_count = cnt;
  *out_dev = dev;
  free(jobs); free(tids); free(order); free(buf); free(ids);
  return 0;
}

typedef struct {
  const double *x, *y;
  int64_t n;
  double thr, reach;
  int nthreads, tid;
  uint64_t count;
} occ_job;

static void *occ_worker(void *arg) {
  occ_job *J = (occ_job *)arg;
  uint64_t cnt = 0;
  for (int64_t base = (int64_t)J->tid * 256; base < J->n; base += (int64_t)J->nthreads * 256) {
    int64_t end = base + 256 < J->n ? base + 256 : J->n;
    for (int64_t i = base; i < end; ++i) {
      const double xi = J->x[i], yi = J->y[i];
      for (int64_t j = i + 1; j < J->n; ++j) {
        double dx = J->x[j] - xi;
        if (dx >= J->reach) break;
        double dy = J->y[j] - yi;
        if (dx * dx + dy * dy < J->thr) ++cnt;
      }
    }
  }
  J->count = cnt;
  return NULL;
}

/* Occluding vertex pairs: thr = (2r)^2 as computed by the caller in Python,
 * reach = 2r.  Returns 0 on success. */
int oracle_node_occlusion(const double *xy, int64_t n, double thr, double reach,
                          int nthreads, uint64_t *out_count) {
  *out_count = 0;
  if (n < 2) return 0;
  int64_t *order = (int64_t *)malloc(sizeof(int64_t) * n);
  double *buf = (double *)malloc(sizeof(double) * n * 3);
  if (!order || !buf) { free(order); free(buf); return 1; }
  for (int64_t k = 0; k < n; ++k) { buf[k] = xy[2 * k]; order[k] = k; }
  g_sort_key = buf;
  qsort(order, (size_t)n, sizeof(int64_t), cmp_by_key);
  double *x = buf + n, *y = buf + 2 * n;
  for (int64_t k = 0; k < n; ++k) { x[k] = xy[2 * order[k]]; y[k] = xy[2 * order[k] + 1]; }
  if (nthreads < 1) nthreads = 1;
  occ_job *jobs = (occ_job *)calloc((size_t)nthreads, sizeof(occ_job));
  pthread_t *tids = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
  for (int t = 0; t < nthreads; ++t) {
    occ_job *J = &jobs[t];
    J->x = x; J->y = y; J->n = n; J->thr = thr; J->reach = reach;
    J->nthreads = nthreads; J->tid = t;
    pthread_create(&tids[t], NULL, occ_worker, J);
  }
  uint64_t cnt = 0;
  for (int t = 0; t < nthreads; ++t) { pthread_join(tids[t], NULL); cnt += jobs[t].count; }
  *out_count = cnt;
  free(jobs); free(tids); free(order); free(buf);
  return 0;
}
