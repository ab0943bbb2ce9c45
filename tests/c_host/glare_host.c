/* A non-Python host of the C ABI (include/glare_b200.h): what a Go (cgo),
 * Java (JNI) or Rust (FFI) caller of the library does, in plain C.
 *
 *   glare_host <input.bin> <world>
 *
 * input.bin: int64 n, int64 m, double r, double ideal, then xy (n*2 float64)
 * and edges (m*2 int64, normalised as LayoutGraph does).  The program
 * copies the arrays to the device, evaluates all five metrics through the
 * C entry points, evaluates the crossing pass a second time as `world`
 * interleaved shards (glr_crossing_pairs_interleaved, the multi-GPU unit
 * rule) summed on the device, combines that sum through the library's NCCL
 * entry points (a one-rank communicator here), and prints one JSON line.
 * Exit status 0 on success. */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "glare_b200.h"

#define CK(call)                                                                  \
  do {                                                                            \
    int rc_ = (call);                                                             \
    if (rc_ != 0) {                                                               \
      fprintf(stderr, "%s failed (%d): %s\n", #call, rc_, glr_last_error());      \
      return 2;                                                                   \
    }                                                                             \
  } while (0)
#define CU(call)                                                                  \
  do {                                                                            \
    cudaError_t e_ = (call);                                                      \
    if (e_ != cudaSuccess) {                                                      \
      fprintf(stderr, "%s: %s\n", #call, cudaGetErrorString(e_));                 \
      return 3;                                                                   \
    }                                                                             \
  } while (0)

int main(int argc, char **argv) {
  if (argc < 3) {
    fprintf(stderr, "usage: %s input.bin world\n", argv[0]);
    return 1;
  }
  const int world = atoi(argv[2]);
  FILE *f = fopen(argv[1], "rb");
  if (!f) return 1;
  int64_t nm[2];
  double rp[2];
  if (fread(nm, sizeof(int64_t), 2, f) != 2 || fread(rp, sizeof(double), 2, f) != 2) return 1;
  const int64_t n = nm[0], m = nm[1];
  const double r = rp[0], ideal = rp[1];
  double *xy = (double *)malloc(sizeof(double) * 2 * n);
  int64_t *edges = (int64_t *)malloc(sizeof(int64_t) * 2 * m);
  if (fread(xy, sizeof(double), 2 * n, f) != (size_t)(2 * n) ||
      fread(edges, sizeof(int64_t), 2 * m, f) != (size_t)(2 * m))
    return 1;
  fclose(f);

  cudaStream_t st;
  CU(cudaStreamCreate(&st));
  double *d_xy, *d_out;
  int64_t *d_edges;
  CU(cudaMalloc((void **)&d_xy, sizeof(double) * 2 * n));
  CU(cudaMalloc((void **)&d_edges, sizeof(int64_t) * 2 * m));
  CU(cudaMalloc((void **)&d_out, sizeof(double) * 16));
  CU(cudaMemsetAsync(d_out, 0, sizeof(double) * 16, st));
  CU(cudaMemcpyAsync(d_xy, xy, sizeof(double) * 2 * n, cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(d_edges, edges, sizeof(int64_t) * 2 * m, cudaMemcpyHostToDevice, st));

  /* node_occlusion: thr = (2r)^2 as exact.py:63 computes it */
  const double thr = (2.0 * r) * (2.0 * r);
  CK(glr_occlusion_count(d_xy, n, thr, 0, glr_occlusion_units(n), d_out + 0, st));
  /* _crossing_scan with the ideal angle: (count, dev_sum) */
  CK(glr_crossing_scan(d_xy, n, d_edges, m, 1, ideal, 0, glr_crossing_units(m), d_out + 1, st));
  /* M_a: (sum d_v, vertices of degree >= 1, M_a); M_l: (mean, S, M_l) */
  CK(glr_minimum_angle(d_xy, n, d_edges, m, d_out + 3, st));
  CK(glr_edge_length_variation(d_xy, n, d_edges, m, d_out + 6, st));

  /* the same crossing pass as `world` interleaved shards, summed */
  void *d_rec;
  CU(cudaMalloc(&d_rec, glr_crossing_records_bytes(n, m)));
  CK(glr_crossing_prepare(d_xy, n, d_edges, m, d_rec, st));
  double *d_share;
  CU(cudaMalloc((void **)&d_share, sizeof(double) * 2 * (size_t)world));
  for (int rank = 0; rank < world; ++rank)
    CK(glr_crossing_pairs_interleaved(d_rec, n, m, 1, ideal, NULL, 0, rank, world,
                                      d_share + 2 * rank, st));
  double *share = (double *)malloc(sizeof(double) * 2 * (size_t)world);
  CU(cudaMemcpyAsync(share, d_share, sizeof(double) * 2 * world, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  double sum[2] = {0.0, 0.0};
  for (int rank = 0; rank < world; ++rank) {
    sum[0] += share[2 * rank];
    sum[1] += share[2 * rank + 1];
  }
  /* combine through the library's NCCL entry points (one-rank communicator) */
  CU(cudaMemcpyAsync(d_out + 9, sum, sizeof(sum), cudaMemcpyHostToDevice, st));
  unsigned char id[256];
  if (glr_nccl_id_bytes() > (int)sizeof(id)) return 4;
  CK(glr_nccl_unique_id(id));
  void *comm = NULL;
  CK(glr_nccl_comm_init(id, 0, 1, &comm));
  CK(glr_allreduce_sum_f64_comm(comm, d_out + 9, 2, st));
  int dev = 0;
  CU(cudaGetDevice(&dev));
  double *bufs[1] = {d_out + 9};
  CU(cudaStreamSynchronize(st));
  CK(glr_allreduce_sum_f64(1, &dev, bufs, 2));

  double out[16];
  CU(cudaMemcpyAsync(out, d_out, sizeof(out), cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  CK(glr_nccl_comm_destroy(comm));
  printf("{\"nc\": %.17g, \"ec\": %.17g, \"dev\": %.17g, \"ma\": %.17g, \"ml\": %.17g, "
         "\"ec_sharded\": %.17g, \"dev_sharded\": %.17g, \"world\": %d, \"chunk\": %llu}\n",
         out[0], out[1], out[2], out[5], out[8], out[9], out[10], world,
         (unsigned long long)glr_crossing_chunk(glr_crossing_units(m), world));
  return 0;
}
