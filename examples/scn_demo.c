/* scn_demo.c — a plain C program using libscn.so through include/scn.h only
 * (no Python, no torch): the caller owns device memory (cudaMalloc), the
 * library only enqueues work.
 *
 * Workload: 3 tables of constant-colour frames (closed-form results, no oracle
 * needed): table t, row r has every pixel = colour(t, r/5) — a new "shot"
 * every 5 rows. Sample stride 2 per table, concatenate,
 * shard into 2 "ranks" (scn_shard_range) and run HIST + shot-diff per shard
 * (the second shard recomputes its [-1,0] halo). Checks:
 *   H[j][c][bin(colour_c)] = W*H and 0 elsewhere            (HIST)
 *   D[j] = 2*W*H*#{c : bin changes vs previous position}, 0 at table starts
 * Build: make examples/scn_demo ; run: examples/scn_demo (needs a GPU). */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "scn.h"

#define W 96
#define H 40
#define ROWS 23
#define TABLES 3
#define BINS 16

#define CHECK_SCN(x)                                                               \
  do {                                                                             \
    scn_status st_ = (x);                                                          \
    if (st_ != SCN_OK) {                                                           \
      fprintf(stderr, "%s failed: %d %s\n", #x, (int)st_, scn_last_error());       \
      return 1;                                                                    \
    }                                                                              \
  } while (0)
#define CHECK_CUDA(x)                                                              \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      fprintf(stderr, "%s failed: %s\n", #x, cudaGetErrorString(e_));              \
      return 1;                                                                    \
    }                                                                              \
  } while (0)

static uint8_t colour(int t, int shot, int c) { return (uint8_t)((37 * t + 61 * shot + 97 * c) % 256); }

int main(void) {
  const size_t F = (size_t)W * H * 3, stride = (F + 15) / 16 * 16;
  uint8_t* h = (uint8_t*)malloc(stride * ROWS);
  uint8_t* d_frames[TABLES];
  scn_table* tables[TABLES];
  scn_seq* parts[TABLES];
  for (int t = 0; t < TABLES; ++t) {
    for (int r = 0; r < ROWS; ++r)
      for (size_t i = 0; i < F; ++i) h[r * stride + i] = colour(t, r / 5, (int)(i % 3));
    CHECK_CUDA(cudaMalloc((void**)&d_frames[t], stride * ROWS));
    CHECK_CUDA(cudaMemcpy(d_frames[t], h, stride * ROWS, cudaMemcpyHostToDevice));
    CHECK_SCN(scn_table_create(ROWS, W, H, 3, SCN_MEM_DEVICE, d_frames[t], (int64_t)stride, NULL, &tables[t]));
    CHECK_SCN(scn_sample_stride(tables[t], 2, &parts[t]));
  }
  scn_seq* seq;
  CHECK_SCN(scn_seq_concat((const scn_seq* const*)parts, TABLES, &seq));
  const int64_t m = scn_seq_length(seq);
  void* d_ws;
  CHECK_CUDA(cudaMalloc(&d_ws, scn_seq_device_bytes(seq)));
  CHECK_SCN(scn_seq_upload(seq, d_ws, scn_seq_device_bytes(seq), NULL));

  uint32_t *d_hist, *d_diff, *d_scratch;
  CHECK_CUDA(cudaMalloc((void**)&d_hist, sizeof(uint32_t) * 3 * BINS * (size_t)m));
  CHECK_CUDA(cudaMalloc((void**)&d_diff, sizeof(uint32_t) * (size_t)m));
  CHECK_CUDA(cudaMalloc((void**)&d_scratch, sizeof(uint32_t) * 3 * BINS));
  for (int rank = 0; rank < 2; ++rank) {
    int64_t b, e;
    CHECK_SCN(scn_shard_range(m, 2, rank, &b, &e));
    CHECK_SCN(scn_run_hist_shotdiff(seq, b, e, BINS, d_hist + 3 * BINS * b, d_diff + b, d_scratch, NULL));
    CHECK_CUDA(cudaDeviceSynchronize());  /* d_scratch is reused by the next shard */
  }
  uint32_t* hist = (uint32_t*)malloc(sizeof(uint32_t) * 3 * BINS * (size_t)m);
  uint32_t* diff = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)m);
  CHECK_CUDA(cudaMemcpy(hist, d_hist, sizeof(uint32_t) * 3 * BINS * (size_t)m, cudaMemcpyDeviceToHost));
  CHECK_CUDA(cudaMemcpy(diff, d_diff, sizeof(uint32_t) * (size_t)m, cudaMemcpyDeviceToHost));

  int32_t* part = (int32_t*)malloc(sizeof(int32_t) * (size_t)m);
  int64_t* row = (int64_t*)malloc(sizeof(int64_t) * (size_t)m);
  CHECK_SCN(scn_seq_rows(seq, part, row));
  int bad = 0;
  for (int64_t j = 0; j < m; ++j) {
    const int t = part[j], shot = (int)(row[j] / 5);
    uint32_t expect_d = 0;
    for (int c = 0; c < 3; ++c) {
      const int bin = colour(t, shot, c) * BINS / 256;
      for (int b = 0; b < BINS; ++b) {
        const uint32_t want = b == bin ? (uint32_t)(W * H) : 0u;
        if (hist[(j * 3 + c) * BINS + b] != want) ++bad;
      }
      if (j > 0 && part[j - 1] == t) {
        const int pbin = colour(t, (int)(row[j - 1] / 5), c) * BINS / 256;
        if (pbin != bin) expect_d += 2u * W * H;
      }
    }
    if (diff[j] != expect_d) {
      fprintf(stderr, "D[%lld] = %u, expected %u\n", (long long)j, diff[j], expect_d);
      ++bad;
    }
  }
  printf("scn_demo: %s (%lld positions over %d tables, 2 shards, %s)\n", bad ? "FAIL" : "ok", (long long)m, TABLES,
         scn_version());
  scn_seq_destroy(seq);
  for (int t = 0; t < TABLES; ++t) {
    scn_seq_destroy(parts[t]);
    scn_table_destroy(tables[t]);
    cudaFree(d_frames[t]);
  }
  cudaFree(d_ws);
  cudaFree(d_hist);
  cudaFree(d_diff);
  cudaFree(d_scratch);
  free(h);
  free(hist);
  free(diff);
  free(part);
  free(row);
  return bad ? 1 : 0;
}
