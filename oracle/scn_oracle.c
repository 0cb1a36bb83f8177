/* scn_oracle.c — the CPU ORACLE for the Scanner (arXiv 1805.07339) HIST /
 * shot-diff / downsample hot path.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load or execute anything
 * under oracle/. The product path (paper_1805_07339_b200/) never calls it and
 * shares no code with it; the only shared module is the seeded input
 * generator scn_synth/ (frames and index lists, none of the method's
 * arithmetic).
 *
 * Plain, slow, single-threaded, obviously correct: every function is the
 * definition it cites written out with nested loops, in the order the paper
 * states it. All results are exact integers (u32 counts, u8 pixels), so no
 * floating point is involved anywhere.
 *
 * Citations: P:L### = /root/reference/PAPER.md line, S:L### = SPEC.md line.
 * Readings of silent/ambiguous passages are the Q-numbers of DESIGN.md §3
 * (= SURVEY.md §8(c)).
 *
 * Pins (tests/test_oracle_*.py, -m "not gpu"): brute-force enumeration of
 * sampled indices, the paper's 1800/30 -> 60 and 18000/10 -> 1800 examples,
 * closed-form histograms of constant and x-gradient frames, the bin-sum
 * invariant, a range-predicate (bin edge) formulation on random frames, the
 * hand-worked golden fixtures in tests/golden/, closed-form shot-diffs of
 * constant-frame cuts, planted cuts, and closed-form downsamples. No function
 * here is "parity unpinned".
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include "../scn_synth/scn_synth.h"

#define OR_OK 0
#define OR_EINVAL 1
#define OR_ERANGE 2
#define OR_EUNSUPPORTED 4

/* ------------------------------------------------------------------------
 * Sampling (§3.2 "Sampling/spacing operations ... Both sampling and
 * spacing operations can be defined by strides, ranges, or index lists";
 * "sampling every 30th row from a table representing a one-minute long,
 * 30 FPS video (1800 frames) yields a length 60 sequence").
 * A sequence over a table of N rows is the domain [0,N).
 * ------------------------------------------------------------------------ */

/* Stride s: rows {0, s, 2s, ...} < N (reading Q8: start at row 0).
 * Writes up to cap rows to out (out may be NULL); *m = number of rows. */
int oracle_sample_stride(int64_t n_rows, int64_t s, int64_t* out, int64_t cap, int64_t* m) {
  if (n_rows < 0 || s < 1) return OR_EINVAL;
  int64_t k = 0;
  for (int64_t r = 0; r < n_rows; ++r) {
    if (r % s == 0) {            /* "every s-th row" */
      if (out && k < cap) out[k] = r;
      ++k;
    }
  }
  *m = k;
  return OR_OK;
}

/* Range: blocks [a_i, b_i) (half-open, sorted, disjoint, reading Q9), each
 * walked with step k ("Blocks of 2,000 consecutive frames"). */
int oracle_sample_range(int64_t n_rows, const int64_t* blocks, int64_t n_blocks, int64_t step, int64_t* out,
                        int64_t cap, int64_t* m) {
  if (n_rows < 0 || step < 1 || n_blocks < 0) return OR_EINVAL;
  for (int64_t i = 0; i < n_blocks; ++i) {
    int64_t a = blocks[2 * i], b = blocks[2 * i + 1];
    if (a > b) return OR_EINVAL;
    if (i > 0 && a < blocks[2 * i - 1]) return OR_EINVAL; /* sorted and disjoint */
    if (a < 0 || b > n_rows) return OR_ERANGE;
  }
  int64_t k = 0;
  for (int64_t i = 0; i < n_blocks; ++i) {
    int64_t a = blocks[2 * i], b = blocks[2 * i + 1];
    for (int64_t r = a; r < b; ++r) {
      if ((r - a) % step == 0) {
        if (out && k < cap) out[k] = r;
        ++k;
      }
    }
  }
  *m = k;
  return OR_OK;
}

/* Gather: an explicit index list ("index lists", "A random list
 * of frames"); strictly increasing, in [0,N) (reading Q10). */
int oracle_sample_gather(int64_t n_rows, const int64_t* rows, int64_t n, int64_t* out, int64_t cap, int64_t* m) {
  if (n_rows < 0 || n < 0) return OR_EINVAL;
  for (int64_t i = 0; i < n; ++i) {
    if (i > 0 && rows[i] <= rows[i - 1]) return OR_EINVAL;
  }
  for (int64_t i = 0; i < n; ++i) {
    if (rows[i] < 0 || rows[i] >= n_rows) return OR_ERANGE;
  }
  for (int64_t i = 0; i < n && out; ++i)
    if (i < cap) out[i] = rows[i];
  *m = n;
  return OR_OK;
}

/* ------------------------------------------------------------------------
 * HIST (§5.1.2: "Compute and store the pixel color histogram for all
 * frames"; "color histograms on every frame"). Readings Q1-Q3: B bins
 * per channel, bin(v) = floor(v*B/256), three per-channel marginals in stored
 * channel order, layout out[c][b].
 * frame: H rows of W pixels of 3 bytes (HWC), row-major, contiguous.
 * ------------------------------------------------------------------------ */
int oracle_hist(const uint8_t* frame, int32_t w, int32_t h, int32_t bins, uint32_t* out) {
  if (bins < 1 || bins > 256) return OR_EUNSUPPORTED;
  if (w < 1 || h < 1) return OR_EINVAL;
  for (int32_t c = 0; c < 3; ++c)
    for (int32_t b = 0; b < bins; ++b) out[c * bins + b] = 0;
  for (int32_t y = 0; y < h; ++y) {
    for (int32_t x = 0; x < w; ++x) {
      for (int32_t c = 0; c < 3; ++c) {
        uint32_t v = frame[((int64_t)y * w + x) * 3 + c];
        uint32_t b = (v * (uint32_t)bins) / 256u;  /* bin = floor(v*B/256) */
        out[c * bins + b] += 1u;
      }
    }
  }
  return OR_OK;
}

/* ------------------------------------------------------------------------
 * NEXT N4, joint-colour variant (SURVEY §8(f) N4 "256-bin per-channel (or
 * joint-colour) histogram"; "pixel color histogram", reading Q3's
 * alternative): one histogram over colour triples, J bins per channel,
 * bin_J(v) = floor(v*J/256) as in reading Q2, joint bin
 * k = bin_J(R)*J*J + bin_J(G)*J + bin_J(B), layout out[k], k < J^3.
 * frame: H rows of W pixels of 3 bytes (HWC), row-major, contiguous.
 * ------------------------------------------------------------------------ */
int oracle_hist_joint(const uint8_t* frame, int32_t w, int32_t h, int32_t j, uint32_t* out) {
  if (j < 1 || j > 16) return OR_EUNSUPPORTED;
  if (w < 1 || h < 1) return OR_EINVAL;
  const int32_t n = j * j * j;
  for (int32_t k = 0; k < n; ++k) out[k] = 0;
  for (int32_t y = 0; y < h; ++y) {
    for (int32_t x = 0; x < w; ++x) {
      const uint8_t* px = frame + ((int64_t)y * w + x) * 3;
      uint32_t b[3];
      for (int32_t c = 0; c < 3; ++c) b[c] = ((uint32_t)px[c] * (uint32_t)j) / 256u;  /* floor(v*J/256) */
      out[(b[0] * (uint32_t)j + b[1]) * (uint32_t)j + b[2]] += 1u;
    }
  }
  return OR_OK;
}

/* Joint histograms of the synthetic frames at sampled positions [p0, p1)
 * (the frames oracle_run generates): out [p1-p0][J^3]. */
int oracle_run_joint(const synth_spec* spec, const int32_t* videos, const int64_t* rows, int64_t p0, int64_t p1,
                     int32_t j, uint32_t* out) {
  if (j < 1 || j > 16) return OR_EUNSUPPORTED;
  if (p0 < 0 || p1 < p0) return OR_EINVAL;
  const int64_t F = (int64_t)spec->width * spec->height * 3, n = (int64_t)j * j * j;
  uint8_t* frame = (uint8_t*)malloc((size_t)(F > 0 ? F : 1));
  if (!frame) return OR_EINVAL;
  for (int64_t p = p0; p < p1; ++p) {
    synth_frame_desc d = synth_describe(spec, videos[p], rows[p]);
    synth_fill_frame_host(spec, &d, frame);
    int rc = oracle_hist_joint(frame, spec->width, spec->height, j, out + (p - p0) * n);
    if (rc) { free(frame); return rc; }
  }
  free(frame);
  return OR_OK;
}

/* ------------------------------------------------------------------------
 * Shot-diff: a [-1,0] stencil over the SAMPLED sequence ("Stencil
 * operations gain access to a window of elements from the input sequence
 * defined by a constant-offset stencil"; sample-then-stencil composition,
 * fig:sampling-f; reading Q7) of an L1 histogram difference ("detect
 * shot boundaries (via histogram differences)"; reading Q4).
 * Boundary (reading Q6, S:L152 repeat-edge clamp): at the first element of a
 * segment (a video/table, which acts as a slice) the stencil's -1
 * neighbour clamps to the element itself, so D = 0.
 * hist: [m][3*bins]; seg_start[p] != 0 iff p is the first position of a part.
 * ------------------------------------------------------------------------ */
int oracle_shotdiff(const uint32_t* hist, const uint8_t* seg_start, int64_t m, int32_t bins, uint32_t* diff) {
  if (bins < 1 || bins > 256) return OR_EUNSUPPORTED;
  const int64_t k = 3 * (int64_t)bins;
  for (int64_t p = 0; p < m; ++p) {
    int64_t q = (p == 0 || seg_start[p]) ? p : p - 1; /* clamp the -1 offset */
    uint32_t d = 0;
    for (int64_t i = 0; i < k; ++i) {
      uint32_t a = hist[p * k + i], b = hist[q * k + i];
      d += a > b ? a - b : b - a;
    }
    diff[p] = d;
  }
  return OR_OK;
}

/* Shot-diff over joint-colour histograms (NEXT N4's joint variant with the same
 * [-1,0] L1 stencil of P:L455 / P:L210, readings Q4, Q6, Q7): diff[p] =
 * sum_k |hist[p][k] - hist[p-1][k]| over the J^3 counters, 0 at segment starts.
 * hist: [m][J^3]. */
int oracle_shotdiff_joint(const uint32_t* hist, const uint8_t* seg_start, int64_t m, int32_t j, uint32_t* diff) {
  if (j < 1 || j > 16) return OR_EUNSUPPORTED;
  const int64_t k = (int64_t)j * j * j;
  for (int64_t p = 0; p < m; ++p) {
    int64_t q = (p == 0 || seg_start[p]) ? p : p - 1; /* clamp the -1 offset */
    uint32_t d = 0;
    for (int64_t i = 0; i < k; ++i) {
      uint32_t a = hist[p * k + i], b = hist[q * k + i];
      d += a > b ? a - b : b - a;
    }
    diff[p] = d;
  }
  return OR_OK;
}

/* ------------------------------------------------------------------------
 * Downsample: integer 2x box ("downsamples the resulting frames
 * (Resize)", "Downsample and transform an input frame"). Reading Q11:
 * O[y][x][c] = (P(2y,2x)+P(2y,2x+1)+P(2y+1,2x)+P(2y+1,2x+1)+2) >> 2 (round half
 * up), output floor(W/2) x floor(H/2), a trailing odd row/column is dropped.
 * ------------------------------------------------------------------------ */
int oracle_downsample(const uint8_t* frame, int32_t w, int32_t h, uint8_t* out) {
  if (w < 1 || h < 1) return OR_EINVAL;
  const int32_t ow = w / 2, oh = h / 2;
  for (int32_t y = 0; y < oh; ++y) {
    for (int32_t x = 0; x < ow; ++x) {
      for (int32_t c = 0; c < 3; ++c) {
        uint32_t s = 0;
        for (int32_t dy = 0; dy < 2; ++dy)
          for (int32_t dx = 0; dx < 2; ++dx) s += frame[((int64_t)(2 * y + dy) * w + (2 * x + dx)) * 3 + c];
        out[((int64_t)y * ow + x) * 3 + c] = (uint8_t)((s + 2u) / 4u);
      }
    }
  }
  return OR_OK;
}

/* ------------------------------------------------------------------------
 * Whole-job driver over synthetic input: the sampled sequence is given as
 * per-position (video, row) pairs plus segment-start flags (a multi-video
 * job concatenates one sampled sequence per table: "one job for
 * each video"; each table is its own slice for the stencil).
 * Frames are regenerated one at a time from scn_synth (streaming, O(frame)
 * host memory), exactly as decode would deliver them.
 * Outputs (any may be NULL): hist [m][3*bins], diff [m], ds [m][H/2][W/2][3].
 * The positions computed are [p0, p1); the shot-diff of p0 uses position
 * p0-1 (the halo) when p0 is not a segment start.
 * ------------------------------------------------------------------------ */
int oracle_run(const synth_spec* spec, const int32_t* videos, const int64_t* rows, const uint8_t* seg_start,
               int64_t p0, int64_t p1, int32_t bins, uint32_t* hist, uint32_t* diff, uint8_t* ds) {
  if (bins < 1 || bins > 256) return OR_EUNSUPPORTED;
  if (p0 < 0 || p1 < p0) return OR_EINVAL;
  const int64_t F = (int64_t)spec->width * spec->height * 3;
  const int64_t dsb = (int64_t)(spec->width / 2) * (spec->height / 2) * 3;
  const int64_t k = 3 * (int64_t)bins;
  uint8_t* frame = (uint8_t*)malloc((size_t)(F > 0 ? F : 1));
  uint32_t* prev = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)k);
  uint32_t* cur = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)k);
  if (!frame || !prev || !cur) { free(frame); free(prev); free(cur); return OR_EINVAL; }
  int have_prev = 0;
  if (p0 < p1 && p0 > 0 && !seg_start[p0] && diff) {
    synth_frame_desc d = synth_describe(spec, videos[p0 - 1], rows[p0 - 1]);
    synth_fill_frame_host(spec, &d, frame);
    oracle_hist(frame, spec->width, spec->height, bins, prev);
    have_prev = 1;
  }
  for (int64_t p = p0; p < p1; ++p) {
    synth_frame_desc d = synth_describe(spec, videos[p], rows[p]);
    synth_fill_frame_host(spec, &d, frame);
    oracle_hist(frame, spec->width, spec->height, bins, cur);
    if (hist) memcpy(hist + (p - p0) * k, cur, sizeof(uint32_t) * (size_t)k);
    if (diff) {
      uint8_t pair_seg[2] = {1, 0};
      uint32_t pair[2 * 3 * 256];
      uint32_t dd[2];
      if (p == 0 || seg_start[p] || !have_prev) {
        diff[p - p0] = 0;
      } else {
        memcpy(pair, prev, sizeof(uint32_t) * (size_t)k);
        memcpy(pair + k, cur, sizeof(uint32_t) * (size_t)k);
        oracle_shotdiff(pair, pair_seg, 2, bins, dd);
        diff[p - p0] = dd[1];
      }
    }
    if (ds) oracle_downsample(frame, spec->width, spec->height, ds + (p - p0) * dsb);
    memcpy(prev, cur, sizeof(uint32_t) * (size_t)k);
    have_prev = 1;
  }
  free(frame); free(prev); free(cur);
  return OR_OK;
}

/* Same as oracle_run but only the per-frame compute is timed by the caller:
 * generation of each frame happens into `frames` beforehand (bench.py's
 * cpu_baseline, which times hist+diff on pre-generated frames exactly as the
 * GPU path times them on frames already resident in HBM). frames: n frames of
 * F bytes, contiguous. seg_first: nonzero if position 0 starts a segment. */
int oracle_hist_diff_frames(const uint8_t* frames, int64_t n, int32_t w, int32_t h, int32_t bins, int seg_first,
                            uint32_t* hist, uint32_t* diff) {
  if (bins < 1 || bins > 256) return OR_EUNSUPPORTED;
  const int64_t F = (int64_t)w * h * 3;
  const int64_t k = 3 * (int64_t)bins;
  for (int64_t p = 0; p < n; ++p) {
    int rc = oracle_hist(frames + p * F, w, h, bins, hist + p * k);
    if (rc) return rc;
  }
  uint8_t* seg = (uint8_t*)calloc((size_t)(n > 0 ? n : 1), 1);
  if (!seg) return OR_EINVAL;
  if (n > 0) seg[0] = (uint8_t)(seg_first ? 1 : 0);
  int rc = oracle_shotdiff(hist, seg, n, bins, diff);
  free(seg);
  return rc;
}

/* ------------------------------------------------------------------------
 * NEXT N2 — stencil BEFORE sampling (fig:sampling-e; "sampling after
 * the flow operation yields a sparse set of flow fields computed from
 * differences between original video frames"). Graph: table -> HIST ->
 * stencil [offset, 0] -> Sample. The stencil neighbour of sampled row r is
 * row clamp(r + offset, 0, N-1) of the ORIGINAL table (repeat-edge clamp,
 * S:L152; reading Q6).
 *
 * Per-element dependency analysis ("determine the exact set of
 * required points"): the HIST input rows required by the sampled rows S are
 * R = { r, clamp(r + offset) : r in S }, sorted and deduplicated.
 * ------------------------------------------------------------------------ */
static int cmp_i64_or(const void* a, const void* b) {
  int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return (x > y) - (x < y);
}

static int64_t clamp_row(int64_t r, int64_t n_rows) { return r < 0 ? 0 : (r >= n_rows ? n_rows - 1 : r); }

int oracle_required_rows(const int64_t* rows, int64_t m, int32_t offset, int64_t n_rows, int64_t* out, int64_t cap,
                         int64_t* count) {
  if (m < 0 || n_rows < 0) return OR_EINVAL;
  int64_t* tmp = (int64_t*)malloc(sizeof(int64_t) * (size_t)(2 * m + 1));
  if (!tmp) return OR_EINVAL;
  int64_t k = 0;
  for (int64_t j = 0; j < m; ++j) {
    if (rows[j] < 0 || rows[j] >= n_rows) { free(tmp); return OR_ERANGE; }
    tmp[k++] = rows[j];                              /* the sampled row itself (stencil offset 0) */
    tmp[k++] = clamp_row(rows[j] + offset, n_rows);  /* its stencil neighbour */
  }
  qsort(tmp, (size_t)k, sizeof(int64_t), cmp_i64_or);
  int64_t u = 0;
  for (int64_t i = 0; i < k; ++i) {
    if (i == 0 || tmp[i] != tmp[i - 1]) {
      if (out && u < cap) out[u] = tmp[i];
      ++u;
    }
  }
  free(tmp);
  *count = u;
  return OR_OK;
}

/* D'[j] = sum_c sum_b |H(frame S_j)[c][b] - H(frame clamp(S_j + offset))[c][b]| for
 * positions j of a (multi-table) sampled sequence; frames from scn_synth. */
int oracle_stencil_then_sample(const synth_spec* spec, const int32_t* videos, const int64_t* rows, int64_t m,
                               int32_t offset, int64_t n_rows, int32_t bins, uint32_t* diff) {
  if (bins < 1 || bins > 256) return OR_EUNSUPPORTED;
  const int64_t F = (int64_t)spec->width * spec->height * 3;
  const int64_t k = 3 * (int64_t)bins;
  uint8_t* frame = (uint8_t*)malloc((size_t)(F > 0 ? F : 1));
  uint32_t* pair = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(2 * k));
  if (!frame || !pair) { free(frame); free(pair); return OR_EINVAL; }
  const uint8_t seg2[2] = {1, 0};
  for (int64_t j = 0; j < m; ++j) {
    const int64_t nb = clamp_row(rows[j] + offset, n_rows);
    synth_frame_desc d = synth_describe(spec, videos[j], nb);
    synth_fill_frame_host(spec, &d, frame);
    oracle_hist(frame, spec->width, spec->height, bins, pair);      /* neighbour */
    d = synth_describe(spec, videos[j], rows[j]);
    synth_fill_frame_host(spec, &d, frame);
    oracle_hist(frame, spec->width, spec->height, bins, pair + k);  /* sampled frame */
    uint32_t dd[2];
    oracle_shotdiff(pair, seg2, 2, bins, dd);
    diff[j] = dd[1];
  }
  free(frame);
  free(pair);
  return OR_OK;
}

/* ------------------------------------------------------------------------
 * NEXT N3 — a bounded-state operation with warmup W ("Scanner
 * guarantees that prior to invoking an instance of a bounded state operation
 * to generate output element i, the operation will have previously been
 * invoked to produce at least the previous W elements"
 * sliding_mean, S:L361-364 threshold_detector). The op is an adaptive shot
 * detector over the shot-diff column D: its state is the window of the last
 * W_eff = min(W, p - s0) values of D in the current table (s0 = the table's
 * first position; slices reset state), and
 *   cut[p] = W_eff > 0  and  D[p]*W_eff*k_den > k_num*sum(window) + floor*W_eff*k_den
 * i.e. D[p] > (k_num/k_den)*mean(window) + floor, evaluated exactly in 64-bit.
 * diff/seg: [m]; cut: [m] (0/1).
 * ------------------------------------------------------------------------ */
int oracle_adaptive_cuts(const uint32_t* diff, const uint8_t* seg_start, int64_t m, int32_t warmup, uint32_t k_num,
                         uint32_t k_den, uint32_t floor_, uint8_t* cut) {
  if (warmup < 1 || k_den < 1 || m < 0) return OR_EINVAL;
  for (int64_t p = 0; p < m; ++p) {
    int64_t s0 = p;
    while (s0 > 0 && !seg_start[s0]) --s0;          /* first position of p's table */
    int64_t weff = p - s0;
    if (weff > warmup) weff = warmup;
    uint64_t sum = 0;
    for (int64_t i = 1; i <= weff; ++i) sum += diff[p - i];
    uint64_t lhs = (uint64_t)diff[p] * (uint64_t)weff * k_den;
    uint64_t rhs = (uint64_t)k_num * sum + (uint64_t)floor_ * (uint64_t)weff * k_den;
    cut[p] = (uint8_t)(weff > 0 && lhs > rhs ? 1 : 0);
  }
  return OR_OK;
}

/* ------------------------------------------------------------------------
 * NEXT N1 — two-job shot montage ("detect shot boundaries (via
 * histogram differences) ... produce film summaries via montage"; P:L457:
 * "compute color histograms on every frame ... (to detect shot boundaries),
 * and then sparsely computed ... on a single frame per shot"; two jobs because
 * graphs cannot filter data-dependently).
 * Job 1 -> D. Selection (reading Q5 threshold_detector): the first
 * position of every shot = positions p with seg_start[p] or D[p] > tau.
 * Job 2: Gather those frames, 2x downsample (reading Q11), place tile k of the
 * K keyframes at tile-row k / cols, tile-column k % cols of a zeroed canvas of
 * ceil(K/cols)*(H/2) rows x cols*(W/2) pixels (RGB8 HWC).
 * ------------------------------------------------------------------------ */
int oracle_shot_starts(const uint32_t* diff, const uint8_t* seg_start, int64_t m, uint32_t tau, int64_t* out,
                       int64_t cap, int64_t* count) {
  int64_t k = 0;
  for (int64_t p = 0; p < m; ++p) {
    if (seg_start[p] || diff[p] > tau) {
      if (out && k < cap) out[k] = p;
      ++k;
    }
  }
  *count = k;
  return OR_OK;
}

int oracle_montage(const synth_spec* spec, const int32_t* videos, const int64_t* rows, int64_t k, int32_t cols,
                   uint8_t* canvas) {
  if (cols < 1 || k < 0) return OR_EINVAL;
  const int32_t ow = spec->width / 2, oh = spec->height / 2;
  const int64_t tile_rows = (k + cols - 1) / cols;
  const int64_t pitch = (int64_t)cols * ow * 3;
  memset(canvas, 0, (size_t)(tile_rows * oh * pitch));
  const int64_t F = (int64_t)spec->width * spec->height * 3;
  uint8_t* frame = (uint8_t*)malloc((size_t)(F > 0 ? F : 1));
  uint8_t* ds = (uint8_t*)malloc((size_t)((int64_t)ow * oh * 3 + 1));
  if (!frame || !ds) { free(frame); free(ds); return OR_EINVAL; }
  for (int64_t i = 0; i < k; ++i) {
    synth_frame_desc d = synth_describe(spec, videos[i], rows[i]);
    synth_fill_frame_host(spec, &d, frame);
    oracle_downsample(frame, spec->width, spec->height, ds);
    const int64_t ty = i / cols, tx = i % cols;
    for (int32_t y = 0; y < oh; ++y)
      for (int32_t x = 0; x < ow; ++x)
        for (int32_t c = 0; c < 3; ++c)
          canvas[(ty * oh + y) * pitch + (tx * ow + x) * 3 + c] = ds[((int64_t)y * ow + x) * 3 + c];
  }
  free(frame);
  free(ds);
  return OR_OK;
}
