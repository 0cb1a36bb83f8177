/* synth_host.c — host side of the seeded input generator (see scn_synth.h). INPUT ONLY. */
#include "scn_synth.h"
#include <stdlib.h>
#include <string.h>

static int32_t shot_len(const synth_spec* s, int32_t scene, int32_t shot) {
  uint32_t r = synth_key3(s->seed ^ 0x5EEDU, (uint32_t)scene, (uint32_t)shot);
  int32_t span = s->len_max - s->len_min + 1;
  if (span < 1) span = 1;
  return s->len_min + (int32_t)(r % (uint32_t)span);
}

synth_frame_desc synth_describe(const synth_spec* s, int32_t video, int64_t row) {
  synth_frame_desc d;
  d.video = video;
  d.row = row;
  d.x_offset = 0;
  int32_t scene = video;
  if (s->shared_scene) {
    scene = 0;
    int32_t nv = s->n_videos_scene > 0 ? s->n_videos_scene : 1;
    d.x_offset = (int32_t)(((int64_t)video * s->width) / nv);
  }
  int32_t shot = 0;
  int64_t start = 0;
  if (s->n_cuts >= 0) {
    for (int32_t i = 0; i < s->n_cuts; ++i) {
      if (s->cuts[i] <= row) { shot = i + 1; start = s->cuts[i]; }
    }
  } else {
    for (;;) {
      int64_t len = shot_len(s, scene, shot);
      if (start + len > row) break;
      start += len;
      ++shot;
    }
  }
  d.shot = shot;
  d.t = (int32_t)(row - start);
  (void)scene;
  return d;
}

int64_t synth_cut_rows(const synth_spec* s, int32_t video, int64_t num_rows, int64_t* out, int64_t cap) {
  int64_t n = 0;
  if (s->n_cuts >= 0) {
    for (int32_t i = 0; i < s->n_cuts; ++i)
      if (s->cuts[i] > 0 && s->cuts[i] < num_rows) { if (n < cap) out[n] = s->cuts[i]; ++n; }
    return n;
  }
  int32_t scene = s->shared_scene ? 0 : video;
  int64_t start = 0;
  for (int32_t shot = 0;; ++shot) {
    start += shot_len(s, scene, shot);
    if (start >= num_rows) break;
    if (n < cap) out[n] = start;
    ++n;
  }
  return n;
}

void synth_fill_frame_host(const synth_spec* s, const synth_frame_desc* d, uint8_t* dst) {
  int32_t scene = s->shared_scene ? 0 : d->video;
  synth_shot_params sp = synth_shot(s->seed, s->width, s->height, scene, d->shot);
  uint32_t fk = synth_frame_key(s->seed, d->video, d->row);
  size_t i = 0;
  for (int32_t y = 0; y < s->height; ++y)
    for (int32_t x = 0; x < s->width; ++x)
      for (int32_t c = 0; c < 3; ++c) dst[i++] = synth_pixel(s->mode, fk, &sp, s->width, d, y, x, c);
}

static uint64_t splitmix64(uint64_t* st) {
  uint64_t z = (*st += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

static int cmp_i64(const void* a, const void* b) {
  int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return (x > y) - (x < y);
}

/* Floyd's sampling without replacement; membership via a sorted probe of the chosen set is
 * O(k^2) in the worst case, so use a simple open-addressing hash set. */
int synth_gather_rows(uint64_t seed, int64_t n, int64_t k, int64_t* out) {
  if (k < 0 || k > n) return -1;
  if (k == 0) return 0;
  int64_t cap = 1;
  while (cap < 4 * k) cap <<= 1;
  int64_t* set = (int64_t*)malloc(sizeof(int64_t) * (size_t)cap);
  if (!set) return -2;
  for (int64_t i = 0; i < cap; ++i) set[i] = -1;
  uint64_t st = seed;
  int64_t m = 0;
  for (int64_t j = n - k; j < n; ++j) {
    int64_t t = (int64_t)(splitmix64(&st) % (uint64_t)(j + 1));
    /* if t already chosen, choose j */
    int64_t h = (int64_t)((uint64_t)t * 0x9E3779B97F4A7C15ULL >> 1) & (cap - 1);
    int found = 0;
    while (set[h] != -1) { if (set[h] == t) { found = 1; break; } h = (h + 1) & (cap - 1); }
    int64_t v = found ? j : t;
    h = (int64_t)((uint64_t)v * 0x9E3779B97F4A7C15ULL >> 1) & (cap - 1);
    while (set[h] != -1) h = (h + 1) & (cap - 1);
    set[h] = v;
    out[m++] = v;
  }
  free(set);
  qsort(out, (size_t)m, sizeof(int64_t), cmp_i64);
  return 0;
}

/* Fill many frames (one per descriptor) into host buffers dst[i] (nbytes each >= W*H*3). */
void synth_fill_frames_host(const synth_spec* s, const synth_frame_desc* d, int64_t n, uint8_t* const* dst) {
  for (int64_t i = 0; i < n; ++i) synth_fill_frame_host(s, d + i, dst[i]);
}
