/* scn_synth.h — seeded synthetic RGB8 video generator (INPUT ONLY).
 *
 * This module is the only code shared by the CUDA path and the CPU oracle
 * (task rule ③: "only the seeded input generators serve both, from a module of
 * their own that holds none of the method's arithmetic"). It produces frame
 * bytes, shot structure and gather index lists; it computes no histogram,
 * difference or downsample.
 *
 * Recipe (DESIGN.md §"Input recipe"):
 *   - decode is out of scope (BASELINE.json north_star), so frames are
 *     generated directly as RGB8 HWC bytes;
 *   - mode SYNTH_SHOTS: each video is a sequence of shots. Shot k has a base
 *     colour per channel (even shots in [0,31], odd shots in [96,159], so
 *     adjacent shots differ by >= 65 levels = >= 4 bins at B=16), an integer
 *     gradient spanning <= 96 levels across the frame, a horizontal drift of
 *     -4..4 px/frame applied cyclically (so the within-shot histogram changes
 *     only through the per-pixel noise), and +-4 per-byte noise;
 *   - mode SYNTH_UNIFORM: independent uniform bytes (adversarial for
 *     warp aggregation);
 *   - mode SYNTH_CONSTANT: every byte of a channel equals the shot's base
 *     colour (adversarial for per-bin contention);
 *   - mode SYNTH_XGRAD: v = x mod 256 in every channel (closed-form histogram).
 *
 * All arithmetic is uint32/int32 and defined identically on host and device.
 */
#ifndef SCN_SYNTH_H
#define SCN_SYNTH_H

#include <stdint.h>

#ifdef __CUDACC__
#define SYNTH_HD __host__ __device__ __forceinline__
#else
#define SYNTH_HD static inline
#endif

#ifdef __cplusplus
extern "C" {
#endif

enum { SYNTH_SHOTS = 0, SYNTH_UNIFORM = 1, SYNTH_CONSTANT = 2, SYNTH_XGRAD = 3 };

/* Per-video content spec. Shot boundaries are either an explicit list of cut
 * rows (n_cuts >= 0; a cut row is the first frame of a new shot) or random
 * shot lengths uniform in [len_min, len_max] drawn from the seed (n_cuts < 0). */
typedef struct {
  uint32_t seed;
  int32_t width, height;
  int32_t mode;
  int32_t n_cuts;           /* < 0: random shot lengths */
  const int64_t* cuts;      /* sorted cut rows when n_cuts >= 0 */
  int32_t len_min, len_max; /* random shot lengths */
  int32_t shared_scene;     /* nonzero: all videos share shot content (VR rig), with a per-video x offset */
  int32_t n_videos_scene;   /* x offset = video * width / n_videos_scene when shared_scene */
} synth_spec;

/* Per-frame descriptor: which content the frame shows. */
typedef struct {
  int32_t video;
  int32_t shot;      /* shot index within the video (or scene) */
  int32_t t;         /* frame index within the shot */
  int32_t x_offset;  /* horizontal offset (VR rig cameras) */
  int64_t row;       /* row index within the video table */
} synth_frame_desc;

SYNTH_HD uint32_t synth_mix32(uint32_t x) {
  /* lowbias32 (public-domain integer hash) */
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

SYNTH_HD uint32_t synth_key3(uint32_t seed, uint32_t a, uint32_t b) {
  return synth_mix32(seed ^ synth_mix32(a * 0x9E3779B1U ^ synth_mix32(b + 0x632BE5ABU)));
}

/* floor(a / 256) for signed a without relying on implementation-defined >> */
SYNTH_HD int32_t synth_floor_div256(int32_t a) { return a >= 0 ? a / 256 : -((-a + 255) / 256); }

SYNTH_HD int32_t synth_mod(int32_t a, int32_t m) { int32_t r = a % m; return r < 0 ? r + m : r; }

/* Shot parameters for (video-or-scene, shot). */
typedef struct {
  int32_t base[3];
  int32_t gx[3], gy[3];
  int32_t drift;
} synth_shot_params;

SYNTH_HD synth_shot_params synth_shot(uint32_t seed, int32_t width, int32_t height, int32_t scene, int32_t shot) {
  synth_shot_params p;
  uint32_t sh = synth_key3(seed, (uint32_t)scene + 0x51ED27U, (uint32_t)shot);
  int32_t gmx = (96 * 256) / (width > 0 ? width : 1);
  int32_t gmy = (96 * 256) / (height > 0 ? height : 1);
  for (int c = 0; c < 3; ++c) {
    uint32_t r = synth_mix32(sh ^ (0x1000193U * (uint32_t)(c + 1)));
    p.base[c] = (shot & 1) ? 96 + (int32_t)(r % 64U) : (int32_t)(r % 32U);
    uint32_t r2 = synth_mix32(r ^ 0xA5A5A5A5U);
    uint32_t r3 = synth_mix32(r2 ^ 0x5A5A5A5AU);
    p.gx[c] = (int32_t)(r2 % (uint32_t)(2 * gmx + 1)) - gmx;
    p.gy[c] = (int32_t)(r3 % (uint32_t)(2 * gmy + 1)) - gmy;
  }
  p.drift = (int32_t)(synth_mix32(sh ^ 0xC0FFEEU) % 9U) - 4;
  return p;
}

SYNTH_HD uint32_t synth_frame_key(uint32_t seed, int32_t video, int64_t row) {
  return synth_key3(seed ^ 0xF00DU, (uint32_t)video, (uint32_t)row ^ (uint32_t)(row >> 32));
}

/* The byte at (y, x, c) of the frame described by d. sp = synth_shot(...) for d. */
SYNTH_HD uint8_t synth_pixel(int32_t mode, uint32_t fkey, const synth_shot_params* sp, int32_t width,
                             const synth_frame_desc* d, int32_t y, int32_t x, int32_t c) {
  if (mode == SYNTH_XGRAD) return (uint8_t)(x & 255);
  if (mode == SYNTH_UNIFORM) {
    uint32_t idx = ((uint32_t)y * (uint32_t)width + (uint32_t)x) * 3U + (uint32_t)c;
    return (uint8_t)(synth_mix32(fkey ^ synth_mix32(idx)) & 255U);
  }
  if (mode == SYNTH_CONSTANT) return (uint8_t)sp->base[c];
  int32_t xs = synth_mod(x + sp->drift * d->t + d->x_offset, width);
  uint32_t nz = synth_mix32(fkey ^ ((uint32_t)y * (uint32_t)width + (uint32_t)x));
  int32_t noise = (int32_t)((nz >> (3 * c)) & 7U) - 4;
  int32_t v = sp->base[c] + synth_floor_div256(sp->gx[c] * xs + sp->gy[c] * y) + noise;
  return (uint8_t)(v < 0 ? 0 : (v > 255 ? 255 : v));
}

/* ---- host-only helpers (shot lookup, gather lists); defined in synth_host.c ---- */
#ifndef __CUDA_ARCH__
/* Describe row `row` of video `video`. */
synth_frame_desc synth_describe(const synth_spec* spec, int32_t video, int64_t row);
/* Shot start rows of a video with num_rows rows (cuts). Returns number written (<= cap). */
int64_t synth_cut_rows(const synth_spec* spec, int32_t video, int64_t num_rows, int64_t* out, int64_t cap);
/* Write one full frame (HWC, width*height*3 bytes) to dst. */
void synth_fill_frame_host(const synth_spec* spec, const synth_frame_desc* d, uint8_t* dst);
/* k distinct rows from [0, n), drawn with Floyd's algorithm on splitmix64(seed), sorted ascending. */
int synth_gather_rows(uint64_t seed, int64_t n, int64_t k, int64_t* out);
#endif

#ifdef __cplusplus
}
#endif
#endif /* SCN_SYNTH_H */
