// kernels.cu — sm_100a kernels of the Scanner HIST / shot-diff / downsample
// hot path (arXiv 1805.07339 P:L331 HIST, P:L455 shot boundaries via
// histogram differences over a [-1,0] stencil P:L210, P:L183/P:L335 resize).
//
// K1+K2 hist_tma_kernel<0, LOGB>  (bins = 2^LOGB <= 16; the configs' B = 16)
//   Persistent, one CTA per SM (227 KB smem). Warp 16 is a TMA producer: one
//   elected lane streams 43,008-byte tiles of the sampled frames with 1-D bulk
//   copies (cp.async.bulk -> UBLKCP) into a 3-stage shared-memory ring guarded
//   by full/empty mbarriers. Warps 0-15 consume: each thread takes 48-byte
//   units (16 pixels, 3 x LDS.128, channel of byte j = j mod 3) and counts
//   PAIRS of same-channel pixels (p, p+8) — bytes j and j+24, same position in
//   their words, so one SHF + one LOP3 select makes four keys at once —
//   key = bin(a) | bin(b) << LOGB into a lane-private table (bank == lane:
//   conflict-free for any content; at B = 16 channels 0/1 share 256-byte key rows
//   so one PRMT turns a key byte into its address) with one red.shared.add per
//   pair, i.e. 0.5 shared atomics per byte, 75 instructions per 48 bytes. Pairs halve the atomics and the issue slots per byte against a
//   single key per byte; measured on B200 (profiles/r01_tune.jsonl) pairs
//   sustain 6.3-6.4 TB/s vs 5.6-5.8 TB/s for one key per byte at B = 16
//   (the shared-atomic pipe itself, 31.8 lane-ops/clk/SM by the ILP K0
//   microbenchmark, is not the bound). On a frame change the CTA's consumer warps
//   marginalise the table (sum over lanes and the partner bin) into 3*B
//   counters and merge them with one red.global.add each ("one global merge
//   per block" per frame segment).
// K2g MODE 1: any bins in [1,256], one atomic per byte, bin = (v*B)>>8, same ring.
// K2a MODE 5: the north_star's design, kept selectable (SCN_HIST_IMPL=match) and
//   measured: per-warp bins, __match_any_sync peer aggregation, leader atomics,
//   __reduce_add_sync merge, one global add per key per block.
// K2s MODE 4 (NEXT N4): B = 32..256 power of two, one shifted key per byte
//   (table | bin << 7 | lane << 2), e.g. 256 bins at 6.86 TB/s on C2.
// K2f hist_tma_kernel<2, LOGB>: K1+K2 with the 2x box downsample fused into the
//   consumer (a thread takes the two vertically adjacent 48-byte units of a
//   row pair, histograms both and emits 8 output pixels), so each sampled
//   frame is read from HBM once (reading Q12). At B = 16 (VAR bit 128, default)
//   it uses the split layout (make_layout_split): channel 2's pair keys in 16 KB
//   of half-lane rows and ring slots on both sides of the 64 KB PRMT block, so
//   1080p and 4K both get 3 stages of 46 KB row-pair tiles.
// K3 shotdiff_kernel: one warp per position, L1 over 3*B counters with
//   __reduce_add_sync.
// K4 hist_tma_kernel<3, 4>: the same ring without the table (downsample only);
//   downsample_vec_kernel (LDG.128) and downsample_generic_kernel (any W) otherwise.
//
// Why not the north_star's per-warp bins + __match_any_sync aggregation: on
// this B200 MATCH.ANY issues at 0.035 warp-instr/clk/SM (profiles/
// r01_k0_micro_v2.json), i.e. ~1.1 bytes/clk/SM if applied per byte, ~5% of the
// HBM roofline. DESIGN.md §5 records the deviation and the evidence.
#include "kernels.h"
#include "ptx.cuh"

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <utility>

namespace scn {

constexpr int kDefaultConsWarps = 16;  // consumer warps per CTA (+1 producer warp)
constexpr uint32_t kTile = 43008;  // 896 x 48 bytes: a multiple of 48 (channel phase) and 16 (TMA); 3 stages.
                                   // Measured best of 24,576..64,512 on B200 (profiles/r01_tune.jsonl)
constexpr uint32_t kFusedTile = 64512;  // target bytes per row-pair tile, fused hist+downsample (measured)
constexpr uint32_t kDsTile = 23040;     // downsample-only kernel: no table, so smaller tiles and a deeper ring win
constexpr int kMaxStages = 8;
constexpr uint32_t kCtrlBytes = 1024;
constexpr uint32_t kBarId = 1;     // named barrier among consumer warps

struct HistParams {
  FrameSrc src;
  int64_t n_items;
  int32_t n_halo;
  uint32_t* out;
  uint32_t* halo_out;
  uint8_t* ds_out;
  int64_t ds_pitch;  // bytes between output rows
  int32_t ds_cols;   // > 0: montage tiles (NEXT N1)
  int64_t F;
  int32_t width, height, bins;
  uint32_t tile;          // bytes per full tile
  int32_t rows_per_tile;  // fused kernel: rows per tile (even); 0 otherwise
  int32_t tpf;            // tiles per frame
  int64_t total_tiles;
  uint32_t smem_bytes;
  uint32_t table_bytes;
  uint32_t table_align;
  uint32_t stage_bytes;  // VAR bit 32: per-slot staging of the tile's downsample output (after its input bytes)
  int32_t l2_hint;  // 1: TMA loads carry an L2 evict_first policy (SCN_TMA_HINT)
  int32_t l2_prefetch;  // > 0: the producer bulk-prefetches tile t + l2_prefetch into L2 (SCN_L2_PREFETCH)
  int32_t max_stages;   // > 0: cap on the ring depth (SCN_MAX_STAGES)
  int32_t n_dest;   // > 0: results go to every dest[g] (fused all-gather over peer memory)
  uint64_t dest[kMaxDest];
};

__device__ __forceinline__ uint64_t frame_addr(const FrameSrc& s, int64_t i) {
  return s.ptrs ? s.ptrs[i] : s.base + (uint64_t)i * s.stride;
}

// First output byte of downsampled frame io: contiguous frames (cols == 0) or
// tile (io / cols, io % cols) of a montage canvas with row pitch `pitch` (NEXT N1).
__device__ __forceinline__ uint8_t* ds_frame_base(uint8_t* base, int64_t io, int64_t oh, int64_t ow3, int64_t pitch,
                                                  int32_t cols) {
  if (cols > 0) return base + (io / cols) * oh * pitch + (io % cols) * ow3;
  return base + io * oh * pitch;
}

struct Layout {
  uint32_t ctrl;   // [full bars][empty bars][hsum]
  uint32_t table;
  uint32_t ring, stride;
  int stages;
  uint32_t ring_hi = 0;  // split layout: slots n_lo.. live above the table
  int n_lo = 0;
  __device__ __forceinline__ uint32_t slot(int s) const { return ring + (uint32_t)s * stride; }
  __device__ __forceinline__ uint32_t slot_split(int s) const {
    return s < n_lo ? ring + (uint32_t)s * stride : ring_hi + (uint32_t)(s - n_lo) * stride;
  }
};

// Shared-memory layout: 1 KB control block at the bottom, the lane-private table at
// the highest table_align-aligned address that fits (so bin fields can be OR-ed into
// its address), and one contiguous ring of tile slots in between (each slot: the tile's
// input bytes, then stage_bytes of staged downsample output when the TMA-store path is on).
__device__ __forceinline__ Layout make_layout(uint32_t base, uint32_t smem_bytes, uint32_t tile, uint32_t tb_bytes,
                                              uint32_t tb_align, uint32_t stage_bytes) {
  Layout L;
  L.ctrl = base;
  const uint32_t end = base + smem_bytes;
  L.table = (end - tb_bytes) & ~(tb_align - 1);
  L.ring = (base + kCtrlBytes + 127) & ~127u;
  L.stride = ((tile + 127) & ~127u) + ((stage_bytes + 127) & ~127u);
  const uint32_t need = stage_bytes ? L.stride : tile;  // the last slot's footprint
  L.stages = L.table >= L.ring + need ? (int)((L.table - L.ring - need) / L.stride) + 1 : 0;
  if (L.stages > kMaxStages) L.stages = kMaxStages;
  if (L.table < base + kCtrlBytes) L.stages = 0;
  return L;
}

// Split layout of the fused hist + downsample kernel at B = 16 (VAR bit 128): the
// 64 KB PRMT block of channels 0/1 at the first 64 KB boundary above the control
// block, channel 2's pair keys in 16 KB right below it as tab2[key][lane / 2] (64-byte
// rows of 16 counters shared by lanes 2l, 2l+1), and ring slots both below tab2 and
// above the block. Against the 96 KB table this frees 16 KB and the 64 KB alignment
// waste, so 4K row-pair tiles get 3 stages instead of 2 (1080p: 8-row tiles instead of
// 6). Lanes 2l and 2l+1 hit the same bank only when their channel-2 keys differ with
// equal parity (a 2-way conflict); equal keys are one address (aggregated).
constexpr uint32_t kTab2Bytes = 16384;
constexpr uint32_t kSplitTab2 = kTab2Bytes;
__device__ __forceinline__ Layout make_layout_split(uint32_t base, uint32_t smem_bytes, uint32_t tile) {
  Layout L;
  L.ctrl = base;
  const uint32_t end = base + smem_bytes;
  const uint32_t block = (base + kCtrlBytes + kTab2Bytes + 65535u) & ~65535u;
  L.table = block - kTab2Bytes;
  L.ring = (base + kCtrlBytes + 127) & ~127u;
  L.stride = (tile + 127) & ~127u;
  L.ring_hi = block + 65536u;
  const int lo = L.table >= L.ring + tile ? (int)((L.table - L.ring - tile) / L.stride) + 1 : 0;
  const int hi = end >= L.ring_hi + tile ? (int)((end - L.ring_hi - tile) / L.stride) + 1 : 0;
  L.stages = lo + hi > kMaxStages ? kMaxStages : lo + hi;
  L.n_lo = lo < L.stages ? lo : L.stages;
  if (L.ring_hi > end) L.stages = 0;
  return L;
}

template <int OFF>
__device__ __forceinline__ void red_shared_add_off(uint32_t addr) {
  asm volatile("red.shared.add.u32 [%0+%1], 1;" ::"r"(addr), "n"(OFF) : "memory");
}

// Byte J of the unit shifted so its top LOGB bits (its bin) land at bit DST (unmasked).
template <int J, int DST, int LOGB>
__device__ __forceinline__ uint32_t bin_shift(const uint32_t* w) {
  constexpr int src = 8 * (J & 3) + 8 - LOGB;
  const uint32_t x = w[J >> 2];
  if constexpr (src >= DST) return x >> (src - DST);
  else return x << (DST - src);
}
// (a & b) | c in one LOP3
template <uint32_t MASK>
__device__ __forceinline__ uint32_t lop3_and_or(uint32_t a, uint32_t c) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(a), "n"(MASK), "r"(c));
  return d;
}

// Count the 24 same-channel pixel pairs of one 48-byte unit (16 pixels).
// lane4 = table base | lane << 2. Pair (2q, 2q+1) of channel c: bytes 6q+c, 6q+3+c.
template <int LOGB, int P>
__device__ __forceinline__ void pair_unit_step(const uint32_t* w, uint32_t lane4) {
  constexpr int q = P / 3, c = P % 3;
  constexpr int JA = 6 * q + c, JB = 6 * q + 3 + c;
  constexpr int B = 1 << LOGB;
  // addr = (yA & maskA) | ((yB & maskB) | lane4): two LOP3s (forced; the compiler emits three)
  const uint32_t lo = lop3_and_or<((1u << LOGB) - 1u) << 7>(bin_shift<JB, 7, LOGB>(w), lane4);
  const uint32_t addr = lop3_and_or<((1u << LOGB) - 1u) << (7 + LOGB)>(bin_shift<JA, 7 + LOGB, LOGB>(w), lo);
  red_shared_add_off<c * B * B * 128>(addr);
}
template <int LOGB, int... P>
__device__ __forceinline__ void pair_unit_all(const uint32_t* w, uint32_t lane4, std::integer_sequence<int, P...>) {
  (pair_unit_step<LOGB, P>(w, lane4), ...);
}
// Word-parallel pairing (default): pixel p pairs with pixel p+8 of the unit, i.e. byte j
// with byte j+24 — same channel (24 = 0 mod 3) and same position within its word, so
// one SHF + one LOP3 select builds a word K of four 2*LOGB-bit keys:
//   K = ((w[k] >> (8-LOGB)) & M1) | ((w[k+6] >> (8-2*LOGB)) & M2)   (M1/M2: per-byte fields)
// and each key costs one shift + one LOP3 (mask | lane4) to become an address.
// Which pixels are paired does not matter: the flush adds each key's count to both
// of its bins (same channel), so the marginals are exact for any same-channel pairing.
//
// B = 16 layout (kPrmtTable): the 256 keys of channels 0 and 1 share 256-byte rows of a
// 64 KB-aligned block, tab01[key][c][lane], so key byte I of K drops straight into byte 1
// of the address with ONE PRMT (byte 0 = lane << 2, bytes 2-3 = the block's high bits;
// c * 128 is the ATOMS immediate); channel 2 keeps 128-byte rows, tab2[key][lane], in the
// 32 KB after the block (table | key << 7 | lane << 2 + 64 KB: shift + LOP3). 16 of the
// unit's 24 keys cost one instruction instead of two; the table is still 96 KB.
template <int LOGB, int K_, int I, bool PRMT, bool H2>
__device__ __forceinline__ void wpair_key_step(uint32_t K, uint32_t lane4, uint32_t lane4h) {
  constexpr int J = 4 * K_ + I;  // byte of the first pixel of the pair
  constexpr int c = J % 3;
  constexpr int B = 1 << LOGB;
  constexpr uint32_t kmask = ((1u << (2 * LOGB)) - 1u) << 7;
  if constexpr (PRMT && c < 2) {
    red_shared_add_off<c * 128>(__byte_perm(K, lane4, 0x7604u | (I << 4)));
    return;
  }
  if constexpr (H2 && c == 2) {  // split layout: tab2 | key << 6 | (lane / 2) << 2
    constexpr uint32_t kmask6 = ((1u << (2 * LOGB)) - 1u) << 6;
    uint32_t x;
    if constexpr (8 * I >= 6) x = K >> (8 * I - 6);
    else x = K << (6 - 8 * I);
    red_shared_add_off<0>(lop3_and_or<kmask6>(x, lane4h));
    return;
  }
  uint32_t x;
  if constexpr (8 * I >= 7) x = K >> (8 * I - 7);
  else x = K << (7 - 8 * I);
  red_shared_add_off<(PRMT ? 65536 : c * B * B * 128)>(lop3_and_or<kmask>(x, lane4));
}
template <int LOGB, int K_, bool PRMT, bool H2>
__device__ __forceinline__ void wpair_word(const uint32_t* w, uint32_t lane4, uint32_t lane4h) {
  constexpr uint32_t f = (1u << LOGB) - 1u;
  constexpr uint32_t M1 = f * 0x01010101u, M2 = (f << LOGB) * 0x01010101u;
  const uint32_t a = w[K_] >> (8 - LOGB);
  const uint32_t b = (8 - 2 * LOGB) > 0 ? (w[K_ + 6] >> (8 - 2 * LOGB)) : w[K_ + 6];
  uint32_t Kw;
  if constexpr (M2 == (~M1)) {
    // per bit: M1 ? a : b  (LUT for operands (b, a, M1): (0xCC & 0xAA) | (0xF0 & ~0xAA) = 0xD8)
    asm("lop3.b32 %0, %1, %2, %3, 0xD8;" : "=r"(Kw) : "r"(b), "r"(a), "n"(M1));
  } else {
    Kw = (a & M1) | (b & M2);
  }
  wpair_key_step<LOGB, K_, 0, PRMT, H2>(Kw, lane4, lane4h);
  wpair_key_step<LOGB, K_, 1, PRMT, H2>(Kw, lane4, lane4h);
  wpair_key_step<LOGB, K_, 2, PRMT, H2>(Kw, lane4, lane4h);
  wpair_key_step<LOGB, K_, 3, PRMT, H2>(Kw, lane4, lane4h);
}
template <int LOGB, int VAR = 0>
__device__ __forceinline__ void hist_unit_pair(const uint32_t* w, uint32_t lane4, uint32_t lane4h = 0) {
  if constexpr ((VAR & 8) || LOGB == 0) {  // adjacent-pixel pairing (previous default, SCN_HIST_VAR=8)
    pair_unit_all<LOGB>(w, lane4, std::make_integer_sequence<int, 24>{});
  } else {
    constexpr bool P = LOGB == 4 && !(VAR & 64);  // B = 16: PRMT table layout (VAR bit 64: the previous one)
    constexpr bool H = P && (VAR & 128);          // split layout: channel 2 in half-lane rows
    wpair_word<LOGB, 0, P, H>(w, lane4, lane4h); wpair_word<LOGB, 1, P, H>(w, lane4, lane4h);
    wpair_word<LOGB, 2, P, H>(w, lane4, lane4h); wpair_word<LOGB, 3, P, H>(w, lane4, lane4h);
    wpair_word<LOGB, 4, P, H>(w, lane4, lane4h); wpair_word<LOGB, 5, P, H>(w, lane4, lane4h);
  }
}

// Single-key lane-private counting for B = 2^LOGB in [32, 256] (NEXT N4): byte J of
// channel J % 3 -> tab[c][bin][lane], bin = top LOGB bits; table 32 KB-aligned per
// channel for B = 256 so the address is table | bin << 7 | lane << 2 (one LOP3).
// B = 256 PRMT layout (kPrmt256, default): channels 0 and 1 share 256-byte rows of a
// 64 KB-aligned block, tab01[bin][c][lane], so ONE PRMT drops the byte (its bin) into
// byte 1 of the address (c * 128 is the ATOMS immediate); channel 2 keeps 128-byte rows
// in the 32 KB after the block (PRMT + IMAD as before). 2/3 of the bytes cost one
// instruction instead of two; the table is still 96 KB.
template <int LOGB, int J, bool P256>
__device__ __forceinline__ void single_unit_step(const uint32_t* w, uint32_t lane4) {
  constexpr int c = J % 3;
  constexpr int B = 1 << LOGB;
  uint32_t addr;
  if constexpr (P256 && c < 2) {
    red_shared_add_off<c * 128>(__byte_perm(w[J >> 2], lane4, 0x7604u | ((J & 3) << 4)));
    return;
  } else if constexpr (P256) {
    addr = __byte_perm(w[J >> 2], 0u, 0x4440u + (J & 3)) * 128u + lane4;
    red_shared_add_off<65536>(addr);
    return;
  } else if constexpr (LOGB == 8) {
    // B = 256: the key is the byte; PRMT zero-extends it (ALU), IMAD scales and adds the
    // lane offset (FMA pipe): one op on each pipe instead of two ALU ops
    addr = __byte_perm(w[J >> 2], 0u, 0x4440u + (J & 3)) * 128u + lane4;
  } else {
    addr = lop3_and_or<((1u << LOGB) - 1u) << 7>(bin_shift<J, 7, LOGB>(w), lane4);
  }
  red_shared_add_off<c * B * 128>(addr);
}
template <int LOGB, bool P256, int... J>
__device__ __forceinline__ void single_unit_all(const uint32_t* w, uint32_t lane4, std::integer_sequence<int, J...>) {
  (single_unit_step<LOGB, J, P256>(w, lane4), ...);
}
template <int LOGB, bool P256 = false>
__device__ __forceinline__ void hist_unit_single(const uint32_t* w, uint32_t lane4) {
  single_unit_all<LOGB, P256>(w, lane4, std::make_integer_sequence<int, 48>{});
}

__device__ __forceinline__ void load_unit(uint32_t a, uint32_t* w) {
  const uint4 v0 = lds128(a), v1 = lds128(a + 16), v2 = lds128(a + 32);
  w[0] = v0.x; w[1] = v0.y; w[2] = v0.z; w[3] = v0.w;
  w[4] = v1.x; w[5] = v1.y; w[6] = v1.z; w[7] = v1.w;
  w[8] = v2.x; w[9] = v2.y; w[10] = v2.z; w[11] = v2.w;
}

// ---- 2x box downsample of a 2 x 48-byte unit pair -> 24 output bytes --------
// O = (a+b+c+d+2)>>2 per channel byte; output byte m of the 8-pixel group averages source
// bytes i = 2m - (m % 3) and i + 3 of both rows.
// Fast 2x2 average of 16 pixels x 2 rows (t, b: 12 words each) -> 8 pixels (6 words).
// Per word: vertical partial sums of the high 6 bits (hv) and low 2 bits (lv) of
// each byte; a funnel shift by 3 bytes aligns pixel 2x+1 over pixel 2x, so
// A = hv + hv>>24b + (((lv + lv>>24b + 2) >> 2) & 3) is the exact average at every
// byte position p with p mod 6 in {0,1,2}; ten PRMTs compact those bytes.
__device__ __forceinline__ void ds_unit(const uint32_t* t, const uint32_t* b, uint32_t* o) {
  uint32_t hv[13], lv[13], A[12];
#pragma unroll
  for (int k = 0; k < 12; ++k) {
    hv[k] = ((t[k] >> 2) & 0x3F3F3F3Fu) + ((b[k] >> 2) & 0x3F3F3F3Fu);  // <= 126 per byte
    lv[k] = (t[k] & 0x03030303u) + (b[k] & 0x03030303u);                // <= 6 per byte
  }
  hv[12] = 0;
  lv[12] = 0;
#pragma unroll
  for (int k = 0; k < 12; ++k) {
    const uint32_t H = hv[k] + __funnelshift_r(hv[k], hv[k + 1], 24);               // <= 252
    const uint32_t Lo = lv[k] + __funnelshift_r(lv[k], lv[k + 1], 24) + 0x02020202u;  // <= 14
    A[k] = H + ((Lo >> 2) & 0x03030303u);                                            // <= 255
  }
  // output byte m <- stream byte 2m - (m mod 3)
  o[0] = __byte_perm(A[0], A[1], 0x6210);
  o[1] = __byte_perm(__byte_perm(A[1], A[2], 0x0043), A[3], 0x5410);
  o[2] = __byte_perm(__byte_perm(A[3], A[4], 0x0762), A[5], 0x4210);
  o[3] = __byte_perm(A[6], A[7], 0x6210);
  o[4] = __byte_perm(__byte_perm(A[7], A[8], 0x0043), A[9], 0x5410);
  o[5] = __byte_perm(__byte_perm(A[9], A[10], 0x0762), A[11], 0x4210);
}
// dp4a variant: output byte m = (T_i + T_{i+3} + B_i + B_{i+3} + 2) >> 2 with i = 2m - m%3,
// each pair taken from a 4-byte window (funnel shift) by one IDP.4A with weights
// (1,0,0,1); the sums run on the FMA pipe instead of the ALU pipe.
template <int I>
__device__ __forceinline__ uint32_t win4(const uint32_t* w) {
  if constexpr ((I & 3) == 0) return w[I >> 2];
  else return __funnelshift_r(w[I >> 2], w[(I >> 2) + 1], 8 * (I & 3));
}
// The weights are 64, not 1: the result is (sum + 2) * 64 <= 65,408, so the output byte
// (sum + 2) >> 2 sits exactly in bits 8-15 — no shift and no mask afterwards.
template <int M>
__device__ __forceinline__ uint32_t ds_sum(const uint32_t* t, const uint32_t* b) {  // (sum + 2) * 64
  constexpr int I = 2 * M - (M % 3);
  return __dp4a(win4<I>(b), 0x40000040u, __dp4a(win4<I>(t), 0x40000040u, 128u));
}
// Packing: two scaled sums at 16-bit spacing (one IMAD: no carry, each < 2^16) put output
// bytes m and m+2 in bytes 1 and 3; one PRMT interleaves the two words' bytes 1 and 3.
template <int Q>
__device__ __forceinline__ uint32_t ds_word4(const uint32_t* t, const uint32_t* b) {
  const uint32_t t02 = ds_sum<4 * Q + 2>(t, b) * 65536u + ds_sum<4 * Q>(t, b);
  const uint32_t t13 = ds_sum<4 * Q + 3>(t, b) * 65536u + ds_sum<4 * Q + 1>(t, b);
  return __byte_perm(t02, t13, 0x7351);
}
// Funnel-free variant (SCN_DS_VAR=2): a pair (X_i, X_{i+3}) that straddles words k, k+1
// is summed by two dp4a on the aligned words with single-byte weights (FMA pipe only).
template <int M>
__device__ __forceinline__ uint32_t ds_sum2(const uint32_t* t, const uint32_t* b) {  // sum + 2, <= 1022
  constexpr int I = 2 * M - (M % 3), K = I >> 2, O = I & 3;
  if constexpr (O == 0) {
    return __dp4a(t[K], 0x01000001u, __dp4a(b[K], 0x01000001u, 2u));
  } else {
    constexpr uint32_t wa = 1u << (8 * O), wb = 1u << (8 * (O - 1));
    return __dp4a(t[K], wa, __dp4a(t[K + 1], wb, __dp4a(b[K], wa, __dp4a(b[K + 1], wb, 2u))));
  }
}
template <int Q>
__device__ __forceinline__ uint32_t ds_word4b(const uint32_t* t, const uint32_t* b) {
  const uint32_t t02 = ((ds_sum2<4 * Q + 2>(t, b) * 65536u + ds_sum2<4 * Q>(t, b)) >> 2) & 0x00FF00FFu;
  const uint32_t t13 = ((ds_sum2<4 * Q + 3>(t, b) * 65536u + ds_sum2<4 * Q + 1>(t, b)) >> 2) & 0x00FF00FFu;
  return __byte_perm(t02, t13, 0x6240);
}
__device__ __forceinline__ void ds_unit_dp4a_nofunnel(const uint32_t* t, const uint32_t* b, uint32_t* o) {
  o[0] = ds_word4b<0>(t, b); o[1] = ds_word4b<1>(t, b); o[2] = ds_word4b<2>(t, b);
  o[3] = ds_word4b<3>(t, b); o[4] = ds_word4b<4>(t, b); o[5] = ds_word4b<5>(t, b);
}
__device__ __forceinline__ void ds_unit_dp4a(const uint32_t* t, const uint32_t* b, uint32_t* o) {
  o[0] = ds_word4<0>(t, b); o[1] = ds_word4<1>(t, b); o[2] = ds_word4<2>(t, b);
  o[3] = ds_word4<3>(t, b); o[4] = ds_word4<4>(t, b); o[5] = ds_word4<5>(t, b);
}
template <int DSV>
__device__ __forceinline__ void ds_unit_v(const uint32_t* t, const uint32_t* b, uint32_t* o) {
  if constexpr (DSV == 2) ds_unit_dp4a_nofunnel(t, b, o);
  else if constexpr (DSV == 1) ds_unit_dp4a(t, b, o);
  else ds_unit(t, b, o);
}

__device__ __forceinline__ void st_global_24(uint8_t* dst, const uint32_t* o) {
  uint2* d = reinterpret_cast<uint2*>(dst);
  d[0] = make_uint2(o[0], o[1]);
  d[1] = make_uint2(o[2], o[3]);
  d[2] = make_uint2(o[4], o[5]);
}

// ---------------------------------------------------------------------------
// The persistent TMA-ring histogram kernel. MODE 0: pair-key table (B = 2^LOGB
// <= 16); MODE 1: single-key table, any B (LOGB unused); MODE 2: pair-key +
// fused downsample; MODE 3: downsample only (no table). VAR bit 2: dp4a downsample;
// bit 32: downsample output staged in the slot and written by the producer's TMA bulk stores.
// ---------------------------------------------------------------------------
template <int MODE, int LOGB, int NW, int VAR = 0>
__global__ void __launch_bounds__(NW * 32 + 32, 1) hist_tma_kernel(const __grid_constant__ HistParams p) {
  constexpr int kConsWarps = NW;
  constexpr int kConsThreads = NW * 32;
  constexpr int kThreads = kConsThreads + 32;
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int BP = 1 << LOGB;
  const uint32_t base = smem_addr(smem);
  constexpr bool kSplit = MODE == 2 && LOGB == 4 && (VAR & 128) && !(VAR & 64) && !(VAR & 32);
  Layout L = kSplit ? make_layout_split(base, p.smem_bytes, p.tile)
                    : make_layout(base, p.smem_bytes, p.tile, p.table_bytes, p.table_align, p.stage_bytes);
  if (p.max_stages > 0 && L.stages > p.max_stages) {  // ring-depth cap (SCN_MAX_STAGES, measurement knob)
    L.stages = p.max_stages;
    if (L.n_lo > L.stages) L.n_lo = L.stages;
  }
  auto slot_of = [&](int s) -> uint32_t {
    if constexpr (kSplit) return L.slot_split(s);
    else return L.slot(s);
  };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t full0 = L.ctrl, empty0 = L.ctrl + 8 * kMaxStages;
  uint32_t* hsum = reinterpret_cast<uint32_t*>(smem + 16 * kMaxStages);
  const int B = (MODE == 1) ? p.bins : BP;
  constexpr bool kSingle = (MODE == 1 || MODE == 4);  // one key per byte: flush rows are (c, bin) directly
  constexpr bool kPrmt256 = MODE == 4 && LOGB == 8 && !(VAR & 64);  // B = 256 PRMT table layout
  // B = 16 pair keys with word-parallel pairing: the PRMT table layout (see wpair_key_step)
  constexpr bool kPrmtTable = (MODE == 0 || MODE == 2) && LOGB == 4 && !(VAR & 8) && !(VAR & 64);
  constexpr bool kTmaStore = (MODE == 2 || MODE == 3) && (VAR & 32);  // downsample out via TMA bulk stores
  const uint32_t sfree0 = L.ctrl + 512;  // kTmaStore: slot's output area read by its bulk store

  if (threadIdx.x == 0) {
    if (L.stages < 2) __trap();
    for (int s = 0; s < L.stages; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, kConsWarps);
      if constexpr (kTmaStore) mbar_init(sfree0 + 8 * s, 1);
    }
    fence_mbar_init();
  }
  // zero the table and the merge counters
  for (uint32_t i = threadIdx.x; i < p.table_bytes / 16; i += kThreads) sts128(L.table + 16 * i, make_uint4(0, 0, 0, 0));
  for (int i = threadIdx.x; i < 3 * 16; i += kThreads) hsum[i] = 0;
  __syncthreads();

  const int64_t t0 = p.total_tiles * blockIdx.x / gridDim.x;
  const int64_t t1 = p.total_tiles * (blockIdx.x + 1) / gridDim.x;

  if constexpr (kTmaStore) {
    if (warp == kConsWarps) {
      // ---- producer with TMA stores: after the consumers release tile q's slot, its staged
      // downsample output is bulk-stored (one copy per tile, or per output row in a montage),
      // issued S tiles behind the loads; sfree[s] tells the consumers the copy has read it ----
      if (lane == 0) {
        const int S = L.stages;
        int s = 0;
        uint32_t ph = 0;
        int64_t item = t0 / p.tpf;
        int32_t k = (int32_t)(t0 - item * p.tpf);
        int64_t sitem = item;  // tile whose output is stored next
        int32_t sk = k;
        const uint32_t in_bytes = (p.tile + 127u) & ~127u;
        const int64_t ow3 = (int64_t)(p.width / 2) * 3;
        const uint32_t last_rows = (uint32_t)(p.height - (p.tpf - 1) * p.rows_per_tile);
        const int64_t tile_out = (int64_t)(p.rows_per_tile / 2) * p.ds_pitch;
        auto store_next = [&](int slot) {
          if (sitem >= p.n_halo) {
            const uint32_t orows = ((sk == p.tpf - 1) ? last_rows : (uint32_t)p.rows_per_tile) / 2u;
            uint8_t* dst = ds_frame_base(p.ds_out, sitem - p.n_halo, p.height / 2, ow3, p.ds_pitch, p.ds_cols) +
                           (int64_t)sk * tile_out;
            const uint32_t src = L.slot(slot) + in_bytes;
            if (p.ds_pitch == ow3) {
              tma_store_1d(dst, src, orows * (uint32_t)ow3);
            } else {
              for (uint32_t r = 0; r < orows; ++r) tma_store_1d(dst + (int64_t)r * p.ds_pitch, src + r * (uint32_t)ow3, (uint32_t)ow3);
            }
          }
          if (++sk == p.tpf) { sk = 0; ++sitem; }
        };
        for (int64_t t = t0; t < t1; ++t, (++k == p.tpf) ? (k = 0, ++item) : 0) {
          const uint64_t off = (uint64_t)k * p.tile;
          const uint64_t len = (uint64_t)p.F - off < p.tile ? (uint64_t)p.F - off : p.tile;
          const uint32_t bytes = (uint32_t)((len + 15) & ~15ull);
          mbar_wait(empty0 + 8 * s, ph ^ 1);
          const bool wrapped = t - t0 >= S;
          if (wrapped) store_next(s);  // tile t - S, released just now
          mbar_arrive_expect_tx(full0 + 8 * s, bytes);
          tma_load_1d(slot_of(s), reinterpret_cast<const void*>(frame_addr(p.src, item) + off), bytes, full0 + 8 * s);
          if (wrapped) {
            bulk_commit();
            bulk_wait_read<0>();
            mbar_arrive(sfree0 + 8 * s);
          }
          if (++s == S) { s = 0; ph ^= 1; }
        }
        // drain: the last min(n, S) tiles
        const int64_t n = t1 - t0;
        for (int64_t q = t1 - (n < S ? n : S); q < t1; ++q) {
          const int slot = (int)((q - t0) % S);
          mbar_wait(empty0 + 8 * slot, (uint32_t)(((q - t0) / S) & 1));
          store_next(slot);
        }
        bulk_commit();
        bulk_wait_all();
      }
      return;
    }
  } else if (warp == kConsWarps) {
    // ---------------- producer: one elected lane issues the bulk copies ----------------
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      int64_t item = t0 / p.tpf;
      int32_t k = (int32_t)(t0 - item * p.tpf);
      const uint64_t policy = l2_policy_evict_first();
      // L2 prefetch cursor, l2_prefetch tiles ahead of the load cursor
      int64_t pitem = item;
      int32_t pk = k;
      for (int32_t i = 0; i < p.l2_prefetch; ++i)
        if (++pk == p.tpf) { pk = 0; ++pitem; }
      // the frame's address is loaded (sparse tables: a global read of the row pointer) once
      // per frame and BEFORE the empty-slot wait, so its latency overlaps the wait instead of
      // delaying the copy once the slot frees
      int64_t base_item = -1;
      uint64_t base = 0;
      for (int64_t t = t0; t < t1; ++t, (++k == p.tpf) ? (k = 0, ++item) : 0) {
        const uint64_t off = (uint64_t)k * p.tile;
        const uint64_t len = (uint64_t)p.F - off < p.tile ? (uint64_t)p.F - off : p.tile;
        const uint32_t bytes = (uint32_t)((len + 15) & ~15ull);
        if (item != base_item) {
          base_item = item;
          base = frame_addr(p.src, item);
        }
        if (p.l2_prefetch > 0) {
          if (t + p.l2_prefetch < t1) {
            const uint64_t poff = (uint64_t)pk * p.tile;
            const uint64_t plen = (uint64_t)p.F - poff < p.tile ? (uint64_t)p.F - poff : p.tile;
            tma_prefetch_l2(reinterpret_cast<const void*>(frame_addr(p.src, pitem) + poff), (uint32_t)((plen + 15) & ~15ull));
          }
          if (++pk == p.tpf) { pk = 0; ++pitem; }
        }
        const void* src = reinterpret_cast<const void*>(base + off);
        mbar_wait(empty0 + 8 * s, ph ^ 1);
        mbar_arrive_expect_tx(full0 + 8 * s, bytes);
        if (p.l2_hint) tma_load_1d_hint(slot_of(s), src, bytes, full0 + 8 * s, policy);  // frames are read once
        else tma_load_1d(slot_of(s), src, bytes, full0 + 8 * s);
        if (++s == L.stages) { s = 0; ph ^= 1; }
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  const int ctid = threadIdx.x;  // 0 .. kConsThreads-1
  // split layout: channels 0/1 in the 64 KB block after tab2, channel 2 in tab2 (half lanes)
  const uint32_t lane4 = (kSplit ? L.table + kTab2Bytes : L.table) | ((uint32_t)lane << 2);
  const uint32_t lane4h = L.table | ((uint32_t)lane >> 1 << 2);
  int s = 0;
  uint32_t ph = 0;
  // Units are dealt round-robin over the consumer threads across tile boundaries: a thread's
  // next unit (pair) index in the current tile is carried from the previous tile (minus
  // that tile's unit count), so every warp shares the work and a tile costs no division.
  uint32_t ucur = (uint32_t)ctid;
  int64_t cur = -1;

  auto out_row = [&](int64_t item) -> uint32_t* {
    return item < p.n_halo ? p.halo_out + item * 3 * B : p.out + (item - p.n_halo) * 3 * B;
  };
  // add v to counter idx of item's row: locally, or (fused all-gather) into the same row of
  // every rank's result column through peer memory (NVLink when the dest is on another GPU)
  auto emit = [&](int64_t item, int idx, uint32_t v) {
    if (p.n_dest == 0 || item < p.n_halo) {
      red_global_add(out_row(item) + idx, v);
    } else {
      const int64_t off = (item - p.n_halo) * 3 * B + idx;
      for (int g = 0; g < p.n_dest; ++g) red_global_add(reinterpret_cast<uint32_t*>(p.dest[g]) + off, v);
    }
  };

  // Flush without zeroing (default): the lane-private counters keep accumulating over the
  // CTA's frames and a frame's count of a row is its 32-lane sum minus the sum at the
  // previous flush (exact mod 2^32). Each thread always flushes the same rows
  // (r = ctid + i * kConsThreads), so the previous sums live in registers and the flush
  // reads the table without writing it back (half the shared-memory traffic).
  // VAR bit 256: the previous flush that re-zeroes every row (A/B).
  constexpr bool kZeroFlush = (VAR & 256) != 0;
  constexpr int kSnapN = (768 + kConsThreads - 1) / kConsThreads;  // rows <= 3 * 256
  uint32_t snap[kSnapN];
#pragma unroll
  for (int i = 0; i < kSnapN; ++i) snap[i] = 0;
  auto flush = [&](int64_t item) {
    if constexpr (MODE == 3) return;
    named_bar(kBarId, kConsThreads);
    if constexpr (MODE == 5) {
      // merge the per-warp bins: lane l < NW holds warp l's count of key k; __reduce_add_sync
      // sums them and lane 0 issues the block's one global add per key
      uint32_t* wbins = reinterpret_cast<uint32_t*>(smem + (L.table - base));
      for (int k = warp; k < 3 * BP; k += kConsWarps) {
        uint32_t v = lane < kConsWarps ? wbins[lane * 3 * BP + k] : 0u;
        if (lane < kConsWarps) wbins[lane * 3 * BP + k] = 0u;
        v = __reduce_add_sync(0xFFFFFFFFu, v);
        if (lane == 0 && v) emit(item, k, v);
      }
      named_bar(kBarId, kConsThreads);
      return;
    }
    const int rows = kSingle ? 3 * B : 3 * BP * BP;
#pragma unroll
    for (int i = 0; i < kSnapN; ++i) {
      const int r = ctid + i * kConsThreads;
      if (r >= rows) break;
      uint32_t ra = L.table + (uint32_t)r * 128u;
      uint32_t sum = 0;
      if constexpr (kSplit) {  // tab01[key][c] in the block after tab2; channel 2: tab2[key], 64-byte rows
        const uint32_t c = (uint32_t)r >> 8, key = (uint32_t)r & 255u;
        if (c < 2) {
          ra = L.table + kTab2Bytes + key * 256u + c * 128u;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint32_t a = ra + (uint32_t)(((j + r) & 7) * 16);
            const uint4 v = lds128(a);
            sum += v.x + v.y + v.z + v.w;
            if constexpr (kZeroFlush) sts128(a, make_uint4(0, 0, 0, 0));
          }
        } else {
          ra = L.table + key * 64u;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t a = ra + (uint32_t)(((j + r) & 3) * 16);
            const uint4 v = lds128(a);
            sum += v.x + v.y + v.z + v.w;
            if constexpr (kZeroFlush) sts128(a, make_uint4(0, 0, 0, 0));
          }
        }
      } else {
      if constexpr (kPrmtTable || kPrmt256) {  // row (c, key): tab01[key][c] for c < 2, tab2[key] after the block
        const uint32_t c = (uint32_t)r >> 8, key = (uint32_t)r & 255u;
        ra = c < 2 ? L.table + key * 256u + c * 128u : L.table + 65536u + key * 128u;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t a = ra + (uint32_t)(((j + r) & 7) * 16);
        const uint4 v = lds128(a);
        sum += v.x + v.y + v.z + v.w;
        if constexpr (kZeroFlush) sts128(a, make_uint4(0, 0, 0, 0));
      }
      }
      if constexpr (!kZeroFlush) {  // this frame's count = the row sum since the previous flush
        const uint32_t total = sum;
        sum = total - snap[i];
        snap[i] = total;
      }
      if (sum) {
        if (kSingle) {
          emit(item, r, sum);
        } else {
          const int c = r / (BP * BP), key = r % (BP * BP);
          atomicAdd(&hsum[c * BP + (key >> LOGB)], sum);
          atomicAdd(&hsum[c * BP + (key & (BP - 1))], sum);
        }
      }
    }
    if (!kSingle) {
      named_bar(kBarId, kConsThreads);
      if (ctid < 3 * BP) {
        const uint32_t v = hsum[ctid];
        hsum[ctid] = 0;
        if (v) emit(item, ctid, v);
      }
    }
    named_bar(kBarId, kConsThreads);
  };

  // row-pair tiling constants of the downsample modes (unused otherwise)
  struct {
    uint32_t rowb, upr, dq, dr, last_rows, in_bytes, ow3s;
    int64_t pitch, ow3, tile_out;
    uint8_t* ds_frame;
  } rg{};
  if constexpr (MODE == 2 || MODE == 3) {
    rg.rowb = (uint32_t)p.width * 3u;
    rg.upr = (uint32_t)p.width / 16u;
    rg.dq = (uint32_t)kConsThreads / rg.upr;
    rg.dr = (uint32_t)kConsThreads - rg.dq * rg.upr;
    rg.last_rows = (uint32_t)(p.height - (p.tpf - 1) * p.rows_per_tile);
    rg.pitch = p.ds_pitch;
    rg.ow3 = (int64_t)(p.width / 2) * 3;
    rg.tile_out = (int64_t)(p.rows_per_tile / 2) * rg.pitch;
    rg.in_bytes = (p.tile + 127u) & ~127u;
    rg.ow3s = (uint32_t)rg.ow3;
  }
  // MODE 2/3: the carried unit pair as (row pair, column unit), ucur = rpc * upr + xcc
  uint32_t rpc = 0, xcc = 0;
  if constexpr (MODE == 2 || MODE == 3) {
    rpc = (uint32_t)ctid / rg.upr;
    xcc = (uint32_t)ctid - rpc * rg.upr;
  }
  int64_t item = t0 / p.tpf;
  int32_t k = (int32_t)(t0 - item * p.tpf);
  const int32_t ntiles = (int32_t)(t1 - t0);  // < 2^31 tiles per CTA
  for (int32_t i = 0; i < ntiles; ++i, (++k == p.tpf) ? (k = 0, ++item) : 0) {
    if (k == 0 || i == 0) {  // a new frame (item changes exactly when k wraps)
      if (cur >= 0) flush(cur);
      cur = item;
      if constexpr (MODE == 2 || MODE == 3) {
        if (item >= p.n_halo)
          rg.ds_frame = ds_frame_base(p.ds_out, item - p.n_halo, p.height / 2, rg.ow3, rg.pitch, p.ds_cols);
      }
    }
    const uint64_t off = (uint64_t)k * p.tile;
    const uint32_t len = (uint32_t)((uint64_t)p.F - off < p.tile ? (uint64_t)p.F - off : p.tile);
    mbar_wait(full0 + 8 * s, ph);
    if constexpr (kTmaStore) {
      if (i >= L.stages) mbar_wait(sfree0 + 8 * s, ph ^ 1);  // the slot's previous output is stored
    }
    const uint32_t slot = slot_of(s);

    if constexpr (MODE == 2 || MODE == 3) {
      // fused: rows [k*R, k*R + rows) of the frame; unit pairs over row pairs.
      // Per-frame constants (rg.*) are hoisted out of the tile loop; rows of the last
      // tile and the frame's output base are precomputed, so a tile costs no division.
      const uint32_t rows = (k == p.tpf - 1) ? rg.last_rows : (uint32_t)p.rows_per_tile;
      const uint32_t npairs = (rows / 2) * rg.upr;
      uint8_t* dsf = (item >= p.n_halo) ? rg.ds_frame + (int64_t)k * rg.tile_out : nullptr;
      // unit pair u -> (row pair rp, column unit xc), carried from the previous tile and
      // advanced incrementally (no division)
      uint32_t u = ucur, rp = rpc, xc = xcc;
      for (; u < npairs; u += kConsThreads, rp += rg.dq, xc += rg.dr, (xc >= rg.upr) ? (xc -= rg.upr, ++rp) : 0) {
        const uint32_t a = slot + rp * 2u * rg.rowb + xc * 48u;
        uint32_t wt[12], wb[12], o[6];
        load_unit(a, wt);
        load_unit(a + rg.rowb, wb);
        if constexpr (MODE == 2) {
          hist_unit_pair<LOGB, VAR & (64 | 128)>(wt, lane4, lane4h);
          hist_unit_pair<LOGB, VAR & (64 | 128)>(wb, lane4, lane4h);
        }
        if (dsf) {
          ds_unit_v<(VAR & 16) ? 2 : ((VAR >> 2) & 1)>(wt, wb, o);
          if constexpr (kTmaStore) {  // staged in the slot's output area; the producer bulk-stores the tile
            const uint32_t d = slot + rg.in_bytes + rp * rg.ow3s + xc * 24u;
            sts64(d, o[0], o[1]);
            sts64(d + 8, o[2], o[3]);
            sts64(d + 16, o[4], o[5]);
          } else {
            st_global_24(dsf + (int64_t)rp * rg.pitch + xc * 24, o);
          }
        }
      }
      ucur = u - npairs;  // same column unit, rows / 2 row pairs earlier in the next tile
      rpc = rp - rows / 2;
      xcc = xc;
      if (MODE == 2 && (rows & 1)) {  // odd last row of an odd-height frame: histogram only
        for (uint32_t v = (uint32_t)ctid; v < rg.upr; v += kConsThreads) {
          uint32_t w[12];
          load_unit(slot + (rows - 1) * rg.rowb + v * 48u, w);
          hist_unit_pair<LOGB, VAR & (64 | 128)>(w, lane4, lane4h);
        }
      }
    } else {
      const uint32_t nunits = len / 48u;
      uint32_t u = ucur;
      for (; u < nunits; u += kConsThreads) {
        uint32_t w[12];
        load_unit(slot + u * 48u, w);
        if constexpr (MODE == 0) {
          hist_unit_pair<LOGB, VAR>(w, lane4);
        } else if constexpr (MODE == 5) {
          // north_star K2a: per-warp bins, peers found with __match_any_sync, one leader
          // atomic of popc(peers) per peer group
          const uint32_t am = __activemask();
          const uint32_t lt = (1u << lane) - 1u;
          uint32_t* wb = reinterpret_cast<uint32_t*>(smem + (L.table - base)) + (uint32_t)warp * 3u * BP;
#pragma unroll
          for (int j = 0; j < 48; ++j) {
            const uint32_t v = (w[j >> 2] >> (8 * (j & 3))) & 0xFFu;
            const uint32_t key = (uint32_t)(j % 3) * BP + (v >> (8 - LOGB));
            const uint32_t peers = __match_any_sync(am, key);
            if ((peers & lt) == 0) atomicAdd(wb + key, (uint32_t)__popc(peers));
          }
        } else if constexpr (MODE == 4) {
          hist_unit_single<LOGB, kPrmt256>(w, lane4);
        } else {
          const uint32_t Bu = (uint32_t)B;
#pragma unroll
          for (int j = 0; j < 48; ++j) {
            const uint32_t v = (w[j >> 2] >> (8 * (j & 3))) & 0xFFu;
            const uint32_t bin = (v * Bu) >> 8;
            red_shared_add(lane4 + (((uint32_t)(j % 3) * Bu + bin) << 7), 1u);
          }
        }
      }
      // tail bytes (frame size not a multiple of 48): direct global counts
      const uint32_t rem = len - nunits * 48u;
      if ((uint32_t)ctid < rem) {
        const uint32_t j = nunits * 48u + (uint32_t)ctid;
        uint32_t v;
        asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(slot + j));
        const uint32_t bin = (v * (uint32_t)B) >> 8;
        emit(item, (int)((j % 3) * B + bin), 1u);
      }
      ucur = u - nunits;
    }
    if constexpr (kTmaStore) fence_proxy_async_smem();  // staged output visible to the bulk store
    __syncwarp();
    if (lane == 0) mbar_arrive(empty0 + 8 * s);
    if (++s == L.stages) { s = 0; ph ^= 1; }
  }
  if (cur >= 0) flush(cur);
}

// ---------------------------------------------------------------------------
// K3: shot-diff. One warp per position.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) shotdiff_kernel(const uint32_t* __restrict__ hist,
                                                        const uint32_t* __restrict__ halo,
                                                        const uint8_t* __restrict__ seg, int64_t n, int32_t bins,
                                                        uint32_t* __restrict__ diff) {
  const int64_t pos = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (pos >= n) return;
  const int K = 3 * bins;
  uint32_t s = 0;
  if (!seg[pos]) {
    const uint32_t* cur = hist + pos * K;
    const uint32_t* prev = pos == 0 ? halo : cur - K;
    for (int i = lane; i < K; i += 32) {
      const uint32_t a = cur[i], b = prev[i];
      s += a > b ? a - b : b - a;
    }
  }
  s = __reduce_add_sync(0xFFFFFFFFu, s);
  if (lane == 0) diff[pos] = s;
}

// K3e: D[j] = sum |H[a_j] - H[b_j]| over explicit row pairs (NEXT N2, fig:sampling-e):
// the histogram column covers the required set R; a_j / b_j index the sampled row
// and its stencil neighbour in R.
__global__ void __launch_bounds__(256) diff_pairs_kernel(const uint32_t* __restrict__ hist,
                                                          const int64_t* __restrict__ ia,
                                                          const int64_t* __restrict__ ib, int64_t n, int32_t bins,
                                                          uint32_t* __restrict__ diff) {
  const int64_t pos = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (pos >= n) return;
  const int K = 3 * bins;
  const uint32_t* x = hist + ia[pos] * K;
  const uint32_t* y = hist + ib[pos] * K;
  uint32_t s = 0;
  for (int i = lane; i < K; i += 32) {
    const uint32_t a = x[i], b = y[i];
    s += a > b ? a - b : b - a;
  }
  s = __reduce_add_sync(0xFFFFFFFFu, s);
  if (lane == 0) diff[pos] = s;
}

// ---------------------------------------------------------------------------
// K4: downsample. Vectorised path (W % 16 == 0): one thread per 8 output pixels
// from two 48-byte LDG.128 x3 loads; generic path: one thread per output byte.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void ldg_unit(const uint8_t* p, uint32_t* w) {
  const uint4* q = reinterpret_cast<const uint4*>(p);
  const uint4 v0 = __ldcs(q), v1 = __ldcs(q + 1), v2 = __ldcs(q + 2);
  w[0] = v0.x; w[1] = v0.y; w[2] = v0.z; w[3] = v0.w;
  w[4] = v1.x; w[5] = v1.y; w[6] = v1.z; w[7] = v1.w;
  w[8] = v2.x; w[9] = v2.y; w[10] = v2.z; w[11] = v2.w;
}

// one block per (output row y = blockIdx.x, frame = item0 + blockIdx.y); threads over 48-byte column units
__global__ void __launch_bounds__(128) downsample_vec_kernel(FrameSrc src, int64_t item0, int32_t width,
                                                             int32_t height, uint8_t* __restrict__ out,
                                                             int64_t pitch, int32_t cols) {
  const uint32_t upr = (uint32_t)width / 16u, oh = (uint32_t)height / 2u;
  const uint32_t y = blockIdx.x;
  const int64_t item = item0 + blockIdx.y;
  const uint32_t rowb = (uint32_t)width * 3u, ow3 = (uint32_t)(width / 2) * 3u;
  const uint8_t* f = reinterpret_cast<const uint8_t*>(frame_addr(src, item)) + (size_t)(2u * y) * rowb;
  uint8_t* o = ds_frame_base(out, item, oh, ow3, pitch, cols) + (int64_t)y * pitch;
  for (uint32_t xc = threadIdx.x; xc < upr; xc += blockDim.x) {
    uint32_t wt[12], wb[12], r[6];
    ldg_unit(f + xc * 48u, wt);
    ldg_unit(f + rowb + xc * 48u, wb);
    ds_unit(wt, wb, r);
    st_global_24(o + xc * 24u, r);
  }
}

__global__ void __launch_bounds__(256) downsample_generic_kernel(FrameSrc src, int64_t n, int32_t width,
                                                                 int32_t height, uint8_t* __restrict__ out,
                                                                 int64_t pitch, int32_t cols) {
  const int32_t ow = width / 2, oh = height / 2;
  const int64_t per = (int64_t)ow * oh * 3;
  const int64_t total = per * n;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t item = g / per;
    const int64_t o = g - item * per;
    const int64_t pix = o / 3;
    const int c = (int)(o - pix * 3);
    const int64_t y = pix / ow, x = pix - y * ow;
    const uint8_t* f = reinterpret_cast<const uint8_t*>(frame_addr(src, item));
    const int64_t i00 = ((2 * y) * width + 2 * x) * 3 + c;
    const uint32_t s = (uint32_t)f[i00] + f[i00 + 3] + f[i00 + (int64_t)width * 3] + f[i00 + (int64_t)width * 3 + 3];
    ds_frame_base(out, item, oh, (int64_t)ow * 3, pitch, cols)[y * pitch + x * 3 + c] = (uint8_t)((s + 2u) >> 2);
  }
}

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------
static int g_num_sms = 0;
static int g_smem_optin = 0;
static int g_smem_reserved = 0;  // shared memory the system reserves per block (dynamic smem starts after it)
static int g_grid_cap = 0;       // SCN_GRID=G: persistent CTAs (default: one per SM; measurement knob)

// Queried once per process (all GPUs of a B200 box are identical) and published together:
// concurrent first calls from several host threads serialize on the mutex, and a failed
// query (e.g. no device yet) is retried by the next call.
static std::mutex g_props_mu;
static std::atomic<bool> g_props_ok{false};
static cudaError_t device_props() {
  if (g_props_ok.load(std::memory_order_acquire)) return cudaSuccess;
  std::lock_guard<std::mutex> lk(g_props_mu);
  if (g_props_ok.load(std::memory_order_relaxed)) return cudaSuccess;
  int dev = 0, sms = 0, optin = 0, reserved = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&reserved, cudaDevAttrReservedSharedMemoryPerBlock, dev);
  if (e != cudaSuccess) return e;
  g_num_sms = sms;
  g_smem_optin = optin;
  g_smem_reserved = reserved;
  g_props_ok.store(true, std::memory_order_release);
  return cudaSuccess;
}

static int log2_exact(int b) {
  for (int l = 0; l <= 4; ++l)
    if ((1 << l) == b) return l;
  return -1;
}

const char* hist_variant_name(int32_t bins) {
  if (log2_exact(bins) >= 0) return "tma_pair_lane_private";
  if (bins >= 32 && (bins & (bins - 1)) == 0) return "tma_single_shift_lane_private";
  return "tma_single_lane_private";
}

template <int MODE, int LOGB, int NW = kDefaultConsWarps, int VAR = 0>
static cudaError_t launch_tma(HistParams p, cudaStream_t st) {
  auto fn = hist_tma_kernel<MODE, LOGB, NW, VAR>;
  static unsigned configured = 0;  // per instantiation: bit d = smem opt-in done on device d
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const unsigned bit = 1u << (dev & 31);
  if (!(__atomic_load_n(&configured, __ATOMIC_ACQUIRE) & bit)) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem_bytes);
    if (e != cudaSuccess) return e;
    __atomic_fetch_or(&configured, bit, __ATOMIC_RELEASE);
  }
  int grid = g_num_sms;
  if (g_grid_cap > 0 && g_grid_cap < grid) grid = g_grid_cap;  // SCN_GRID (measurement knob)
  if (p.total_tiles < grid) grid = (int)p.total_tiles;
  if (grid < 1) return cudaSuccess;
  fn<<<grid, NW * 32 + 32, p.smem_bytes, st>>>(p);
  return cudaGetLastError();
}

// Tuning knobs (env, read once; defaults are the measured best):
// SCN_HIST_TILE tile bytes of the B = 16 kernel (multiple of 48), SCN_FUSED_TILE
// target bytes of the row-pair tiles, SCN_HIST_VAR=8 the previous adjacent-pixel
// pairing, SCN_HIST_VAR=64 the pre-PRMT table layout, SCN_HIST_SINGLE=1 one key per byte at B = 16, SCN_DS_VAR=0 the bytewise
// SWAR downsample, SCN_DS_IMPL=1 the LDG downsample kernel, SCN_HIST_WARPS (8/12/16)
// and SCN_FUSED_WARPS (8/12/16) consumer warps. (Measured and removed: 20/24 consumer
// warps, right shifts as mul.hi, two units per loop iteration.)
static int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v && *v ? atoi(v) : dflt;
}
static int g_tune_warps = -1;
static uint32_t g_tune_tile = 0;
static uint32_t g_fused_tile = 0;  // SCN_FUSED_TILE: target bytes per row-pair tile (fused)
static uint32_t g_ds_tile = 0;     // SCN_DS_TILE: target bytes per row-pair tile (downsample only)
static uint32_t g_fused_tile_env = 0, g_ds_tile_env = 0;  // explicit overrides (0 = rows_per_tile rule)
static int g_tune_var = 0;  // SCN_HIST_VAR: 8 = adjacent-pixel pairing
static int g_ds_var = 1;    // SCN_DS_VAR: 0 = SWAR hi/lo + funnel, 1 = dp4a (measured faster)
static int g_ds_impl = 0;   // SCN_DS_IMPL: 0 = TMA ring (MODE 3), 1 = LDG kernel
static int g_hist_single = 0;  // SCN_HIST_SINGLE: B = 16 with one key per byte instead of pair keys
static int g_fused_warps = 8;  // SCN_FUSED_WARPS: consumer warps of the fused / ds-only kernels (measured best: 8)
static int g_tma_hint = 0;     // SCN_TMA_HINT=1: L2 evict_first policy on the frame loads
static int g_l2_prefetch = -1;  // SCN_L2_PREFETCH=P: bulk L2 prefetch P tiles ahead (default: fused 1, else 0)
static int g_hist_match = 0;   // SCN_HIST_IMPL=match: the north_star's per-warp bins + __match_any_sync (K2a)
static int g_ds_store = 0;     // SCN_DS_STORE=1: downsample output by producer TMA bulk stores (measured slower)
static int g_fused_split = 1;  // SCN_FUSED_SPLIT=0: the fused kernel's previous 96 KB table layout
static int g_flush_zero = 0;   // SCN_FLUSH_ZERO=1: the previous flush that re-zeroes the table (A/B)
static int g_max_stages = 0;   // SCN_MAX_STAGES=S: ring-depth cap (default 3; measurement knob)
static std::once_flag g_tuning_once;
static void read_tuning_once() {
  g_tune_warps = env_int("SCN_HIST_WARPS", kDefaultConsWarps);
  int t = env_int("SCN_HIST_TILE", (int)kTile);
  if (t < 48 || t % 48 != 0 || t > 65536) t = (int)kTile;
  g_tune_tile = (uint32_t)t;
  int f = env_int("SCN_FUSED_TILE", (int)kFusedTile);
  if (f < 96 || f > 65536) f = (int)kTile;
  g_fused_tile = (uint32_t)f;
  g_fused_tile_env = getenv("SCN_FUSED_TILE") ? g_fused_tile : 0;
  int dt = env_int("SCN_DS_TILE", (int)kDsTile);
  if (dt < 96 || dt > 65536) dt = (int)kDsTile;
  g_ds_tile = (uint32_t)dt;
  g_ds_tile_env = getenv("SCN_DS_TILE") ? g_ds_tile : 0;
  g_tune_var = env_int("SCN_HIST_VAR", 0);
  g_ds_var = env_int("SCN_DS_VAR", 1);
  g_ds_impl = env_int("SCN_DS_IMPL", 0);
  g_hist_single = env_int("SCN_HIST_SINGLE", 0);
  g_fused_warps = env_int("SCN_FUSED_WARPS", 8);
  g_tma_hint = env_int("SCN_TMA_HINT", 0);
  g_l2_prefetch = env_int("SCN_L2_PREFETCH", -1);
  g_ds_store = env_int("SCN_DS_STORE", 0);
  g_fused_split = env_int("SCN_FUSED_SPLIT", 1);
  g_flush_zero = env_int("SCN_FLUSH_ZERO", 0);
  g_max_stages = env_int("SCN_MAX_STAGES", 0);
  g_grid_cap = env_int("SCN_GRID", 0);
  {
    const char* impl = getenv("SCN_HIST_IMPL");
    g_hist_match = impl && strcmp(impl, "match") == 0;
  }
}
static void read_tuning() { std::call_once(g_tuning_once, read_tuning_once); }

// Rows per row-pair tile (measured): the largest even row count whose tiles
// give `stages` ring stages next to a table of table_bytes, unless that is under 4 rows, in
// which case the largest even count that still gives 2 stages (1080p fused: 6 rows x 3
// stages; 4K fused: 4 rows x 2; downsample-only 1080p: 8 rows x 4). An explicit tile size
// from the environment (env_tile > 0) wins.
// With the TMA-store path each slot also holds the tile's output (rows/2 rows of 1.5 W
// bytes), so a row costs rowb + ow3 / 2 bytes of ring.
static int rows_per_tile(int64_t rowb, uint32_t table_bytes, int stages, uint32_t env_tile, bool staged) {
  if (env_tile) return (int)((int64_t)env_tile / rowb) & ~1;
  const int64_t cost = staged ? rowb + rowb / 4 : rowb;  // one ow3 = rowb / 2 output row per row pair
  const int64_t ring = (int64_t)g_smem_optin - (int64_t)kCtrlBytes - (int64_t)table_bytes - 2048 - (staged ? 256 * stages : 0);
  int r = (int)(ring / stages / cost) & ~1;
  if (r < 4) r = (int)(ring / 2 / cost) & ~1;
  return r;
}

// Rows per tile for the split layout (make_layout_split, mirrored here with the dynamic
// smem base = the per-block reserved size): the largest even row count (tile <= 64 KB)
// whose tiles give >= 3 ring stages over the two ring segments; 0 if none. The device
// recomputes the same layout and traps on < 2 stages.
static int rows_per_tile_split(int64_t rowb, uint32_t env_tile) {
  const uint32_t base = (uint32_t)g_smem_reserved, end = base + (uint32_t)g_smem_optin;
  const uint32_t block = (base + kCtrlBytes + kSplitTab2 + 65535u) & ~65535u;
  const uint32_t tab2 = block - kSplitTab2, ring = (base + kCtrlBytes + 127u) & ~127u, hi = block + 65536u;
  if (hi > end) return 0;
  auto stages = [&](int r) {
    const uint32_t tile = (uint32_t)(r * rowb), stride = (tile + 127u) & ~127u;
    const int lo = tab2 >= ring + tile ? (int)((tab2 - ring - tile) / stride) + 1 : 0;
    const int up = end >= hi + tile ? (int)((end - hi - tile) / stride) + 1 : 0;
    return lo + up;
  };
  if (env_tile) {
    const int r = (int)((int64_t)env_tile / rowb) & ~1;
    return r >= 2 && stages(r) >= 2 ? r : 0;
  }
  for (int r = (int)(65536 / rowb) & ~1; r >= 2; r -= 2)
    if (stages(r) >= 3) return r;
  return 0;
}

// TMA bulk stores of the downsample output need every output row segment 16-byte aligned:
// W % 32 == 0 (rows of 1.5 W bytes, segments of 24-byte units starting at even units),
// a 16-byte multiple row pitch and a 16-byte aligned output base.
static bool ds_store_ok(int32_t width, int64_t pitch, const uint8_t* out) {
  return g_ds_store && width % 32 == 0 && pitch % 16 == 0 && ((uintptr_t)out & 15u) == 0;
}

static HistParams base_params(const HistJob& j) {
  HistParams p{};
  p.src = j.src;
  p.n_items = j.n_items;
  p.n_halo = j.n_halo;
  p.out = j.out;
  p.halo_out = j.halo_out;
  p.ds_out = j.ds_out;
  p.ds_pitch = j.ds_pitch > 0 ? j.ds_pitch : (int64_t)(j.width / 2) * 3;
  p.ds_cols = j.ds_cols;
  p.F = (int64_t)j.width * j.height * 3;
  p.width = j.width;
  p.height = j.height;
  p.bins = j.bins;
  p.smem_bytes = (uint32_t)g_smem_optin;
  read_tuning();
  p.l2_hint = g_tma_hint;
  p.l2_prefetch = g_l2_prefetch > 0 ? g_l2_prefetch : 0;
  // at most three ring stages: deeper rings stream slower on B200 (pure TMA reads, the
  // downsample-only kernel, and the kernels whose smaller tables leave room for 4-8 stages:
  // bins 8 / 32 / 64 / 128 run +5-9 % with 3; profiles/r01_tune.jsonl, SCN_MAX_STAGES A/B)
  p.max_stages = g_max_stages >= 2 ? g_max_stages : 3;
  p.n_dest = j.n_dest;
  for (int g = 0; g < kMaxDest; ++g) p.dest[g] = j.dest[g];
  return p;
}

cudaError_t launch_histogram(const HistJob& j, cudaStream_t st, int* launches) {
  cudaError_t e = device_props();
  if (e != cudaSuccess) return e;
  if (j.n_items <= 0) return cudaSuccess;
  HistParams p = base_params(j);
  p.ds_out = nullptr;
  read_tuning();
  p.tile = (j.bins == 16) ? g_tune_tile : kTile;
  p.rows_per_tile = 0;
  p.tpf = (int32_t)((p.F + p.tile - 1) / p.tile);
  p.total_tiles = p.n_items * p.tpf;
  const int lb = log2_exact(j.bins);
  *launches += 1;
  if (lb >= 0) {
    const int Bp = 1 << lb;
    p.table_bytes = 3u * Bp * Bp * 128u;
    p.table_align = lb == 4 ? 65536u : (uint32_t)Bp * Bp * 128u;  // B = 16: the PRMT layout's 64 KB block
    switch (lb) {
      case 0: return launch_tma<0, 0>(p, st);
      case 1: return launch_tma<0, 1>(p, st);
      case 2: return launch_tma<0, 2>(p, st);
      case 3: return launch_tma<0, 3>(p, st);
      default:
        if (g_hist_match) {  // north_star K2a: per-warp bins + __match_any_sync (SCN_HIST_IMPL=match)
          p.table_bytes = (uint32_t)kDefaultConsWarps * 3u * 16u * 4u;
          p.table_align = 128u;
          return launch_tma<5, 4>(p, st);
        }
        if (g_hist_single) {  // single shifted key per byte, 6 KB table (SCN_HIST_SINGLE=1)
          p.table_bytes = 3u * 16u * 128u;
          p.table_align = 16u * 128u;
          return launch_tma<4, 4>(p, st);
        }
        if (g_tune_var == 8) return launch_tma<0, 4, 16, 8>(p, st);
        if (g_tune_var == 64) return launch_tma<0, 4, 16, 64>(p, st);  // previous table layout (A/B)
        if (g_tune_warps == 12) return launch_tma<0, 4, 12>(p, st);
        if (g_tune_warps == 8) return launch_tma<0, 4, 8>(p, st);
        if (g_flush_zero) return launch_tma<0, 4, 16, 256>(p, st);
        return launch_tma<0, 4>(p, st);
    }
  }
  if (j.bins >= 32 && (j.bins & (j.bins - 1)) == 0) {  // NEXT N4: B = 32..256, one shifted key per byte
    p.table_bytes = 3u * (uint32_t)j.bins * 128u;
    p.table_align = (uint32_t)j.bins * 128u;
    switch (j.bins) {
      case 32: return launch_tma<4, 5>(p, st);
      case 64: return launch_tma<4, 6>(p, st);
      case 128: return launch_tma<4, 7>(p, st);
      default:
        if (g_tune_var == 64) return launch_tma<4, 8, 16, 64>(p, st);  // previous shifted-key layout (A/B)
        p.table_align = 65536u;  // the PRMT layout's 64 KB block
        return launch_tma<4, 8>(p, st);
    }
  }
  p.table_bytes = 3u * (uint32_t)j.bins * 128u;
  p.table_align = 128u;
  return launch_tma<1, 0>(p, st);
}

static cudaError_t launch_ds_tma(const FrameSrc& src, int64_t n, int32_t width, int32_t height, uint8_t* out,
                                 cudaStream_t st, int64_t pitch, int32_t cols);

cudaError_t launch_downsample(const FrameSrc& src, int64_t n, int32_t width, int32_t height, uint8_t* out,
                              cudaStream_t st, int* launches, int64_t ds_pitch, int32_t ds_cols, bool allow_vec) {
  const int64_t pitch = ds_pitch > 0 ? ds_pitch : (int64_t)(width / 2) * 3;
  cudaError_t e = device_props();
  if (e != cudaSuccess) return e;
  if (n <= 0 || width < 2 || height < 2) return cudaSuccess;
  read_tuning();
  if (allow_vec && width % 16 == 0 && g_ds_impl == 0 && (int64_t)width * 6 <= 65536) {
    *launches += 1;
    return launch_ds_tma(src, n, width, height, out, st, pitch, ds_cols);
  }
  if (allow_vec && width % 16 == 0) {
    *launches += (int)((n + 65534) / 65535);
    const int threads = width / 16 >= 128 ? 128 : ((width / 16 + 31) / 32) * 32;
    for (int64_t i0 = 0; i0 < n; i0 += 65535) {
      const int64_t cnt = n - i0 < 65535 ? n - i0 : 65535;
      dim3 grid((unsigned)(height / 2), (unsigned)cnt);
      downsample_vec_kernel<<<grid, threads, 0, st>>>(src, i0, width, height, out, pitch, ds_cols);
    }
  } else {
    *launches += 1;
    const int grid = g_num_sms * 8;
    downsample_generic_kernel<<<grid, 256, 0, st>>>(src, n, width, height, out, pitch, ds_cols);
  }
  return cudaGetLastError();
}

cudaError_t launch_hist_downsample(const HistJob& j, cudaStream_t st, int* launches) {
  cudaError_t e = device_props();
  if (e != cudaSuccess) return e;
  if (j.n_items <= 0) return cudaSuccess;
  const int lb = log2_exact(j.bins);
  const int64_t rowb = (int64_t)j.width * 3;
  read_tuning();
  const int64_t pitch = j.ds_pitch > 0 ? j.ds_pitch : (int64_t)(j.width / 2) * 3;
  const bool tstore = lb == 4 && g_fused_warps == 8 && g_ds_var == 1 && ds_store_ok(j.width, pitch, j.ds_out);
  // split layout (default at B = 16 with the 8-warp dp4a kernel): more ring for the same table
  const int rsplit = (lb == 4 && !tstore && g_fused_split && g_ds_var == 1 && g_tune_var == 0 &&
                      (g_fused_warps == 8 || g_fused_warps == 12 || g_fused_warps == 16))
                         ? rows_per_tile_split(rowb, g_fused_tile_env) : 0;
  int rpt = rsplit ? rsplit : rows_per_tile(rowb, 3u * 256u * 128u, 3, g_fused_tile_env, tstore);
  if (rpt > j.height) rpt = j.height + (j.height & 1);  // whole frame in one tile
  const bool fused = lb >= 0 && j.width % 16 == 0 && rpt >= 2 && j.n_halo == 0;
  if (!fused) {
    HistJob h = j;
    h.ds_out = nullptr;
    e = launch_histogram(h, st, launches);
    if (e != cudaSuccess) return e;
    FrameSrc src = j.src;
    return launch_downsample(src, j.n_items, j.width, j.height, j.ds_out, st, launches, j.ds_pitch, j.ds_cols);
  }
  HistParams p = base_params(j);
  // one tile of L2 bulk prefetch ahead of the ring (measured: C4 +0.8 %, C5 +1.7 %; it
  // slows the read-only histogram kernel, which keeps 0)
  p.l2_prefetch = g_l2_prefetch >= 0 ? g_l2_prefetch : 1;
  p.rows_per_tile = rpt;
  p.tile = (uint32_t)(rpt * rowb);
  p.tpf = (j.height + rpt - 1) / rpt;
  p.total_tiles = p.n_items * p.tpf;
  const int Bp = 1 << lb;
  p.table_bytes = 3u * Bp * Bp * 128u;
  p.table_align = lb == 4 ? 65536u : (uint32_t)Bp * Bp * 128u;  // B = 16: the PRMT layout's 64 KB block
  *launches += 1;
  switch (lb) {
    case 0: return launch_tma<2, 0>(p, st);
    case 1: return launch_tma<2, 1>(p, st);
    case 2: return launch_tma<2, 2>(p, st);
    case 3: return launch_tma<2, 3>(p, st);
    default:
      if (tstore) {
        p.stage_bytes = (uint32_t)(rpt / 2) * (uint32_t)(j.width / 2) * 3u;
        return launch_tma<2, 4, 8, 4 | 32>(p, st);
      }
      if (rsplit) {
        p.table_bytes = kSplitTab2 + 65536u;  // tab2 + the channel 0/1 block, zeroed as one range
        if (g_flush_zero && g_fused_warps == 8) return launch_tma<2, 4, 8, 4 | 128 | 256>(p, st);
        if (g_fused_warps == 12) return launch_tma<2, 4, 12, 4 | 128>(p, st);
        if (g_fused_warps == 16) return launch_tma<2, 4, 16, 4 | 128>(p, st);
        return launch_tma<2, 4, 8, 4 | 128>(p, st);
      }
      if (g_fused_warps == 8 && g_ds_var == 2) return launch_tma<2, 4, 8, 16>(p, st);
      if (g_fused_warps == 8 && g_ds_var == 1 && g_tune_var == 64) return launch_tma<2, 4, 8, 4 | 64>(p, st);
      if (g_fused_warps == 8 && g_ds_var == 1) return launch_tma<2, 4, 8, 4>(p, st);
      if (g_fused_warps == 12 && g_ds_var == 1) return launch_tma<2, 4, 12, 4>(p, st);
      if (g_ds_var == 1) return launch_tma<2, 4, kDefaultConsWarps, 4>(p, st);
      return launch_tma<2, 4>(p, st);
  }
}

// downsample-only TMA ring (MODE 3): same row-pair tiles, no table
static cudaError_t launch_ds_tma(const FrameSrc& src, int64_t n, int32_t width, int32_t height, uint8_t* out,
                                 cudaStream_t st, int64_t pitch, int32_t cols) {
  read_tuning();
  HistJob j{};
  j.ds_pitch = pitch;
  j.ds_cols = cols;
  j.src = src;
  j.n_items = n;
  j.ds_out = out;
  j.width = width;
  j.height = height;
  j.bins = 16;
  HistParams p = base_params(j);
  const int64_t rowb = (int64_t)width * 3;
  const bool tstore = g_fused_warps == 8 && g_ds_var == 1 && ds_store_ok(width, pitch, out);
  int rpt = rows_per_tile(rowb, 0u, 4, g_ds_tile_env, tstore);
  if (rpt < 2) rpt = 2;
  if (rpt > height) rpt = height + (height & 1);
  p.rows_per_tile = rpt;
  p.tile = (uint32_t)(rpt * rowb);
  p.tpf = (height + rpt - 1) / rpt;
  p.total_tiles = n * p.tpf;
  p.table_bytes = 0;
  p.table_align = 128;
  if (tstore) {
    p.stage_bytes = (uint32_t)(rpt / 2) * (uint32_t)(width / 2) * 3u;
    return launch_tma<3, 4, 8, 4 | 32>(p, st);
  }
  if (g_ds_var == 2 && g_fused_warps == 8) return launch_tma<3, 4, 8, 16>(p, st);
  if (g_ds_var == 1 && g_fused_warps == 8) return launch_tma<3, 4, 8, 4>(p, st);
  if (g_ds_var == 1) return launch_tma<3, 4, kDefaultConsWarps, 4>(p, st);
  return launch_tma<3, 4>(p, st);
}

cudaError_t launch_shotdiff(const uint32_t* hist, const uint32_t* halo_row, const uint8_t* seg, int64_t n,
                            int32_t bins, uint32_t* diff, cudaStream_t st, int* launches) {
  if (n <= 0) return cudaSuccess;
  *launches += 1;
  const int64_t blocks = (n + 7) / 8;
  shotdiff_kernel<<<(unsigned)blocks, 256, 0, st>>>(hist, halo_row, seg, n, bins, diff);
  return cudaGetLastError();
}

}  // namespace scn

namespace scn {
cudaError_t launch_diff_pairs(const uint32_t* hist, const int64_t* a, const int64_t* b, int64_t n, int32_t bins,
                              uint32_t* diff, cudaStream_t st, int* launches) {
  if (n <= 0) return cudaSuccess;
  *launches += 1;
  diff_pairs_kernel<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(hist, a, b, n, bins, diff);
  return cudaGetLastError();
}
}  // namespace scn

namespace scn {
// NEXT N3: adaptive shot detector, a bounded-state op with warmup W.
// State = window of the last W_eff = min(W, q - table start) shot-diffs; the
// shard's first W positions before q0 are warmup: read, never written.
__global__ void __launch_bounds__(256) adaptive_cuts_kernel(const uint32_t* __restrict__ diff,
                                                             const uint8_t* __restrict__ seg, int64_t q0, int64_t n,
                                                             int32_t warmup, uint32_t k_num, uint32_t k_den,
                                                             uint32_t floor_, uint8_t* __restrict__ cut) {
  const int64_t q = q0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  uint64_t sum = 0;
  int32_t weff = 0;
  for (int32_t i = 1; i <= warmup; ++i) {
    if (seg[q - i + 1]) break;  // the window never crosses the table's first position
    sum += diff[q - i];
    weff = i;
  }
  const uint64_t lhs = (uint64_t)diff[q] * (uint64_t)weff * k_den;
  const uint64_t rhs = (uint64_t)k_num * sum + (uint64_t)floor_ * (uint64_t)weff * k_den;
  cut[q - q0] = (weff > 0 && lhs > rhs) ? 1 : 0;
}

cudaError_t launch_adaptive_cuts(const uint32_t* diff, const uint8_t* seg, int64_t q0, int64_t n, int32_t warmup,
                                 uint32_t k_num, uint32_t k_den, uint32_t floor_, uint8_t* cut, cudaStream_t st,
                                 int* launches) {
  const int64_t cnt = n - q0;
  if (cnt <= 0) return cudaSuccess;
  *launches += 1;
  adaptive_cuts_kernel<<<(unsigned)((cnt + 255) / 256), 256, 0, st>>>(diff, seg, q0, n, warmup, k_num, k_den, floor_,
                                                                      cut);
  return cudaGetLastError();
}
}  // namespace scn

namespace scn {
__global__ void __launch_bounds__(256) zero_dests_kernel(DestList d, int64_t words) {
  const int g = blockIdx.y;
  uint32_t* q = reinterpret_cast<uint32_t*>(d.p[g]);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < words; i += (int64_t)gridDim.x * blockDim.x)
    q[i] = 0u;
}

cudaError_t launch_zero_dests(const DestList& d, int64_t words, cudaStream_t st, int* launches) {
  if (d.n <= 0 || words <= 0) return cudaSuccess;
  *launches += 1;
  int64_t bx = (words + 255) / 256;
  if (bx > 1024) bx = 1024;
  zero_dests_kernel<<<dim3((unsigned)bx, (unsigned)d.n), 256, 0, st>>>(d, words);
  return cudaGetLastError();
}

// K3 with the fused all-gather: D[p] goes to every destination column
__global__ void __launch_bounds__(256) shotdiff_dests_kernel(const uint32_t* __restrict__ hist,
                                                              const uint32_t* __restrict__ halo,
                                                              const uint8_t* __restrict__ seg, int64_t n,
                                                              int32_t bins, DestList d) {
  const int64_t pos = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (pos >= n) return;
  const int K = 3 * bins;
  uint32_t s = 0;
  if (!seg[pos]) {
    const uint32_t* cur = hist + pos * K;
    const uint32_t* prev = pos == 0 ? halo : cur - K;
    for (int i = lane; i < K; i += 32) {
      const uint32_t a = cur[i], b = prev[i];
      s += a > b ? a - b : b - a;
    }
  }
  s = __reduce_add_sync(0xFFFFFFFFu, s);
  if (lane < d.n) reinterpret_cast<uint32_t*>(d.p[lane])[pos] = s;
}

cudaError_t launch_shotdiff_dests(const uint32_t* hist, const uint32_t* halo_row, const uint8_t* seg, int64_t n,
                                  int32_t bins, const DestList& d, cudaStream_t st, int* launches) {
  if (n <= 0) return cudaSuccess;
  *launches += 1;
  shotdiff_dests_kernel<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(hist, halo_row, seg, n, bins, d);
  return cudaGetLastError();
}
}  // namespace scn
