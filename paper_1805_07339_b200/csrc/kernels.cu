// kernels.cu — sm_100a kernels of the Scanner HIST / shot-diff / downsample
// hot path (arXiv 1805.07339 P:L331 HIST, P:L455 shot boundaries via
// histogram differences over a [-1,0] stencil P:L210, P:L183/P:L335 resize).
//
// One persistent TMA-ring kernel template, hist_tma_kernel<MODE, NW, VAR>, one CTA
// per SM (227 KB smem). Warp NW is the producer: one elected lane streams tiles of
// the sampled frames with 1-D bulk copies (cp.async.bulk -> SASS UBLKCP) into a
// 3-stage shared-memory ring guarded by full/empty mbarriers; warps 0..NW-1 consume.
//
// K1+K2  MODE kPair   (bins B dividing 16; the configs' B = 16). Each consumer thread
//   takes 48-byte units (16 pixels, 3 x LDS.128, channel of byte j = j mod 3) and counts
//   PAIRS of same-channel pixels (p, p+8) — bytes j and j+24, same position in their
//   words, so one SHF + one LOP3 select makes four 8-bit keys (bin16(a) | bin16(b) << 4)
//   at once — into a lane-private table (bank == lane: conflict-free for any content;
//   channels 0/1 share 256-byte key rows so one PRMT turns a key byte into its address):
//   one red.shared.add per pair, 0.5 shared atomics per byte, 75 instructions per 48 B.
//   On a frame change the consumer warps marginalise the table (row sums over lanes,
//   each key's count added to both of its 16-level bins) and merge the frame's 3*B
//   counters with one red.global.add each ("one global merge per block" per frame
//   segment). B = 1, 2, 4, 8 merge 16/B adjacent 16-level bins at that flush:
//   bin_B(v) = (v*B) >> 8 = (v >> 4) >> (4 - log2 B) (reading Q2).
// K2b    MODE kPairB  (B < 16 not dividing 16): the K1 pair keys with B-level fields, the bins of
//   four bytes from two 16-bit-lane IMADs (v*B)>>8: 0.5 shared atomics per byte for every B <= 16.
// K2r    MODE kRaw    (B in [17,256]): one key per byte, the byte value itself
//   (256 lane-private rows per channel, PRMT addresses: byte -> address byte 1). The flush
//   maps value rows to bins, bin = (v*B) >> 8, in shared counters above the table, so any
//   B runs at the 256-bin kernel's rate (no per-byte multiply).
// K2f    MODE kFused  (any B; VAR kVarBins = K2b keys, kVarRaw = raw keys with the bin counters at
//   the top of shared memory; default B dividing 16): K1+K2 with the 2x box downsample fused into the
//   consumer over row-pair tiles (a thread takes two vertically adjacent 48-byte units,
//   histograms both and emits 8 output pixels with dp4a window sums), so each sampled
//   frame is read from HBM once (reading Q12). Split table layout: 3 stages of ~46 KB.
// K4     MODE kDs     the same row-pair ring without the table (downsample only).
//   VAR kVarGen (both row-pair modes): any width and any output alignment — rows are
//   re-aligned in registers after the bulk copy (4 x LDS.128 + 12 funnel shifts per
//   unit), the W mod 16 tail pixels of each row take a bytewise path. Output: the
//   downsample-only kernel stages each tile's output rows in its ring slot and the
//   producer writes them with one TMA bulk store (cp.async.bulk.global.shared::cta);
//   the fused kernel (and montage canvases) write aligned 8-byte words assembled across
//   neighbouring lanes with one shuffle pair. VAR kVarHalf (fused, where it buys a bigger
//   tile): a half-lane 64 KB key block, every key one PRMT.
// K2a    MODE kMatch  the north_star's design, selectable (scn_set_hist_impl): per-warp
//   bins, __match_any_sync peer groups per byte, leader atomicAdd(popc), __reduce_add_sync
//   merge across warps, one global add per key per block.
// K2a'   MODE kMatchPacked  K2a amortised: one __match_any_sync per packed word of four
//   pair keys (8 bytes), so MATCH issues 1/8 as often; per-warp pair-key bins.
// K2j    MODE kJoint (NEXT N4's joint-colour variant): one key per pixel,
//   k = bin(R)*J*J + bin(G)*J + bin(B), J <= 8, into J^3 lane-private 128-byte rows; four bytes
//   are binned per two 16-bit-lane IMADs and a pixel keyed with one IDP.4A.
// K3     shotdiff_kernel: one warp per position, L1 over 3*B (or J^3) counters, __reduce_add_sync.
//
// Why not the north_star's per-warp bins + __match_any_sync aggregation as the default:
// on this B200 MATCH.ANY issues at 0.035 warp-instr/clk/SM (profiles/r01_k0_micro_v2.json),
// i.e. ~1.1 bytes/clk/SM if applied per byte, ~5% of the HBM roofline. DESIGN.md §5.
#include "kernels.h"
#include "ptx.cuh"

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <utility>

namespace scn {

enum : int {
  kModePair = 0, kModeFused = 2, kModeDs = 3, kModeRaw = 4, kModeMatch = 5, kModeMatchPacked = 6, kModeJoint = 7,
  kModePairB = 8
};
constexpr int kVarGen = 1;   // row-pair modes: any width / output alignment
constexpr int kVarHalf = 2;  // fused kVarGen: half-lane 64 KB key block (see pair_key_step)
constexpr int kVarBins = 4;  // fused: pair keys of B-level bins (B < 16 not dividing 16, see K2b)
constexpr int kVarRaw = 8;   // fused: raw byte keys in the half-lane block (B > 16, see K2r)

constexpr int kHistWarps = 16;  // consumer warps of the hist-only kernels (+1 producer warp)
constexpr int kDsWarps = 8;     // consumer warps of the fused / downsample-only kernels
// kVarGen kernels: more warps hide the longer dependency chains of the realigned loads and
// stores (measured, profiles/r02_tune_gen.jsonl: ds-only 1366x768 5.51 / 6.32 / 6.76 TB/s with
// 8 / 12 / 16 warps on the direct cross-lane stores; with the staged bulk stores 12 warps
// are best, profiles/r02_tune_gen2.jsonl: 6.95 / 6.83 / 6.93 for 12 / 16 / 20).
constexpr int kGenDsWarps = 12;
constexpr int kGenFusedWarps = 12;
constexpr int kGenHalfWarps = 16;  // half-lane fused kernel (1366x768: 12 rows x 85 units = 510 unit pairs per tile)
constexpr uint32_t kTile = 43008;  // 896 x 48 bytes: a multiple of 48 (channel phase) and 16 (TMA); 3 stages.
                                   // Measured best of 24,576..64,512 on B200 (profiles/r01_tune.jsonl)
constexpr uint32_t kGenSlack = 64;  // kVarGen slots: 15 B of leading misalignment + 15 B rounding + 16 B overread
constexpr int kMaxStages = 8;
constexpr int kDefaultStages = 3;  // deeper rings stream slower on B200 (DESIGN.md §5 "Ring depth")
constexpr uint32_t kCtrlBytes = 1024;
constexpr uint32_t kRemapBytes = 3u * 256u * 4u;  // kRaw: 3*B bin counters kept above the table
constexpr uint32_t kBarId = 1;  // named barrier among consumer warps
constexpr uint32_t kTab2Bytes = 16384;

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
  int32_t joint;          // kModeJoint: J bins per channel (the output row holds J^3 counters)
  uint32_t tile;          // frame bytes per full tile (row-pair modes: rows_per_tile * W * 3)
  uint32_t slot;          // shared-memory bytes per ring slot (>= tile; + kGenSlack for kVarGen)
  uint32_t out_off;       // kVarGen staged stores: offset of the slot's output stage (0 = direct stores)
  int32_t rows_per_tile;  // row-pair modes: rows per tile (even); 0 otherwise
  int32_t tpf;            // tiles per frame
  int64_t total_tiles;
  uint32_t smem_bytes;
  uint32_t table_bytes;
  uint32_t table_align;
  int32_t l2_prefetch;  // > 0: the producer bulk-prefetches tile t + l2_prefetch into L2
  int32_t max_stages;   // cap on the ring depth
  uint32_t prod_sleep;  // > 0: the producer waits for a free slot with this suspend-time hint (ns)
  int32_t n_dest;       // > 0: results go to every dest[g] (fused all-gather over peer memory)
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
  __device__ __forceinline__ uint32_t slot(int s) const {
    return s < n_lo ? ring + (uint32_t)s * stride : ring_hi + (uint32_t)(s - n_lo) * stride;
  }
};

// Shared-memory layout: 1 KB control block at the bottom, the lane-private table at the
// highest table_align-aligned address that leaves `above` bytes over it (so bin fields can
// be OR-ed into its address), and one contiguous ring of tile slots in between.
__device__ __forceinline__ Layout make_layout(uint32_t base, uint32_t smem_bytes, uint32_t slot, uint32_t tb_bytes,
                                              uint32_t tb_align, uint32_t above) {
  Layout L;
  L.ctrl = base;
  const uint32_t end = base + smem_bytes;
  L.table = (end - tb_bytes - above) & ~(tb_align - 1);
  L.ring = (base + kCtrlBytes + 127) & ~127u;
  L.stride = (slot + 127) & ~127u;
  L.stages = L.table >= L.ring + slot ? (int)((L.table - L.ring - slot) / L.stride) + 1 : 0;
  if (L.stages > kMaxStages) L.stages = kMaxStages;
  if (L.table < base + kCtrlBytes) L.stages = 0;
  L.n_lo = L.stages;
  return L;
}

// Split layout of the fused hist + downsample kernel: the 64 KB PRMT block of channels
// 0/1 at the first 64 KB boundary above the control block, channel 2's pair keys in 16 KB
// right below it as tab2[key][lane / 2] (64-byte rows of 16 counters shared by lanes 2l,
// 2l+1), and ring slots both below tab2 and above the block. Against a 96 KB table this
// frees 16 KB and the 64 KB alignment waste, so 4K row-pair tiles get 3 stages instead of
// 2 (1080p: 8-row tiles instead of 6). Lanes 2l and 2l+1 hit the same bank only when their
// channel-2 keys differ with equal parity (a 2-way conflict); equal keys are one address.
__device__ __forceinline__ Layout make_layout_split(uint32_t base, uint32_t smem_bytes, uint32_t slot) {
  Layout L;
  L.ctrl = base;
  const uint32_t end = base + smem_bytes;
  const uint32_t block = (base + kCtrlBytes + kTab2Bytes + 65535u) & ~65535u;
  L.table = block - kTab2Bytes;
  L.ring = (base + kCtrlBytes + 127) & ~127u;
  L.stride = (slot + 127) & ~127u;
  L.ring_hi = block + 65536u;
  const int lo = L.table >= L.ring + slot ? (int)((L.table - L.ring - slot) / L.stride) + 1 : 0;
  const int hi = end >= L.ring_hi + slot ? (int)((end - L.ring_hi - slot) / L.stride) + 1 : 0;
  L.stages = lo + hi > kMaxStages ? kMaxStages : lo + hi;
  L.n_lo = lo < L.stages ? lo : L.stages;
  if (L.ring_hi > end) L.stages = 0;
  return L;
}

// Half-lane layout of the realigning fused kernel: the 64 KB key block at the first 64 KB
// boundary above the control block, ring slots below and above it.
__device__ __forceinline__ Layout make_layout_half(uint32_t base, uint32_t smem_bytes, uint32_t slot) {
  Layout L;
  L.ctrl = base;
  const uint32_t end = base + smem_bytes;
  L.table = (base + kCtrlBytes + 65535u) & ~65535u;
  L.ring = (base + kCtrlBytes + 127) & ~127u;
  L.stride = (slot + 127) & ~127u;
  L.ring_hi = L.table + 65536u;
  const int lo = L.table >= L.ring + slot ? (int)((L.table - L.ring - slot) / L.stride) + 1 : 0;
  const int hi = end >= L.ring_hi + slot ? (int)((end - L.ring_hi - slot) / L.stride) + 1 : 0;
  L.stages = lo + hi > kMaxStages ? kMaxStages : lo + hi;
  L.n_lo = lo < L.stages ? lo : L.stages;
  if (L.ring_hi > end) L.stages = 0;
  return L;
}

template <int OFF>
__device__ __forceinline__ void red_shared_add_off(uint32_t addr) {
  asm volatile("red.shared.add.u32 [%0+%1], 1;" ::"r"(addr), "n"(OFF) : "memory");
}

// ---- K2 pair keys (B = 16 levels) -----------------------------------------------------
// Pixel p of a 48-byte unit pairs with pixel p+8, i.e. byte j with byte j+24 — same channel
// (24 = 0 mod 3) and same position within its word, so one SHF + one LOP3 select builds a
// word K of four 8-bit keys:  K = ((w[k] >> 4) & 0x0F0F0F0F) | (w[k+6] & 0xF0F0F0F0).
// Which pixels are paired does not matter: the flush adds each key's count to both of its
// bins (same channel), so the marginals are exact for any same-channel pairing.
//
// Table (kPair, non-split): the 256 keys of channels 0 and 1 share 256-byte rows of a
// 64 KB-aligned block, tab01[key][c][lane], so key byte I of K drops straight into byte 1
// of the address with ONE PRMT (byte 0 = lane << 2, bytes 2-3 = the block's high bits;
// c * 128 is the ATOMS immediate); channel 2 keeps 128-byte rows, tab2[key][lane], in the
// 32 KB after the block (table | key << 7 | lane << 2 + 64 KB: shift + LOP3).
// Split layout (kFused, H2): channel 2 in tab2[key][lane / 2] below the block.
template <uint32_t MASK>
__device__ __forceinline__ uint32_t lop3_and_or(uint32_t a, uint32_t c) {  // (a & MASK) | c in one LOP3
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(a), "n"(MASK), "r"(c));
  return d;
}
__device__ __forceinline__ uint32_t pair_key_word(uint32_t a, uint32_t b) {
  uint32_t K;  // per bit: 0x0F0F0F0F ? (a >> 4) : b   (LUT 0xD8 for operands (b, a>>4, M))
  asm("lop3.b32 %0, %1, %2, %3, 0xD8;" : "=r"(K) : "r"(b), "r"(a >> 4), "n"(0x0F0F0F0Fu));
  return K;
}
// Half-lane block (H2 == 2, the realigning fused kernel when it buys a bigger tile): all
// three channels in one 64 KB-aligned block of 256-byte key rows tab[key][c][lane / 2] (16
// counters per channel, a 64-byte spare), so every key takes ONE PRMT (key -> address byte 1,
// (lane / 2) << 2 in byte 0, c * 64 as the ATOMS immediate). 64 KB instead of the split
// layout's 80 KB: at 1366 wide the ring takes 12-row tiles instead of 10.
template <int K_, int I, int H2>
__device__ __forceinline__ void pair_key_step(uint32_t K, uint32_t lane4, uint32_t lane4h) {
  constexpr int c = (4 * K_ + I) % 3;  // channel of byte 4*K_ + I
  if constexpr (H2 == 2) {
    red_shared_add_off<c * 64>(__byte_perm(K, lane4, 0x7604u | (I << 4)));
  } else if constexpr (c < 2) {
    red_shared_add_off<c * 128>(__byte_perm(K, lane4, 0x7604u | (I << 4)));
  } else if constexpr (H2) {  // split layout: tab2 | key << 6 | (lane / 2) << 2
    uint32_t x;
    if constexpr (8 * I >= 6) x = K >> (8 * I - 6);
    else x = K << (6 - 8 * I);
    red_shared_add_off<0>(lop3_and_or<0xFFu << 6>(x, lane4h));
  } else {
    uint32_t x;
    if constexpr (8 * I >= 7) x = K >> (8 * I - 7);
    else x = K << (7 - 8 * I);
    red_shared_add_off<65536>(lop3_and_or<0xFFu << 7>(x, lane4));
  }
}
template <int K_, int H2>
__device__ __forceinline__ void pair_word(const uint32_t* w, uint32_t lane4, uint32_t lane4h) {
  const uint32_t Kw = pair_key_word(w[K_], w[K_ + 6]);
  pair_key_step<K_, 0, H2>(Kw, lane4, lane4h);
  pair_key_step<K_, 1, H2>(Kw, lane4, lane4h);
  pair_key_step<K_, 2, H2>(Kw, lane4, lane4h);
  pair_key_step<K_, 3, H2>(Kw, lane4, lane4h);
}
template <int H2>
__device__ __forceinline__ void hist_unit_pair(const uint32_t* w, uint32_t lane4, uint32_t lane4h = 0) {
  pair_word<0, H2>(w, lane4, lane4h); pair_word<1, H2>(w, lane4, lane4h); pair_word<2, H2>(w, lane4, lane4h);
  pair_word<3, H2>(w, lane4, lane4h); pair_word<4, H2>(w, lane4, lane4h); pair_word<5, H2>(w, lane4, lane4h);
}

// ---- K2r raw byte keys (256 levels, PRMT layout) ------------------------------------------
// Byte J of channel J % 3: channels 0 and 1 share 256-byte rows of a 64 KB-aligned block,
// tab01[v][c][lane], so ONE PRMT drops the byte into byte 1 of the address (c * 128 is the
// ATOMS immediate); channel 2 keeps 128-byte rows in the 32 KB after the block (PRMT + IMAD).
template <int J>
__device__ __forceinline__ void raw_unit_step(const uint32_t* w, uint32_t lane4) {
  constexpr int c = J % 3;
  if constexpr (c < 2) {
    red_shared_add_off<c * 128>(__byte_perm(w[J >> 2], lane4, 0x7604u | ((J & 3) << 4)));
  } else {
    red_shared_add_off<65536>(__byte_perm(w[J >> 2], 0u, 0x4440u + (J & 3)) * 128u + lane4);
  }
}
template <int... J>
__device__ __forceinline__ void raw_unit_all(const uint32_t* w, uint32_t lane4, std::integer_sequence<int, J...>) {
  (raw_unit_step<J>(w, lane4), ...);
}
__device__ __forceinline__ void hist_unit_raw(const uint32_t* w, uint32_t lane4) {
  raw_unit_all(w, lane4, std::make_integer_sequence<int, 48>{});
}

// ---- K2a' packed match: one MATCH per word of four pair keys --------------------------------
template <int K_>
__device__ __forceinline__ void match_packed_word(const uint32_t* w, uint32_t am, uint32_t lt, uint32_t* wb) {
  const uint32_t Kw = pair_key_word(w[K_], w[K_ + 6]);
  const uint32_t peers = __match_any_sync(am, Kw);
  if ((peers & lt) == 0) {  // the group's leader adds the group size to its four keys
    const uint32_t n = (uint32_t)__popc(peers);
#pragma unroll
    for (int I = 0; I < 4; ++I) atomicAdd(wb + ((4 * K_ + I) % 3) * 256 + ((Kw >> (8 * I)) & 0xFFu), n);
  }
}

// ---- NEXT N4 joint-colour keys: one key per pixel, k = (bR * J + bG) * J + bB ------------
// Pixel P of a unit is bytes 3P..3P+2 (reading Q2 bins, (v * J) >> 8); the key picks a 128-byte
// lane-private row.
// Any J, SIMD: the bins of a word's four bytes come from two 16-bit-lane products,
// (v * J) >> 8 for bytes 0/2 and 1/3 at once (v * J < 2^16), i.e. 2 PRMT + 2 IMAD + SHF + LOP3
// per 4 bytes; a pixel's key bin(R)*J^2 + bin(G)*J + bin(B) is then ONE IDP.4A of its 4-byte
// window of bins (a funnel shift for 12 of the 16 pixels) against (J^2, J, 1, 0), and its row
// address one LEA: ~2.75 instructions per byte. Measured (profiles/r02_tune_joint.jsonl, same
// box): every J at 7.24-7.33 TB/s; a multiply per channel byte ran J = 3/5/7 at 5.5 TB/s, and
// the shift-and-OR bin fields for J = 2^L (3 SHF + 3 LOP3 per pixel) 6.4-6.9 TB/s.
__device__ __forceinline__ uint32_t joint_bins4(uint32_t w, uint32_t J) {
  const uint32_t lo = __byte_perm(w, 0u, 0x4240u) * J;  // [0, b2, 0, b0] * J
  const uint32_t hi = __byte_perm(w, 0u, 0x4341u) * J;  // [0, b3, 0, b1] * J
  uint32_t B;  // (lo >> 8) & 0x00FF00FF | hi & 0xFF00FF00: one LOP3 (LUT 0xCA = M ? a : b per bit)
  asm("lop3.b32 %0, %1, %2, %3, 0xCA;" : "=r"(B) : "r"(0x00FF00FFu), "r"(lo >> 8), "r"(hi));
  return B;
}
template <int P>
__device__ __forceinline__ void joint_simd_step(const uint32_t* b, uint32_t lane4, uint32_t wts) {
  constexpr int i = 3 * P;
  const uint32_t win = (i & 3) ? __funnelshift_r(b[i >> 2], b[(i >> 2) + 1], 8 * (i & 3)) : b[i >> 2];
  red_shared_add_off<0>(lane4 + (__dp4a(win, wts, 0u) << 7));
}
template <int... P>
__device__ __forceinline__ void joint_simd_all(const uint32_t* b, uint32_t lane4, uint32_t wts,
                                               std::integer_sequence<int, P...>) {
  (joint_simd_step<P>(b, lane4, wts), ...);
}
// ---- K2b: any B <= 16 as pair keys of SIMD bins ---------------------------------------------
// The bins of bytes j and j+24 (same channel) of a unit, from joint_bins4 (B <= 16: bins < 16),
// form the key word bins(w[k]) | bins(w[k+6]) << 4 (one IMAD: no carries), i.e. the K1 pair
// keys with B-level instead of 16-level fields: 0.5 shared atomics per byte for every B <= 16
// (K2r, one atomic per byte, keeps B > 16). The flush adds each key to both of its bins.
__device__ __forceinline__ uint32_t joint_bins4(uint32_t w, uint32_t J);
template <int K_, int H2>
__device__ __forceinline__ void pair_word_bins(const uint32_t* w, uint32_t lane4, uint32_t lane4h, uint32_t B) {
  const uint32_t Kw = joint_bins4(w[K_ + 6], B) * 16u + joint_bins4(w[K_], B);
  pair_key_step<K_, 0, H2>(Kw, lane4, lane4h);
  pair_key_step<K_, 1, H2>(Kw, lane4, lane4h);
  pair_key_step<K_, 2, H2>(Kw, lane4, lane4h);
  pair_key_step<K_, 3, H2>(Kw, lane4, lane4h);
}
template <int H2>
__device__ __forceinline__ void hist_unit_pair_bins(const uint32_t* w, uint32_t lane4, uint32_t lane4h, uint32_t B) {
  pair_word_bins<0, H2>(w, lane4, lane4h, B); pair_word_bins<1, H2>(w, lane4, lane4h, B);
  pair_word_bins<2, H2>(w, lane4, lane4h, B); pair_word_bins<3, H2>(w, lane4, lane4h, B);
  pair_word_bins<4, H2>(w, lane4, lane4h, B); pair_word_bins<5, H2>(w, lane4, lane4h, B);
}
// kVarRaw: one raw byte key per byte in the fused kernels' split table (K2r's keys in 80 KB
// instead of 96 KB so a fused ring still fits): channels 0/1 full-lane in the 64 KB PRMT block
// (one PRMT: byte -> address byte 1, c * 128 the ATOMS immediate), channel 2 in the half-lane
// tab2[v][lane / 2] (SHF + LOP3); the flush maps value rows to bins as K2r does.
template <int J>
__device__ __forceinline__ void raw_split_step(const uint32_t* w, uint32_t lane4, uint32_t lane4h) {
  constexpr int c = J % 3, sh = 8 * (J & 3);
  if constexpr (c < 2) {
    red_shared_add_off<c * 128>(__byte_perm(w[J >> 2], lane4, 0x7604u | ((J & 3) << 4)));
  } else {  // tab2 | v << 6 | (lane / 2) << 2
    uint32_t x;
    if constexpr (sh >= 6) x = w[J >> 2] >> (sh - 6);
    else x = w[J >> 2] << (6 - sh);
    red_shared_add_off<0>(lop3_and_or<0xFFu << 6>(x, lane4h));
  }
}
template <int... J>
__device__ __forceinline__ void raw_split_all(const uint32_t* w, uint32_t lane4, uint32_t lane4h,
                                              std::integer_sequence<int, J...>) {
  (raw_split_step<J>(w, lane4, lane4h), ...);
}
// the fused kernels' histogram of one 48-byte unit: 16-level pair keys, (kVarBins) pair keys of
// B-level bins for B < 16 not dividing 16, or (kVarRaw) raw byte keys for B > 16
template <int H2, bool BINS, bool RAW>
__device__ __forceinline__ void hist_unit_fused(const uint32_t* w, uint32_t lane4, uint32_t lane4h, uint32_t B) {
  if constexpr (RAW) raw_split_all(w, lane4, lane4h, std::make_integer_sequence<int, 48>{});
  else if constexpr (BINS) hist_unit_pair_bins<H2>(w, lane4, lane4h, B);
  else hist_unit_pair<H2>(w, lane4, lane4h);
}

__device__ __forceinline__ void hist_unit_joint(const uint32_t* w, uint32_t lane4, uint32_t J) {
  uint32_t b[13];
#pragma unroll
  for (int k = 0; k < 12; ++k) b[k] = joint_bins4(w[k], J);
  b[12] = 0u;  // pixel 15's window reads bytes 45..48: byte 48 has weight 0
  joint_simd_all(b, lane4, J * J | J << 8 | 1u << 16, std::make_integer_sequence<int, 16>{});
}
__device__ __forceinline__ void load_unit(uint32_t a, uint32_t* w) {  // 48 bytes at a 16-byte aligned address
  const uint4 v0 = lds128(a), v1 = lds128(a + 16), v2 = lds128(a + 32);
  w[0] = v0.x; w[1] = v0.y; w[2] = v0.z; w[3] = v0.w;
  w[4] = v1.x; w[5] = v1.y; w[6] = v1.z; w[7] = v1.w;
  w[8] = v2.x; w[9] = v2.y; w[10] = v2.z; w[11] = v2.w;
}
// 48 bytes at ANY address: four aligned LDS.128 (<= 16 bytes past the unit), then funnel
// shifts by the byte misalignment (kVarGen; a warp-uniform branch except across rows)
template <int J>
__device__ __forceinline__ void realign(const uint32_t* q, uint32_t* w, uint32_t bits) {
#pragma unroll
  for (int k = 0; k < 12; ++k) w[k] = __funnelshift_r(q[k + J], q[k + J + 1], bits);
}
__device__ __forceinline__ void load_unit_any(uint32_t a, uint32_t* w) {
  const uint32_t a16 = a & ~15u, sh = a & 15u;
  uint32_t q[16];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint4 v = lds128(a16 + 16 * i);
    q[4 * i] = v.x; q[4 * i + 1] = v.y; q[4 * i + 2] = v.z; q[4 * i + 3] = v.w;
  }
  const uint32_t bits = (sh & 3u) * 8u;
  switch (sh >> 2) {
    case 0: realign<0>(q, w, bits); break;
    case 1: realign<1>(q, w, bits); break;
    case 2: realign<2>(q, w, bits); break;
    default: realign<3>(q, w, bits); break;
  }
}

// ---- 2x box downsample of a 2 x 48-byte unit pair -> 24 output bytes --------
// Output byte m of the 8-pixel group = (T_i + T_{i+3} + B_i + B_{i+3} + 2) >> 2 with
// i = 2m - m%3, each pair taken from a 4-byte window (funnel shift) by one IDP.4A; the
// sums run on the FMA pipe. The weights are 64, not 1: the result is (sum + 2) * 64 <=
// 65,408, so the output byte sits exactly in bits 8-15 — no shift and no mask afterwards.
template <int I>
__device__ __forceinline__ uint32_t win4(const uint32_t* w) {
  if constexpr ((I & 3) == 0) return w[I >> 2];
  else return __funnelshift_r(w[I >> 2], w[(I >> 2) + 1], 8 * (I & 3));
}
template <int M>
__device__ __forceinline__ uint32_t ds_sum(const uint32_t* t, const uint32_t* b) {  // (sum + 2) * 64
  constexpr int I = 2 * M - (M % 3);
  return __dp4a(win4<I>(b), 0x40000040u, __dp4a(win4<I>(t), 0x40000040u, 128u));
}
// Two scaled sums at 16-bit spacing (one IMAD: no carry, each < 2^16) put output bytes m and
// m+2 in bytes 1 and 3; one PRMT interleaves the two words' bytes 1 and 3.
template <int Q>
__device__ __forceinline__ uint32_t ds_word4(const uint32_t* t, const uint32_t* b) {
  const uint32_t t02 = ds_sum<4 * Q + 2>(t, b) * 65536u + ds_sum<4 * Q>(t, b);
  const uint32_t t13 = ds_sum<4 * Q + 3>(t, b) * 65536u + ds_sum<4 * Q + 1>(t, b);
  return __byte_perm(t02, t13, 0x7351);
}
__device__ __forceinline__ void ds_unit(const uint32_t* t, const uint32_t* b, uint32_t* o) {
  o[0] = ds_word4<0>(t, b); o[1] = ds_word4<1>(t, b); o[2] = ds_word4<2>(t, b);
  o[3] = ds_word4<3>(t, b); o[4] = ds_word4<4>(t, b); o[5] = ds_word4<5>(t, b);
}

__device__ __forceinline__ void st_global_24(uint8_t* dst, const uint32_t* o) {  // dst 8-byte aligned
  uint2* d = reinterpret_cast<uint2*>(dst);
  d[0] = make_uint2(o[0], o[1]);
  d[1] = make_uint2(o[2], o[3]);
  d[2] = make_uint2(o[4], o[5]);
}
__device__ __forceinline__ void st_pred_u8(uint8_t* p, uint32_t v, bool pr) {
  asm volatile("{ .reg .pred q; setp.ne.u32 q, %2, 0; @q st.global.u8 [%0], %1; }" ::"l"(p), "r"(v),
               "r"((uint32_t)pr) : "memory");
}
__device__ __forceinline__ void st_pred_u16(uint8_t* p, uint32_t v, bool pr) {
  asm volatile("{ .reg .pred q; setp.ne.u32 q, %2, 0; @q st.global.u16 [%0], %1; }" ::"l"(p), "r"(v),
               "r"((uint32_t)pr) : "memory");
}
__device__ __forceinline__ void st_pred_u32(uint8_t* p, uint32_t v, bool pr) {
  asm volatile("{ .reg .pred q; setp.ne.u32 q, %2, 0; @q st.global.u32 [%0], %1; }" ::"l"(p), "r"(v),
               "r"((uint32_t)pr) : "memory");
}
// 24 output bytes at ANY address (kVarGen). Lanes of one row write consecutive 24-byte
// chunks; each lane stores the three aligned 8-byte words that START inside its chunk —
// when the chunk is not 8-aligned the third one ends in the next lane's chunk, whose first
// 8 bytes come by one shuffle pair. The words are cut from the 32-bit stream (o, next) by
// funnel shifts after a select on the word offset, so every lane runs the same code for
// any alignment. Bytes of a word whose neighbour is missing (row ends, warp edges, idle
// lanes) are written as naturally aligned 1/2/4-byte pieces. All 32 lanes call this
// (full-warp shuffles); only `act` lanes store.
__device__ __forceinline__ void st_global_24_any(uint8_t* dst, const uint32_t* o, bool act, bool has_next,
                                                 bool has_prev) {
  const uint32_t n0 = __shfl_down_sync(0xFFFFFFFFu, o[0], 1), n1 = __shfl_down_sync(0xFFFFFFFFu, o[1], 1);
  if (!act) return;
  const uint32_t b = (8u - ((uint32_t)(uintptr_t)dst & 7u)) & 7u;  // bytes before the first aligned word
  const uint32_t s = 8u * (b & 3u);
  const bool hi = b >= 4u;
  const uint32_t w[8] = {o[0], o[1], o[2], o[3], o[4], o[5], n0, n1};
  uint32_t t[7];
#pragma unroll
  for (int i = 0; i < 7; ++i) t[i] = hi ? w[i + 1] : w[i];
  uint32_t v[6];  // v[i] = stream bytes [4i + b, 4i + b + 4)
#pragma unroll
  for (int i = 0; i < 6; ++i) v[i] = __funnelshift_r(t[i], t[i + 1], s);
  uint2* d = reinterpret_cast<uint2*>(dst + b);
  d[0] = make_uint2(v[0], v[1]);
  d[1] = make_uint2(v[2], v[3]);
  if (b == 0u || has_next) d[2] = make_uint2(v[4], v[5]);
  // Words without a neighbour, written as naturally aligned 4/2/1-byte pieces by predicated
  // stores (branch-free: the edge lanes of a warp would otherwise serialise two branches).
  // Tail: own bytes [b + 16, 24) = n = 8 - b bytes at the aligned q = dst + b + 16.
  const bool tl = b != 0u && !has_next;
  const uint32_t n = 8u - b;
  uint8_t* q = dst + b + 16u;
  st_pred_u32(q, v[4], tl && (n & 4u));
  const uint32_t t2 = (n & 4u) ? v[5] : v[4];
  st_pred_u16(q + (n & 4u), t2, tl && (n & 2u));
  st_pred_u8(q + (n & 6u), t2 >> (8u * (n & 2u)), tl && (n & 1u));
  // Head: bytes [0, b) at dst (alignment a = 8 - b): a 1-byte piece up to 2-alignment, a
  // 2-byte piece up to 4-alignment, a 4-byte piece up to the first aligned word.
  const bool hd = b != 0u && !has_prev;
  const uint32_t a = 8u - b, a1 = a + (a & 1u), a2 = a1 + (a1 & 2u);
  st_pred_u8(dst, o[0], hd && (a & 1u));
  st_pred_u16(dst + (a1 - a), __funnelshift_r(o[0], o[1], 8u * (a1 - a)), hd && (a1 & 2u));
  st_pred_u32(dst + (a2 - a), __funnelshift_r(o[0], o[1], 8u * (a2 - a)), hd && (a2 & 4u));
}

// 24 output bytes at ANY shared-memory address (kVarGen staged stores): the bytes up to the
// next 4-byte boundary as a 1/2/4-byte head, five aligned words cut by one funnel shift each
// (__funnelshift_rc: shift 32 = the high word, so m = 0 needs no special case), and the last
// m bytes as a 1/2-byte tail — branch-free predicated stores, 8 at most, 5-7 executed.
__device__ __forceinline__ void sts_24_any(uint32_t a, const uint32_t* o) {
  const uint32_t m = a & 3u, sh = 8u * (4u - m), al = a + 4u - m;
  sts_pred_u32(a, o[0], m == 0u);
  sts_pred_u8(a, o[0], m & 1u);
  sts_pred_u16(a + (m & 1u), o[0] >> (8u * (m & 1u)), m == 1u || m == 2u);
#pragma unroll
  for (int j = 0; j < 5; ++j) sts32(al + 4u * j, __funnelshift_rc(o[j], o[j + 1], sh));
  sts_pred_u16(al + 20u, o[5] >> sh, m >= 2u);
  sts_pred_u8(al + 20u + (m & 2u), o[5] >> 24, m & 1u);
}

// ---------------------------------------------------------------------------
// The persistent TMA-ring kernel (modes: see the file header).
// ---------------------------------------------------------------------------
template <int MODE, int NW, int VAR = 0>
__global__ void __launch_bounds__(NW * 32 + 32, 1) hist_tma_kernel(const __grid_constant__ HistParams p) {
  constexpr int kConsWarps = NW;
  constexpr int kConsThreads = NW * 32;
  constexpr int kThreads = kConsThreads + 32;
  constexpr bool kRowPair = MODE == kModeFused || MODE == kModeDs;
  constexpr bool kGen = kRowPair && (VAR & kVarGen);
  constexpr bool kRawF = MODE == kModeFused && (VAR & kVarRaw);  // fused raw byte keys (B > 16)
  constexpr bool kRawAny = MODE == kModeRaw || kRawF;
  constexpr bool kHalf = MODE == kModeFused && (VAR & kVarHalf);  // half-lane 64 KB block
  constexpr bool kBins = MODE == kModePairB || (MODE == kModeFused && (VAR & kVarBins));  // B-level pair keys
  constexpr bool kSplit = MODE == kModeFused && !kHalf;
  constexpr int kH2 = kHalf ? 2 : 1;
  constexpr bool kTable = MODE != kModeDs;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t base = smem_addr(smem);
  // kRawF keeps its 3 x B bin counters in the top kRemapBytes of shared memory, out of the ring
  Layout L = kSplit  ? make_layout_split(base, p.smem_bytes - (kRawF ? kRemapBytes : 0u), p.slot)
             : kHalf ? make_layout_half(base, p.smem_bytes, p.slot)
                     : make_layout(base, p.smem_bytes, p.slot, p.table_bytes, p.table_align,
                                  MODE == kModeRaw ? kRemapBytes : 0u);
  if (p.max_stages > 0 && L.stages > p.max_stages) {
    L.stages = p.max_stages;
    if (L.n_lo > L.stages) L.n_lo = L.stages;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t full0 = L.ctrl, empty0 = L.ctrl + 8 * kMaxStages;
  uint32_t* hsum = reinterpret_cast<uint32_t*>(smem + 16 * kMaxStages);  // 3 x 16 bins (pair modes)
  // bin counters of the raw-key modes: kRaw right above the table, kRawF at the top of shared memory
  uint32_t* const remap_base = kRawF ? reinterpret_cast<uint32_t*>(smem + p.smem_bytes - kRemapBytes)
                                     : reinterpret_cast<uint32_t*>(smem + (L.table + p.table_bytes - base));
  auto remap = [&](uint32_t i) -> uint32_t* { return remap_base + i; };
  const int B = p.bins;
  const int RS = MODE == kModeJoint ? p.joint * p.joint * p.joint : 3 * B;  // counters per output row

  if (threadIdx.x == 0) {
    if (L.stages < 2) __trap();
    for (int s = 0; s < L.stages; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, kConsWarps);
    }
    fence_mbar_init();
  }
  if constexpr (kTable) {  // zero the table and the merge counters
    for (uint32_t i = threadIdx.x; i < p.table_bytes / 16; i += kThreads) sts128(L.table + 16 * i, make_uint4(0, 0, 0, 0));
    for (int i = threadIdx.x; i < 3 * 16; i += kThreads) hsum[i] = 0;
    if constexpr (kRawAny)
      for (int i = threadIdx.x; i < 3 * 256; i += kThreads) *remap((uint32_t)i) = 0;
  }
  __syncthreads();

  const int64_t t0 = p.total_tiles * blockIdx.x / gridDim.x;
  const int64_t t1 = p.total_tiles * (blockIdx.x + 1) / gridDim.x;
  // kVarGen staged stores (contiguous output rows): each ring slot holds an input tile and,
  // at out_off, the image of that tile's output bytes at the destination's alignment mod 16;
  // the producer writes its 16-byte-aligned interior with one bulk store, the consumers write
  // the < 16-byte head and tail fragments (shared with the neighbouring tiles) directly.
  // (downsample-only kernel only: the fused one keeps direct stores and none of this code)
  constexpr bool kCanStage = kGen && MODE == kModeDs;
  const bool kStaged = kCanStage && p.out_off != 0u;
  const int64_t ow3 = (int64_t)(p.width / 2) * 3;

  if (warp == kConsWarps) {
    // output tile (sitem, sk) of slot s: bytes [g0, g0 + n) of the destination frame
    int64_t sitem = t0 / p.tpf;
    int32_t sk = (int32_t)(t0 - sitem * p.tpf);
    auto stage_store = [&](int ss, int64_t& it, int32_t& kk) {
      if (it >= p.n_halo) {
        const uint32_t rows = kk == p.tpf - 1 ? (uint32_t)(p.height - (p.tpf - 1) * p.rows_per_tile)
                                              : (uint32_t)p.rows_per_tile;
        const uint64_t g0 = (uint64_t)(uintptr_t)(p.ds_out + (it - p.n_halo) * (int64_t)(p.height / 2) * ow3 +
                                                  (int64_t)kk * (p.rows_per_tile / 2) * ow3);
        const uint64_t a = (g0 + 15) & ~15ull, b = (g0 + (uint64_t)(rows / 2) * (uint64_t)ow3) & ~15ull;
        if (b > a) {
          tma_store_1d(reinterpret_cast<void*>(a), L.slot(ss) + p.out_off + 16u, (uint32_t)(b - a));
          bulk_commit();
        }
      }
      if (++kk == p.tpf) { kk = 0; ++it; }
    };
    // ---------------- producer: one elected lane issues the bulk copies ----------------
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      int64_t item = t0 / p.tpf;
      int32_t k = (int32_t)(t0 - item * p.tpf);
      int64_t pitem = item;  // L2 prefetch cursor, l2_prefetch tiles ahead of the load cursor
      int32_t pk = k;
      for (int32_t i = 0; i < p.l2_prefetch; ++i)
        if (++pk == p.tpf) { pk = 0; ++pitem; }
      // the frame's address (sparse tables: a global read of the row pointer) is loaded once
      // per frame and BEFORE the empty-slot wait, so its latency overlaps the wait
      int64_t base_item = -1;
      uint64_t fbase = 0;
      int defer = -1;  // kStaged: slot whose full-barrier arrive waits for the last store's read
      for (int64_t t = t0; t < t1; ++t, (++k == p.tpf) ? (k = 0, ++item) : 0) {
        const uint64_t off = (uint64_t)k * p.tile;
        const uint64_t len = (uint64_t)p.F - off < p.tile ? (uint64_t)p.F - off : p.tile;
        if (item != base_item) {
          base_item = item;
          fbase = frame_addr(p.src, item);
        }
        if (p.l2_prefetch > 0) {
          if (t + p.l2_prefetch < t1) {
            const uint64_t poff = (uint64_t)pk * p.tile;
            const uint64_t plen = (uint64_t)p.F - poff < p.tile ? (uint64_t)p.F - poff : p.tile;
            const uint64_t pa = frame_addr(p.src, pitem) + poff;
            tma_prefetch_l2(reinterpret_cast<const void*>(pa & ~15ull),
                            (uint32_t)(((pa + plen + 15) & ~15ull) - (pa & ~15ull)));
          }
          if (++pk == p.tpf) { pk = 0; ++pitem; }
        }
        // the 16-byte granules covering [off, off + len): the tile start is aligned unless
        // the row-pair tiling of a kVarGen frame puts it mid-granule (frames are 16-aligned)
        const uint64_t a0 = (fbase + off) & ~15ull;
        const uint32_t bytes = (uint32_t)(((fbase + off + len + 15) & ~15ull) - a0);
        if (p.prod_sleep) mbar_wait_sleep(empty0 + 8 * s, ph ^ 1, p.prod_sleep);
        else mbar_wait(empty0 + 8 * s, ph ^ 1);
        if (kStaged) {
          // The consumers released slot s: store the output tile they staged in it and load the
          // next input tile into the slot's input region. The consumers may rewrite the output
          // region only after the store has READ it, so the slot's full-barrier arrive waits for
          // that — deferred to the next iteration (a consumer tile later, after the next empty
          // wait), where the read is long done, so the producer never blocks on its own store.
          if (defer >= 0) {
            bulk_wait_read0();
            mbar_arrive(full0 + 8 * defer);
            defer = -1;
          }
          const bool st_out = t - t0 >= L.stages;
          if (st_out) stage_store(s, sitem, sk);
          mbar_expect_tx(full0 + 8 * s, bytes);
          tma_load_1d(L.slot(s), reinterpret_cast<const void*>(a0), bytes, full0 + 8 * s);
          if (st_out) defer = s;
          else mbar_arrive(full0 + 8 * s);
        } else {
          mbar_arrive_expect_tx(full0 + 8 * s, bytes);
          tma_load_1d(L.slot(s), reinterpret_cast<const void*>(a0), bytes, full0 + 8 * s);
        }
        if (++s == L.stages) { s = 0; ph ^= 1; }
      }
      if (kStaged) {  // the last min(stages, tiles) output tiles
        if (defer >= 0) {
          bulk_wait_read0();
          mbar_arrive(full0 + 8 * defer);
        }
        const int64_t nt = t1 - t0;
        if (nt < L.stages) {  // slots 0 .. nt-1 hold their first tiles (phase 0)
          s = 0;
          ph = 1;
        }
        for (int64_t t = nt > L.stages ? nt - L.stages : 0; t < nt; ++t) {
          mbar_wait(empty0 + 8 * s, ph ^ 1);
          stage_store(s, sitem, sk);
          if (++s == L.stages) { s = 0; ph ^= 1; }
        }
        bulk_wait0();
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  const int ctid = threadIdx.x;  // 0 .. kConsThreads-1
  // split layout: channels 0/1 in the 64 KB block after tab2, channel 2 in tab2 (half lanes)
  const uint32_t lane4 = kHalf ? L.table | ((uint32_t)lane >> 1 << 2)
                              : (kSplit ? L.table + kTab2Bytes : L.table) | ((uint32_t)lane << 2);
  const uint32_t lane4h = L.table | ((uint32_t)lane >> 1 << 2);
  int s = 0;
  uint32_t ph = 0;
  // Units are dealt round-robin over the consumer threads across tile boundaries: a thread's
  // next unit (pair) index in the current tile is carried from the previous tile (minus
  // that tile's unit count), so every warp shares the work and a tile costs no division.
  uint32_t ucur = (uint32_t)ctid;
  int64_t cur = -1;

  auto out_row = [&](int64_t item) -> uint32_t* {
    return item < p.n_halo ? p.halo_out + item * RS : p.out + (item - p.n_halo) * RS;
  };
  // add v to counter idx of item's row: locally, or (fused all-gather) into the same row of
  // every rank's result column through peer memory (NVLink when the dest is on another GPU)
  auto emit = [&](int64_t item, int idx, uint32_t v) {
    if (p.n_dest == 0 || item < p.n_halo) {
      red_global_add(out_row(item) + idx, v);
    } else {
      const int64_t off = (item - p.n_halo) * RS + idx;
      for (int g = 0; g < p.n_dest; ++g) red_global_add(reinterpret_cast<uint32_t*>(p.dest[g]) + off, v);
    }
  };

  // Flush at a frame change. The lane-private counters are never re-zeroed: they keep
  // accumulating over the CTA's frames and a frame's count of a row is its 32-lane sum minus
  // the sum at the previous flush (exact mod 2^32). Each thread always flushes the same rows
  // (r = ctid + i * kConsThreads), so the previous sums live in registers and the flush only
  // reads shared memory.
  constexpr int kSnapN = (768 + kConsThreads - 1) / kConsThreads;  // rows <= 3 * 256
  uint32_t snap[kSnapN];
#pragma unroll
  for (int i = 0; i < kSnapN; ++i) snap[i] = 0;
  auto flush = [&](int64_t item) {
    if constexpr (!kTable) return;
    named_bar(kBarId, kConsThreads);
    if constexpr (MODE == kModeMatch) {
      // per-warp bins wbins[warp][c][bin16]: lane l < NW holds warp l's count, __reduce_add_sync
      // sums them, lane 0 adds the block's total to the 16-level merge counters
      uint32_t* wbins = reinterpret_cast<uint32_t*>(smem + (L.table - base));
      for (int k = warp; k < 48; k += kConsWarps) {
        uint32_t v = lane < kConsWarps ? wbins[lane * 48 + k] : 0u;
        if (lane < kConsWarps) wbins[lane * 48 + k] = 0u;
        v = __reduce_add_sync(0xFFFFFFFFu, v);
        if (lane == 0) hsum[k] += v;
      }
    } else if constexpr (MODE == kModeMatchPacked) {
      // per-warp pair-key bins wbins[warp][c][key]; the block's count of (c, key) goes to both bins
      uint32_t* wbins = reinterpret_cast<uint32_t*>(smem + (L.table - base));
      for (int r = warp; r < 768; r += kConsWarps) {
        uint32_t v = lane < kConsWarps ? wbins[lane * 768 + r] : 0u;
        if (lane < kConsWarps) wbins[lane * 768 + r] = 0u;
        v = __reduce_add_sync(0xFFFFFFFFu, v);
        if (lane == 0 && v) {
          const int c = r >> 8, key = r & 255;
          atomicAdd(&hsum[c * 16 + (key & 15)], v);
          atomicAdd(&hsum[c * 16 + (key >> 4)], v);
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < kSnapN; ++i) {
        const int r = ctid + i * kConsThreads;  // row (c, key) = (r >> 8, r & 255); kModeJoint: the joint bin
        if (r >= (MODE == kModeJoint ? RS : 768)) break;
        if constexpr (MODE == kModeJoint) {
          uint32_t sum = 0;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint4 v = lds128(L.table + (uint32_t)r * 128u + (uint32_t)(((j + r) & 7) * 16));
            sum += v.x + v.y + v.z + v.w;
          }
          const uint32_t total = sum;
          sum = total - snap[i];
          snap[i] = total;
          if (sum) emit(item, r, sum);
          continue;
        }
        const uint32_t c = (uint32_t)r >> 8, key = (uint32_t)r & 255u;
        uint32_t sum = 0;
        if (kHalf) {  // tab[key][c]: 64-byte half-lane rows in 256-byte key rows
          const uint32_t ra = L.table + key * 256u + c * 64u;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint4 v = lds128(ra + (uint32_t)(((j + r) & 3) * 16));
            sum += v.x + v.y + v.z + v.w;
          }
        } else if (kSplit && c == 2) {  // tab2[key]: 64-byte rows
          const uint32_t ra = L.table + key * 64u;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint4 v = lds128(ra + (uint32_t)(((j + r) & 3) * 16));
            sum += v.x + v.y + v.z + v.w;
          }
        } else {  // tab01[key][c] in the 64 KB block; non-split channel 2: tab2[key] after it
          const uint32_t blk = kSplit ? L.table + kTab2Bytes : L.table;
          const uint32_t ra = c < 2 ? blk + key * 256u + c * 128u : blk + 65536u + key * 128u;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint4 v = lds128(ra + (uint32_t)(((j + r) & 7) * 16));
            sum += v.x + v.y + v.z + v.w;
          }
        }
        const uint32_t total = sum;  // this frame's count = the row sum since the previous flush
        sum = total - snap[i];
        snap[i] = total;
        if (sum) {
          if constexpr (kRawAny) {  // value row -> bin (v * B) >> 8
            if (B == 256) emit(item, r, sum);
            else atomicAdd(remap(c * B + ((key * (uint32_t)B) >> 8)), sum);
          } else {  // a pair key counts once in each of its two 16-level bins
            atomicAdd(&hsum[c * 16 + (key >> 4)], sum);
            atomicAdd(&hsum[c * 16 + (key & 15u)], sum);
          }
        }
      }
    }
    named_bar(kBarId, kConsThreads);
    if constexpr (kRawAny) {
      if (B != 256) {
        for (int i = ctid; i < 3 * B; i += kConsThreads) {
          const uint32_t v = *remap((uint32_t)i);
          *remap((uint32_t)i) = 0;
          if (v) emit(item, i, v);
        }
      }
    } else if (MODE != kModeJoint && ctid < 3 * B) {  // B divides 16: bin b of channel c merges 16/B adjacent 16-level bins
      const int c = ctid / B, b = ctid - c * B, g = kBins ? 1 : 16 / B;
      uint32_t v = 0;
      for (int k = 0; k < g; ++k) {
        v += hsum[c * 16 + b * g + k];
        hsum[c * 16 + b * g + k] = 0;
      }
      if (v) emit(item, ctid, v);
    }
    named_bar(kBarId, kConsThreads);
  };

  // row-pair tiling constants of the downsample modes (unused otherwise)
  struct {
    uint32_t rowb, upr, dq, dr, last_rows, tin, tob;
    uint32_t hq, hr, hdq, hdr, oq, orr, odq, odr;  // kVarGen tails: divmod(ctid, tin / tob), divmod(threads, ...)
    int64_t pitch, ow3, tile_out;
    uint8_t* ds_frame;
  } rg{};
  uint32_t rpc = 0, xcc = 0;  // the carried unit pair as (row pair, column unit), ucur = rpc * upr + xcc
  if constexpr (kRowPair) {
    rg.rowb = (uint32_t)p.width * 3u;
    rg.upr = (uint32_t)p.width / 16u;
    if (rg.upr) {
      rg.dq = (uint32_t)kConsThreads / rg.upr;
      rg.dr = (uint32_t)kConsThreads - rg.dq * rg.upr;
      rpc = (uint32_t)ctid / rg.upr;
      xcc = (uint32_t)ctid - rpc * rg.upr;
    }
    rg.last_rows = (uint32_t)(p.height - (p.tpf - 1) * p.rows_per_tile);
    rg.pitch = p.ds_pitch;
    rg.ow3 = (int64_t)(p.width / 2) * 3;
    rg.tile_out = (int64_t)(p.rows_per_tile / 2) * rg.pitch;
    rg.tin = ((uint32_t)p.width - 16u * rg.upr) * 3u;          // tail input bytes per row
    rg.tob = ((uint32_t)p.width / 2u - 8u * rg.upr) * 3u;      // tail output bytes per output row
    if (rg.tin) {
      rg.hq = (uint32_t)ctid / rg.tin, rg.hr = (uint32_t)ctid - rg.hq * rg.tin;
      rg.hdq = (uint32_t)kConsThreads / rg.tin, rg.hdr = (uint32_t)kConsThreads - rg.hdq * rg.tin;
    }
    if (rg.tob) {
      rg.oq = (uint32_t)ctid / rg.tob, rg.orr = (uint32_t)ctid - rg.oq * rg.tob;
      rg.odq = (uint32_t)kConsThreads / rg.tob, rg.odr = (uint32_t)kConsThreads - rg.odq * rg.tob;
    }
  }
  int64_t item = t0 / p.tpf;
  int32_t k = (int32_t)(t0 - item * p.tpf);
  const int32_t ntiles = (int32_t)(t1 - t0);  // < 2^31 tiles per CTA
  for (int32_t i = 0; i < ntiles; ++i, (++k == p.tpf) ? (k = 0, ++item) : 0) {
    if (k == 0 || i == 0) {  // a new frame (item changes exactly when k wraps)
      if (cur >= 0) flush(cur);
      cur = item;
      if constexpr (kRowPair) {
        if (item >= p.n_halo)
          rg.ds_frame = ds_frame_base(p.ds_out, item - p.n_halo, p.height / 2, rg.ow3, rg.pitch, p.ds_cols);
      }
    }
    const uint64_t off = (uint64_t)k * p.tile;
    const uint32_t len = (uint32_t)((uint64_t)p.F - off < p.tile ? (uint64_t)p.F - off : p.tile);
    mbar_wait(full0 + 8 * s, ph);
    const uint32_t slot = L.slot(s) + (uint32_t)(off & 15u);  // the tile's first byte

    if constexpr (kRowPair) {
      // rows [k*R, k*R + rows) of the frame; unit pairs over row pairs. Per-frame constants
      // (rg.*) are hoisted out of the tile loop, so a tile costs no division.
      const uint32_t rows = (k == p.tpf - 1) ? rg.last_rows : (uint32_t)p.rows_per_tile;
      const uint32_t npairs = (rows / 2) * rg.upr;
      uint8_t* dsf = (item >= p.n_halo) ? rg.ds_frame + (int64_t)k * rg.tile_out : nullptr;
      uint32_t u = ucur, rp = rpc, xc = xcc;
      // staged stores: tile-local output byte c goes to the stage at ob + c if c is in the
      // bulk-stored interior [hl, tb), else straight to dsf[c] (the fragments, < 16 B each)
      uint32_t ob = 0, hl = 0, tb = 0;
      if (kStaged && dsf) {
        const uint32_t n = (rows / 2) * (uint32_t)ow3, r = (uint32_t)(uintptr_t)dsf & 15u;
        hl = (16u - r) & 15u;
        tb = (uint32_t)((((uint64_t)(uintptr_t)dsf + n) & ~15ull) - (uint64_t)(uintptr_t)dsf);
        if (tb <= hl) hl = tb = n;  // no aligned interior: every byte direct
        ob = L.slot(s) + p.out_off + 16u - hl;
      }
      auto put_byte = [&](uint32_t c, uint32_t v) {
        if (c >= hl && c < tb) sts_u8(ob + c, v);
        else dsf[c] = (uint8_t)v;
      };
      if (kStaged) {
        for (; u < npairs; u += kConsThreads, rp += rg.dq, xc += rg.dr, (xc >= rg.upr) ? (xc -= rg.upr, ++rp) : 0) {
          const uint32_t a = slot + rp * 2u * rg.rowb + xc * 48u;
          uint32_t wt[12], wb[12], o[6];
          load_unit_any(a, wt);
          load_unit_any(a + rg.rowb, wb);
          if constexpr (MODE == kModeFused) {
            hist_unit_fused<kH2, kBins, kRawF>(wt, lane4, lane4h, (uint32_t)B);
            hist_unit_fused<kH2, kBins, kRawF>(wb, lane4, lane4h, (uint32_t)B);
          }
          if (dsf) {
            ds_unit(wt, wb, o);
            const uint32_t c = rp * (uint32_t)ow3 + xc * 24u;
            if (c >= hl && c + 24u <= tb) {
              sts_24_any(ob + c, o);
            } else {  // a fragment edge of the tile (two chunks per tile at most)
#pragma unroll
              for (int q = 0; q < 24; ++q) put_byte(c + (uint32_t)q, o[q >> 2] >> (8 * (q & 3)));
            }
          }
        }
      } else if constexpr (kGen) {
        // Warp-uniform iterations (the shuffles of the realigned stores need every lane): a lane
        // whose units of this tile are done idles without advancing, so the carried (u, rp, xc)
        // are exactly the per-lane loop's. Lanes hold consecutive units except where the
        // round-robin start rotates inside the warp, so a neighbour is checked by its unit index.
        for (;;) {
          const bool act = u < npairs;
          if (!__any_sync(0xFFFFFFFFu, act)) break;
          uint32_t o[6] = {0, 0, 0, 0, 0, 0};
          if (act) {
            const uint32_t a = slot + rp * 2u * rg.rowb + xc * 48u;
            uint32_t wt[12], wb[12];
            load_unit_any(a, wt);
            load_unit_any(a + rg.rowb, wb);
            if constexpr (MODE == kModeFused) {
              hist_unit_fused<kH2, kBins, kRawF>(wt, lane4, lane4h, (uint32_t)B);
              hist_unit_fused<kH2, kBins, kRawF>(wb, lane4, lane4h, (uint32_t)B);
            }
            if (dsf) ds_unit(wt, wb, o);
          }
          if (dsf) {  // uniform per tile
            const uint32_t un = __shfl_down_sync(0xFFFFFFFFu, u, 1), up = __shfl_up_sync(0xFFFFFFFFu, u, 1);
            const bool has_next = lane < 31 && un == u + 1 && u + 1 < npairs && xc + 1 < rg.upr;
            const bool has_prev = lane > 0 && up + 1 == u && xc > 0;
            st_global_24_any(dsf + (int64_t)rp * rg.pitch + xc * 24, o, act, has_next, has_prev);
          }
          if (act) {
            u += kConsThreads;
            rp += rg.dq;
            xc += rg.dr;
            if (xc >= rg.upr) { xc -= rg.upr; ++rp; }
          }
        }
      } else {
        for (; u < npairs; u += kConsThreads, rp += rg.dq, xc += rg.dr, (xc >= rg.upr) ? (xc -= rg.upr, ++rp) : 0) {
          const uint32_t a = slot + rp * 2u * rg.rowb + xc * 48u;
          uint32_t wt[12], wb[12], o[6];
          load_unit(a, wt);
          load_unit(a + rg.rowb, wb);
          if constexpr (MODE == kModeFused) {
            hist_unit_fused<kH2, kBins, kRawF>(wt, lane4, lane4h, (uint32_t)B);
            hist_unit_fused<kH2, kBins, kRawF>(wb, lane4, lane4h, (uint32_t)B);
          }
          if (dsf) {
            ds_unit(wt, wb, o);
            st_global_24(dsf + (int64_t)rp * rg.pitch + xc * 24, o);
          }
        }
      }
      if (rg.upr) {
        ucur = u - npairs;  // same column unit, rows / 2 row pairs earlier in the next tile
        rpc = rp - rows / 2;
        xcc = xc;
      }
      if constexpr (kGen) {
        // W mod 16 tail pixels of each row, bytewise
        if (rg.tin) {
          // items t = ctid + i * kConsThreads as (row, byte) pairs advanced without division
          if constexpr (MODE == kModeFused) {  // histogram of every tail byte, all rows of the tile
            for (uint32_t r = rg.hq, j = rg.hr; r < rows; r += rg.hdq, j += rg.hdr, (j >= rg.tin) ? (j -= rg.tin, ++r) : 0) {
              const uint32_t v = lds_u8(slot + r * rg.rowb + 48u * rg.upr + j);
              if constexpr (kRawF) {
                if (B == 256) emit(item, (int)((j % 3u) * 256u + v), 1u);
                else atomicAdd(remap((j % 3u) * (uint32_t)B + ((v * (uint32_t)B) >> 8)), 1u);
              } else {
                atomicAdd(&hsum[(j % 3u) * 16u + (kBins ? (v * (uint32_t)B) >> 8 : v >> 4)], 1u);
              }
            }
          }
          if (dsf && rg.tob) {
            for (uint32_t y = rg.oq, j = rg.orr; y < rows / 2; y += rg.odq, j += rg.odr, (j >= rg.tob) ? (j -= rg.tob, ++y) : 0) {
              const uint32_t i0 = slot + 2u * y * rg.rowb + 48u * rg.upr + 2u * (j - j % 3u) + j % 3u;
              const uint32_t sum = lds_u8(i0) + lds_u8(i0 + 3) + lds_u8(i0 + rg.rowb) + lds_u8(i0 + rg.rowb + 3);
              if (kStaged) put_byte(y * (uint32_t)ow3 + 24u * rg.upr + j, (sum + 2u) >> 2);
              else dsf[(int64_t)y * rg.pitch + 24 * rg.upr + j] = (uint8_t)((sum + 2u) >> 2);
            }
          }
        }
      }
      if (MODE == kModeFused && (rows & 1)) {  // odd last row of an odd-height frame: histogram only
        for (uint32_t v = (uint32_t)ctid; v < rg.upr; v += kConsThreads) {
          uint32_t w[12];
          if constexpr (kGen) load_unit_any(slot + (rows - 1) * rg.rowb + v * 48u, w);
          else load_unit(slot + (rows - 1) * rg.rowb + v * 48u, w);
          hist_unit_fused<kH2, kBins, kRawF>(w, lane4, lane4h, (uint32_t)B);
        }
      }
    } else {
      const uint32_t nunits = len / 48u;
      uint32_t u = ucur;
      for (; u < nunits; u += kConsThreads) {
        uint32_t w[12];
        load_unit(slot + u * 48u, w);
        if constexpr (MODE == kModePair) {
          hist_unit_pair<false>(w, lane4);
        } else if constexpr (MODE == kModePairB) {
          hist_unit_pair_bins<0>(w, lane4, 0u, (uint32_t)B);
        } else if constexpr (MODE == kModeRaw) {
          hist_unit_raw(w, lane4);
        } else if constexpr (MODE == kModeJoint) {
          hist_unit_joint(w, lane4, (uint32_t)p.joint);
        } else if constexpr (MODE == kModeMatch) {
          // north_star K2a: per-warp bins, peers found with __match_any_sync, one leader
          // atomic of popc(peers) per peer group
          const uint32_t am = __activemask();
          const uint32_t lt = (1u << lane) - 1u;
          uint32_t* wb = reinterpret_cast<uint32_t*>(smem + (L.table - base)) + (uint32_t)warp * 48u;
#pragma unroll
          for (int j = 0; j < 48; ++j) {
            const uint32_t key = (uint32_t)(j % 3) * 16u + ((w[j >> 2] >> (8 * (j & 3) + 4)) & 0xFu);
            const uint32_t peers = __match_any_sync(am, key);
            if ((peers & lt) == 0) atomicAdd(wb + key, (uint32_t)__popc(peers));
          }
        } else if constexpr (MODE == kModeMatchPacked) {
          const uint32_t am = __activemask();
          const uint32_t lt = (1u << lane) - 1u;
          uint32_t* wb = reinterpret_cast<uint32_t*>(smem + (L.table - base)) + (uint32_t)warp * 768u;
          match_packed_word<0>(w, am, lt, wb); match_packed_word<1>(w, am, lt, wb);
          match_packed_word<2>(w, am, lt, wb); match_packed_word<3>(w, am, lt, wb);
          match_packed_word<4>(w, am, lt, wb); match_packed_word<5>(w, am, lt, wb);
        }
      }
      // tail bytes (frame size not a multiple of 48): direct global counts of the true bin
      const uint32_t rem = len - nunits * 48u;
      if constexpr (MODE == kModeJoint) {  // whole pixels (tiles and frames are multiples of 3 bytes)
        if ((uint32_t)ctid < rem / 3u) {
          const uint32_t a = slot + nunits * 48u + 3u * (uint32_t)ctid, J = (uint32_t)p.joint;
          const uint32_t k = (((lds_u8(a) * J) >> 8) * J + ((lds_u8(a + 1) * J) >> 8)) * J + ((lds_u8(a + 2) * J) >> 8);
          emit(item, (int)k, 1u);
        }
      } else if ((uint32_t)ctid < rem) {
        const uint32_t j = nunits * 48u + (uint32_t)ctid;
        const uint32_t v = lds_u8(slot + j);
        emit(item, (int)((j % 3) * B + ((v * (uint32_t)B) >> 8)), 1u);
      }
      ucur = u - nunits;
    }
    if (kStaged) fence_proxy_async_smem();  // staged output bytes -> the producer's bulk store
    __syncwarp();
    if (lane == 0) mbar_arrive(empty0 + 8 * s);
    if (++s == L.stages) { s = 0; ph ^= 1; }
  }
  if (cur >= 0) flush(cur);
}

// ---------------------------------------------------------------------------
// K3: shot-diff. One warp per position, L1 over the K counters of a row (3*B per-channel,
// J^3 joint-colour); D goes to every destination column (d.n == 1 and d.p[0] = the
// caller's column for a plain run).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) shotdiff_kernel(const uint32_t* __restrict__ hist,
                                                        const uint32_t* __restrict__ halo,
                                                        const uint8_t* __restrict__ seg, int64_t n, int32_t K,
                                                        DestList d) {
  const int64_t pos = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (pos >= n) return;
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
// K4w: downsample of frames too wide for row-pair tiles (2 rows > the largest ring
// slot, W > ~10,900): one block per output row of the job, threads over output pixels.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) downsample_wide_kernel(FrameSrc src, int64_t n, int32_t width, int32_t height,
                                                              uint8_t* __restrict__ out, int64_t pitch, int32_t cols) {
  const int32_t ow = width / 2, oh = height / 2;
  const int64_t rowb = (int64_t)width * 3;
  for (int64_t g = blockIdx.x; g < n * oh; g += gridDim.x) {
    const int64_t item = g / oh;
    const int32_t y = (int32_t)(g - item * oh);
    const uint8_t* f0 = reinterpret_cast<const uint8_t*>(frame_addr(src, item)) + (int64_t)(2 * y) * rowb;
    const uint8_t* f1 = f0 + rowb;
    uint8_t* o = ds_frame_base(out, item, oh, (int64_t)ow * 3, pitch, cols) + (int64_t)y * pitch;
    for (int32_t x = threadIdx.x; x < ow; x += blockDim.x) {
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const int64_t i = 6 * (int64_t)x + c;
        o[3 * (int64_t)x + c] = (uint8_t)(((uint32_t)f0[i] + f0[i + 3] + f1[i] + f1[i + 3] + 2u) >> 2);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------
static int g_num_sms = 0;
static int g_smem_optin = 0;
static int g_smem_reserved = 0;  // shared memory the system reserves per block (dynamic smem starts after it)

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

// Measurement knobs. The product library has none: every value below is the measured
// default. `make tuning` builds libscn_tuning.so with -DSCN_TUNING, where
// the same names are read once from the environment for A/B runs (tools/, tests/).
struct Knobs {
  int grid = 0;              // SCN_GRID: persistent CTAs (0 = one per SM)
  uint32_t hist_tile = kTile;  // SCN_HIST_TILE: tile bytes of the hist-only kernels (multiple of 48)
  uint32_t fused_tile = 0;   // SCN_FUSED_TILE: bytes per row-pair tile, fused (0 = rows_per_tile_split rule)
  uint32_t ds_tile = 0;      // SCN_DS_TILE: bytes per row-pair tile, downsample only (0 = rule)
  int max_stages = kDefaultStages;  // SCN_MAX_STAGES: ring-depth cap
  int l2_prefetch_fused = 1;  // SCN_L2_PREFETCH: bulk L2 prefetch distance of the row-pair kernels
  int l2_prefetch_hist = 0;   //   (the read-only histogram keeps 0: the data would cross L2 twice)
  uint32_t prod_sleep = 0;    // SCN_PROD_SLEEP: producer empty-slot wait suspend hint in ns (0 = spin)
  int hist_warps = 0;         // SCN_HIST_WARPS: consumer warps of the hist-only kernels (tuning build: 8/20)
  int gen_stage = 1;          // SCN_GEN_STAGE: kVarGen downsample-only output through the staged bulk
                              // store (0 = the direct cross-lane stores, kept for montage canvases)
  int gen_half = 1;           // SCN_GEN_HALF: 0 = never the half-lane fused layout (A/B)
  int pair_bins = 1;          // SCN_PAIR_BINS: 0 = bins < 16 not dividing 16 on K2r instead of K2b (A/B)
  int fused_raw = 1;          // SCN_FUSED_RAW: 0 = B > 16 as K2r histogram + downsample pass (A/B)
  int gen_warps = 0;          // SCN_GEN_WARPS: consumer warps of the kVarGen kernels (tuning build: 8/12/16;
                              // 0 = the defaults kGenDsWarps / kGenFusedWarps)
};
static Knobs g_knobs;
#ifdef SCN_TUNING
static int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v && *v ? atoi(v) : dflt;
}
static std::once_flag g_knobs_once;
static void read_knobs_once() {
  Knobs k;
  k.grid = env_int("SCN_GRID", 0);
  const int t = env_int("SCN_HIST_TILE", (int)kTile);
  k.hist_tile = (t >= 48 && t % 48 == 0 && t <= 65536) ? (uint32_t)t : kTile;
  k.fused_tile = (uint32_t)env_int("SCN_FUSED_TILE", 0);
  k.ds_tile = (uint32_t)env_int("SCN_DS_TILE", 0);
  const int st = env_int("SCN_MAX_STAGES", kDefaultStages);
  k.max_stages = st >= 2 ? st : kDefaultStages;
  const int pf = env_int("SCN_L2_PREFETCH", -1);
  if (pf >= 0) k.l2_prefetch_fused = k.l2_prefetch_hist = pf;
  k.prod_sleep = (uint32_t)env_int("SCN_PROD_SLEEP", 0);
  k.gen_warps = env_int("SCN_GEN_WARPS", 0);
  k.gen_stage = env_int("SCN_GEN_STAGE", 1);
  k.gen_half = env_int("SCN_GEN_HALF", 1);
  k.pair_bins = env_int("SCN_PAIR_BINS", 1);
  k.fused_raw = env_int("SCN_FUSED_RAW", 1);
  k.hist_warps = env_int("SCN_HIST_WARPS", 0);
  g_knobs = k;
}
static const Knobs& knobs() {
  std::call_once(g_knobs_once, read_knobs_once);
  return g_knobs;
}
#else
static const Knobs& knobs() { return g_knobs; }
#endif

static std::atomic<int> g_hist_impl{0};  // scn_set_hist_impl: 0 lane-private pair keys, 1 K2a, 2 K2a'
void set_hist_impl(int impl) { g_hist_impl.store(impl, std::memory_order_relaxed); }
int hist_impl() { return g_hist_impl.load(std::memory_order_relaxed); }

static bool divides16(int b) { return b == 1 || b == 2 || b == 4 || b == 8 || b == 16; }

const char* hist_variant_name(int32_t bins) {
  if (divides16(bins)) {
    switch (hist_impl()) {
      case 1: return "k2a_match_per_warp";
      case 2: return "k2a_packed_match_per_warp";
      default: return "tma_pair_lane_private";
    }
  }
  if (bins < 16 && knobs().pair_bins != 0) return "tma_pair_bins_lane_private";
  return "tma_raw_lane_private_remap";
}

template <int MODE, int NW, int VAR = 0>
static cudaError_t launch_tma(HistParams p, cudaStream_t st) {
  auto fn = hist_tma_kernel<MODE, NW, VAR>;
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
  if (knobs().grid > 0 && knobs().grid < grid) grid = knobs().grid;
  if (p.total_tiles < grid) grid = (int)p.total_tiles;
  if (grid < 1) return cudaSuccess;
  fn<<<grid, NW * 32 + 32, p.smem_bytes, st>>>(p);
  return cudaGetLastError();
}

// The kVarGen kernels (any width / output alignment) at the knob's warp count.
template <int MODE>
static cudaError_t launch_gen(const HistParams& p, cudaStream_t st) {
  constexpr int kW = MODE == kModeDs ? kGenDsWarps : kGenFusedWarps;
#ifdef SCN_TUNING
  const int w = knobs().gen_warps;
  if (w == 8 && kW != 8) return launch_tma<MODE, 8, kVarGen>(p, st);
  if (w == 12 && kW != 12) return launch_tma<MODE, 12, kVarGen>(p, st);
  if (w == 16 && kW != 16) return launch_tma<MODE, 16, kVarGen>(p, st);
  if (w == 20 && kW != 20) return launch_tma<MODE, 20, kVarGen>(p, st);
  if (w == 24 && kW != 24) return launch_tma<MODE, 24, kVarGen>(p, st);
#endif
  return launch_tma<MODE, kW, kVarGen>(p, st);
}

// Rows per row-pair tile of the downsample-only kernel: the largest even row count whose
// slots give 4 ring stages (1080p: 8 rows; run with 3 of them), or 2 stages if that is
// under 4 rows; 0 if not even 2 rows fit twice. An explicit tile size (knob) wins.
// Ring-slot bytes of a row-pair tile of r rows: the input rows (+ kGenSlack for kVarGen) and,
// for kVarGen staged stores, the output stage at out_off = ceil16(input) holding the tile's
// r/2 output rows after a 16-byte lead (the head fragment's place, never written).
static uint32_t stage_off(int r, int64_t rowb, uint32_t slack) {
  return (uint32_t)(((int64_t)r * rowb + slack + 15) & ~15ll);
}
static uint32_t slot_bytes(int r, int64_t rowb, uint32_t slack, bool staged) {
  const int64_t in = (int64_t)r * rowb + slack;
  if (!staged) return (uint32_t)in;
  return stage_off(r, rowb, slack) + 16u + (uint32_t)((((int64_t)(r / 2) * (rowb / 6) * 3) + 15) & ~15ll);
}

static int rows_per_tile_ds(int64_t rowb, uint32_t slack, uint32_t env_tile, bool staged) {
  if (env_tile) return (int)((int64_t)env_tile / rowb) & ~1;
  const int64_t ring = (int64_t)g_smem_optin - (int64_t)kCtrlBytes - 2048;
  // round 1 sized the input tile at a quarter of the ring; a staged slot (input + output
  // stage, 1.25x) keeps that input size within a third (the ring runs 3 stages)
  const int64_t cap = staged ? ring / 3 : ring / 4;
  int r = (int)((cap - slack) / rowb) & ~1;
  while (r >= 2 && (int64_t)slot_bytes(r, rowb, slack, staged) > cap) r -= 2;
  if (r < 4) {
    r = (int)((ring / 2 - slack) / rowb) & ~1;
    while (r >= 2 && (int64_t)slot_bytes(r, rowb, slack, staged) > ring / 2) r -= 2;
  }
  return r < 2 ? 0 : r;
}

// Rows per tile for the split layout (make_layout_split, mirrored here with the dynamic
// smem base = the per-block reserved size): the largest even row count (tile <= 64 KB)
// whose slots give >= 3 ring stages over the two ring segments; 0 if none. The device
// recomputes the same layout and traps on < 2 stages.
static int rows_per_tile_split(int64_t rowb, uint32_t slack, uint32_t env_tile, bool staged, bool half = false,
                               uint32_t above = 0) {
  const uint32_t base = (uint32_t)g_smem_reserved, end = base + (uint32_t)g_smem_optin - above;
  const uint32_t t2 = half ? 0u : kTab2Bytes;  // make_layout_half: no tab2 below the block
  const uint32_t block = (base + kCtrlBytes + t2 + 65535u) & ~65535u;
  const uint32_t tab2 = block - t2, ring = (base + kCtrlBytes + 127u) & ~127u, hi = block + 65536u;
  if (hi > end) return 0;
  auto stages = [&](int r) {
    const uint32_t slot = slot_bytes(r, rowb, slack, staged), stride = (slot + 127u) & ~127u;
    const int lo = tab2 >= ring + slot ? (int)((tab2 - ring - slot) / stride) + 1 : 0;
    const int up = end >= hi + slot ? (int)((end - hi - slot) / stride) + 1 : 0;
    return lo + up;
  };
  if (env_tile) {
    const int r = (int)((int64_t)env_tile / rowb) & ~1;
    return r >= 2 && stages(r) >= 2 ? r : 0;
  }
  for (int r = (int)(65536 / rowb) & ~1; r >= 2; r -= 2)
    if (stages(r) >= 3) return r;
  for (int r = (int)(65536 / rowb) & ~1; r >= 2; r -= 2)
    if (stages(r) >= 2) return r;
  return 0;
}

// The aligned row-pair path needs 16-byte aligned rows (W % 16 == 0: rows of 48-byte units)
// and 8-byte aligned output units (pitch and base multiples of 8); anything else takes kVarGen.
static bool rowpair_aligned(int32_t width, int64_t pitch, const uint8_t* out) {
  return width % 16 == 0 && pitch % 8 == 0 && ((uintptr_t)out & 7u) == 0;
}

// kVarGen staged stores need each tile's output rows contiguous (no montage canvas pitch)
static bool staged_ok(int32_t width, int64_t pitch, int32_t ds_cols) {
  return ds_cols == 0 && pitch == (int64_t)(width / 2) * 3 && knobs().gen_stage != 0;
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
  p.joint = j.joint;
  p.smem_bytes = (uint32_t)g_smem_optin;
  p.max_stages = knobs().max_stages;
  p.prod_sleep = knobs().prod_sleep;
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
  p.tile = p.slot = divides16(j.bins) ? knobs().hist_tile : kTile;
  p.rows_per_tile = 0;
  p.tpf = (int32_t)((p.F + p.tile - 1) / p.tile);
  p.total_tiles = p.n_items * p.tpf;
  p.l2_prefetch = knobs().l2_prefetch_hist;
  *launches += 1;
  if (divides16(j.bins)) {
    switch (hist_impl()) {
      case 1:  // north_star K2a: per-warp bins + __match_any_sync per byte
        p.table_bytes = (uint32_t)kHistWarps * 48u * 4u;
        p.table_align = 128u;
        return launch_tma<kModeMatch, kHistWarps>(p, st);
      case 2:  // K2a': one __match_any_sync per packed word of four pair keys
        p.table_bytes = (uint32_t)kHistWarps * 768u * 4u;
        p.table_align = 128u;
        return launch_tma<kModeMatchPacked, kHistWarps>(p, st);
      default:
        p.table_bytes = 3u * 256u * 128u;  // 64 KB PRMT block (channels 0/1) + 32 KB channel 2
        p.table_align = 65536u;
#ifdef SCN_TUNING
        if (knobs().hist_warps == 8) return launch_tma<kModePair, 8>(p, st);
        if (knobs().hist_warps == 20) return launch_tma<kModePair, 20>(p, st);
#endif
        return launch_tma<kModePair, kHistWarps>(p, st);
    }
  }
  p.table_bytes = 3u * 256u * 128u;
  p.table_align = 65536u;
  if (j.bins < 16 && knobs().pair_bins != 0) return launch_tma<kModePairB, kHistWarps>(p, st);  // K2b
#ifdef SCN_TUNING
  if (knobs().hist_warps == 8) return launch_tma<kModeRaw, 8>(p, st);
  if (knobs().hist_warps == 20) return launch_tma<kModeRaw, 20>(p, st);
#endif
  return launch_tma<kModeRaw, kHistWarps>(p, st);
}

// NEXT N4 joint-colour histogram: J bins per channel (1..8), J^3 lane-private rows.
cudaError_t launch_histogram_joint(const HistJob& j, cudaStream_t st, int* launches) {
  cudaError_t e = device_props();
  if (e != cudaSuccess) return e;
  if (j.n_items <= 0) return cudaSuccess;
  HistParams p = base_params(j);
  p.ds_out = nullptr;
  p.tile = p.slot = kTile;
  p.rows_per_tile = 0;
  p.tpf = (int32_t)((p.F + p.tile - 1) / p.tile);
  p.total_tiles = p.n_items * p.tpf;
  p.l2_prefetch = knobs().l2_prefetch_hist;
  p.table_bytes = (uint32_t)(j.joint * j.joint * j.joint) * 128u;
  p.table_align = 128u;  // row address = table + key * 128 + lane * 4 (LEA), any alignment
  *launches += 1;
  return launch_tma<kModeJoint, kHistWarps>(p, st);
}

// Row-pair tiling of frames for the fused / downsample-only kernels.
static void rowpair_tiles(HistParams& p, int rpt, bool gen, bool staged) {
  const int64_t rowb = (int64_t)p.width * 3;
  if (rpt > p.height) rpt = p.height + (p.height & 1);  // whole frame in one tile
  p.rows_per_tile = rpt;
  p.tile = (uint32_t)(rpt * rowb);
  const uint32_t slack = gen ? kGenSlack : 0u;
  p.slot = slot_bytes(rpt, rowb, slack, staged);
  p.out_off = staged ? stage_off(rpt, rowb, slack) : 0u;
  p.tpf = (p.height + rpt - 1) / rpt;
  p.total_tiles = p.n_items * p.tpf;
  p.l2_prefetch = knobs().l2_prefetch_fused;
}

cudaError_t launch_downsample(const FrameSrc& src, int64_t n, int32_t width, int32_t height, uint8_t* out,
                              cudaStream_t st, int* launches, int64_t ds_pitch, int32_t ds_cols) {
  const int64_t pitch = ds_pitch > 0 ? ds_pitch : (int64_t)(width / 2) * 3;
  cudaError_t e = device_props();
  if (e != cudaSuccess) return e;
  if (n <= 0 || width < 2 || height < 2) return cudaSuccess;
  const bool gen = !rowpair_aligned(width, pitch, out);
  const bool staged = gen && staged_ok(width, pitch, ds_cols);
  const int rpt = rows_per_tile_ds((int64_t)width * 3, gen ? kGenSlack : 0u, knobs().ds_tile, staged);
  *launches += 1;
  if (rpt < 2) {  // rows too wide for a ring slot
    const int64_t rows = n * (height / 2);
    const int grid = rows < (int64_t)g_num_sms * 8 ? (int)rows : g_num_sms * 8;
    downsample_wide_kernel<<<grid, 256, 0, st>>>(src, n, width, height, out, pitch, ds_cols);
    return cudaGetLastError();
  }
  HistJob j{};
  j.ds_pitch = pitch;
  j.ds_cols = ds_cols;
  j.src = src;
  j.n_items = n;
  j.ds_out = out;
  j.width = width;
  j.height = height;
  j.bins = 16;
  HistParams p = base_params(j);
  rowpair_tiles(p, rpt, gen, staged);
  p.l2_prefetch = 0;  // measured: the downsample-only kernel keeps 0
  p.table_bytes = 0;
  p.table_align = 128;
  return gen ? launch_gen<kModeDs>(p, st) : launch_tma<kModeDs, kDsWarps>(p, st);
}

cudaError_t launch_hist_downsample(const HistJob& j, cudaStream_t st, int* launches) {
  cudaError_t e = device_props();
  if (e != cudaSuccess) return e;
  if (j.n_items <= 0) return cudaSuccess;
  const int64_t pitch = j.ds_pitch > 0 ? j.ds_pitch : (int64_t)(j.width / 2) * 3;
  const bool gen = !rowpair_aligned(j.width, pitch, j.ds_out);
  // the realigning fused kernel keeps direct stores: its ring slots are worth more as input
  // (a staged slot would cost two rows per tile; measured slower, DESIGN.md §5 kVarGen)
  const bool staged = false;
  int rpt = rows_per_tile_split((int64_t)j.width * 3, gen ? kGenSlack : 0u, knobs().fused_tile, staged);
  // The realigning kernel pays a per-tile cost (tails, frame bookkeeping, the slot hand-off) that
  // bigger tiles amortise: where the half-lane 64 KB block admits more rows per tile than the
  // split 80 KB table AND that tile holds at most one unit pair per thread of 16 consumer
  // warps (no warp runs a second, mostly idle iteration and holds the slot), take it
  // (measured same box, profiles/r02_tune_gen2.jsonl: 1366x768 10 -> 12 rows = 510 unit
  // pairs, +6.6 %; 426x240 36 -> 40 rows = 520 pairs, 16 warps -12 %: kept on the split
  // table; 854x480 gains no rows: the half-lane block alone costs 1.5 % in bank conflicts)
  bool half = false;
  if (gen && knobs().fused_tile == 0 && knobs().gen_half != 0) {
    const int rh = rows_per_tile_split((int64_t)j.width * 3, kGenSlack, 0, staged, true);
    const int64_t pairs = (int64_t)(rh / 2) * (j.width / 16);
    if (rh > rpt && rpt < j.height && pairs <= 32 * kGenHalfWarps) {
      half = true;
      rpt = rh;
    }
  }
  // B < 16 not dividing 16 fuse too, with K2b's pair keys of B-level bins (kVarBins); B > 16 with
  // raw byte keys in the split table (kVarRaw; K2r's 96 KB table leaves no ring), the bin counters
  // at the top of shared memory. Measured (profiles/r02_tune_hist_k2b.jsonl): C4 1080p B = 100
  // 5.60 TB/s vs 3.80 for histogram + downsample passes (a half-lane 64 KB block: 4.55),
  // 1366x768 4.12 vs 3.84, 854x480 3.93 vs 3.59
  const bool bins = !divides16(j.bins) && j.bins < 16 && knobs().pair_bins != 0;
  const bool raw = j.bins > 16 && knobs().fused_raw != 0;
  if (raw) {  // the split table with the bin counters reserved at the top (kRemapBytes)
    rpt = rows_per_tile_split((int64_t)j.width * 3, gen ? kGenSlack : 0u, knobs().fused_tile, staged, false,
                              kRemapBytes);
    half = false;
  }
  const bool fused = ((divides16(j.bins) && hist_impl() == 0) || bins || raw) && rpt >= 2 && j.n_halo == 0 &&
                     j.width >= 2 && j.height >= 2;
  if (!fused) {  // two passes: histogram, then downsample
    HistJob h = j;
    h.ds_out = nullptr;
    e = launch_histogram(h, st, launches);
    if (e != cudaSuccess) return e;
    FrameSrc src = j.src;
    src.ptrs = src.ptrs ? src.ptrs + j.n_halo : nullptr;
    src.base += src.ptrs ? 0 : (uint64_t)j.n_halo * src.stride;
    return launch_downsample(src, j.n_items - j.n_halo, j.width, j.height, j.ds_out, st, launches, j.ds_pitch,
                             j.ds_cols);
  }
  HistParams p = base_params(j);
  rowpair_tiles(p, rpt, gen, staged);
  p.table_bytes = half ? 65536u : kTab2Bytes + 65536u;  // (tab2 +) the key block, zeroed as one range
  p.table_align = 65536u;
  *launches += 1;
  if (raw)
    return gen ? launch_tma<kModeFused, kGenFusedWarps, kVarGen | kVarRaw>(p, st)
               : launch_tma<kModeFused, kDsWarps, kVarRaw>(p, st);
  if (bins) {
    if (half) return launch_tma<kModeFused, kGenHalfWarps, kVarGen | kVarHalf | kVarBins>(p, st);
    return gen ? launch_tma<kModeFused, kGenFusedWarps, kVarGen | kVarBins>(p, st)
               : launch_tma<kModeFused, kDsWarps, kVarBins>(p, st);
  }
  if (half) return launch_tma<kModeFused, kGenHalfWarps, kVarGen | kVarHalf>(p, st);
  return gen ? launch_gen<kModeFused>(p, st) : launch_tma<kModeFused, kDsWarps>(p, st);
}

cudaError_t launch_shotdiff(const uint32_t* hist, const uint32_t* halo_row, const uint8_t* seg, int64_t n,
                            int32_t row, const DestList& d, cudaStream_t st, int* launches) {
  if (n <= 0) return cudaSuccess;
  *launches += 1;
  shotdiff_kernel<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(hist, halo_row, seg, n, row, d);
  return cudaGetLastError();
}

cudaError_t launch_diff_pairs(const uint32_t* hist, const int64_t* a, const int64_t* b, int64_t n, int32_t bins,
                              uint32_t* diff, cudaStream_t st, int* launches) {
  if (n <= 0) return cudaSuccess;
  *launches += 1;
  diff_pairs_kernel<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(hist, a, b, n, bins, diff);
  return cudaGetLastError();
}

// NEXT N3: adaptive shot detector, a bounded-state op with warmup W.
// State = window of the last W_eff = min(W, q - table start) shot-diffs; the
// shard's first W positions before q0 are warmup: read, never written. The host
// bounds W * (k_num + k_den) < 2^32, so both sides of the test fit in 64 bits.
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

}  // namespace scn
