// kernels.h — internal launch interface between the C-ABI host code
// (scn_api.cpp) and the sm_100a kernels (kernels.cu). Not part of the ABI.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace scn {

// Where frame i of a launch lives: ptrs[i] if ptrs != nullptr, else base + i*stride.
struct FrameSrc {
  const uint64_t* ptrs;
  uint64_t base;
  uint64_t stride;
};

struct HistJob {
  FrameSrc src;
  int64_t n_items;     // frames in this launch
  int32_t n_halo;      // the first n_halo items write to halo_out instead of out
  uint32_t* out;       // [n_items - n_halo][3][bins]
  uint32_t* halo_out;  // [n_halo][3][bins]
  uint8_t* ds_out;     // fused downsample output [n_items - n_halo][H/2][W/2][3] or nullptr
  int32_t width, height, bins;
  int32_t joint;       // launch_histogram_joint: J bins per channel (rows of J^3 counters)
  int64_t ds_pitch;    // bytes between output rows (0: (W/2)*3, contiguous frames)
  int32_t ds_cols;     // > 0: montage, frame i is tile (i / cols, i % cols) of a canvas (NEXT N1)
  int32_t n_dest;      // > 0: non-halo rows go to every dest[g] (row 0 = item n_halo) instead of out
  uint64_t dest[16];   // device addresses, local or CUDA-IPC-mapped peer memory (fused all-gather)
};
constexpr int kMaxDest = 16;
struct DestList {
  int32_t n;
  uint64_t p[kMaxDest];
};
// zero `words` u32 at each destination (peer stores for mapped peers)
cudaError_t launch_zero_dests(const DestList& d, int64_t words, cudaStream_t st, int* launches);

// Histogram (zeroes nothing: the caller memsets out/halo_out first).
// Returns the number of kernel launches in *launches.
cudaError_t launch_histogram(const HistJob& job, cudaStream_t st, int* launches);
// NEXT N4 joint-colour histogram (job.joint = J in [1, 8]; out rows of J^3 counters, zeroed by the caller).
cudaError_t launch_histogram_joint(const HistJob& job, cudaStream_t st, int* launches);
// Fused HIST + downsample; falls back to two passes for shapes the fused kernel does not take.
cudaError_t launch_hist_downsample(const HistJob& job, cudaStream_t st, int* launches);
// Shot-diff over n positions of `row` u32 counters each (3*B, or J^3 joint), D[p] written to every d.p[g] + p (d.n = 1 for a plain run);
// seg[p] != 0 marks a segment start; halo_row is the histogram of the position before the
// first (used iff !seg[0]).
cudaError_t launch_shotdiff(const uint32_t* hist, const uint32_t* halo_row, const uint8_t* seg, int64_t n,
                            int32_t row, const DestList& d, cudaStream_t st, int* launches);
// D[j] = sum |H[a[j]] - H[b[j]]| (NEXT N2: stencil before sampling)
cudaError_t launch_diff_pairs(const uint32_t* hist, const int64_t* a, const int64_t* b, int64_t n, int32_t bins,
                              uint32_t* diff, cudaStream_t st, int* launches);
// NEXT N3: cut[q - q0] for q in [q0, n) of a window starting at the warmup begin;
// diff/seg are indexed from the warmup begin (0).
cudaError_t launch_adaptive_cuts(const uint32_t* diff, const uint8_t* seg, int64_t q0, int64_t n, int32_t warmup,
                                 uint32_t k_num, uint32_t k_den, uint32_t floor_, uint8_t* cut, cudaStream_t st,
                                 int* launches);
cudaError_t launch_downsample(const FrameSrc& src, int64_t n, int32_t width, int32_t height, uint8_t* out,
                              cudaStream_t st, int* launches, int64_t ds_pitch = 0, int32_t ds_cols = 0);

// Histogram implementation (scn_set_hist_impl): 0 = lane-private pair keys (default),
// 1 = the north_star's per-warp bins + __match_any_sync per byte (K2a), 2 = K2a with one
// MATCH per packed word of four pair keys (K2a'). Applies to bins dividing 16.
void set_hist_impl(int impl);
int hist_impl();

// Variant names for reporting
const char* hist_variant_name(int32_t bins);

}  // namespace scn
