/* scn.h — C ABI of libscn.so: the B200-native data-parallel hot path of
 * Scanner (Poms et al., arXiv 1805.07339): sampled-frame HIST, [-1,0]
 * histogram-difference shot scoring and 2x box downsample over video tables.
 *
 * Citations: P:L### = PAPER.md line (section named), S:L### = SPEC.md line.
 * Readings Q# of silent/ambiguous passages: DESIGN.md §3.
 *
 * Conventions (all entry points):
 *   - Plain C types only; no torch types. Device pointers are CUDA device
 *     addresses owned by the caller (PyTorch allocates them); the library never
 *     allocates device memory and never frees caller memory.
 *   - Host objects (scn_table, scn_seq) are created by scn_*_create /
 *     scn_sample_* / scn_seq_concat and freed by the matching *_destroy.
 *   - scn_run_* only ENQUEUE work on the given stream (cudaStream_t passed as
 *     void*; NULL = legacy default stream); they never synchronise the device.
 *     Results are valid once the stream has been synchronised. Buffers must
 *     stay alive until then.
 *   - Errors: every call returns a scn_status; nothing throws across the ABI.
 *     scn_last_error() returns a thread-local message for the last non-OK
 *     status. A CUDA launch/runtime failure returns SCN_ECUDA.
 *   - Determinism: every output is an exact integer function of the input;
 *     it does not depend on the shard boundaries, the launch configuration or
 *     the number of GPUs.
 *   - Devices: kernels launch on the calling thread's current CUDA device; the
 *     stream and every device buffer passed to a call must belong to it (peer
 *     destinations of scn_run_hist_shotdiff_to excepted: those are mapped peer
 *     addresses). One process per GPU is the intended layout.
 *   - Threads: a table or sequence may be used by several threads at once for
 *     runs (runs only read it); creating, uploading or destroying it must not
 *     race with other use. scn_last_error / scn_last_launch_count are per
 *     thread.
 */
#ifndef SCN_H
#define SCN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SCN_OK = 0,
  SCN_EINVAL = 1,        /* malformed argument (see each call) */
  SCN_ERANGE = 2,        /* index outside [0,N), absent sparse row, end > M */
  SCN_ECUDA = 3,         /* CUDA launch / copy failure */
  SCN_EUNSUPPORTED = 4   /* bins outside [1,256] */
} scn_status;

typedef enum { SCN_MEM_DEVICE = 0, SCN_MEM_HOST = 1 } scn_mem;

typedef struct scn_table scn_table; /* opaque host-side table metadata */
typedef struct scn_seq scn_seq;     /* opaque sampled sequence */
typedef struct { int64_t start, end; } scn_block; /* half-open row block [start,end) */

const char* scn_last_error(void);
const char* scn_version(void);

/* ---------------------------------------------------------------------------
 * Tables. "Scanner represents video collections ... as tables" with "one row
 * per video frame" (§3). A table binds num_rows RGB8 frames,
 * HWC layout (row-major pixels, 3 bytes R,G,B), width*height*3 = F bytes each.
 *   dense mode : base != NULL, row r at base + r*frame_stride_bytes;
 *                frame_stride_bytes >= F and a multiple of 16; base 16-aligned.
 *   sparse mode: base == NULL, row_ptrs[r] = address of row r or 0 if the row
 *                is not resident (only sampled rows need to be, "only a
 *                sparse set of intermediate sequence elements must be
 *                computed"). Non-zero pointers must be 16-aligned. row_ptrs is
 *                copied.
 *   Every resident row must be readable for ceil16(F) bytes (the TMA bulk
 *   copies move whole 16-byte granules).
 *   where = SCN_MEM_DEVICE: rows are in HBM (scn_run_*).
 *   where = SCN_MEM_HOST:   rows are in (preferably pinned) host memory
 *                           (scn_run_pipeline_host only).
 * Errors: EINVAL if num_rows < 0, width/height < 1, channels != 3,
 *   width*height > 715827882 (the u32 shot-diff bound 6*W*H, reading Q13),
 *   a bad stride or misaligned pointer, or both/neither of base/row_ptrs.
 * ------------------------------------------------------------------------- */
scn_status scn_table_create(int64_t num_rows, int32_t width, int32_t height, int32_t channels, int32_t where,
                            const void* base, int64_t frame_stride_bytes, const uint64_t* row_ptrs,
                            scn_table** out);
void scn_table_destroy(scn_table* t);
int64_t scn_table_rows(const scn_table* t);

/* ---------------------------------------------------------------------------
 * Sampling (§3.2 "Sampling operations ... can be defined by strides,
 * ranges, or index lists"). The result is a sequence of M positions [0,M)
 * (P:L201-202), position j bound to one table row. The frame address of each
 * position is resolved at creation, so the table may be destroyed afterwards.
 *   stride : rows {0, s, 2s, ...} < N (reading Q8); EINVAL if s < 1.
 *   range  : for each block [a,b) in order, rows a, a+step, ... < b (reading
 *            Q9); blocks sorted and disjoint (EINVAL), 0 <= a <= b <= N
 *            (ERANGE), step >= 1 (EINVAL).
 *   gather : the given rows, strictly increasing (EINVAL), in [0,N) (ERANGE)
 *            (reading Q10).
 * In sparse mode a sampled row may be absent (pointer 0); any scn_run_* that
 * reads an absent position returns ERANGE (residency is checked per run, i.e.
 * per work packet, "dependency analysis incrementally (at work packet
 * granularity)"), so each rank only materialises its own shard.
 * ------------------------------------------------------------------------- */
scn_status scn_sample_stride(const scn_table* t, int64_t stride, scn_seq** out);
scn_status scn_sample_range(const scn_table* t, const scn_block* blocks, int64_t n_blocks, int64_t step,
                            scn_seq** out);
scn_status scn_sample_gather(const scn_table* t, const int64_t* rows, int64_t n, scn_seq** out);

/* Concatenate per-table sequences into one job sequence (one job
 * per video, all scheduled together). Each part is its own slice: the stencil
 * never crosses parts (reading Q6). Parts must share width, height and
 * memory location (EINVAL). Parts are copied; they may be destroyed after. */
scn_status scn_seq_concat(const scn_seq* const* parts, int32_t n, scn_seq** out);

int64_t scn_seq_length(const scn_seq* s);
/* Introspection: part index and table row of every position (host arrays of
 * length M; either may be NULL), and segment-start flags (1 at the first
 * position of each part). */
scn_status scn_seq_rows(const scn_seq* s, int32_t* part, int64_t* row);
scn_status scn_seq_seg_starts(const scn_seq* s, uint8_t* flags);

/* Contiguous shard of positions for rank r of G (reading
 * Q17): [floor(r*M/G), floor((r+1)*M/G)). EINVAL if G < 1 or r outside [0,G). */
scn_status scn_shard_range(int64_t m, int32_t world, int32_t rank, int64_t* begin, int64_t* end);
/* 1 if the [-1,0] stencil at position `begin` needs the halo position
 * begin-1 (begin > 0 and begin is not a segment start), else 0 (P:L214 warmup
 * as redundant work; P:L255 the warmup is "treated like a stencil"). */
int32_t scn_seq_needs_halo(const scn_seq* s, int64_t begin);

/* Device metadata for scn_run_*: per-position frame address (u64) and
 * segment-start flag (u8). scn_seq_device_bytes() bytes of caller-owned
 * device memory; the upload is enqueued on `stream` and the workspace must
 * stay alive while runs use it. Host-location sequences need no upload. */
size_t scn_seq_device_bytes(const scn_seq* s);
scn_status scn_seq_upload(scn_seq* s, void* d_workspace, size_t bytes, void* stream);
void scn_seq_destroy(scn_seq* s);

/* ---------------------------------------------------------------------------
 * Runs over positions [begin, end) of an uploaded device-location sequence
 * (one rank's shard). Outputs hold rows for [begin,end) only, row j-begin for
 * position j. EINVAL if begin > end, not uploaded, or a host-location seq;
 * ERANGE if end > M; EUNSUPPORTED if bins outside [1,256].
 * ------------------------------------------------------------------------- */

/* HIST (§5.1.2 "Compute and store the pixel color histogram for all
 * frames"): d_hist[j][c][b] (u32, [end-begin][3][bins]) = number of pixels of
 * frame j whose channel c value v has floor(v*bins/256) == b (readings
 * Q1-Q3). d_hist is zeroed by the call. */
scn_status scn_run_histogram(const scn_seq* s, int64_t begin, int64_t end, int32_t bins, uint32_t* d_hist,
                             void* stream);

/* NEXT N4, joint-colour variant (SURVEY §8(f) N4 "256-bin per-channel (or
 * joint-colour) histogram"; "pixel color histogram", the joint
 * alternative of reading Q3): d_hist[j][k] (u32, [end-begin][J^3], J =
 * bins_per_channel) = number of pixels of frame j whose colour (R,G,B) has
 * k = bin(R)*J*J + bin(G)*J + bin(B), bin(v) = floor(v*J/256) (reading Q2).
 * d_hist is zeroed by the call. EUNSUPPORTED if J is outside [1,8] (the
 * lane-private table holds J^3 <= 512 rows). */
scn_status scn_run_histogram_joint(const scn_seq* s, int64_t begin, int64_t end, int32_t bins_per_channel,
                                   uint32_t* d_hist, void* stream);

/* Shot-diff over joint-colour histograms (NEXT N4 joint variant with the same
 * [-1,0] L1 stencil as scn_run_shotdiff, P:L455 / P:L210, readings Q6, Q7):
 * d_hist as scn_run_histogram_joint ([end-begin][J^3] u32, zeroed by the call);
 * d_diff[j] (u32) = sum_k |H[j][k] - H[j-1][k]| over the J^3 counters, 0 at
 * the first position of a part. If scn_seq_needs_halo(s, begin), the joint
 * histogram of position begin-1 rides in the same launch into d_scratch
 * (>= J^3 u32; recomputed, not communicated). EUNSUPPORTED if J is
 * outside [1,8]; EINVAL on NULL d_hist / d_diff (or d_scratch when a halo is
 * needed); ERANGE if a read position is not resident. */
scn_status scn_run_hist_shotdiff_joint(const scn_seq* s, int64_t begin, int64_t end, int32_t bins_per_channel,
                                       uint32_t* d_hist, uint32_t* d_diff, uint32_t* d_scratch, void* stream);

/* Shot-diff ("detect shot boundaries (via histogram differences)") as
 * a [-1,0] stencil over the sampled sequence (fig:sampling-f; reading
 * Q7): d_diff[j] (u32) = sum_c sum_b |H[j][c][b] - H[j-1][c][b]|, and 0 at the
 * first position of a part (reading Q6). d_hist holds rows [begin,end) from
 * scn_run_histogram with the same bins. If scn_seq_needs_halo(s, begin), the
 * histogram of position begin-1 is recomputed into d_scratch (>= 3*bins u32)
 * rather than communicated (the shard's halo). */
scn_status scn_run_shotdiff(const scn_seq* s, int64_t begin, int64_t end, int32_t bins, const uint32_t* d_hist,
                            uint32_t* d_diff, uint32_t* d_scratch, void* stream);

/* HIST and shot-diff in one pass: the halo frame (if any) rides in the same
 * histogram launch as the shard's frames. Same outputs as the two calls. */
scn_status scn_run_hist_shotdiff(const scn_seq* s, int64_t begin, int64_t end, int32_t bins, uint32_t* d_hist,
                                 uint32_t* d_diff, uint32_t* d_scratch, void* stream);

/* HIST + shot-diff with the result all-gather fused in (north_star: "Only the
 * final per-frame result columns are gathered"): instead of writing this
 * rank's rows to a local buffer for a later collective, the histogram flush
 * and the shot-diff kernel write rows [begin,end) straight into every rank's
 * full result columns. h_hist_dests[g] / h_diff_dests[g] (g < n_dest <= 16)
 * are device addresses of rank g's [M][3][bins] u32 and [M] u32 columns —
 * local memory for g == self, CUDA-IPC-mapped peer memory otherwise (NVLink
 * loads/stores/atomics on a multi-GPU node). The call zeroes this rank's rows
 * in every destination, accumulates the histogram with red.global.add, reads
 * its own rows back from h_hist_dests[self] for the [-1,0] stencil (the halo
 * is recomputed into d_scratch) and stores D into every destination.
 * Rows owned by other ranks are never touched, so ranks need no
 * synchronisation until they read the gathered columns (after a barrier).
 * EINVAL if n_dest outside [1,16], self outside [0,n_dest), or a NULL /
 * misaligned destination. */
scn_status scn_run_hist_shotdiff_to(const scn_seq* s, int64_t begin, int64_t end, int32_t bins,
                                    const uint64_t* h_hist_dests, const uint64_t* h_diff_dests, int32_t n_dest,
                                    int32_t self, uint32_t* d_scratch, void* stream);

/* Peer destinations for scn_run_hist_shotdiff_to: map another process's device
 * allocation (a 64-byte cudaIpcMemHandle_t exported by its owner, plus the byte
 * offset of the column inside that allocation) into this process, opened in the
 * calling thread's CURRENT device context with lazy peer access (NVLink P2P when
 * the owner is another GPU). *d_base is the mapping to release, *d_ptr = base +
 * offset. The library allocates nothing: this only maps memory the peer owns. */
scn_status scn_ipc_import(const void* handle, int64_t offset, uint64_t* d_base, uint64_t* d_ptr);
scn_status scn_ipc_release(uint64_t d_base);

/* 2x integer box downsample ("downsamples the resulting frames
 * (Resize)"): d_out[j] (u8, [end-begin][H/2][W/2][3]) with
 * O[y][x][c] = (P(2y,2x)+P(2y,2x+1)+P(2y+1,2x)+P(2y+1,2x+1)+2) >> 2; a
 * trailing odd row/column is dropped (reading Q11). Any width and any d_out
 * alignment (byte granularity): W % 16 == 0 with an 8-byte aligned d_out takes
 * the aligned row-pair kernel, everything else its realigning variant. */
scn_status scn_run_downsample(const scn_seq* s, int64_t begin, int64_t end, uint8_t* d_out, void* stream);

/* HIST + downsample of the same sampled frames in one read of each frame
 * (reading Q12: siblings over the sampled full-resolution frame). Outputs
 * identical to scn_run_histogram + scn_run_downsample. */
scn_status scn_run_hist_downsample(const scn_seq* s, int64_t begin, int64_t end, int32_t bins, uint32_t* d_hist,
                                   uint8_t* d_out, void* stream);

/* ---------------------------------------------------------------------------
 * End-to-end run over a HOST-location sequence: frames are streamed
 * host->device in chunks through the caller's staging buffer, double-buffered
 * so the copy of chunk k+1 overlaps the kernels on chunk k (P:L248
 * "pipelining of CPU-GPU data transfers ... with graph operation execution").
 *   ops: bit 0 = HIST, bit 1 = shot-diff (needs HIST), bit 2 = downsample.
 *   d_staging: caller device memory, 16-byte aligned, staging_bytes >=
 *              ceil16(end - begin) + 2 * ceil16(F): the first ceil16(end-begin)
 *              bytes hold the shard's segment-start flags, the rest two chunk
 *              slots of at least one frame each (more = larger chunks).
 *   d_scratch: >= 3*bins u32 when shot-diff needs a halo.
 *   copy_stream: second stream for the H2D copies (may equal stream).
 * Outputs as the device-location calls. Only enqueues work (host frames
 * must stay valid until `stream` completes).
 * ------------------------------------------------------------------------- */
#define SCN_OP_HIST 1u
#define SCN_OP_SHOTDIFF 2u
#define SCN_OP_DOWNSAMPLE 4u
scn_status scn_run_pipeline_host(const scn_seq* s, int64_t begin, int64_t end, int32_t bins, uint32_t ops,
                                 uint32_t* d_hist, uint32_t* d_diff, uint8_t* d_out, uint32_t* d_scratch,
                                 void* d_staging, size_t staging_bytes, void* stream, void* copy_stream);

/* ---------------------------------------------------------------------------
 * NEXT N2 — stencil BEFORE sampling (fig:sampling-e; "sampling after
 * the flow operation yields a sparse set of flow fields computed from
 * differences between original video frames"). Graph: table -> HIST ->
 * [offset,0] stencil -> Sample. For the sampled sequence s (rows S per part),
 * computes the exact required HIST input set R = S U clamp(S + offset) per
 * table (per-element dependency analysis; repeat-edge clamp to
 * [0, N-1], reading Q6) as a new sequence `required` (per part sorted and
 * unique, rows resolved through the table s was sampled from; the caller
 * destroys it), and for every position j of s the positions in `required` of
 * S_j (h_pos[j]) and of its neighbour (h_nbr[j]); both host arrays hold M.
 * Then D'[j] = sum |H[h_pos[j]] - H[h_nbr[j]]| with scn_run_histogram over
 * `required` and scn_run_diff_pairs.
 * ------------------------------------------------------------------------- */
scn_status scn_seq_stencil_required(const scn_seq* s, int32_t offset, scn_seq** required, int64_t* h_pos,
                                    int64_t* h_nbr);
/* d_diff[j] = sum_c sum_b |d_hist[d_a[j]][c][b] - d_hist[d_b[j]][c][b]| (u32) for j < n;
 * d_a/d_b: device int64 row indices into d_hist ([rows][3][bins]). */
scn_status scn_run_diff_pairs(const uint32_t* d_hist, const int64_t* d_a, const int64_t* d_b, int64_t n,
                              int32_t bins, uint32_t* d_diff, void* stream);

/* ---------------------------------------------------------------------------
 * NEXT N3 — a bounded-state operation with warmup W (the op is
 * guaranteed to have produced "at least the previous W elements"; a split at a
 * packet boundary recomputes W warmup elements and discards them, P:L214,
 * "treated like a stencil operation with the footprint (i-W,...,i-1,i)",
 * P:L255). The op is an adaptive shot detector over the shot-diff column:
 *   cut[p] = W_eff > 0 and D[p]*W_eff*k_den > k_num*sum(D[p-W_eff..p-1]) + floor*W_eff*k_den
 * with W_eff = min(W, p - first position of p's table) (tables are slices,
 * P:L216), evaluated exactly in 64-bit (S:L357-364 sliding_mean/threshold).
 *
 * scn_seq_warmup_begin returns wb = the first position whose D a shard
 * starting at `begin` needs: max(begin - W, first position of begin's table).
 * scn_run_adaptive_cuts: d_diff holds D for positions [wb, end) (e.g. from
 * scn_run_hist_shotdiff over [wb, end), whose own [-1,0] halo is recomputed);
 * d_cut (u8, [end-begin]) gets the flags for [begin, end) only — the warmup
 * outputs are never written. EINVAL if warmup < 1, k_den < 1 or
 * warmup * (k_num + k_den) >= 2^32 (the bound that keeps both sides of the
 * comparison below 2^64, so it is exact).
 * ------------------------------------------------------------------------- */
int64_t scn_seq_warmup_begin(const scn_seq* s, int64_t begin, int32_t warmup);
scn_status scn_run_adaptive_cuts(const scn_seq* s, int64_t begin, int64_t end, int32_t warmup,
                                 const uint32_t* d_diff, uint32_t k_num, uint32_t k_den, uint32_t floor_,
                                 uint8_t* d_cut, void* stream);

/* ---------------------------------------------------------------------------
 * NEXT N1 — two-job shot montage ("detect shot boundaries (via
 * histogram differences) ... produce film summaries via montage"; P:L457:
 * histograms on every frame, then "sparsely computed ... on a single frame per
 * shot"). A graph cannot filter data-dependently, so this is two
 * jobs with host selection in between:
 *   job 1: scn_run_hist_shotdiff -> D (copied to the host);
 *   scn_select_shot_starts: positions p in [begin,end) with seg_start[p] or
 *     h_diff[p-begin] > tau (threshold_detector, reading Q5) are
 *     written to h_pos (up to cap); *count = how many there are;
 *   scn_seq_gather_positions: job 2's Gather over the sequence's own positions
 *     (strictly increasing, EINVAL; in [0,M), ERANGE) -> a new sequence
 *     (sampling composes; a table change starts a new part);
 *   scn_run_montage: 2x box downsample (as scn_run_downsample) of positions
 *     [begin,end), written as tiles into d_canvas: tile k (k = j - begin) at
 *     tile-row k / cols, tile-column k % cols; canvas_pitch = bytes between
 *     canvas rows (>= cols*(W/2)*3, EINVAL); the call zeroes the
 *     ceil(k/cols)*(H/2) canvas rows it covers first.
 * ------------------------------------------------------------------------- */
scn_status scn_select_shot_starts(const scn_seq* s, int64_t begin, int64_t end, const uint32_t* h_diff, uint32_t tau,
                                  int64_t* h_pos, int64_t cap, int64_t* count);
scn_status scn_seq_gather_positions(const scn_seq* s, const int64_t* h_pos, int64_t n, scn_seq** out);
scn_status scn_run_montage(const scn_seq* s, int64_t begin, int64_t end, int32_t cols, uint8_t* d_canvas,
                           int64_t canvas_pitch, void* stream);

/* Launch statistics for the last scn_run_* call on this thread: number of
 * kernels launched (for bench.py's gpu_launches count). */
int32_t scn_last_launch_count(void);

/* ---------------------------------------------------------------------------
 * Histogram implementation for bins dividing 16 (process-wide; results are
 * identical, only the speed differs — DESIGN.md §5):
 *   SCN_HIST_LANE_PAIRS   (default) lane-private pair-key bins, 0.5 shared
 *                         atomics per byte, one global merge per CTA and frame;
 *   SCN_HIST_MATCH        north_star's per-warp bins with __match_any_sync
 *                         aggregation per byte (K2a);
 *   SCN_HIST_MATCH_PACKED K2a with one __match_any_sync per packed word of four
 *                         pair keys (K2a').
 * Other bin counts always take the raw-value kernel (any B in [1,256], bins
 * merged at the per-frame flush). EINVAL for an unknown value.
 * scn_hist_variant names the kernel a run with `bins` takes.
 * ------------------------------------------------------------------------- */
#define SCN_HIST_LANE_PAIRS 0
#define SCN_HIST_MATCH 1
#define SCN_HIST_MATCH_PACKED 2
scn_status scn_set_hist_impl(int32_t impl);
int32_t scn_get_hist_impl(void);
const char* scn_hist_variant(int32_t bins);

#ifdef __cplusplus
}
#endif
#endif /* SCN_H */
