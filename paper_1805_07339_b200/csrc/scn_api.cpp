// scn_api.cpp — host side of the C ABI declared in include/scn.h: tables,
// sampling, sequence concatenation (slices P:L216),
// shard math with the [-1,0] halo, validation, and the
// kernel launches (kernels.cu). No device memory is allocated here.
#include "scn.h"

#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <algorithm>
#include <cstring>
#include <memory>
#include <new>
#include <string>
#include <vector>

#include "kernels.h"

namespace {

thread_local std::string g_err;
thread_local int32_t g_launches = 0;

scn_status fail(scn_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

scn_status cuda_fail(cudaError_t e, const char* what) {
  return fail(SCN_ECUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

constexpr int64_t kMaxPixels = 715827882;  // 6*W*H must fit in u32 (reading Q13)

inline int64_t ceil16(int64_t x) { return (x + 15) & ~int64_t(15); }

}  // namespace

struct scn_table {
  int64_t rows;
  int32_t width, height, where;
  bool dense;
  uint64_t base, stride;
  std::vector<uint64_t> ptrs;
  uint64_t addr(int64_t r) const { return dense ? base + (uint64_t)r * stride : ptrs[(size_t)r]; }
};

struct scn_seq {
  int32_t width = 0, height = 0, where = 0;
  std::vector<std::shared_ptr<const scn_table>> tables;  // per part: the sampled table (rows outside S, N2)
  std::vector<uint64_t> addr;  // frame address per position
  std::vector<int32_t> part;   // part index per position
  std::vector<int64_t> row;    // table row per position
  std::vector<uint8_t> seg;    // 1 at the first position of each part
  void* d_ws = nullptr;        // uploaded metadata (addr[M] then seg[M])
  int64_t frame_bytes() const { return (int64_t)width * height * 3; }
};

extern "C" {

const char* scn_last_error(void) { return g_err.c_str(); }
#ifndef SCN_GIT_SHA
#define SCN_GIT_SHA "unknown"
#endif
const char* scn_version(void) { return "scn-b200 0.1 (sm_100a, " SCN_GIT_SHA ")"; }
int32_t scn_last_launch_count(void) { return g_launches; }

scn_status scn_set_hist_impl(int32_t impl) {
  if (impl < SCN_HIST_LANE_PAIRS || impl > SCN_HIST_MATCH_PACKED) return fail(SCN_EINVAL, "unknown hist impl %d", impl);
  scn::set_hist_impl(impl);
  return SCN_OK;
}
int32_t scn_get_hist_impl(void) { return scn::hist_impl(); }
const char* scn_hist_variant(int32_t bins) { return scn::hist_variant_name(bins); }

// ---------------------------------------------------------------------------
// tables
// ---------------------------------------------------------------------------
scn_status scn_table_create(int64_t num_rows, int32_t width, int32_t height, int32_t channels, int32_t where,
                            const void* base, int64_t frame_stride_bytes, const uint64_t* row_ptrs,
                            scn_table** out) {
  if (!out) return fail(SCN_EINVAL, "out is NULL");
  *out = nullptr;
  if (num_rows < 0) return fail(SCN_EINVAL, "num_rows < 0");
  if (width < 1 || height < 1) return fail(SCN_EINVAL, "width/height must be >= 1");
  if (channels != 3) return fail(SCN_EINVAL, "channels must be 3 (RGB8), got %d", channels);
  if ((int64_t)width * height > kMaxPixels) return fail(SCN_EINVAL, "width*height exceeds the u32 diff bound");
  if (where != SCN_MEM_DEVICE && where != SCN_MEM_HOST) return fail(SCN_EINVAL, "bad memory location %d", where);
  if ((base == nullptr) == (row_ptrs == nullptr) && num_rows > 0)
    return fail(SCN_EINVAL, "exactly one of base (dense) and row_ptrs (sparse) must be given");
  const int64_t F = (int64_t)width * height * 3;
  scn_table* t = new (std::nothrow) scn_table();
  if (!t) return fail(SCN_EINVAL, "out of host memory");
  t->rows = num_rows;
  t->width = width;
  t->height = height;
  t->where = where;
  t->dense = base != nullptr || num_rows == 0;
  t->base = (uint64_t)(uintptr_t)base;
  t->stride = (uint64_t)frame_stride_bytes;
  if (base) {
    if (frame_stride_bytes < F || frame_stride_bytes % 16 != 0) {
      delete t;
      return fail(SCN_EINVAL, "frame stride %lld must be >= F=%lld and a multiple of 16",
                  (long long)frame_stride_bytes, (long long)F);
    }
    if (t->base % 16 != 0) {
      delete t;
      return fail(SCN_EINVAL, "base must be 16-byte aligned");
    }
  } else if (row_ptrs) {
    t->ptrs.assign(row_ptrs, row_ptrs + num_rows);
    for (int64_t r = 0; r < num_rows; ++r) {
      if (t->ptrs[(size_t)r] % 16 != 0) {
        delete t;
        return fail(SCN_EINVAL, "row pointer %lld not 16-byte aligned", (long long)r);
      }
    }
  }
  *out = t;
  return SCN_OK;
}

void scn_table_destroy(scn_table* t) { delete t; }
int64_t scn_table_rows(const scn_table* t) { return t ? t->rows : -1; }

// ---------------------------------------------------------------------------
// sampling
// ---------------------------------------------------------------------------
static scn_status make_seq(const scn_table* t, const std::vector<int64_t>& rows, scn_seq** out) {
  scn_seq* s = new (std::nothrow) scn_seq();
  if (!s) return fail(SCN_EINVAL, "out of host memory");
  s->width = t->width;
  s->height = t->height;
  s->where = t->where;
  const size_t m = rows.size();
  s->addr.resize(m);
  s->part.assign(m, 0);
  s->row = rows;
  s->seg.assign(m, 0);
  if (m) s->seg[0] = 1;
  s->tables.push_back(std::make_shared<const scn_table>(*t));
  // absent sparse rows (address 0) are allowed here; a run that touches one
  // returns SCN_ERANGE (residency is checked per run, i.e. per work packet)
  for (size_t j = 0; j < m; ++j) s->addr[j] = t->addr(rows[j]);
  *out = s;
  return SCN_OK;
}

scn_status scn_sample_stride(const scn_table* t, int64_t stride, scn_seq** out) {
  if (!t || !out) return fail(SCN_EINVAL, "NULL argument");
  *out = nullptr;
  if (stride < 1) return fail(SCN_EINVAL, "stride must be >= 1, got %lld", (long long)stride);
  std::vector<int64_t> rows;
  rows.reserve((size_t)((t->rows + stride - 1) / stride));
  for (int64_t r = 0; r < t->rows; r += stride) rows.push_back(r);
  return make_seq(t, rows, out);
}

scn_status scn_sample_range(const scn_table* t, const scn_block* blocks, int64_t n_blocks, int64_t step,
                            scn_seq** out) {
  if (!t || !out || (n_blocks > 0 && !blocks)) return fail(SCN_EINVAL, "NULL argument");
  *out = nullptr;
  if (step < 1) return fail(SCN_EINVAL, "step must be >= 1");
  if (n_blocks < 0) return fail(SCN_EINVAL, "n_blocks < 0");
  for (int64_t i = 0; i < n_blocks; ++i) {
    if (blocks[i].start > blocks[i].end) return fail(SCN_EINVAL, "block %lld has start > end", (long long)i);
    if (i > 0 && blocks[i].start < blocks[i - 1].end)
      return fail(SCN_EINVAL, "blocks must be sorted and disjoint (block %lld)", (long long)i);
  }
  for (int64_t i = 0; i < n_blocks; ++i)
    if (blocks[i].start < 0 || blocks[i].end > t->rows)
      return fail(SCN_ERANGE, "block %lld outside [0,%lld)", (long long)i, (long long)t->rows);
  std::vector<int64_t> rows;
  for (int64_t i = 0; i < n_blocks; ++i)
    for (int64_t r = blocks[i].start; r < blocks[i].end; r += step) rows.push_back(r);
  return make_seq(t, rows, out);
}

scn_status scn_sample_gather(const scn_table* t, const int64_t* rows, int64_t n, scn_seq** out) {
  if (!t || !out || (n > 0 && !rows)) return fail(SCN_EINVAL, "NULL argument");
  *out = nullptr;
  if (n < 0) return fail(SCN_EINVAL, "n < 0");
  for (int64_t i = 1; i < n; ++i)
    if (rows[i] <= rows[i - 1]) return fail(SCN_EINVAL, "gather rows must be strictly increasing (index %lld)", (long long)i);
  for (int64_t i = 0; i < n; ++i)
    if (rows[i] < 0 || rows[i] >= t->rows)
      return fail(SCN_ERANGE, "gather row %lld outside [0,%lld)", (long long)rows[i], (long long)t->rows);
  return make_seq(t, std::vector<int64_t>(rows, rows + n), out);
}

scn_status scn_seq_concat(const scn_seq* const* parts, int32_t n, scn_seq** out) {
  if (!out || (n > 0 && !parts)) return fail(SCN_EINVAL, "NULL argument");
  *out = nullptr;
  if (n < 1) return fail(SCN_EINVAL, "need at least one part");
  for (int32_t i = 0; i < n; ++i) {
    if (!parts[i]) return fail(SCN_EINVAL, "part %d is NULL", i);
    if (parts[i]->width != parts[0]->width || parts[i]->height != parts[0]->height ||
        parts[i]->where != parts[0]->where)
      return fail(SCN_EINVAL, "part %d differs in frame shape or memory location", i);
  }
  scn_seq* s = new (std::nothrow) scn_seq();
  if (!s) return fail(SCN_EINVAL, "out of host memory");
  s->width = parts[0]->width;
  s->height = parts[0]->height;
  s->where = parts[0]->where;
  for (int32_t i = 0; i < n; ++i) {
    const scn_seq* p = parts[i];
    const size_t m = p->addr.size();
    // an input may itself be a concatenation: keep its inner parts (tables, slices)
    const int32_t base = (int32_t)s->tables.size();
    s->addr.insert(s->addr.end(), p->addr.begin(), p->addr.end());
    s->row.insert(s->row.end(), p->row.begin(), p->row.end());
    for (size_t j = 0; j < m; ++j) {
      s->part.push_back(base + p->part[j]);
      s->seg.push_back(j == 0 ? 1 : p->seg[j]);
    }
    if (p->tables.empty()) s->tables.push_back(nullptr);
    else s->tables.insert(s->tables.end(), p->tables.begin(), p->tables.end());
  }
  *out = s;
  return SCN_OK;
}

int64_t scn_seq_length(const scn_seq* s) { return s ? (int64_t)s->addr.size() : -1; }

scn_status scn_seq_rows(const scn_seq* s, int32_t* part, int64_t* row) {
  if (!s) return fail(SCN_EINVAL, "NULL seq");
  if (part && !s->part.empty()) memcpy(part, s->part.data(), s->part.size() * sizeof(int32_t));
  if (row && !s->row.empty()) memcpy(row, s->row.data(), s->row.size() * sizeof(int64_t));
  return SCN_OK;
}

scn_status scn_seq_seg_starts(const scn_seq* s, uint8_t* flags) {
  if (!s || !flags) return fail(SCN_EINVAL, "NULL argument");
  if (!s->seg.empty()) memcpy(flags, s->seg.data(), s->seg.size());
  return SCN_OK;
}

scn_status scn_shard_range(int64_t m, int32_t world, int32_t rank, int64_t* begin, int64_t* end) {
  if (!begin || !end) return fail(SCN_EINVAL, "NULL argument");
  if (m < 0 || world < 1 || rank < 0 || rank >= world) return fail(SCN_EINVAL, "bad shard (m=%lld, G=%d, r=%d)",
                                                                  (long long)m, world, rank);
  // floor(r*M/G) without overflow for M up to 2^62/G
  *begin = (int64_t)((__int128)m * rank / world);
  *end = (int64_t)((__int128)m * (rank + 1) / world);
  return SCN_OK;
}

int32_t scn_seq_needs_halo(const scn_seq* s, int64_t begin) {
  if (!s || begin <= 0 || begin >= (int64_t)s->seg.size()) return 0;
  return s->seg[(size_t)begin] ? 0 : 1;
}

size_t scn_seq_device_bytes(const scn_seq* s) {
  if (!s) return 0;
  const size_t m = s->addr.size();
  return ((8 * m + m) + 15) & ~size_t(15);
}

scn_status scn_seq_upload(scn_seq* s, void* d_ws, size_t bytes, void* stream) {
  if (!s) return fail(SCN_EINVAL, "NULL seq");
  if (s->where != SCN_MEM_DEVICE) return fail(SCN_EINVAL, "host-location sequences are not uploaded");
  const size_t need = scn_seq_device_bytes(s);
  if (bytes < need) return fail(SCN_EINVAL, "workspace of %zu bytes < %zu", bytes, need);
  if (need && (!d_ws || (uintptr_t)d_ws % 8 != 0)) return fail(SCN_EINVAL, "workspace NULL or not 8-byte aligned");
  const size_t m = s->addr.size();
  cudaStream_t st = (cudaStream_t)stream;
  if (m) {
    cudaError_t e = cudaMemcpyAsync(d_ws, s->addr.data(), 8 * m, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync((uint8_t*)d_ws + 8 * m, s->seg.data(), m, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return cuda_fail(e, "scn_seq_upload");
  }
  s->d_ws = d_ws;
  return SCN_OK;
}

void scn_seq_destroy(scn_seq* s) { delete s; }

// ---------------------------------------------------------------------------
// NEXT N2: stencil before sampling (fig:sampling-e) — exact required set
// ---------------------------------------------------------------------------
scn_status scn_seq_stencil_required(const scn_seq* s, int32_t offset, scn_seq** required, int64_t* h_pos,
                                    int64_t* h_nbr) {
  if (!s || !required) return fail(SCN_EINVAL, "NULL argument");
  *required = nullptr;
  const size_t m = s->addr.size();
  if (m && (!h_pos || !h_nbr)) return fail(SCN_EINVAL, "h_pos/h_nbr must hold M entries");
  scn_seq* r = new (std::nothrow) scn_seq();
  if (!r) return fail(SCN_EINVAL, "out of host memory");
  r->width = s->width;
  r->height = s->height;
  r->where = s->where;
  size_t j0 = 0;
  int32_t part = 0;
  while (j0 < m) {
    size_t j1 = j0 + 1;
    while (j1 < m && !s->seg[j1]) ++j1;  // positions [j0, j1) are one part (one table)
    const std::shared_ptr<const scn_table>& t = s->tables[(size_t)s->part[j0]];
    if (!t) {
      delete r;
      return fail(SCN_EINVAL, "sequence part has no table");
    }
    // required rows of this table: S and clamp(S + offset) (repeat-edge, reading Q6), sorted, unique
    std::vector<int64_t> rows;
    rows.reserve(2 * (j1 - j0));
    for (size_t j = j0; j < j1; ++j) {
      const int64_t x = s->row[j];
      int64_t nb = x + offset;
      nb = nb < 0 ? 0 : (nb >= t->rows ? t->rows - 1 : nb);
      rows.push_back(x);
      rows.push_back(nb);
    }
    std::sort(rows.begin(), rows.end());
    rows.erase(std::unique(rows.begin(), rows.end()), rows.end());
    const int64_t base = (int64_t)r->addr.size();
    for (size_t i = 0; i < rows.size(); ++i) {
      r->addr.push_back(t->addr(rows[i]));
      r->row.push_back(rows[i]);
      r->part.push_back(part);
      r->seg.push_back(i == 0 ? 1 : 0);
    }
    r->tables.push_back(t);
    for (size_t j = j0; j < j1; ++j) {
      const int64_t x = s->row[j];
      int64_t nb = x + offset;
      nb = nb < 0 ? 0 : (nb >= t->rows ? t->rows - 1 : nb);
      h_pos[j] = base + (std::lower_bound(rows.begin(), rows.end(), x) - rows.begin());
      h_nbr[j] = base + (std::lower_bound(rows.begin(), rows.end(), nb) - rows.begin());
    }
    ++part;
    j0 = j1;
  }
  *required = r;
  return SCN_OK;
}

scn_status scn_run_diff_pairs(const uint32_t* d_hist, const int64_t* d_a, const int64_t* d_b, int64_t n,
                              int32_t bins, uint32_t* d_diff, void* stream) {
  g_launches = 0;
  if (n < 0) return fail(SCN_EINVAL, "n < 0");
  if (bins < 1 || bins > 256) return fail(SCN_EUNSUPPORTED, "bins must be in [1,256], got %d", bins);
  if (n == 0) return SCN_OK;
  if (!d_hist || !d_a || !d_b || !d_diff) return fail(SCN_EINVAL, "NULL device buffer");
  int nl = 0;
  cudaError_t e = scn::launch_diff_pairs(d_hist, d_a, d_b, n, bins, d_diff, (cudaStream_t)stream, &nl);
  g_launches += nl;
  if (e != cudaSuccess) return cuda_fail(e, "diff_pairs launch");
  return SCN_OK;
}

static scn_status check_run(const scn_seq* s, int64_t begin, int64_t end, int32_t bins, bool need_bins);
static const uint8_t* d_seg(const scn_seq* s);

// ---------------------------------------------------------------------------
// NEXT N3: bounded-state op with warmup W
// ---------------------------------------------------------------------------
int64_t scn_seq_warmup_begin(const scn_seq* s, int64_t begin, int32_t warmup) {
  if (!s || begin < 0 || warmup < 0) return -1;
  const int64_t m = (int64_t)s->seg.size();
  if (begin >= m) return begin;
  int64_t p = begin;
  for (int32_t i = 0; i < warmup && p > 0 && !s->seg[(size_t)p]; ++i) --p;  // stop at the table's start
  return p;
}

scn_status scn_run_adaptive_cuts(const scn_seq* s, int64_t begin, int64_t end, int32_t warmup,
                                 const uint32_t* d_diff, uint32_t k_num, uint32_t k_den, uint32_t floor_,
                                 uint8_t* d_cut, void* stream) {
  scn_status rc = check_run(s, begin, end, 1, false);
  if (rc) return rc;
  if (warmup < 1 || k_den < 1) return fail(SCN_EINVAL, "warmup and k_den must be >= 1");
  // both sides of the test are < 2^64 iff W * (k_num + k_den) < 2^32 (D, floor < 2^32)
  if ((uint64_t)warmup * ((uint64_t)k_num + k_den) >= (1ull << 32))
    return fail(SCN_EINVAL, "warmup * (k_num + k_den) must be < 2^32 (64-bit exact comparison)");
  if (end == begin) return SCN_OK;
  if (!d_diff || !d_cut) return fail(SCN_EINVAL, "d_diff/d_cut is NULL");
  const int64_t wb = scn_seq_warmup_begin(s, begin, warmup);
  int nl = 0;
  cudaError_t e = scn::launch_adaptive_cuts(d_diff, d_seg(s) + wb, begin - wb, end - wb, warmup, k_num, k_den,
                                            floor_, d_cut, (cudaStream_t)stream, &nl);
  g_launches += nl;
  if (e != cudaSuccess) return cuda_fail(e, "adaptive_cuts launch");
  return SCN_OK;
}

// ---------------------------------------------------------------------------
// NEXT N1: two-job shot montage (two jobs because graphs cannot
// filter data-dependently)
// ---------------------------------------------------------------------------
scn_status scn_select_shot_starts(const scn_seq* s, int64_t begin, int64_t end, const uint32_t* h_diff, uint32_t tau,
                                  int64_t* h_pos, int64_t cap, int64_t* count) {
  if (!s || !count) return fail(SCN_EINVAL, "NULL argument");
  if (begin < 0 || begin > end) return fail(SCN_EINVAL, "bad range");
  if (end > (int64_t)s->seg.size()) return fail(SCN_ERANGE, "end > sequence length");
  if (end > begin && !h_diff) return fail(SCN_EINVAL, "h_diff is NULL");
  int64_t k = 0;
  for (int64_t p = begin; p < end; ++p) {
    if (s->seg[(size_t)p] || h_diff[p - begin] > tau) {  // threshold_detector (reading Q5)
      if (h_pos && k < cap) h_pos[k] = p;
      ++k;
    }
  }
  *count = k;
  return SCN_OK;
}

scn_status scn_seq_gather_positions(const scn_seq* s, const int64_t* h_pos, int64_t n, scn_seq** out) {
  if (!s || !out || (n > 0 && !h_pos)) return fail(SCN_EINVAL, "NULL argument");
  *out = nullptr;
  if (n < 0) return fail(SCN_EINVAL, "n < 0");
  const int64_t m = (int64_t)s->addr.size();
  for (int64_t i = 0; i < n; ++i) {
    if (i > 0 && h_pos[i] <= h_pos[i - 1]) return fail(SCN_EINVAL, "positions must be strictly increasing");
    if (h_pos[i] < 0 || h_pos[i] >= m) return fail(SCN_ERANGE, "position %lld outside [0,%lld)", (long long)h_pos[i],
                                                    (long long)m);
  }
  scn_seq* r = new (std::nothrow) scn_seq();
  if (!r) return fail(SCN_EINVAL, "out of host memory");
  r->width = s->width;
  r->height = s->height;
  r->where = s->where;
  int32_t last_part = -1, np = -1;
  for (int64_t i = 0; i < n; ++i) {
    const size_t p = (size_t)h_pos[i];
    if (s->part[p] != last_part) {  // a new table starts a new part (slice)
      last_part = s->part[p];
      ++np;
      r->tables.push_back(s->tables.empty() ? nullptr : s->tables[(size_t)last_part]);
      r->seg.push_back(1);
    } else {
      r->seg.push_back(0);
    }
    r->addr.push_back(s->addr[p]);
    r->row.push_back(s->row[p]);
    r->part.push_back(np);
  }
  *out = r;
  return SCN_OK;
}

// ---------------------------------------------------------------------------
// runs
// ---------------------------------------------------------------------------
static scn_status check_run(const scn_seq* s, int64_t begin, int64_t end, int32_t bins, bool need_bins) {
  g_launches = 0;
  if (!s) return fail(SCN_EINVAL, "NULL seq");
  if (s->where != SCN_MEM_DEVICE) return fail(SCN_EINVAL, "scn_run_* needs a device-location sequence");
  if (begin < 0 || begin > end) return fail(SCN_EINVAL, "bad range [%lld,%lld)", (long long)begin, (long long)end);
  if (end > (int64_t)s->addr.size())
    return fail(SCN_ERANGE, "end %lld > sequence length %zu", (long long)end, s->addr.size());
  if (need_bins && (bins < 1 || bins > 256)) return fail(SCN_EUNSUPPORTED, "bins must be in [1,256], got %d", bins);
  if (end > begin && !s->d_ws) return fail(SCN_EINVAL, "sequence not uploaded (scn_seq_upload)");
  return SCN_OK;
}

// every position the run reads must be resident (sparse tables)
static scn_status check_resident(const scn_seq* s, int64_t first, int64_t end) {
  for (int64_t j = first; j < end; ++j)
    if (s->addr[(size_t)j] == 0)
      return fail(SCN_ERANGE, "position %lld (table row %lld) is not resident", (long long)j,
                  (long long)s->row[(size_t)j]);
  return SCN_OK;
}

static scn::DestList one_dest(uint32_t* p) {
  scn::DestList d{};
  d.n = 1;
  d.p[0] = (uint64_t)(uintptr_t)p;
  return d;
}

static const uint64_t* d_addr(const scn_seq* s) { return (const uint64_t*)s->d_ws; }
static const uint8_t* d_seg(const scn_seq* s) { return (const uint8_t*)s->d_ws + 8 * s->addr.size(); }

static scn_status run_hist(const scn_seq* s, int64_t first, int64_t n_items, int32_t n_halo, int32_t bins,
                           uint32_t* d_hist, uint32_t* d_halo, uint8_t* d_ds, cudaStream_t st) {
  const size_t row = (size_t)3 * bins * sizeof(uint32_t);
  cudaError_t e = cudaSuccess;
  if (n_items - n_halo > 0) e = cudaMemsetAsync(d_hist, 0, row * (size_t)(n_items - n_halo), st);
  if (e == cudaSuccess && n_halo) e = cudaMemsetAsync(d_halo, 0, row * (size_t)n_halo, st);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(hist)");
  scn::HistJob j{};
  j.src.ptrs = d_addr(s) + first;
  j.n_items = n_items;
  j.n_halo = n_halo;
  j.out = d_hist;
  j.halo_out = d_halo;
  j.ds_out = d_ds;
  j.width = s->width;
  j.height = s->height;
  j.bins = bins;
  int nl = 0;
  e = d_ds ? scn::launch_hist_downsample(j, st, &nl) : scn::launch_histogram(j, st, &nl);
  g_launches += nl;
  if (e != cudaSuccess) return cuda_fail(e, "histogram launch");
  return SCN_OK;
}

scn_status scn_run_histogram(const scn_seq* s, int64_t begin, int64_t end, int32_t bins, uint32_t* d_hist,
                             void* stream) {
  scn_status rc = check_run(s, begin, end, bins, true);
  if (rc) return rc;
  if (end == begin) return SCN_OK;
  if (!d_hist) return fail(SCN_EINVAL, "d_hist is NULL");
  if ((rc = check_resident(s, begin, end))) return rc;
  return run_hist(s, begin, end - begin, 0, bins, d_hist, nullptr, nullptr, (cudaStream_t)stream);
}

// joint-colour histograms of n_items positions from `first`; the first n_halo go to d_halo
static scn_status run_hist_joint(const scn_seq* s, int64_t first, int64_t n_items, int32_t n_halo, int32_t J,
                                 uint32_t* d_hist, uint32_t* d_halo, cudaStream_t st) {
  const size_t row = (size_t)J * J * J * sizeof(uint32_t);
  cudaError_t e = cudaSuccess;
  if (n_items - n_halo > 0) e = cudaMemsetAsync(d_hist, 0, row * (size_t)(n_items - n_halo), st);
  if (e == cudaSuccess && n_halo) e = cudaMemsetAsync(d_halo, 0, row * (size_t)n_halo, st);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(joint hist)");
  scn::HistJob j{};
  j.src.ptrs = d_addr(s) + first;
  j.n_items = n_items;
  j.n_halo = n_halo;
  j.out = d_hist;
  j.halo_out = d_halo;
  j.width = s->width;
  j.height = s->height;
  j.bins = J;
  j.joint = J;
  int nl = 0;
  e = scn::launch_histogram_joint(j, st, &nl);
  g_launches += nl;
  if (e != cudaSuccess) return cuda_fail(e, "joint histogram launch");
  return SCN_OK;
}

static scn_status check_joint(int32_t J) {
  if (J < 1 || J > 8) return fail(SCN_EUNSUPPORTED, "joint bins per channel must be in [1,8], got %d", J);
  return SCN_OK;
}

scn_status scn_run_histogram_joint(const scn_seq* s, int64_t begin, int64_t end, int32_t bins_per_channel,
                                   uint32_t* d_hist, void* stream) {
  scn_status rc = check_run(s, begin, end, 0, false);
  if (rc || (rc = check_joint(bins_per_channel))) return rc;
  if (end == begin) return SCN_OK;
  if (!d_hist) return fail(SCN_EINVAL, "d_hist is NULL");
  if ((rc = check_resident(s, begin, end))) return rc;
  return run_hist_joint(s, begin, end - begin, 0, bins_per_channel, d_hist, nullptr, (cudaStream_t)stream);
}

scn_status scn_run_hist_shotdiff_joint(const scn_seq* s, int64_t begin, int64_t end, int32_t bins_per_channel,
                                       uint32_t* d_hist, uint32_t* d_diff, uint32_t* d_scratch, void* stream) {
  scn_status rc = check_run(s, begin, end, 0, false);
  if (rc || (rc = check_joint(bins_per_channel))) return rc;
  if (end == begin) return SCN_OK;
  if (!d_hist || !d_diff) return fail(SCN_EINVAL, "d_hist/d_diff is NULL");
  cudaStream_t st = (cudaStream_t)stream;
  const int32_t halo = scn_seq_needs_halo(s, begin);
  if (halo && !d_scratch) return fail(SCN_EINVAL, "d_scratch needed for the halo histogram");
  if ((rc = check_resident(s, begin - halo, end))) return rc;
  const int32_t J = bins_per_channel;
  // the halo frame (position begin-1) is recomputed in the same launch
  rc = run_hist_joint(s, begin - halo, end - begin + halo, halo, J, d_hist, d_scratch, st);
  if (rc) return rc;
  int nl = 0;
  cudaError_t e = scn::launch_shotdiff(d_hist, halo ? d_scratch : nullptr, d_seg(s) + begin, end - begin,
                                       J * J * J, one_dest(d_diff), st, &nl);
  g_launches += nl;
  if (e != cudaSuccess) return cuda_fail(e, "joint shotdiff launch");
  return SCN_OK;
}

static scn_status run_diff(const scn_seq* s, int64_t begin, int64_t end, int32_t bins, const uint32_t* d_hist,
                           const uint32_t* halo, uint32_t* d_diff, cudaStream_t st) {
  int nl = 0;
  cudaError_t e = scn::launch_shotdiff(d_hist, halo, d_seg(s) + begin, end - begin, 3 * bins, one_dest(d_diff), st, &nl);
  g_launches += nl;
  if (e != cudaSuccess) return cuda_fail(e, "shotdiff launch");
  return SCN_OK;
}

scn_status scn_run_shotdiff(const scn_seq* s, int64_t begin, int64_t end, int32_t bins, const uint32_t* d_hist,
                            uint32_t* d_diff, uint32_t* d_scratch, void* stream) {
  scn_status rc = check_run(s, begin, end, bins, true);
  if (rc) return rc;
  if (end == begin) return SCN_OK;
  if (!d_hist || !d_diff) return fail(SCN_EINVAL, "d_hist/d_diff is NULL");
  cudaStream_t st = (cudaStream_t)stream;
  const int32_t halo = scn_seq_needs_halo(s, begin);
  if (halo) {
    if (!d_scratch) return fail(SCN_EINVAL, "d_scratch needed for the halo histogram");
    if ((rc = check_resident(s, begin - 1, begin))) return rc;
    // recompute the halo (position begin-1) rather than communicate it
    rc = run_hist(s, begin - 1, 1, 1, bins, nullptr, d_scratch, nullptr, st);
    if (rc) return rc;
  }
  return run_diff(s, begin, end, bins, d_hist, halo ? d_scratch : nullptr, d_diff, st);
}

scn_status scn_run_hist_shotdiff(const scn_seq* s, int64_t begin, int64_t end, int32_t bins, uint32_t* d_hist,
                                 uint32_t* d_diff, uint32_t* d_scratch, void* stream) {
  scn_status rc = check_run(s, begin, end, bins, true);
  if (rc) return rc;
  if (end == begin) return SCN_OK;
  if (!d_hist || !d_diff) return fail(SCN_EINVAL, "d_hist/d_diff is NULL");
  cudaStream_t st = (cudaStream_t)stream;
  const int32_t halo = scn_seq_needs_halo(s, begin);
  if (halo && !d_scratch) return fail(SCN_EINVAL, "d_scratch needed for the halo histogram");
  if ((rc = check_resident(s, begin - halo, end))) return rc;
  rc = run_hist(s, begin - halo, end - begin + halo, halo, bins, d_hist, d_scratch, nullptr, st);
  if (rc) return rc;
  return run_diff(s, begin, end, bins, d_hist, halo ? d_scratch : nullptr, d_diff, st);
}

scn_status scn_run_hist_shotdiff_to(const scn_seq* s, int64_t begin, int64_t end, int32_t bins,
                                    const uint64_t* h_hist_dests, const uint64_t* h_diff_dests, int32_t n_dest,
                                    int32_t self, uint32_t* d_scratch, void* stream) {
  scn_status rc = check_run(s, begin, end, bins, true);
  if (rc) return rc;
  if (n_dest < 1 || n_dest > scn::kMaxDest) return fail(SCN_EINVAL, "n_dest must be in [1,%d]", scn::kMaxDest);
  if (self < 0 || self >= n_dest) return fail(SCN_EINVAL, "self must be in [0,n_dest)");
  if (!h_hist_dests || !h_diff_dests) return fail(SCN_EINVAL, "destination lists are NULL");
  for (int32_t g = 0; g < n_dest; ++g)
    if (!h_hist_dests[g] || !h_diff_dests[g] || h_hist_dests[g] % 4 || h_diff_dests[g] % 4)
      return fail(SCN_EINVAL, "destination %d is NULL or misaligned", g);
  if (end == begin) return SCN_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int32_t halo = scn_seq_needs_halo(s, begin);
  if (halo && !d_scratch) return fail(SCN_EINVAL, "d_scratch needed for the halo histogram");
  if ((rc = check_resident(s, begin - halo, end))) return rc;
  const int64_t n = end - begin, K = 3 * (int64_t)bins;
  // this rank owns rows [begin,end) of every destination: zero them (peer stores), then
  // the histogram flush accumulates straight into all of them
  scn::DestList dh{}, dd{};
  dh.n = dd.n = n_dest;
  for (int32_t g = 0; g < n_dest; ++g) {
    dh.p[g] = h_hist_dests[g] + (uint64_t)(begin * K) * sizeof(uint32_t);
    dd.p[g] = h_diff_dests[g] + (uint64_t)begin * sizeof(uint32_t);
  }
  int nl = 0;
  cudaError_t e = scn::launch_zero_dests(dh, n * K, st, &nl);
  if (e == cudaSuccess && halo) e = cudaMemsetAsync(d_scratch, 0, (size_t)K * sizeof(uint32_t), st);
  if (e != cudaSuccess) {
    g_launches += nl;
    return cuda_fail(e, "zero destinations");
  }
  scn::HistJob j{};
  j.src.ptrs = d_addr(s) + begin - halo;
  j.n_items = n + halo;
  j.n_halo = halo;
  j.out = reinterpret_cast<uint32_t*>(dh.p[self]);
  j.halo_out = d_scratch;
  j.width = s->width;
  j.height = s->height;
  j.bins = bins;
  j.n_dest = n_dest;
  for (int32_t g = 0; g < n_dest; ++g) j.dest[g] = dh.p[g];
  e = scn::launch_histogram(j, st, &nl);
  if (e == cudaSuccess)
    e = scn::launch_shotdiff(reinterpret_cast<const uint32_t*>(dh.p[self]), halo ? d_scratch : nullptr,
                             d_seg(s) + begin, n, (int32_t)K, dd, st, &nl);
  g_launches += nl;
  if (e != cudaSuccess) return cuda_fail(e, "hist_shotdiff_to launch");
  return SCN_OK;
}

scn_status scn_ipc_import(const void* handle, int64_t offset, uint64_t* d_base, uint64_t* d_ptr) {
  if (!handle || !d_base || !d_ptr || offset < 0) return fail(SCN_EINVAL, "NULL argument or negative offset");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof h);
  void* base = nullptr;
  // opened in the CURRENT device's context; peer access to the owner's GPU is enabled lazily
  cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle");
  *d_base = (uint64_t)(uintptr_t)base;
  *d_ptr = *d_base + (uint64_t)offset;
  return SCN_OK;
}

scn_status scn_ipc_release(uint64_t d_base) {
  if (!d_base) return fail(SCN_EINVAL, "NULL base");
  cudaError_t e = cudaIpcCloseMemHandle((void*)(uintptr_t)d_base);
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcCloseMemHandle");
  return SCN_OK;
}

scn_status scn_run_downsample(const scn_seq* s, int64_t begin, int64_t end, uint8_t* d_out, void* stream) {
  scn_status rc = check_run(s, begin, end, 0, false);
  if (rc) return rc;
  if (end == begin) return SCN_OK;
  if (!d_out && s->width >= 2 && s->height >= 2) return fail(SCN_EINVAL, "d_out is NULL");
  if ((rc = check_resident(s, begin, end))) return rc;
  scn::FrameSrc src{d_addr(s) + begin, 0, 0};
  int nl = 0;
  cudaError_t e = scn::launch_downsample(src, end - begin, s->width, s->height, d_out, (cudaStream_t)stream, &nl);
  g_launches += nl;
  if (e != cudaSuccess) return cuda_fail(e, "downsample launch");
  return SCN_OK;
}

scn_status scn_run_montage(const scn_seq* s, int64_t begin, int64_t end, int32_t cols, uint8_t* d_canvas,
                           int64_t canvas_pitch, void* stream) {
  scn_status rc = check_run(s, begin, end, 0, false);
  if (rc) return rc;
  if (cols < 1) return fail(SCN_EINVAL, "cols must be >= 1");
  const int64_t ow3 = (int64_t)(s->width / 2) * 3, oh = s->height / 2;
  if (canvas_pitch < cols * ow3) return fail(SCN_EINVAL, "canvas pitch %lld < cols*(W/2)*3", (long long)canvas_pitch);
  if (end == begin || oh == 0 || ow3 == 0) return SCN_OK;
  if (!d_canvas) return fail(SCN_EINVAL, "d_canvas is NULL");
  if ((rc = check_resident(s, begin, end))) return rc;
  const int64_t k = end - begin, tile_rows = (k + cols - 1) / cols;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(d_canvas, 0, (size_t)(tile_rows * oh * canvas_pitch), st);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(canvas)");
  // any canvas alignment: unaligned tiles take the kernel's realigned-store path
  scn::FrameSrc src{d_addr(s) + begin, 0, 0};
  int nl = 0;
  e = scn::launch_downsample(src, k, s->width, s->height, d_canvas, st, &nl, canvas_pitch, cols);
  g_launches += nl;
  if (e != cudaSuccess) return cuda_fail(e, "montage launch");
  return SCN_OK;
}

scn_status scn_run_hist_downsample(const scn_seq* s, int64_t begin, int64_t end, int32_t bins, uint32_t* d_hist,
                                   uint8_t* d_out, void* stream) {
  scn_status rc = check_run(s, begin, end, bins, true);
  if (rc) return rc;
  if (end == begin) return SCN_OK;
  if (!d_hist) return fail(SCN_EINVAL, "d_hist is NULL");
  if ((rc = check_resident(s, begin, end))) return rc;
  if (!d_out) {
    if (s->width >= 2 && s->height >= 2) return fail(SCN_EINVAL, "d_out is NULL");
    return run_hist(s, begin, end - begin, 0, bins, d_hist, nullptr, nullptr, (cudaStream_t)stream);
  }
  return run_hist(s, begin, end - begin, 0, bins, d_hist, nullptr, d_out, (cudaStream_t)stream);
}

// ---------------------------------------------------------------------------
// end-to-end over host frames: double-buffered H2D staging
// ---------------------------------------------------------------------------
scn_status scn_run_pipeline_host(const scn_seq* s, int64_t begin, int64_t end, int32_t bins, uint32_t ops,
                                 uint32_t* d_hist, uint32_t* d_diff, uint8_t* d_out, uint32_t* d_scratch,
                                 void* d_staging, size_t staging_bytes, void* stream, void* copy_stream) {
  g_launches = 0;
  if (!s) return fail(SCN_EINVAL, "NULL seq");
  if (s->where != SCN_MEM_HOST) return fail(SCN_EINVAL, "scn_run_pipeline_host needs a host-location sequence");
  if (begin < 0 || begin > end) return fail(SCN_EINVAL, "bad range");
  if (end > (int64_t)s->addr.size()) return fail(SCN_ERANGE, "end > sequence length");
  const bool do_hist = ops & SCN_OP_HIST, do_diff = ops & SCN_OP_SHOTDIFF, do_ds = ops & SCN_OP_DOWNSAMPLE;
  if (ops & ~7u) return fail(SCN_EINVAL, "unknown op bits 0x%x", ops);
  if (do_diff && !do_hist) return fail(SCN_EINVAL, "shot-diff needs HIST");
  if ((do_hist || do_diff) && (bins < 1 || bins > 256)) return fail(SCN_EUNSUPPORTED, "bins must be in [1,256]");
  if (end == begin) return SCN_OK;
  if ((do_hist && !d_hist) || (do_diff && !d_diff) || (do_ds && !d_out && s->width >= 2 && s->height >= 2))
    return fail(SCN_EINVAL, "missing output buffer");
  const int64_t n = end - begin;
  const int32_t halo = do_diff ? scn_seq_needs_halo(s, begin) : 0;
  if (halo && !d_scratch) return fail(SCN_EINVAL, "d_scratch needed for the halo histogram");
  for (int64_t j = begin - halo; j < end; ++j)
    if (s->addr[(size_t)j] == 0) return fail(SCN_ERANGE, "position %lld is not resident", (long long)j);
  const int64_t F = s->frame_bytes(), F16 = ceil16(F);
  const size_t hdr = (size_t)ceil16(n);
  if (!d_staging || (uintptr_t)d_staging % 16 != 0) return fail(SCN_EINVAL, "staging NULL or not 16-aligned");
  if (staging_bytes < hdr + 2 * (size_t)F16) return fail(SCN_EINVAL, "staging buffer too small");
  const size_t slot_bytes = ((staging_bytes - hdr) / 2) & ~size_t(15);
  const int64_t per_chunk = (int64_t)(slot_bytes / (size_t)F16);
  uint8_t* slots[2] = {(uint8_t*)d_staging + hdr, (uint8_t*)d_staging + hdr + slot_bytes};
  cudaStream_t st = (cudaStream_t)stream, cst = copy_stream ? (cudaStream_t)copy_stream : st;

  cudaError_t e = cudaSuccess;
  cudaEvent_t copied[2], freed[2];
  for (int i = 0; i < 2; ++i) {
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&copied[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&freed[i], cudaEventDisableTiming);
  }
  if (e != cudaSuccess) return cuda_fail(e, "cudaEventCreate");
  if (do_diff) e = cudaMemcpyAsync(d_staging, s->seg.data() + begin, (size_t)n, cudaMemcpyHostToDevice, st);
  const size_t row = (size_t)3 * bins * sizeof(uint32_t);
  if (e == cudaSuccess && do_hist) e = cudaMemsetAsync(d_hist, 0, row * (size_t)n, st);
  if (e == cudaSuccess && halo) e = cudaMemsetAsync(d_scratch, 0, row, st);
  // the copy stream must not overwrite the slots while earlier work queued on
  // `stream` (e.g. the previous call's kernels) may still read them
  if (e == cudaSuccess && cst != st) {
    e = cudaEventRecord(freed[0], st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(cst, freed[0], 0);
  }
  bool first_use[2] = {true, true};
  int64_t item = begin - halo;  // next position to stage
  int chunk = 0;
  while (e == cudaSuccess && item < end) {
    const int b = chunk & 1;
    const int64_t k = (end - item) < per_chunk ? (end - item) : per_chunk;
    if (!first_use[b]) e = cudaStreamWaitEvent(cst, freed[b], 0);
    first_use[b] = false;
    // coalesce runs of host frames that are contiguous with stride F16
    for (int64_t i = 0; i < k && e == cudaSuccess;) {
      int64_t r = 1;
      const uint64_t a0 = s->addr[(size_t)(item + i)];
      while (i + r < k && s->addr[(size_t)(item + i + r)] == a0 + (uint64_t)r * F16) ++r;
      if (r > 1)
        e = cudaMemcpyAsync(slots[b] + i * F16, (const void*)a0, (size_t)(r * F16), cudaMemcpyHostToDevice, cst);
      else
        e = cudaMemcpyAsync(slots[b] + i * F16, (const void*)a0, (size_t)F, cudaMemcpyHostToDevice, cst);
      i += r;
    }
    if (e == cudaSuccess) e = cudaEventRecord(copied[b], cst);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, copied[b], 0);
    if (e != cudaSuccess) break;
    const int32_t h = (item < begin) ? 1 : 0;  // only the first chunk can carry the halo
    scn::FrameSrc src{nullptr, (uint64_t)(uintptr_t)slots[b], (uint64_t)F16};
    int nl = 0;
    if (do_hist) {
      scn::HistJob j{};
      j.src = src;
      j.n_items = k;
      j.n_halo = h;
      j.out = d_hist + (size_t)(item + h - begin) * 3 * bins;
      j.halo_out = d_scratch;
      j.width = s->width;
      j.height = s->height;
      j.bins = bins;
      if (do_ds && !h) {
        j.ds_out = d_out + (size_t)(item - begin) * (size_t)((s->width / 2) * (s->height / 2) * 3);
        e = scn::launch_hist_downsample(j, st, &nl);
      } else {
        e = scn::launch_histogram(j, st, &nl);
        if (e == cudaSuccess && do_ds && k - h > 0) {
          scn::FrameSrc s2{nullptr, src.base + (uint64_t)h * F16, (uint64_t)F16};
          e = scn::launch_downsample(s2, k - h, s->width, s->height,
                                     d_out + (size_t)(item + h - begin) * (size_t)((s->width / 2) * (s->height / 2) * 3),
                                     st, &nl);
        }
      }
    } else if (do_ds) {
      e = scn::launch_downsample(src, k, s->width, s->height,
                                 d_out + (size_t)(item - begin) * (size_t)((s->width / 2) * (s->height / 2) * 3), st,
                                 &nl);
    }
    g_launches += nl;
    if (e == cudaSuccess) e = cudaEventRecord(freed[b], st);
    item += k;
    ++chunk;
  }
  if (e == cudaSuccess && do_diff) {
    int nl = 0;
    e = scn::launch_shotdiff(d_hist, halo ? d_scratch : nullptr, (const uint8_t*)d_staging, n, 3 * bins,
                             one_dest(d_diff), st, &nl);
    g_launches += nl;
  }
  for (int i = 0; i < 2; ++i) {
    cudaEventDestroy(copied[i]);
    cudaEventDestroy(freed[i]);
  }
  if (e != cudaSuccess) return cuda_fail(e, "scn_run_pipeline_host");
  return SCN_OK;
}

}  // extern "C"
