// K0 microbenchmarks (SURVEY.md §7 step 3, §8(d) "K0 microbenchmarks").
// Not part of the product path: measures the rooflines that decide the
// histogram design on the actual B200 before any kernel is tuned.
//   (i)   HBM streaming read: TMA 1-D bulk ring and LDG.128
//   (ii)  red.shared.add.u32 lane-private (conflict-free) lane-ops/clk/SM
//   (iii) red.shared.add.u32 all lanes same address
//   (iv)  red.shared.add.u32 random addresses over 48 / 768 words
//   (v)   __match_any_sync and __reduce_add_sync warp-instr/clk/SM
//   (vi)  non-atomic LDS+IADD+STS lane-private RMW
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o k0 k0.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// ---------------- shared atomics ----------------
// mode 0: lane-private (addr = key*32+lane, key varies) ; mode 1: same address ;
// mode 2: random over 48 words ; mode 3: random over 768 words ; mode 4: LDS/STS RMW lane-private (per-warp table)
template <int MODE>
__global__ void k_atoms(uint32_t* out, long long* cycles, int iters) {
  extern __shared__ uint32_t tab[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwords = (MODE == 4) ? (blockDim.x / 32) * 48 * 32 : 768 * 32;
  for (int i = threadIdx.x; i < nwords; i += blockDim.x) tab[i] = 0;
  __syncthreads();
  uint32_t x = threadIdx.x * 2654435761u + blockIdx.x * 97u + 12345u;
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      x = x * 1664525u + 1013904223u;
      uint32_t addr;
      if (MODE == 0) addr = (((x >> 20) & 767u) << 5) | lane;
      else if (MODE == 1) addr = 5;
      else if (MODE == 2) addr = (x >> 20) % 48u;
      else if (MODE == 3) addr = (x >> 20) % 768u;
      else addr = (uint32_t)warp * 48 * 32 + ((((x >> 20) % 48u)) << 5) + lane;
      if (MODE == 4) {
        tab[addr] += 1;
      } else {
        asm volatile("red.shared.add.u32 [%0], %1;" :: "r"(smem_u32(tab + addr)), "r"(1u) : "memory");
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  uint32_t s = 0;
  for (int i = threadIdx.x; i < nwords; i += blockDim.x) s += tab[i];
  atomicAdd(out, s);
}

// Same, without the serial LCG: 16 independent addresses per thread precomputed in registers, so the
// loop is ATOMS-issue bound (the LCG version above is bound by its dependent IMAD chain).
template <int MODE>
__global__ void k_atoms_ilp(uint32_t* out, long long* cycles, int iters) {
  extern __shared__ uint32_t tab[];
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 768 * 32; i += blockDim.x) tab[i] = 0;
  __syncthreads();
  uint32_t a[16];
  uint32_t x = threadIdx.x * 2654435761u + blockIdx.x * 97u + 12345u;
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    x = x * 1664525u + 1013904223u;
    uint32_t key = MODE == 0 ? ((x >> 20) % 768u) : (MODE == 1 ? (uint32_t)(u % 16) : ((x >> 20) % 48u));
    a[u] = smem_u32(tab + key * 32 + lane);
  }
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) asm volatile("red.shared.add.u32 [%0], %1;" :: "r"(a[u]), "r"(1u) : "memory");
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  uint32_t s = 0;
  for (int i = threadIdx.x; i < 768 * 32; i += blockDim.x) s += tab[i];
  atomicAdd(out, s);
}

// ---------------- match_any / reduce_add ----------------
template <int MODE>
__global__ void k_warp(uint32_t* out, long long* cycles, int iters) {
  const int lane = threadIdx.x & 31;
  uint32_t x = threadIdx.x * 2654435761u + blockIdx.x;
  uint32_t acc = 0;
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      x = x * 1664525u + 1013904223u;
      if (MODE == 0) acc += __match_any_sync(0xffffffffu, (x >> 28) + lane * 0);
      else acc += __reduce_add_sync(0xffffffffu, x);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  if (acc == 0x12345678u) out[0] = acc;
}

// ---------------- HBM read: LDG.128 ----------------
__global__ void k_ldg(const uint4* __restrict__ in, size_t n16, uint32_t* out) {
  uint32_t acc = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n16; i += 4 * stride) {
    uint4 a = __ldcs(in + i), b = __ldcs(in + i + stride), c = __ldcs(in + i + 2 * stride), d = __ldcs(in + i + 3 * stride);
    acc ^= a.x ^ a.y ^ a.z ^ a.w ^ b.x ^ b.y ^ b.z ^ b.w ^ c.x ^ c.y ^ c.z ^ c.w ^ d.x ^ d.y ^ d.z ^ d.w;
  }
  for (; i < n16; i += stride) { uint4 a = __ldcs(in + i); acc ^= a.x ^ a.y ^ a.z ^ a.w; }
  if (acc == 0x9e3779b9u) out[0] = acc;
}

// ---------------- HBM read: TMA bulk ring ----------------
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" :: "r"(smem_u32(b)), "r"(phase) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

__global__ void k_tma(const uint8_t* __restrict__ in, size_t ntiles, uint32_t tile, int stages, uint32_t* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* full = (uint64_t*)sm;
  uint64_t* empty = full + 16;
  uint8_t* ring = sm + 256;
  const int nwarps = blockDim.x / 32, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ncons = nwarps - 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, ncons); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  size_t t0 = ntiles * blockIdx.x / gridDim.x, t1 = ntiles * (blockIdx.x + 1) / gridDim.x;
  if (warp == 0) {
    if (lane == 0) {
      int s = 0; uint32_t ph = 0;
      for (size_t t = t0; t < t1; ++t) {
        mbar_wait(empty + s, ph ^ 1);
        mbar_expect_tx(full + s, tile);
        bulk_g2s(ring + (size_t)s * tile, in + t * tile, tile, full + s);
        if (++s == stages) { s = 0; ph ^= 1; }
      }
    }
  } else {
    uint32_t acc = 0;
    int s = 0; uint32_t ph = 0;
    const int ct = threadIdx.x - 32, nct = ncons * 32;
    for (size_t t = t0; t < t1; ++t) {
      mbar_wait(full + s, ph);
      const uint4* p = (const uint4*)(ring + (size_t)s * tile);
      for (uint32_t i = ct; i < tile / 16; i += nct) { uint4 v = p[i]; acc ^= v.x ^ v.y ^ v.z ^ v.w; }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + s);
      if (++s == stages) { s = 0; ph ^= 1; }
    }
    if (acc == 0x9e3779b9u) out[0] = acc;
  }
}

static double median_cycles(std::vector<long long>& c) {
  std::vector<long long> v = c; std::sort(v.begin(), v.end()); return (double)v[v.size() / 2];
}
#include <algorithm>

static int sustained(int reps) {
  // sustained TMA read (tile 43008, 3 stages, 17 warps) of 48 GB, reps times: is the HBM side stable?
  int nsm; CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  size_t bytes = (size_t)48 << 30; uint8_t* buf; CK(cudaMalloc(&buf, bytes)); CK(cudaMemset(buf, 1, bytes));
  uint32_t* dout; CK(cudaMalloc(&dout, 64));
  uint32_t tile = 43008; int stages = 3; size_t smem = 256 + (size_t)stages * tile; size_t ntiles = bytes / tile;
  CK(cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  printf("{\"sustained_tma_read_GBps\": [");
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0); k_tma<<<nsm, 17 * 32, smem>>>(buf, ntiles, tile, stages, dout); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%s%.0f", r ? ", " : "", (double)ntiles * tile / (ms * 1e6));
  }
  printf("]}\n");
  return 0;
}

int main(int argc, char** argv) {
  if (argc > 1) return sustained(atoi(argv[1]));
  int dev = 0; CK(cudaSetDevice(dev));
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, dev));
  const int nsm = prop.multiProcessorCount;
  printf("{\"device\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"smem_optin\": %zu,\n", prop.name, nsm, prop.l2CacheSize,
         prop.sharedMemPerBlockOptin);
  uint32_t* dout; CK(cudaMalloc(&dout, 64)); long long* dcyc; CK(cudaMalloc(&dcyc, sizeof(long long) * 4096));
  std::vector<long long> hc(4096);
  // ---- shared atomics
  const char* names[5] = {"atoms_lane_private_768keys", "atoms_same_addr", "atoms_rand48", "atoms_rand768", "lds_sts_rmw_lane_private"};
  for (int mode = 0; mode < 5; ++mode) {
    for (int threads : {256, 512, 1024}) {
      int iters = (mode == 1) ? 64 : 512;
      size_t smem = (mode == 4) ? (size_t)(threads / 32) * 48 * 32 * 4 : 768 * 32 * 4;
      if (smem > prop.sharedMemPerBlockOptin) continue;
      void (*fn)(uint32_t*, long long*, int) = nullptr;
      switch (mode) { case 0: fn = k_atoms<0>; break; case 1: fn = k_atoms<1>; break; case 2: fn = k_atoms<2>; break;
        case 3: fn = k_atoms<3>; break; default: fn = k_atoms<4>; }
      CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      fn<<<nsm, threads, smem>>>(dout, dcyc, iters / 8);
      CK(cudaDeviceSynchronize());
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      fn<<<nsm, threads, smem>>>(dout, dcyc, iters);
      cudaEventRecord(e1); CK(cudaDeviceSynchronize());
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      CK(cudaMemcpy(hc.data(), dcyc, sizeof(long long) * nsm, cudaMemcpyDeviceToHost));
      std::vector<long long> v(hc.begin(), hc.begin() + nsm);
      double cyc = median_cycles(v);
      double lane_ops = (double)threads * iters * 16;
      printf("\"%s_t%d\": {\"lane_ops_per_clk_per_sm\": %.3f, \"ms\": %.4f, \"clk_mhz_implied\": %.0f},\n", names[mode], threads,
             lane_ops / cyc, ms, cyc / (ms * 1e3));
    }
  }
  // ---- shared atomics, independent addresses (no dependent chain)
  for (int mode = 0; mode < 3; ++mode) {
    for (int threads : {512, 1024}) {
      int iters = 512;
      size_t smem = 768 * 32 * 4;
      void (*fn)(uint32_t*, long long*, int) = mode == 0 ? k_atoms_ilp<0> : (mode == 1 ? k_atoms_ilp<1> : k_atoms_ilp<2>);
      CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      fn<<<nsm, threads, smem>>>(dout, dcyc, 8); CK(cudaDeviceSynchronize());
      fn<<<nsm, threads, smem>>>(dout, dcyc, iters); CK(cudaDeviceSynchronize());
      CK(cudaMemcpy(hc.data(), dcyc, sizeof(long long) * nsm, cudaMemcpyDeviceToHost));
      std::vector<long long> v(hc.begin(), hc.begin() + nsm);
      double cyc = median_cycles(v);
      const char* nm = mode == 0 ? "atoms_ilp_lane_private_768keys" : (mode == 1 ? "atoms_ilp_lane_private_16keys_repeat" : "atoms_ilp_lane_private_48keys");
      printf("\"%s_t%d\": {\"lane_ops_per_clk_per_sm\": %.3f},\n", nm, threads, (double)threads * iters * 16 / cyc);
    }
  }
  // ---- warp intrinsics
  for (int mode = 0; mode < 2; ++mode) {
    int threads = 1024, iters = 256;
    void (*fn)(uint32_t*, long long*, int) = mode == 0 ? k_warp<0> : k_warp<1>;
    fn<<<nsm, threads>>>(dout, dcyc, 8); CK(cudaDeviceSynchronize());
    fn<<<nsm, threads>>>(dout, dcyc, iters); CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(hc.data(), dcyc, sizeof(long long) * nsm, cudaMemcpyDeviceToHost));
    std::vector<long long> v(hc.begin(), hc.begin() + nsm);
    double cyc = median_cycles(v);
    double warp_ops = (double)(threads / 32) * iters * 16;
    printf("\"%s\": {\"warp_instr_per_clk_per_sm\": %.3f},\n", mode == 0 ? "match_any" : "reduce_add", warp_ops / cyc);
  }
  // ---- HBM read
  size_t bytes = (size_t)16 << 30;
  uint8_t* buf; CK(cudaMalloc(&buf, bytes)); CK(cudaMemset(buf, 1, bytes));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int blocks_per_sm : {2, 4, 8}) {
    int g = nsm * blocks_per_sm;
    k_ldg<<<g, 512>>>((const uint4*)buf, bytes / 16, dout); CK(cudaDeviceSynchronize());
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); k_ldg<<<g, 512>>>((const uint4*)buf, bytes / 16, dout); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); best = std::min(best, ms);
    }
    printf("\"ldg128_read_b%d\": {\"GBps\": %.1f},\n", blocks_per_sm, bytes / (best * 1e6));
  }
  for (uint32_t tile : {16384u, 32768u, 46080u}) {
    for (int stages : {3, 4, 6}) {
      for (int warps : {5, 9, 17}) {
        size_t smem = 256 + (size_t)stages * tile;
        if (smem > prop.sharedMemPerBlockOptin) continue;
        size_t ntiles = bytes / tile;
        CK(cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_tma<<<nsm, warps * 32, smem>>>(buf, ntiles, tile, stages, dout); CK(cudaDeviceSynchronize());
        float best = 1e9;
        for (int r = 0; r < 3; ++r) {
          cudaEventRecord(e0); k_tma<<<nsm, warps * 32, smem>>>(buf, ntiles, tile, stages, dout); cudaEventRecord(e1);
          CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); best = std::min(best, ms);
        }
        printf("\"tma_read_t%u_s%d_w%d\": {\"GBps\": %.1f},\n", tile, stages, warps, (double)ntiles * tile / (best * 1e6));
      }
    }
  }
  printf("\"done\": true}\n");
  return 0;
}
