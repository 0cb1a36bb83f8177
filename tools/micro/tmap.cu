// Feasibility probe: can a 2-D TMA tensor map with an OVERLAPPING view (dims {512, N},
// row stride 256 B) load a byte row that starts at ANY address into 16-byte aligned
// shared memory (box {256, k} at coordinate (addr % 256, addr / 256))? Prints the encode
// status, then checks the landed bytes against global memory for many misalignments.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cstdlib>

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const __grid_constant__ CUtensorMap tm, int x0, int y0, int nbytes, uint8_t* out) {
  __shared__ __align__(128) uint8_t buf[256 * 20];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&bar)), "r"(nbytes));
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        ::"r"(smem_addr(buf)), "l"(&tm), "r"(x0), "r"(y0), "r"(smem_addr(&bar)) : "memory");
  }
  asm volatile(
      "{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0; @!p bra W; }" ::"r"(smem_addr(&bar)));
  for (int i = threadIdx.x; i < nbytes; i += blockDim.x) out[i] = buf[i];
}

int main(int argc, char** argv) {
  const int only = argc > 1 ? atoi(argv[1]) : -1;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto encode = (CUresult(*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill))fn;
  const size_t bytes = 1 << 20;
  uint8_t* d;
  cudaMalloc(&d, bytes + 4096);
  std::vector<uint8_t> h(bytes);
  for (size_t i = 0; i < bytes; ++i) h[i] = (uint8_t)(i * 2654435761u >> 24);
  cudaMemcpy(d, h.data(), bytes, cudaMemcpyHostToDevice);
  CUtensorMap tm;
  const int K = 17;
  cuuint64_t dims[2] = {512, (bytes - 512) / 256 + 1};
  cuuint64_t strides[1] = {256};
  cuuint32_t box[2] = {256, (cuuint32_t)K};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode overlapping view: %d\n", (int)r);
  if (r != CUDA_SUCCESS) return 1;
  uint8_t* dout;
  cudaMalloc(&dout, 256 * K);
  int bad = 0;
  for (int off : {0, 1, 2, 3, 7, 13, 255, 256 + 5, 4098 * 3, 4098 * 7 + 1, 100000}) {
    if (only >= 0 && off != only) continue;
    probe<<<1, 128>>>(tm, off % 256, off / 256, 256 * K, dout);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<uint8_t> o(256 * K);
    cudaMemcpy(o.data(), dout, o.size(), cudaMemcpyDeviceToHost);
    int mism = 0;
    for (int i = 0; i < 256 * K; ++i) mism += o[i] != h[off + i];
    printf("off %d: %s, mismatches %d\n", off, cudaGetErrorString(e), mism);
    bad += mism;
  }
  printf("%s\n", bad ? "FAIL" : "PASS");
  return 0;
}
