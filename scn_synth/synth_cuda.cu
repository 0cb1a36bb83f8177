// synth_cuda.cu — device fill of synthetic frames (INPUT ONLY, untimed).
// Same generator as synth_host.c (scn_synth.h); used by bench.py and the GPU
// tests to materialise sampled rows directly in HBM, since decode is out of
// scope (BASELINE.json north_star). Holds none of the method's arithmetic.
#include "scn_synth.h"
#include "synth_host.c"  // host helpers compiled into the same .so
#include <cuda_runtime.h>
#include <stdlib.h>

typedef struct {
  synth_frame_desc d;
  synth_shot_params sp;
  uint32_t fkey;
  uint32_t pad;
  uint64_t dst;  // device address of the frame
} synth_job;

__global__ void synth_fill_kernel(const synth_job* __restrict__ jobs, int32_t mode, int32_t width, int32_t height) {
  const synth_job& j = jobs[blockIdx.y];
  const int64_t F = (int64_t)width * height * 3;
  uint8_t* dst = (uint8_t*)j.dst;
  synth_shot_params sp = j.sp;
  synth_frame_desc d = j.d;
  for (int64_t chunk = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; chunk * 16 < F;
       chunk += (int64_t)gridDim.x * blockDim.x) {
    int64_t o = chunk * 16;
    uint8_t b[16];
    int64_t pix = o / 3;
    int32_t c = (int32_t)(o - pix * 3);
    int32_t y = (int32_t)(pix / width), x = (int32_t)(pix - (int64_t)y * width);
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      b[k] = (o + k < F) ? synth_pixel(mode, j.fkey, &sp, width, &d, y, x, c) : 0;
      if (++c == 3) { c = 0; if (++x == width) { x = 0; ++y; } }
    }
    if (o + 16 <= F) {
      uint4 v;
      v.x = b[0] | (b[1] << 8) | (b[2] << 16) | ((uint32_t)b[3] << 24);
      v.y = b[4] | (b[5] << 8) | (b[6] << 16) | ((uint32_t)b[7] << 24);
      v.z = b[8] | (b[9] << 8) | (b[10] << 16) | ((uint32_t)b[11] << 24);
      v.w = b[12] | (b[13] << 8) | (b[14] << 16) | ((uint32_t)b[15] << 24);
      *(uint4*)(dst + o) = v;
    } else {
      for (int k = 0; k < 16 && o + k < F; ++k) dst[o + k] = b[k];
    }
  }
}

extern "C" {

// Fill n frames. h_rows[i] = row of video h_videos[i]; d_dst[i] = device address.
// d_jobs: device scratch of n * sizeof(synth_job) bytes (caller-owned). Returns cudaError_t.
size_t synth_job_bytes(void) { return sizeof(synth_job); }

int synth_fill_frames_device(const synth_spec* spec, const int32_t* h_videos, const int64_t* h_rows,
                             const uint64_t* h_dst, int64_t n, void* d_jobs, cudaStream_t stream) {
  if (n <= 0) return 0;
  synth_job* h = (synth_job*)malloc(sizeof(synth_job) * (size_t)n);
  if (!h) return (int)cudaErrorMemoryAllocation;
  for (int64_t i = 0; i < n; ++i) {
    h[i].d = synth_describe(spec, h_videos[i], h_rows[i]);
    int32_t scene = spec->shared_scene ? 0 : h_videos[i];
    h[i].sp = synth_shot(spec->seed, spec->width, spec->height, scene, h[i].d.shot);
    h[i].fkey = synth_frame_key(spec->seed, h_videos[i], h_rows[i]);
    h[i].pad = 0;
    h[i].dst = h_dst[i];
  }
  cudaError_t e = cudaMemcpyAsync(d_jobs, h, sizeof(synth_job) * (size_t)n, cudaMemcpyHostToDevice, stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  free(h);
  if (e != cudaSuccess) return (int)e;
  const int64_t F = (int64_t)spec->width * spec->height * 3;
  int64_t chunks = (F + 15) / 16;
  int bx = (int)((chunks + 255) / 256);
  if (bx > 1024) bx = 1024;
  for (int64_t off = 0; off < n; off += 65535) {
    int64_t cnt = n - off < 65535 ? n - off : 65535;
    dim3 grid(bx, (unsigned)cnt);
    synth_fill_kernel<<<grid, 256, 0, stream>>>((const synth_job*)d_jobs + off, spec->mode, spec->width, spec->height);
  }
  return (int)cudaGetLastError();
}
}
