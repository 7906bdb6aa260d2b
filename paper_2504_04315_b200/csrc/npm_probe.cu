// npm_probe.cu -- measurement probe, not part of the method: the peak rate of
// random 16-byte float4 gathers and float4 scatter-adds (red.global.add.v4.f32)
// into a table of a given size.  SURVEY 8(d) asks for a measured L2
// random-gather peak next to the HBM peak: the c2-c4 grid tables (10.2 MB)
// are L2-resident, so the gathers/scatters of the fused kernels are bounded by
// L1TEX/L2 access throughput, not by DRAM bandwidth.  bench.py reports the
// fused kernels' grid accesses against this probe.
//
// Access pattern: each thread handles "samples" of 8 x `levels` accesses;
// corner c of level l of sample s reads entry hash(s, l, c) mod T (uniform
// random, no spatial coherence: the unbinned training order is random).
// 16 accesses are in flight per thread, as in the fused kernels.
#include <cuda_runtime.h>
#include <stdint.h>

#include "npm.h"

namespace {

__device__ __forceinline__ uint32_t mix32(uint32_t x) {   // lowbias32
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
  return x;
}

__global__ void __launch_bounds__(256) probe_gather_kernel(const float4* __restrict__ tab, uint32_t T,
                                                           int64_t n, int levels, float* __restrict__ out) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (int l = 0; l < levels; l += 2) {
      float4 v[16];
#pragma unroll
      for (int c = 0; c < 16; ++c)
        v[c] = __ldg(tab + mix32((uint32_t)s * 0x9E3779B9u + (uint32_t)(l * 8 + c)) % T);
#pragma unroll
      for (int c = 0; c < 16; ++c) acc += v[c].x + v[c].y + v[c].z + v[c].w;
    }
    out[s] = acc;
  }
}

__global__ void __launch_bounds__(256) probe_scatter_kernel(float4* __restrict__ tab, uint32_t T, int64_t n,
                                                            int levels) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
    for (int l = 0; l < levels; l += 2) {
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        float4* p = tab + mix32((uint32_t)s * 0x9E3779B9u + (uint32_t)(l * 8 + c)) % T;
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(1e-7f), "f"(1e-7f),
                     "f"(1e-7f), "f"(1e-7f)
                     : "memory");
      }
    }
  }
}

}  // namespace

extern "C" npm_status npm_probe_grid_access(int cuda_device, int64_t table_entries, int64_t n_samples,
                                            int levels, int kind, int reps, double* ms_per_rep) {
  if (table_entries <= 0 || table_entries > 0xFFFFFFFFll || n_samples <= 0 || levels <= 0 || (levels & 1) ||
      (kind != 0 && kind != 1) || reps <= 0 || !ms_per_rep)
    return NPM_ERR_INVALID;
  int prev = 0;
  cudaGetDevice(&prev);
  if (cudaSetDevice(cuda_device) != cudaSuccess) return NPM_ERR_CUDA;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cuda_device);
  float4* tab = nullptr;
  float* out = nullptr;
  cudaStream_t st = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  npm_status r = NPM_OK;
  if (cudaMalloc(&tab, (size_t)table_entries * sizeof(float4)) != cudaSuccess ||
      cudaMalloc(&out, (size_t)n_samples * sizeof(float)) != cudaSuccess ||
      cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess) {
    r = NPM_ERR_CUDA;
  } else {
    cudaMemsetAsync(tab, 0, (size_t)table_entries * sizeof(float4), st);
    const int blocks = sms * 8;   // 2048 threads per SM
    auto launch = [&]() {
      if (kind == 0)
        probe_gather_kernel<<<blocks, 256, 0, st>>>(tab, (uint32_t)table_entries, n_samples, levels, out);
      else
        probe_scatter_kernel<<<blocks, 256, 0, st>>>(tab, (uint32_t)table_entries, n_samples, levels);
    };
    launch();   // warm-up: the table becomes L2-resident if it fits
    cudaEventRecord(e0, st);
    for (int i = 0; i < reps; ++i) launch();
    cudaEventRecord(e1, st);
    float ms = 0.f;
    if (cudaEventSynchronize(e1) != cudaSuccess || cudaEventElapsedTime(&ms, e0, e1) != cudaSuccess ||
        cudaGetLastError() != cudaSuccess)
      r = NPM_ERR_CUDA;
    *ms_per_rep = (double)ms / reps;
  }
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  if (st) cudaStreamDestroy(st);
  cudaFree(out);
  cudaFree(tab);
  cudaSetDevice(prev);
  return r;
}
