// npm_bin.cu -- spatial binning of a sample batch: counting sort by the Morton
// code of the sample's cell in a 16^3 grid over the scene AABB.  Not part of
// the method: it only reorders the processing of independent samples so that
// the 32 samples of a warp are spatially clustered and their grid gathers hit
// few cache lines.  Results are independent of
// the order up to fp32 summation order.
//
// Pass 1 (bin_count): each CTA histograms its contiguous span in smem and
//   adds its non-zero bins to the global histogram (one atomic per
//   (CTA, bin), not per sample: the samples lie on surfaces, so a few bins
//   are hot and per-sample atomics serialise on them).
// Pass 2 (bin_place): each CTA scans its chunk's histogram row in smem,
//   re-histograms its span, reserves its range in every non-zero bin with one
//   atomic, then places its samples with smem atomics.
// Sort chunks: batches above kSortChunk samples are sorted in independent
// consecutive chunks (histogram row = chunk, chunk-major scan), so that the
// scattered per-sample input reads and output writes of a binned launch stay
// inside one chunk's window (~44 MB of SoA I/O at 2^20 queries), which the
// 126 MB L2 merges before write-back.  Measured on B200 (c3, 8.4 M queries):
// one global sort made the query kernel 44 % slower per query than at c2.
#include <cstdlib>

#include "npm_kernels.cuh"

namespace npm {
namespace {

constexpr int kBins = 1 << kBinBits;
constexpr int kThreads = 512;

__device__ __forceinline__ uint32_t spread3(uint32_t v) {   // 5 bits -> every third bit
  v &= 0x1Fu;
  v = (v | (v << 8)) & 0x0100F00Fu;
  v = (v | (v << 4)) & 0x010C30C3u;
  v = (v | (v << 2)) & 0x01249249u;
  return v;
}

__device__ __forceinline__ uint32_t bin_key(const float* px, const float* py, const float* pz, int64_t i,
                                            const GridDesc& g) {
  const float ux = normalize_axis(__ldg(px + i), g.lo[0], g.inv[0]);
  const float uy = normalize_axis(__ldg(py + i), g.lo[1], g.inv[1]);
  const float uz = normalize_axis(__ldg(pz + i), g.lo[2], g.inv[2]);
  // 15-bit Morton code of a 32^3 cell grid: bin = top 12 bits (16^3 cells),
  // sub-cell = low 3 bits (bin_refine orders each bin by it)
  const uint32_t cx = min((uint32_t)(ux * 32.0f), 31u), cy = min((uint32_t)(uy * 32.0f), 31u),
                 cz = min((uint32_t)(uz * 32.0f), 31u);
  return spread3(cx) | (spread3(cy) << 1) | (spread3(cz) << 2);
}

__global__ void __launch_bounds__(kThreads) bin_count_kernel(const float* __restrict__ px,
                                                             const float* __restrict__ py,
                                                             const float* __restrict__ pz, int64_t n,
                                                             int64_t chunk, int64_t sort_chunk, GridDesc g,
                                                             uint32_t* __restrict__ keys, uint32_t* __restrict__ hist) {
  __shared__ uint32_t h[kBins];
  for (int b = threadIdx.x; b < kBins; b += blockDim.x) h[b] = 0;
  __syncthreads();
  const int64_t i0 = (int64_t)blockIdx.x * chunk, i1 = min(i0 + chunk, n);
  for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
    const uint32_t k = bin_key(px, py, pz, i, g);
    keys[i] = k;
    atomicAdd(h + (k >> (15 - kBinBits)), 1u);
  }
  __syncthreads();
  hist += (i0 / sort_chunk) * kBins;   // this span's sort-chunk row
  for (int b = threadIdx.x; b < kBins; b += blockDim.x)
    if (h[b]) atomicAdd(hist + b, h[b]);
}

// Pass 2+3 fused: every CTA scans its sort-chunk's histogram row itself (4096
// counts, block scan in smem) instead of a separate single-CTA scan launch,
// then reserves its range in each non-zero bin (cursor atomics) and places.
__global__ void __launch_bounds__(kThreads) bin_place_kernel(const uint32_t* __restrict__ keys, int64_t n,
                                                             int64_t chunk, int64_t sort_chunk,
                                                             const uint32_t* __restrict__ hist,
                                                             uint32_t* __restrict__ cursor,
                                                             uint32_t* __restrict__ bstart,
                                                             uint32_t* __restrict__ perm, bool pack) {
  constexpr int PER = kBins / kThreads;
  __shared__ uint32_t h[kBins];
  __shared__ uint32_t base[kBins];
  __shared__ uint32_t warp_tot[kThreads / 32];
  const int t = threadIdx.x;
  const int64_t i0 = (int64_t)blockIdx.x * chunk, i1 = min(i0 + chunk, n);
  const int64_t row = i0 / sort_chunk;
  // exclusive scan of this chunk's counts; chunk row r starts at slot r * sort_chunk
  {
    uint32_t v[PER], sum = 0;
#pragma unroll
    for (int j = 0; j < PER; ++j) { v[j] = hist[row * kBins + t * PER + j]; sum += v[j]; }
    uint32_t inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
      if ((t & 31) >= o) inc += y;
    }
    if ((t & 31) == 31) warp_tot[t >> 5] = inc;
    for (int b2 = t; b2 < kBins; b2 += blockDim.x) h[b2] = 0;
    __syncthreads();
    if (t < 32) {
      const uint32_t w = t < kThreads / 32 ? warp_tot[t] : 0u;
      uint32_t wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
        if (t >= o) wi += y;
      }
      if (t < kThreads / 32) warp_tot[t] = wi - w;
    }
    __syncthreads();
    uint32_t run = (uint32_t)(row * sort_chunk) + warp_tot[t >> 5] + inc - sum;
    const bool publish = i0 == row * sort_chunk;   // the row's first CTA
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      base[t * PER + j] = run;
      if (publish) bstart[row * kBins + t * PER + j] = run;
      run += v[j];
    }
  }
  __syncthreads();
  for (int64_t i = i0 + t; i < i1; i += blockDim.x) atomicAdd(h + (keys[i] >> (15 - kBinBits)), 1u);
  __syncthreads();
  cursor += row * kBins;
  for (int b2 = t; b2 < kBins; b2 += blockDim.x) {
    const uint32_t c = h[b2];
    h[b2] = c ? base[b2] + atomicAdd(cursor + b2, c) : 0u;   // this CTA's range in bin b2
  }
  __syncthreads();
  for (int64_t i = i0 + t; i < i1; i += blockDim.x) {
    const uint32_t k = keys[i];
    const uint32_t slot = atomicAdd(h + (k >> (15 - kBinBits)), 1u);
    // pack: the sub-cell rides in the top 3 bits for bin_refine (n < 2^29)
    perm[slot] = (uint32_t)i | (pack ? (k & 7u) << 29 : 0u);
  }
}

// Pass 3 (bin_refine, HBM-resident tables only): one CTA per bin orders the
// bin's samples by their 32^3 sub-cell (3-bit counting sort in smem), so a
// 128-sample tile covers an eighth of a bin's volume: more corners shared at
// the mid levels.  Measured on B200: c5 query 3.15 -> 3.08 ms, binned train
// 5.10 -> 4.80 ms for +89 us of refinement; with L2-resident tables (c2, c3)
// the refinement costs more than the queries gain (c2 +26 us vs -11 us).
constexpr int kRefineMax = 8192;   // larger bins keep the place order
__global__ void __launch_bounds__(256) bin_refine_kernel(const uint32_t* __restrict__ hist,
                                                         const uint32_t* __restrict__ bstart, int nb,
                                                         uint32_t* __restrict__ perm) {
  __shared__ uint32_t sp[kRefineMax];
  __shared__ uint32_t cnt[8], off[8];
  constexpr uint32_t kIdx = (1u << 29) - 1u;
  const int b = blockIdx.x;
  if (b >= nb) return;
  const uint32_t c = hist[b];
  if (c == 0) return;
  const uint32_t s0 = bstart[b];
  const int t = threadIdx.x;
  if (c <= 128 || c > (uint32_t)kRefineMax) {   // keep the place order; strip the packed sub-cells
    for (uint32_t j = t; j < c; j += blockDim.x) perm[s0 + j] &= kIdx;
    return;
  }
  if (t < 8) cnt[t] = 0;
  __syncthreads();
  for (uint32_t j = t; j < c; j += blockDim.x) {
    const uint32_t v = perm[s0 + j];
    sp[j] = v;
    atomicAdd(cnt + (v >> 29), 1u);
  }
  __syncthreads();
  if (t == 0) {
    uint32_t run = 0;
    for (int k = 0; k < 8; ++k) { off[k] = run; run += cnt[k]; }
  }
  __syncthreads();
  for (uint32_t j = t; j < c; j += blockDim.x) {
    const uint32_t v = sp[j];
    perm[s0 + atomicAdd(off + (v >> 29), 1u)] = v & kIdx;
  }
}

}  // namespace

// counts [chunks][kBins], cursors [chunks][kBins], bin starts [chunks][kBins]
int bin_hist_entries(int64_t n, int64_t sort_chunk) {
  const int64_t chunks = n <= sort_chunk ? 1 : (n + sort_chunk - 1) / sort_chunk;
  return (int)(3 * chunks * kBins);
}

// sort_chunk: n (one global sort) or kSortChunk (a multiple of 32 * 4096)
int launch_bin(const float* px, const float* py, const float* pz, int64_t n, int64_t sort_chunk, bool refine,
               const GridDesc& g, uint32_t* keys, uint32_t* hist, uint32_t* perm, int sms, cudaStream_t st) {
  if (n == 0) return 0;
  if (sort_chunk >= n) sort_chunk = n;
  const int nb = bin_hist_entries(n, sort_chunk) / 3;
  cudaMemsetAsync(hist, 0, (size_t)2 * nb * sizeof(uint32_t), st);   // counts + cursors
  // samples per CTA: small spans (short per-thread loops of dependent loads and
  // smem atomics, many CTAs in flight) against the per-CTA fixed cost of
  // scanning / flushing the 4096-bin row (B200 c2, one sort: 4096 per CTA
  // 33 us, 2048 41 us, 1024 50 us).  NPM_BIN_SPAN (measurement knob): samples
  // per CTA, a power of two >= 512.
  static int64_t knob = -1;
  if (knob < 0) {
    const char* e = getenv("NPM_BIN_SPAN");
    knob = e ? atoll(e) : 0;
  }
  const int64_t per = knob >= 512 ? knob : 4096;
  int64_t span;
  if (sort_chunk == n) {   // one sort over the whole batch
    const int64_t want = (n + per - 1) / per;
    const int64_t cap = knob >= 512 ? want : (int64_t)sms * 2;
    const int blocks = (int)(want < cap ? want : cap);
    span = (n + blocks - 1) / blocks;
  } else {                 // chunks of sort_chunk; CTA spans never straddle a chunk
    // sort_chunk / 128 = 8192 samples (B200 c3 bin 130 -> 106 us; / 256: 120 us)
    span = knob >= 512 && sort_chunk % knob == 0 ? knob : sort_chunk / 128;
  }
  const int blocks = (int)((n + span - 1) / span);
  bin_count_kernel<<<blocks, kThreads, 0, st>>>(px, py, pz, n, span, sort_chunk, g, keys, hist);
  refine = refine && n < (int64_t(1) << 29);
  bin_place_kernel<<<blocks, kThreads, 0, st>>>(keys, n, span, sort_chunk, hist, hist + nb, hist + 2 * nb, perm,
                                                refine);
  if (!refine) return 2;
  bin_refine_kernel<<<nb, 256, 0, st>>>(hist, hist + 2 * nb, nb, perm);
  return 3;
}

}  // namespace npm
