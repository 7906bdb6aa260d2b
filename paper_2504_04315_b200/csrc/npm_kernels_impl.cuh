// npm_kernels_impl.cuh -- decoder shape descriptor, the encode-only kernel
// (npm_encode / npm_encode_debug) and warp reductions shared by the fused
// tcgen05 kernels (npm_tc_kernels.cuh).  The round-1 CUDA-core (FFMA) decoder
// path was removed in round 2; the fused tensor-core kernels are the only
// decoder path.
//
// Layout in HBM: SoA inputs; flat fp32 parameters
// [MLP layers W[out][in], b[out] ... | grid levels [entries][4]].
#pragma once
#include "npm_kernels.cuh"

namespace npm {
namespace detail {

constexpr int kThreads = 128;

__host__ __device__ constexpr int pad4(int x) { return (x + 3) & ~3; }

// Compile-time decoder shape.
template <int NIN_, int W_, int NL_, int NOUT_>
struct Net {
  static constexpr int NIN = NIN_, W = W_, NL = NL_, NOUT = NOUT_, K = NOUT_ / 4;
  static constexpr bool PRODUCT = (NIN_ == 65);
  static constexpr int NGRID = PRODUCT ? 32 : NIN_;   // L*F grid features
  static constexpr int L = NGRID / 4;
  static constexpr int NINP = pad4(NIN_);
  // smem float offsets: layer k weights [out][inp] then bias [out]
  __host__ __device__ static constexpr int in_dim(int k) { return k == 0 ? NIN : W; }
  __host__ __device__ static constexpr int inp_dim(int k) { return k == 0 ? NINP : W; }
  __host__ __device__ static constexpr int out_dim(int k) { return k == NL - 1 ? NOUT : W; }
  // sum of out_dim(j) for j < k (k <= NL).  Offsets below are closed forms, not
  // recursions: nvcc emits recursive constexpr functions as real device calls
  // when the argument is an unrolled loop index.
  __host__ __device__ static constexpr int osum(int k) { return k < NL ? k * W : (NL - 1) * W + NOUT; }
  __host__ __device__ static constexpr int w_off(int k) {
    return k == 0 ? 0 : out_dim(0) * (NINP + 1) + (W + 1) * (osum(k) - out_dim(0));
  }
  __host__ __device__ static constexpr int b_off(int k) { return w_off(k) + out_dim(k) * inp_dim(k); }
  static constexpr int SMEM_FLOATS = b_off(NL - 1) + NOUT;
  // offsets in the global (logical, unpadded) layout
  __host__ __device__ static constexpr int gw_off(int k) {
    return k == 0 ? 0 : out_dim(0) * (NIN + 1) + (W + 1) * (osum(k) - out_dim(0));
  }
  __host__ __device__ static constexpr int gb_off(int k) { return gw_off(k) + out_dim(k) * in_dim(k); }
  static constexpr int N_MLP = gb_off(NL - 1) + NOUT;
};

// Eq. 13 for one sample: z[0 .. 4L) = concat_l sum_c w_c E_l[idx_c].
template <int L>
__device__ __forceinline__ void encode_sample(const GridDesc& g, const float4* __restrict__ tab, float x, float y,
                                              float z, float* out, uint32_t* dbg_idx, float* dbg_w, int64_t n,
                                              int64_t i) {
  const float ux = normalize_axis(x, g.lo[0], g.inv[0]);
  const float uy = normalize_axis(y, g.lo[1], g.inv[1]);
  const float uz = normalize_axis(z, g.lo[2], g.inv[2]);
#pragma unroll
  for (int l = 0; l < L; ++l) {
    LevelCorners lc;
    level_corners(g, l, ux, uy, uz, lc);
    const float4* t = tab + g.off[l];
    float4 v[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) v[c] = __ldg(t + lc.idx[c]);
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      a0 = fmaf(lc.w[c], v[c].x, a0);
      a1 = fmaf(lc.w[c], v[c].y, a1);
      a2 = fmaf(lc.w[c], v[c].z, a2);
      a3 = fmaf(lc.w[c], v[c].w, a3);
    }
    out[4 * l + 0] = a0; out[4 * l + 1] = a1; out[4 * l + 2] = a2; out[4 * l + 3] = a3;
    if (dbg_idx) {
#pragma unroll
      for (int c = 0; c < 8; ++c) dbg_idx[(int64_t)(l * 8 + c) * n + i] = lc.idx[c];
    }
    if (dbg_w) {
#pragma unroll
      for (int c = 0; c < 8; ++c) dbg_w[(int64_t)(l * 8 + c) * n + i] = lc.w[c];
    }
  }
}

// Encode-only kernel (any L, no MLP): Eq. 13 + debug corner export.
template <int L>
__global__ void __launch_bounds__(kThreads) encode_kernel(QueryArgs a) {
  const float4* tab = reinterpret_cast<const float4*>(a.params);  // points at the grid section
  const int64_t n = a.n;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float z[4 * L];
    encode_sample<L>(a.grid, tab, __ldg(a.px + i), __ldg(a.py + i), __ldg(a.pz + i), z, a.dbg_idx, a.dbg_w, n, i);
    if (a.feat) {
#pragma unroll
      for (int j = 0; j < 4 * L; ++j) a.feat[(int64_t)j * n + i] = z[j];
    }
  }
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ unsigned warp_sum_u(unsigned v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace detail
}  // namespace npm
