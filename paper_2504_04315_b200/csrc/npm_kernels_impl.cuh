// npm_kernels_impl.cuh -- templated sm_100a kernels of the NPM hot path (CUDA-core path).
// Instantiated once per decoder shape in npm_net_*.cu (parallel compilation).
//
// Stages (Fig. 2 (1)-(5)):
//   encode   Eq. 13 grid gather + trilinear blend
//   decode   Eq. 14 MLP, fp32 FFMA with weights in smem
//   head     Table 1 mappings, Eq. 4 pdf, Jakob sampling
//   train    Eq. 9 head -> backprop -> grid scatter-add
//   adam     Adam + EMA
//
// Layout in HBM: SoA inputs; flat fp32 parameters
// [MLP layers W[out][in], b[out] ... | grid levels [entries][4]]; training
// scratch feature-major [rows][n] so that thread-per-sample accesses coalesce.
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

template <class N>
__device__ __forceinline__ void stage_weights(const float* __restrict__ g, float* s) {
#pragma unroll
  for (int k = 0; k < N::NL; ++k) {
    const int in = N::in_dim(k), inp = N::inp_dim(k), out = N::out_dim(k);
    for (int e = threadIdx.x; e < out * inp; e += blockDim.x) {
      const int o = e / inp, i = e - o * inp;
      s[N::w_off(k) + e] = i < in ? __ldg(g + N::gw_off(k) + o * in + i) : 0.0f;
    }
    for (int o = threadIdx.x; o < out; o += blockDim.x) s[N::b_off(k) + o] = __ldg(g + N::gb_off(k) + o);
  }
}

// out = act(W in + b), W [OUT][INP] in smem, broadcast reads (all lanes read
// the same weight): one LDS.128 feeds four FFMAs.
template <int INP, int OUT, bool RELU>
__device__ __forceinline__ void dense_fwd(const float* __restrict__ sw, const float* __restrict__ sb,
                                          const float* in, float* out) {
#pragma unroll
  for (int o = 0; o < OUT; ++o) {
    const float4* w4 = reinterpret_cast<const float4*>(sw + o * INP);
    float a0 = sb[o], a1 = 0.0f;
#pragma unroll
    for (int i = 0; i < INP / 4; ++i) {
      const float4 w = w4[i];
      a0 = fmaf(w.x, in[4 * i + 0], a0);
      a1 = fmaf(w.y, in[4 * i + 1], a1);
      a0 = fmaf(w.z, in[4 * i + 2], a0);
      a1 = fmaf(w.w, in[4 * i + 3], a1);
    }
    const float a = a0 + a1;
    out[o] = RELU ? fmaxf(a, 0.0f) : a;
  }
}

// din[i] = sum_o W[o][i] dout[o]  (W^T dout), masked by act_in > 0 if MASK.
template <int INP, int IN, int OUT, bool MASK>
__device__ __forceinline__ void dense_bwd(const float* __restrict__ sw, const float* dout, const float* act_in,
                                          float* din) {
#pragma unroll
  for (int i = 0; i < IN; ++i) din[i] = 0.0f;
#pragma unroll
  for (int o = 0; o < OUT; ++o) {
    const float d = dout[o];
    const float4* w4 = reinterpret_cast<const float4*>(sw + o * INP);
#pragma unroll
    for (int i = 0; i < INP / 4; ++i) {
      const float4 w = w4[i];
      if (4 * i + 0 < IN) din[4 * i + 0] = fmaf(w.x, d, din[4 * i + 0]);
      if (4 * i + 1 < IN) din[4 * i + 1] = fmaf(w.y, d, din[4 * i + 1]);
      if (4 * i + 2 < IN) din[4 * i + 2] = fmaf(w.z, d, din[4 * i + 2]);
      if (4 * i + 3 < IN) din[4 * i + 3] = fmaf(w.w, d, din[4 * i + 3]);
    }
  }
  if (MASK) {
#pragma unroll
    for (int i = 0; i < IN; ++i) din[i] = act_in[i] > 0.0f ? din[i] : 0.0f;
  }
}

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

// Network input z (radiance: G(x); product: [G, SH4(w_o), SH4(n), roughness]).
template <class N>
__device__ __forceinline__ void network_input(const GridDesc& g, const float4* tab, const float* px,
                                              const float* py, const float* pz, const float* wox,
                                              const float* woy, const float* woz, const float* nx,
                                              const float* ny, const float* nz, const float* rough,
                                              int64_t i, float* z, uint32_t* dbg_idx, float* dbg_w, int64_t n) {
  encode_sample<N::L>(g, tab, __ldg(px + i), __ldg(py + i), __ldg(pz + i), z, dbg_idx, dbg_w, n, i);
  if (N::PRODUCT) {
    sh4(__ldg(wox + i), __ldg(woy + i), __ldg(woz + i), z + 32);
    sh4(__ldg(nx + i), __ldg(ny + i), __ldg(nz + i), z + 48);
    z[64] = __ldg(rough + i);
  }
#pragma unroll
  for (int j = N::NIN; j < N::NINP; ++j) z[j] = 0.0f;
}

template <class N>
__device__ __forceinline__ void mlp_forward(const float* sw, const float* z, float* raw, float* h1, float* h2) {
  if constexpr (N::NL == 2) {
    dense_fwd<N::NINP, N::W, true>(sw + N::w_off(0), sw + N::b_off(0), z, h1);
    dense_fwd<N::W, N::NOUT, false>(sw + N::w_off(1), sw + N::b_off(1), h1, raw);
  } else {
    dense_fwd<N::NINP, N::W, true>(sw + N::w_off(0), sw + N::b_off(0), z, h1);
    dense_fwd<N::W, N::W, true>(sw + N::w_off(1), sw + N::b_off(1), h1, h2);
    dense_fwd<N::W, N::NOUT, false>(sw + N::w_off(N::NL - 1), sw + N::b_off(N::NL - 1), h2, raw);
  }
}

// ---------------------------------------------------------------------------
// Fused query kernel: encode -> decode -> Table 1 -> {pdf, sample}.
// Persistent grid-stride loop, thread per sample, weights staged once per CTA.
template <class N>
__global__ void __launch_bounds__(kThreads) query_kernel(QueryArgs a) {
  extern __shared__ float4 smem4[];
  float* sw = reinterpret_cast<float*>(smem4);
  const bool need_mlp = a.raw || a.lambda || a.kappa || a.mu || a.pdf || a.do_sample;
  if (need_mlp) {
    stage_weights<N>(a.params, sw);
    __syncthreads();
  }
  const float4* tab = reinterpret_cast<const float4*>(a.params + N::N_MLP);
  const int64_t n = a.n;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float z[N::NINP];
    if (a.feat_in) {
#pragma unroll
      for (int j = 0; j < N::NGRID; ++j) z[j] = __ldg(a.feat_in + (int64_t)j * n + i);
#pragma unroll
      for (int j = N::NGRID; j < N::NINP; ++j) z[j] = 0.0f;
    } else {
      network_input<N>(a.grid, tab, a.px, a.py, a.pz, a.wox, a.woy, a.woz, a.nx, a.ny, a.nz, a.rough, i, z,
                       a.dbg_idx, a.dbg_w, n);
    }
    if (a.feat) {
#pragma unroll
      for (int j = 0; j < N::NGRID; ++j) a.feat[(int64_t)j * n + i] = z[j];
    }
    if (!need_mlp) continue;
    float raw[N::NOUT];
    {
      float h1[N::W], h2[N::W];
      mlp_forward<N>(sw, z, raw, h1, h2);
    }
    if (a.raw) {
#pragma unroll
      for (int j = 0; j < N::NOUT; ++j) a.raw[(int64_t)j * n + i] = raw[j];
    }
    Mixture<N::K> m;
    activate<N::K>(raw, a.log_kmin, a.log_kmax, m);
    if (a.lambda) {
#pragma unroll
      for (int j = 0; j < N::K; ++j) a.lambda[(int64_t)j * n + i] = m.lam[j];
    }
    if (a.kappa) {
#pragma unroll
      for (int j = 0; j < N::K; ++j) a.kappa[(int64_t)j * n + i] = m.kap[j];
    }
    if (a.mu) {
#pragma unroll
      for (int j = 0; j < N::K; ++j) {
        a.mu[(int64_t)(0 * N::K + j) * n + i] = m.mx[j];
        a.mu[(int64_t)(1 * N::K + j) * n + i] = m.my[j];
        a.mu[(int64_t)(2 * N::K + j) * n + i] = m.mz[j];
      }
    }
    if (a.pdf) a.pdf[i] = mixture_pdf<N::K>(m, __ldg(a.wx + i), __ldg(a.wy + i), __ldg(a.wz + i));
    if (a.do_sample) {
      float3 u;
      if (a.u) u = make_float3(__ldg(a.u + i), __ldg(a.u + n + i), __ldg(a.u + 2 * n + i));
      else u = philox_uniforms(a.seed, (uint64_t)i + a.offset);
      float wx, wy, wz;
      mixture_sample<N::K>(m, u.x, u.y, u.z, wx, wy, wz);
      a.sx[i] = wx; a.sy[i] = wy; a.sz[i] = wz;
      a.spdf[i] = mixture_pdf<N::K>(m, wx, wy, wz);
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

// ---------------------------------------------------------------------------
// Training forward: z, h_k stored feature-major; Eq. 9 head -> delta[NL-1].
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

template <class N>
__global__ void __launch_bounds__(kThreads) train_forward_kernel(TrainArgs a) {
  extern __shared__ float4 smem4[];
  float* sw = reinterpret_cast<float*>(smem4);
  stage_weights<N>(a.params, sw);
  __syncthreads();
  const float4* tab = reinterpret_cast<const float4*>(a.params + N::N_MLP);
  const int64_t n = a.n;
  double loss = 0.0;
  unsigned c_used = 0, c_zero = 0, c_drop = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t n_iter = (n + stride - 1) / stride;
  for (int64_t it = 0; it < n_iter; ++it) {
    const int64_t i = it * stride + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
      float z[N::NINP];
      network_input<N>(a.grid, tab, a.px, a.py, a.pz, a.wox, a.woy, a.woz, a.nx, a.ny, a.nz, a.rough, i, z,
                       nullptr, nullptr, n);
#pragma unroll
      for (int j = 0; j < N::NIN; ++j) a.act[0][(int64_t)j * n + i] = z[j];
      float raw[N::NOUT];
      {
        float h1[N::W], h2[N::W];
        mlp_forward<N>(sw, z, raw, h1, h2);
#pragma unroll
        for (int j = 0; j < N::W; ++j) a.act[1][(int64_t)j * n + i] = h1[j];
        if constexpr (N::NL == 3) {
#pragma unroll
          for (int j = 0; j < N::W; ++j) a.act[2][(int64_t)j * n + i] = h2[j];
        }
      }
      // C-O12: a = D^/p~ (luminance if RGB, C-A11); drop if non-finite / p~ <= 0.
      float t = __ldg(a.target + i);
      bool all_zero = t == 0.0f;
      if (a.channels == 3) {
        const float tg = __ldg(a.target + a.target_stride + i), tb = __ldg(a.target + 2 * a.target_stride + i);
        all_zero = all_zero && tg == 0.0f && tb == 0.0f;   // D^ = 0 iff every channel is 0
        t = 0.2126f * t + 0.7152f * tg + 0.0722f * tb;
      }
      const float p = __ldg(a.spdf + i);
      const float ratio = t / p;
      const bool drop = !isfinite(ratio) || !isfinite(p) || !(p > 0.0f);
      const bool zero = !drop && all_zero;
      float draw[N::NOUT];
      if (drop || zero) {
#pragma unroll
        for (int j = 0; j < N::NOUT; ++j) draw[j] = 0.0f;
        c_drop += drop; c_zero += zero;
      } else {
        const float s = (float)(-(double)ratio * a.inv_n_global);
        const float logv = grad_head<N::K>(raw, a.log_kmin, a.log_kmax, __ldg(a.wx + i), __ldg(a.wy + i),
                                           __ldg(a.wz + i), s, draw);
        loss += (double)s * (double)logv;
        c_used += 1;
      }
#pragma unroll
      for (int j = 0; j < N::NOUT; ++j) a.delta[N::NL - 1][(int64_t)j * n + i] = draw[j];
    }
  }
  loss = warp_sum_d(loss);
  c_used = warp_sum_u(c_used); c_zero = warp_sum_u(c_zero); c_drop = warp_sum_u(c_drop);
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(a.stats, loss);
    atomicAdd(a.counters + 0, (unsigned long long)c_used);
    atomicAdd(a.counters + 1, (unsigned long long)c_zero);
    atomicAdd(a.counters + 2, (unsigned long long)c_drop);
  }
}

// Training backward (dX chain) + grid scatter-add (C-O14, C-O15).
template <class N>
__global__ void __launch_bounds__(kThreads) train_backward_kernel(TrainArgs a) {
  extern __shared__ float4 smem4[];
  float* sw = reinterpret_cast<float*>(smem4);
  stage_weights<N>(a.params, sw);
  __syncthreads();
  float4* gtab = reinterpret_cast<float4*>(a.grads + N::N_MLP);
  const int64_t n = a.n;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float d_out[N::NOUT];
#pragma unroll
    for (int j = 0; j < N::NOUT; ++j) d_out[j] = a.delta[N::NL - 1][(int64_t)j * n + i];
    float d1[N::W];
    if constexpr (N::NL == 3) {
      float h2[N::W], d2[N::W], h1[N::W];
#pragma unroll
      for (int j = 0; j < N::W; ++j) h2[j] = a.act[2][(int64_t)j * n + i];
      dense_bwd<N::W, N::W, N::NOUT, true>(sw + N::w_off(2), d_out, h2, d2);
#pragma unroll
      for (int j = 0; j < N::W; ++j) a.delta[1][(int64_t)j * n + i] = d2[j];
#pragma unroll
      for (int j = 0; j < N::W; ++j) h1[j] = a.act[1][(int64_t)j * n + i];
      dense_bwd<N::W, N::W, N::W, true>(sw + N::w_off(1), d2, h1, d1);
    } else {
      float h1[N::W];
#pragma unroll
      for (int j = 0; j < N::W; ++j) h1[j] = a.act[1][(int64_t)j * n + i];
      dense_bwd<N::W, N::W, N::NOUT, true>(sw + N::w_off(1), d_out, h1, d1);
    }
#pragma unroll
    for (int j = 0; j < N::W; ++j) a.delta[0][(int64_t)j * n + i] = d1[j];
    float dz[N::NGRID];
    dense_bwd<N::NINP, N::NGRID, N::W, false>(sw + N::w_off(0), d1, nullptr, dz);
    // scatter dz into the grid gradient: dE_l[idx_c] += w_c dz_l
    const float ux = normalize_axis(__ldg(a.px + i), a.grid.lo[0], a.grid.inv[0]);
    const float uy = normalize_axis(__ldg(a.py + i), a.grid.lo[1], a.grid.inv[1]);
    const float uz = normalize_axis(__ldg(a.pz + i), a.grid.lo[2], a.grid.inv[2]);
#pragma unroll
    for (int l = 0; l < N::L; ++l) {
      const float g0 = dz[4 * l], g1 = dz[4 * l + 1], g2 = dz[4 * l + 2], g3 = dz[4 * l + 3];
      if (g0 == 0.0f && g1 == 0.0f && g2 == 0.0f && g3 == 0.0f) continue;
      LevelCorners lc;
      level_corners(a.grid, l, ux, uy, uz, lc);
      float4* t = gtab + a.grid.off[l];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const float w = lc.w[c];
        atomicAdd(t + lc.idx[c], make_float4(w * g0, w * g1, w * g2, w * g3));
      }
    }
  }
}

// dW_k[o][i] += sum_n delta_k[o][n] act_k[i][n];  db_k[o] += sum_n delta_k[o][n].
// One CTA per (sample chunk, layer); 4x4 register micro-tiles over [OUT][INP].
constexpr int kDwTile = 32;    // samples per smem stage
template <class N>
__global__ void __launch_bounds__(256) weight_grad_kernel(TrainArgs a) {
  const int k = blockIdx.y;
  const int in = k == 0 ? N::NIN : N::W;
  const int inp = k == 0 ? N::NINP : N::W;
  const int out = k == N::NL - 1 ? N::NOUT : N::W;
  constexpr int MAXI = N::NINP > N::W ? N::NINP : N::W;
  constexpr int MAXO = N::NOUT > N::W ? N::NOUT : N::W;
  __shared__ __align__(16) float sd[kDwTile][MAXO + 4];
  __shared__ __align__(16) float sa[kDwTile][MAXI + 4];
  const float* D = a.delta[k];
  const float* A = a.act[k];
  const int64_t n = a.n;
  const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  const int64_t n0 = (int64_t)blockIdx.x * chunk;
  const int64_t n1 = n0 + chunk < n ? n0 + chunk : n;
  const int tiles_o = out / 4, tiles_i = inp / 4, n_mt = tiles_o * tiles_i;
  float acc[2][16];
  float accb[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[r][j] = 0.0f;
  for (int64_t s0 = n0; s0 < n1; s0 += kDwTile) {
    __syncthreads();
    for (int e = threadIdx.x; e < kDwTile * MAXO; e += blockDim.x) {
      const int s = e % kDwTile, o = e / kDwTile;
      if (o < out) sd[s][o] = (s0 + s < n1) ? D[(int64_t)o * n + s0 + s] : 0.0f;
    }
    for (int e = threadIdx.x; e < kDwTile * MAXI; e += blockDim.x) {
      const int s = e % kDwTile, c = e / kDwTile;
      if (c < inp) sa[s][c] = (s0 + s < n1 && c < in) ? A[(int64_t)c * n + s0 + s] : 0.0f;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int mt = threadIdx.x + r * 256;
      if (mt < n_mt) {
        const int to = mt / tiles_i, ti = mt - to * tiles_i;
#pragma unroll 8
        for (int s = 0; s < kDwTile; ++s) {
          const float4 dv = *reinterpret_cast<const float4*>(&sd[s][4 * to]);
          const float4 av = *reinterpret_cast<const float4*>(&sa[s][4 * ti]);
          const float dd[4] = {dv.x, dv.y, dv.z, dv.w}, aa[4] = {av.x, av.y, av.z, av.w};
#pragma unroll
          for (int p = 0; p < 4; ++p)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[r][p * 4 + q] = fmaf(dd[p], aa[q], acc[r][p * 4 + q]);
        }
      }
    }
    if (threadIdx.x < tiles_o) {
      for (int s = 0; s < kDwTile; ++s) {
        const float4 dv = *reinterpret_cast<const float4*>(&sd[s][4 * threadIdx.x]);
        accb[0] += dv.x; accb[1] += dv.y; accb[2] += dv.z; accb[3] += dv.w;
      }
    }
  }
  // flush: grads layout W[out][in] then b[out] (logical, unpadded)
  const int gw = N::gw_off(k), gb = N::gb_off(k);
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int mt = threadIdx.x + r * 256;
    if (mt < n_mt) {
      const int to = mt / tiles_i, ti = mt - to * tiles_i;
#pragma unroll
      for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int o = 4 * to + p, i = 4 * ti + q;
          if (i < in) atomicAdd(a.grads + gw + o * in + i, acc[r][p * 4 + q]);
        }
    }
  }
  if (threadIdx.x < tiles_o) {
#pragma unroll
    for (int p = 0; p < 4; ++p) atomicAdd(a.grads + gb + 4 * threadIdx.x + p, accb[p]);
  }
}

template <class N>
struct Launch {
  static void attrs() {
    const int smem = (int)(N::SMEM_FLOATS * sizeof(float));
    if (smem <= 48 * 1024) return;
    cudaFuncSetAttribute(query_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(train_forward_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(train_backward_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  }
  static int query(const QueryArgs& a, int sms, cudaStream_t st) {
    const size_t smem = N::SMEM_FLOATS * sizeof(float);
    attrs();
    const int64_t need = (a.n + kThreads - 1) / kThreads;
    const int blocks = (int)(need < (int64_t)sms * 8 ? need : (int64_t)sms * 8);
    query_kernel<N><<<blocks, kThreads, smem, st>>>(a);
    return 1;
  }
  static int train_fwd(const TrainArgs& a, int sms, cudaStream_t st) {
    attrs();
    const size_t smem = N::SMEM_FLOATS * sizeof(float);
    const int64_t need = (a.n + kThreads - 1) / kThreads;
    const int blocks = (int)(need < (int64_t)sms * 8 ? need : (int64_t)sms * 8);
    train_forward_kernel<N><<<blocks, kThreads, smem, st>>>(a);
    return 1;
  }
  static int train_bwd(const TrainArgs& a, int sms, cudaStream_t st) {
    attrs();
    const size_t smem = N::SMEM_FLOATS * sizeof(float);
    const int64_t need = (a.n + kThreads - 1) / kThreads;
    const int blocks = (int)(need < (int64_t)sms * 8 ? need : (int64_t)sms * 8);
    train_backward_kernel<N><<<blocks, kThreads, smem, st>>>(a);
    return 1;
  }
  static int dw(const TrainArgs& a, int sms, cudaStream_t st) {
    const int64_t need = (a.n + 1023) / 1024;
    const int bx = (int)(need < (int64_t)sms * 2 ? need : (int64_t)sms * 2);
    weight_grad_kernel<N><<<dim3(bx > 0 ? bx : 1, N::NL), 256, 0, st>>>(a);
    return 1;
  }
};

}  // namespace detail
}  // namespace npm
