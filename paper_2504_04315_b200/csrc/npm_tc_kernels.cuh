// npm_tc_kernels.cuh -- fused NPM kernels with the decoder on tcgen05/TMEM.
//
// One CTA = 128 threads = one 128-sample tile in flight; thread r owns sample
// (row) r of the tile, which is TMEM lane r of every accumulator, so each
// epilogue is thread-per-sample (Table 1 mappings, Eq. 9 head, sampling).
// Persistent grid, tiles strided over CTAs.
//
// Decoder precision: every MMA operand x is split x = hi + lo in bf16 and the
// product is hi*hi + hi*lo + lo*hi accumulated in fp32 in TMEM ("split-bf16",
// single-pass bf16/TF32 miss the 1e-4 parameter tolerance).
//
// Train tile (Eq. 9 -> backprop):
//   encode   z -> X0 (smem, chunk-major), ones feature at n_in (bias grads)
//   forward  for k: TMEM <- X_k W_k^T (MMA), epilogue +b, ReLU -> X_{k+1}
//   head     raw -> Eq. 9 head -> delta_L (smem)
//   backward for k = L..0 (one MMA batch each):
//              TMEM      <- delta_k W_k          (dX; k = 0: dz, grid part)
//              dW_k^T    += X_k^T delta_k        (persistent TMEM accumulator,
//                                                 the ones row of X_k gives db_k)
//            epilogue: delta_{k-1} = dX * ReLU'(X_k) -> smem (over X_k)
//   scatter  dz -> red.global.add.v4.f32 on the 8L corners (C-O15)
// CTA end: dW/db accumulators -> one fp32 atomic add per element to GRADS.
#pragma once
#include "npm_kernels_impl.cuh"
#include "npm_tc.cuh"

namespace npm {
namespace tck {

using namespace detail;

constexpr int R = 128;          // rows (samples) per tile = MMA M
constexpr uint32_t CH = R * 16; // bytes of one 8-feature chunk of a tile

__host__ __device__ constexpr int r16(int x) { return (x + 15) & ~15; }

template <class N>
struct TC {
  static constexpr int NL = N::NL, W = N::W, NOUT = N::NOUT, NIN = N::NIN;
  static constexpr int KIN = r16(NIN);          // layer-0 MMA K
  static constexpr int ZF = r16(NIN + 1);       // train X0 features (ones at NIN)
  static constexpr int HF = r16(W + 1);         // train hidden features (ones at W)
  __host__ __device__ static constexpr int in_p(int k) { return k == 0 ? KIN : W; }   // padded MMA K of layer k
  __host__ __device__ static constexpr int out(int k) { return k == NL - 1 ? NOUT : W; }
  __host__ __device__ static constexpr int in(int k) { return k == 0 ? NIN : W; }
  // bf16 weight bytes of layer k (hi or lo)
  __host__ __device__ static constexpr uint32_t wbytes(int k) { return (uint32_t)(in_p(k) * out(k) * 2); }
  __host__ __device__ static constexpr uint32_t woff(int k) {  // offset of layer k (hi, then lo)
    return k == 0 ? 0u : woff(k - 1) + 2u * wbytes(k - 1);
  }
  static constexpr uint32_t WBYTES = woff(NL);
  __host__ __device__ static constexpr uint32_t boff(int k) { return k == 0 ? 0u : boff(k - 1) + 4u * out(k - 1); }
  static constexpr uint32_t BBYTES = boff(NL);
  // TMEM columns: scratch [0, 64), dW^T accumulators after it
  static constexpr int SCR = 64;
  __host__ __device__ static constexpr int dwcol(int k) { return k == 0 ? SCR : dwcol(k - 1) + out(k - 1); }
  static constexpr int TCOLS_TRAIN = 256;
  static constexpr int TCOLS_QUERY = 64;
  // ---- train smem map: X_0 (ZF), X_1..X_{NL-1} (HF), D_last (NOUT), weights, bias
  __host__ __device__ static constexpr uint32_t xfeat(int k) { return k == 0 ? ZF : HF; }
  __host__ __device__ static constexpr uint32_t xoff(int k) {  // hi at xoff, lo at xoff + xfeat/8*CH
    return k == 0 ? 0u : xoff(k - 1) + 2u * (xfeat(k - 1) / 8) * CH;
  }
  static constexpr uint32_t DOFF = xoff(NL);
  static constexpr uint32_t WOFF_T = DOFF + 2u * (NOUT / 8) * CH;
  static constexpr uint32_t BOFF_T = WOFF_T + WBYTES;
  static constexpr uint32_t MISC_T = (BOFF_T + BBYTES + 127u) & ~127u;
  // every X_k^T MMA reads 16 chunks from its lo base: keep them inside the allocation
  __host__ __device__ static constexpr uint32_t overread(int k) {
    return xoff(k) + (xfeat(k) / 8) * CH + 16u * CH;
  }
  __host__ __device__ static constexpr uint32_t max_overread(int k) {
    return k < 0 ? 0u : (overread(k) > max_overread(k - 1) ? overread(k) : max_overread(k - 1));
  }
  static constexpr uint32_t SMEM_TRAIN_RAW = MISC_T + 64;
  static constexpr uint32_t SMEM_TRAIN =
      SMEM_TRAIN_RAW > max_overread(NL - 1) ? SMEM_TRAIN_RAW : max_overread(NL - 1);
  // ---- query smem map: buffer A (max(KIN, W) feats), buffer B (W feats), weights, bias
  static constexpr int QAF = KIN > W ? KIN : W;
  static constexpr uint32_t QA = 0, QB = 2u * (QAF / 8) * CH;
  static constexpr uint32_t WOFF_Q = QB + 2u * (W / 8) * CH;
  static constexpr uint32_t BOFF_Q = WOFF_Q + WBYTES;
  static constexpr uint32_t MISC_Q = (BOFF_Q + BBYTES + 127u) & ~127u;
  static constexpr uint32_t SMEM_QUERY = MISC_Q + 64;
};

// Convert fp32 weights (global, [out][in]) into split-bf16 chunk-major smem and
// stage the biases.  Weight element (o, i): byte (i/8)*out*16 + o*16 + (i%8)*2.
template <class N>
__device__ __forceinline__ void stage_weights_tc(const float* __restrict__ g, uint8_t* smem, uint32_t woff,
                                                 uint32_t boff) {
  using T = TC<N>;
  const uint32_t sbase = tc::smem_u32(smem);
#pragma unroll
  for (int k = 0; k < N::NL; ++k) {
    const int in = T::in(k), inp = T::in_p(k), out = T::out(k);
    const float* gw = g + N::gw_off(k);
    const uint32_t hi = sbase + woff + T::woff(k), lo = hi + T::wbytes(k);
    for (int e = threadIdx.x; e < out * (inp / 8); e += blockDim.x) {
      const int o = e % out, j = e / out;
      float v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int i = 8 * j + q;
        v[q] = i < in ? __ldg(gw + o * in + i) : 0.0f;
      }
      uint32_t h[4], l[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) tc::split_pack(v[2 * q], v[2 * q + 1], h[q], l[q]);
      const uint32_t off = (uint32_t)(j * out * 16 + o * 16);
      tc::st_shared_v4(hi + off, h[0], h[1], h[2], h[3]);
      tc::st_shared_v4(lo + off, l[0], l[1], l[2], l[3]);
    }
    float* sb = reinterpret_cast<float*>(smem + boff + T::boff(k));
    for (int o = threadIdx.x; o < out; o += blockDim.x) sb[o] = __ldg(g + N::gb_off(k) + o);
  }
}

// Issue the 3 split-bf16 MMAs of one K step: hi*hi, hi*lo, lo*hi.
__device__ __forceinline__ void mma3(uint32_t d, uint64_t ahi, uint64_t alo, uint64_t bhi, uint64_t blo,
                                     uint32_t idesc, uint32_t acc) {
  tc::mma_bf16(d, ahi, bhi, idesc, acc);
  tc::mma_bf16(d, ahi, blo, idesc, 1u);
  tc::mma_bf16(d, alo, bhi, idesc, 1u);
}

// Forward MMA: D[R x out] = X[R x K] W[out x K]^T, both K-major.
__device__ __forceinline__ void issue_fwd(uint32_t d, uint32_t xhi, uint32_t xlo, uint32_t whi, uint32_t wlo,
                                          int K, int out) {
  const uint32_t idesc = tc::idesc_bf16(R, out, false, false);
  for (int s = 0; s < K / 16; ++s) {
    const uint32_t xa = (uint32_t)s * 2u * CH, wa = (uint32_t)s * 2u * (uint32_t)out * 16u;
    mma3(d, tc::sdesc(xhi + xa, CH, 128), tc::sdesc(xlo + xa, CH, 128), tc::sdesc(whi + wa, out * 16, 128),
         tc::sdesc(wlo + wa, out * 16, 128), idesc, s > 0 ? 1u : 0u);
  }
}

// dX MMA: D[R x nin] = delta[R x out] W[out x nin]: A K-major, B MN-major.
__device__ __forceinline__ void issue_dx(uint32_t d, uint32_t dhi, uint32_t dlo, uint32_t whi, uint32_t wlo,
                                         int out, int nin) {
  const uint32_t idesc = tc::idesc_bf16(R, nin, false, true);
  for (int s = 0; s < out / 16; ++s) {
    const uint32_t da = (uint32_t)s * 2u * CH, wa = (uint32_t)s * 256u;
    mma3(d, tc::sdesc(dhi + da, CH, 128), tc::sdesc(dlo + da, CH, 128), tc::sdesc(whi + wa, 128, out * 16),
         tc::sdesc(wlo + wa, 128, out * 16), idesc, s > 0 ? 1u : 0u);
  }
}

// dW^T MMA: D[128 x out] += X^T[128 feats x R] delta[R x out]: both MN-major.
__device__ __forceinline__ void issue_dw(uint32_t d, uint32_t xhi, uint32_t xlo, uint32_t dhi, uint32_t dlo,
                                         int out, uint32_t first) {
  const uint32_t idesc = tc::idesc_bf16(128, out, true, true);
  for (int s = 0; s < R / 16; ++s) {
    const uint32_t ra = (uint32_t)s * 256u;
    mma3(d, tc::sdesc(xhi + ra, 128, CH), tc::sdesc(xlo + ra, 128, CH), tc::sdesc(dhi + ra, 128, CH),
         tc::sdesc(dlo + ra, 128, CH), idesc, (first && s == 0) ? 0u : 1u);
  }
}

// Read `cols` fp32 TMEM columns of this thread's lane starting at col.
template <int COLS>
__device__ __forceinline__ void tmem_row(uint32_t tbase, int col, float* v) {
  const uint32_t lane = (uint32_t)((threadIdx.x & ~31) << 16);
#pragma unroll
  for (int c = 0; c < COLS; c += 16) tc::tmem_ld16(tbase + lane + (uint32_t)(col + c), v + c);
  tc::tmem_wait_ld();
}

// Make this thread's smem writes visible to the tensor core and its TMEM
// reads ordered before the next MMA, then CTA barrier.
__device__ __forceinline__ void handoff_to_mma() {
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
}

__device__ __forceinline__ void wait_mma(uint64_t* mbar, uint32_t& phase) {
  tc::mbar_wait(mbar, phase);
  phase ^= 1u;
  tc::fence_after_sync();
}

template <class N>
__device__ __forceinline__ void setup_cta(uint8_t* smem, uint32_t misc, int tcols, uint64_t*& mbar,
                                          uint32_t& tbase) {
  mbar = reinterpret_cast<uint64_t*>(smem + misc);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + misc + 8);
  if (threadIdx.x == 0) {
    tc::mbar_init(mbar, 1);
    tc::fence_mbar_init();
  }
  if (threadIdx.x < 32) tc::tmem_alloc(tslot, (uint32_t)tcols);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  tbase = *tslot;
}

__device__ __forceinline__ void teardown_cta(uint32_t tbase, int tcols) {
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  if (threadIdx.x < 32) tc::tmem_dealloc(tbase, (uint32_t)tcols);
}

// ---------------------------------------------------------------------------
// Fused query kernel: encode -> decoder (tcgen05) -> Table 1 -> outputs.
template <class N>
__global__ void __launch_bounds__(R, 1) tc_query_kernel(QueryArgs a) {
  using T = TC<N>;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sb = tc::smem_u32(smem);
  uint64_t* mbar;
  uint32_t tbase;
  setup_cta<N>(smem, T::MISC_Q, T::TCOLS_QUERY, mbar, tbase);
  stage_weights_tc<N>(a.params, smem, T::WOFF_Q, T::BOFF_Q);
  const float4* tab = reinterpret_cast<const float4*>(a.params + N::N_MLP);
  const float* bias = reinterpret_cast<const float*>(smem + T::BOFF_Q);
  const int r = threadIdx.x;
  const int64_t n = a.n;
  const int64_t ntiles = (n + R - 1) / R;
  uint32_t phase = 0;
  const uint32_t xbuf[2] = {sb + T::QA, sb + T::QB};
  const uint32_t xlo[2] = {(uint32_t)(T::QAF / 8) * CH, (uint32_t)(N::W / 8) * CH};
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t i = tile * R + r;
    const bool valid = i < n;
    // ---- encode (Eq. 13) + conditioning -> buffer A
    {
      float z[T::KIN];
      if (valid) {
        if (a.feat_in) {
#pragma unroll
          for (int j = 0; j < N::NGRID; ++j) z[j] = __ldg(a.feat_in + (int64_t)j * n + i);
#pragma unroll
          for (int j = N::NGRID; j < N::NINP; ++j) z[j] = 0.0f;
        } else {
          network_input<N>(a.grid, tab, a.px, a.py, a.pz, a.wox, a.woy, a.woz, a.nx, a.ny, a.nz, a.rough, i,
                           z, nullptr, nullptr, n);
        }
      } else {
#pragma unroll
        for (int j = 0; j < N::NINP; ++j) z[j] = 0.0f;
      }
#pragma unroll
      for (int j = N::NINP; j < T::KIN; ++j) z[j] = 0.0f;
#pragma unroll
      for (int j = 0; j < T::KIN / 8; ++j) tc::store_chunk(xbuf[0], xbuf[0] + xlo[0], R, r, j, z + 8 * j);
    }
    float raw[N::NOUT];
#pragma unroll
    for (int k = 0; k < N::NL; ++k) {
      const int src = k & 1, dst = (k + 1) & 1;
      handoff_to_mma();
      if (r == 0) {
        tc::fence_after_sync();
        const uint32_t w = sb + T::WOFF_Q + T::woff(k);
        issue_fwd(tbase, xbuf[src], xbuf[src] + xlo[src], w, w + T::wbytes(k), T::in_p(k), T::out(k));
        tc::mma_commit(mbar);
      }
      wait_mma(mbar, phase);
      if (k < N::NL - 1) {
        float h[N::W];
        tmem_row<N::W>(tbase, 0, h);
        const float* b = bias + T::boff(k) / 4;
#pragma unroll
        for (int j = 0; j < N::W; ++j) h[j] = fmaxf(h[j] + b[j], 0.0f);
#pragma unroll
        for (int j = 0; j < N::W / 8; ++j) tc::store_chunk(xbuf[dst], xbuf[dst] + xlo[dst], R, r, j, h + 8 * j);
      } else {
        tmem_row<N::NOUT>(tbase, 0, raw);
        const float* b = bias + T::boff(k) / 4;
#pragma unroll
        for (int j = 0; j < N::NOUT; ++j) raw[j] += b[j];
      }
    }
    if (!valid) continue;
    // ---- Table 1 + outputs (thread per sample)
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
  teardown_cta(tbase, T::TCOLS_QUERY);
}

// ---------------------------------------------------------------------------
// Fused training kernel: encode -> forward -> Eq. 9 head -> backward (dX, dW^T)
// -> grid scatter; dW/db flushed once per CTA.
template <class N>
__global__ void __launch_bounds__(R, 1) tc_train_kernel(TrainArgs a) {
  using T = TC<N>;
  constexpr int NL = N::NL;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sb = tc::smem_u32(smem);
  uint64_t* mbar;
  uint32_t tbase;
  setup_cta<N>(smem, T::MISC_T, T::TCOLS_TRAIN, mbar, tbase);
  stage_weights_tc<N>(a.params, smem, T::WOFF_T, T::BOFF_T);
  const float4* tab = reinterpret_cast<const float4*>(a.params + N::N_MLP);
  float4* gtab = reinterpret_cast<float4*>(a.grads + N::N_MLP);
  const float* bias = reinterpret_cast<const float*>(smem + T::BOFF_T);
  const int r = threadIdx.x;
  const int64_t n = a.n;
  const int64_t ntiles = (n + R - 1) / R;
  uint32_t phase = 0, first = 1;
  double loss = 0.0;
  unsigned c_used = 0, c_zero = 0, c_drop = 0;
  // smem addresses of X_k (hi) and its lo offset
  uint32_t xhi[NL], xlo[NL];
#pragma unroll
  for (int k = 0; k < NL; ++k) {
    xhi[k] = sb + T::xoff(k);
    xlo[k] = xhi[k] + (T::xfeat(k) / 8) * CH;
  }
  const uint32_t dlast_hi = sb + T::DOFF, dlast_lo = dlast_hi + (N::NOUT / 8) * CH;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t i = tile * R + r;
    const bool valid = i < n;
    uint64_t mask[NL];   // ReLU masks of X_1..X_{NL-1} (bit j: feature j > 0)
    // ---- encode -> X_0 (features [0, NIN), ones at NIN, zeros to ZF)
    {
      float z[T::ZF];
      if (valid) {
        network_input<N>(a.grid, tab, a.px, a.py, a.pz, a.wox, a.woy, a.woz, a.nx, a.ny, a.nz, a.rough, i, z,
                         nullptr, nullptr, n);
      } else {
#pragma unroll
        for (int j = 0; j < N::NINP; ++j) z[j] = 0.0f;
      }
#pragma unroll
      for (int j = N::NIN; j < T::ZF; ++j) z[j] = j == N::NIN ? 1.0f : 0.0f;
#pragma unroll
      for (int j = 0; j < T::ZF / 8; ++j) tc::store_chunk(xhi[0], xlo[0], R, r, j, z + 8 * j);
    }
    // ---- forward
    float draw[N::NOUT];
#pragma unroll
    for (int k = 0; k < NL; ++k) {
      handoff_to_mma();
      if (r == 0) {
        tc::fence_after_sync();
        const uint32_t w = sb + T::WOFF_T + T::woff(k);
        issue_fwd(tbase, xhi[k], xlo[k], w, w + T::wbytes(k), T::in_p(k), T::out(k));
        tc::mma_commit(mbar);
      }
      wait_mma(mbar, phase);
      const float* b = bias + T::boff(k) / 4;
      if (k < NL - 1) {
        float h[T::HF];
        tmem_row<N::W>(tbase, 0, h);
        uint64_t mk = 0;
#pragma unroll
        for (int j = 0; j < N::W; ++j) {
          h[j] = fmaxf(h[j] + b[j], 0.0f);
          mk |= (h[j] > 0.0f ? 1ull : 0ull) << j;
        }
        mask[k + 1] = mk;
#pragma unroll
        for (int j = N::W; j < T::HF; ++j) h[j] = j == N::W ? 1.0f : 0.0f;
#pragma unroll
        for (int j = 0; j < T::HF / 8; ++j) tc::store_chunk(xhi[k + 1], xlo[k + 1], R, r, j, h + 8 * j);
      } else {
        float raw[N::NOUT];
        tmem_row<N::NOUT>(tbase, 0, raw);
#pragma unroll
        for (int j = 0; j < N::NOUT; ++j) raw[j] += b[j];
        // ---- Eq. 9 head (C-O12, C-O13)
        bool use = false;
        float s = 0.0f;
        if (valid) {
          float t = __ldg(a.target + i);
          bool all_zero = t == 0.0f;
          if (a.channels == 3) {
            const float tg = __ldg(a.target + n + i), tb = __ldg(a.target + 2 * n + i);
            all_zero = all_zero && tg == 0.0f && tb == 0.0f;
            t = 0.2126f * t + 0.7152f * tg + 0.0722f * tb;
          }
          const float p = __ldg(a.spdf + i);
          const float ratio = t / p;
          const bool drop = !isfinite(ratio) || !isfinite(p) || !(p > 0.0f);
          const bool zero = !drop && all_zero;
          c_drop += drop;
          c_zero += zero;
          use = !drop && !zero;
          s = (float)(-(double)ratio * a.inv_n_global);
        }
        if (use) {
          const float logv = grad_head<N::K>(raw, a.log_kmin, a.log_kmax, __ldg(a.wx + i), __ldg(a.wy + i),
                                             __ldg(a.wz + i), s, draw);
          loss += (double)s * (double)logv;
          c_used += 1;
        } else {
#pragma unroll
          for (int j = 0; j < N::NOUT; ++j) draw[j] = 0.0f;
        }
#pragma unroll
        for (int j = 0; j < N::NOUT / 8; ++j) tc::store_chunk(dlast_hi, dlast_lo, R, r, j, draw + 8 * j);
      }
    }
    // ---- backward
    uint32_t dhi = dlast_hi, dlo = dlast_lo;
#pragma unroll
    for (int k = NL - 1; k >= 0; --k) {
      handoff_to_mma();
      const int nin = k > 0 ? N::W : N::NGRID;
      if (r == 0) {
        tc::fence_after_sync();
        const uint32_t w = sb + T::WOFF_T + T::woff(k);
        issue_dx(tbase, dhi, dlo, w, w + T::wbytes(k), T::out(k), nin);
        issue_dw(tbase + (uint32_t)T::dwcol(k), xhi[k], xlo[k], dhi, dlo, T::out(k), first);
        tc::mma_commit(mbar);
      }
      wait_mma(mbar, phase);
      if (k > 0) {
        float d[N::W];
        tmem_row<N::W>(tbase, 0, d);
        const uint64_t mk = mask[k];
#pragma unroll
        for (int j = 0; j < N::W; ++j) d[j] = ((mk >> j) & 1ull) ? d[j] : 0.0f;
        // delta_{k-1} overwrites X_k (dead once its dW MMA completed)
        dhi = xhi[k];
        dlo = xhi[k] + (N::W / 8) * CH;
#pragma unroll
        for (int j = 0; j < N::W / 8; ++j) tc::store_chunk(dhi, dlo, R, r, j, d + 8 * j);
      } else {
        float dz[N::NGRID];
        tmem_row<N::NGRID>(tbase, 0, dz);   // warp-collective: before the validity branch
        if (!valid) continue;
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
    first = 0;
  }
  // ---- flush dW^T / db accumulators: lane r = input feature r (r == in: bias)
  if (!first) {
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
#pragma unroll
    for (int k = 0; k < NL; ++k) {
      constexpr int MAXO = N::NOUT > N::W ? N::NOUT : N::W;
      float v[MAXO];
      const int out = T::out(k), in = T::in(k);
      if (out == N::NOUT) tmem_row<N::NOUT>(tbase, T::dwcol(k), v);
      else tmem_row<N::W>(tbase, T::dwcol(k), v);
      if (r < in) {
        float* g = a.grads + N::gw_off(k) + r;
        for (int o = 0; o < out; ++o) atomicAdd(g + o * in, v[o]);
      } else if (r == in) {
        float* g = a.grads + N::gb_off(k);
        for (int o = 0; o < out; ++o) atomicAdd(g + o, v[o]);
      }
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
  teardown_cta(tbase, T::TCOLS_TRAIN);
}

template <class N>
struct TcLaunch {
  static int query(const QueryArgs& a, int sms, cudaStream_t st) {
    using T = TC<N>;
    cudaFuncSetAttribute(tc_query_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)T::SMEM_QUERY);
    const int64_t ntiles = (a.n + R - 1) / R;
    const int per_sm = (int)((227u * 1024u) / (T::SMEM_QUERY + 1024u));
    const int64_t cap = (int64_t)sms * (per_sm < 1 ? 1 : (per_sm > 4 ? 4 : per_sm));
    const int blocks = (int)(ntiles < cap ? ntiles : cap);
    tc_query_kernel<N><<<blocks, R, T::SMEM_QUERY, st>>>(a);
    return 1;
  }
  static int train(const TrainArgs& a, int sms, cudaStream_t st) {
    using T = TC<N>;
    cudaFuncSetAttribute(tc_train_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)T::SMEM_TRAIN);
    const int64_t ntiles = (a.n + R - 1) / R;
    const int per_sm = (int)((227u * 1024u) / (T::SMEM_TRAIN + 1024u));
    const int64_t cap = (int64_t)sms * (per_sm < 1 ? 1 : (per_sm > 2 ? 2 : per_sm));
    const int blocks = (int)(ntiles < cap ? ntiles : cap);
    tc_train_kernel<N><<<blocks, R, T::SMEM_TRAIN, st>>>(a);
    return 1;
  }
};

}  // namespace tck
}  // namespace npm
