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
  static_assert(N::N_MLP % 8 == 0, "grid tables must start 32-B aligned (paired gathers)");
  static constexpr int KIN = r16(NIN);          // layer-0 MMA K
  // train X0 features: ones at NIN (bias row of dW_0^T), >= KIN for the forward K
  static constexpr int ZF = KIN > ((NIN + 8) & ~7) ? KIN : ((NIN + 8) & ~7);
  static constexpr int HF = W + 8;              // train hidden features (ones at W)
  __host__ __device__ static constexpr int in_p(int k) { return k == 0 ? KIN : W; }   // padded MMA K of layer k
  __host__ __device__ static constexpr int out(int k) { return k == NL - 1 ? NOUT : W; }
  __host__ __device__ static constexpr int in(int k) { return k == 0 ? NIN : W; }
  // bf16 weight bytes of layer k (hi or lo)
  __host__ __device__ static constexpr uint32_t wbytes(int k) { return (uint32_t)(in_p(k) * out(k) * 2); }
  __host__ __device__ static constexpr int osum(int k) { return N::osum(k); }   // sum of out(j), j < k
  __host__ __device__ static constexpr uint32_t woff(int k) {  // offset of layer k (hi, then lo)
    return k == 0 ? 0u : (uint32_t)(4 * (KIN * out(0) + W * (osum(k) - out(0))));
  }
  static constexpr uint32_t WBYTES = woff(NL);
  __host__ __device__ static constexpr uint32_t boff(int k) { return 4u * (uint32_t)osum(k); }
  static constexpr uint32_t BBYTES = boff(NL);
  static constexpr int TCOLS_QUERY = 64;
  // train X_k features
  __host__ __device__ static constexpr uint32_t xfeat(int k) { return k == 0 ? ZF : HF; }
  // ---- query smem map: buffer A (max(KIN, W) feats), buffer B (W feats), weights, bias
  static constexpr int QAF = KIN > W ? KIN : W;
  static constexpr uint32_t QA = 0, QB = 2u * (QAF / 8) * CH;
  static constexpr uint32_t WOFF_Q = QB + 2u * (W / 8) * CH;
  static constexpr uint32_t BOFF_Q = WOFF_Q + WBYTES;
  static constexpr uint32_t RED_Q = (BOFF_Q + BBYTES + 127u) & ~127u;   // head reductions [5][4][R] f32
  static constexpr uint32_t MISC_Q = RED_Q + 5u * 4u * R * 4u;
  static constexpr uint32_t SMEM_QUERY = MISC_Q + 64;
  // ---- two-group query map (one 512-thread CTA per SM, one weight copy):
  // weights, bias | group g: buffer A, buffer B, head reductions | misc
  static constexpr uint32_t QRED_BYTES = (3u * 2u + 3u + 2u + 2u) * R * 4u;   // TPR = 2 slots (+ C-A34 logit parts)
  static constexpr uint32_t QG0 = (WBYTES + BBYTES + 1023u) & ~1023u;
  static constexpr uint32_t QGB = (QB + 2u * (W / 8) * CH + QRED_BYTES + 1023u) & ~1023u;
  static constexpr uint32_t MISC_Q2 = QG0 + 2u * QGB;
  static constexpr uint32_t SMEM_QUERY2 = MISC_Q2 + 64;
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

// Descriptors are built once per batch; a K step only advances the 14-bit
// start-address field (addr >> 4 stays < 2^14 for any smem address), so each
// further MMA costs one 64-bit add on the issuing thread.

// Forward MMA: D[R x out] = X[R x K] W[out x K]^T, both K-major.
__device__ __forceinline__ void issue_fwd(uint32_t d, uint32_t xhi, uint32_t xlo, uint32_t whi, uint32_t wlo,
                                          int K, int out) {
  const uint32_t idesc = tc::idesc_bf16(R, out, false, false);
  const uint64_t ah = tc::sdesc(xhi, CH, 128), al = tc::sdesc(xlo, CH, 128);
  const uint64_t bh = tc::sdesc(whi, out * 16, 128), bl = tc::sdesc(wlo, out * 16, 128);
#pragma unroll
  for (int s = 0; s < K / 16; ++s) {
    const uint64_t xa = (uint64_t)(s * 2 * (int)CH) >> 4, wa = (uint64_t)(s * 2 * out * 16) >> 4;
    mma3(d, ah + xa, al + xa, bh + wa, bl + wa, idesc, s > 0 ? 1u : 0u);
  }
}

__device__ __forceinline__ void wait_mma(uint64_t* mbar, uint32_t& phase) {
  tc::mbar_wait(mbar, phase);
  phase ^= 1u;
  tc::fence_after_sync();
}

template <class N>
__device__ __forceinline__ void setup_cta(uint8_t* smem, uint32_t misc, int tcols, uint64_t*& mbar,
                                          uint32_t& tbase) {
  mbar = reinterpret_cast<uint64_t*>(smem + misc);           // mbar[0]: waited MMA batches
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + misc + 16);   // mbar[1]: deferred dW batches
  if (threadIdx.x == 0) {
    tc::mbar_init(mbar, 1);
    tc::mbar_init(mbar + 1, 1);
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
// Fused query kernel: encode -> decoder (tcgen05) -> Table 1 -> outputs, with
// the train kernel's mapping: 4 threads per sample row (512 threads), quarter q
// owning grid levels [q L/4, ...), accumulator columns [q C/4, ...) and lobes
// [q K/4, ...); softmax, mixture sums and the lobe choice cross quarters
// through smem.  Lobe choice (C-O10, C-A17): quarter boundaries
// B_q = sum_{q'<q} S_q' (S_q = sum of the quarter's e^{lambda'-M}) are
// computed identically by the 4 threads of a row, so exactly one quarter owns
// u1 and picks its first lobe with u1 < C_i (its last lobe at C = B_{q+1}).
template <class N, int TPR, int MODE, int GROUPS>
__global__ void __launch_bounds__(GROUPS * TPR * R, GROUPS == 2 ? 1 : 4 / TPR) tc_query_kernel(QueryArgs a) {
  // MODE (compile time, so the plain query carries none of the variants' code):
  // 0 guide sampling / pdf; 1 combined BSDF/guide MIS (f-1); 2 cosine product (f-2)
  // GROUPS = 2: one 512-thread CTA per SM runs two independent tiles (one per
  // 256-thread group, own buffers / mbarrier / TMEM columns / named barrier)
  // over ONE copy of the weights; the smem saved goes to L1 for the gathers.
  constexpr bool COMBINED = MODE == 1, COSPROD = MODE == 2;
  static_assert(GROUPS == 1 || TPR == 2, "two-group query uses 2 threads per row");
  using T = TC<N>;
  constexpr int NL = N::NL, K = N::K, W = N::W;
  constexpr int KQ = K / TPR, WQ = W / TPR, LQ = N::L / TPR, GQ = 4 * LQ;
  static_assert(K % TPR == 0 && N::L % TPR == 0, "parts");
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sb = tc::smem_u32(smem);
  const int g = GROUPS == 2 ? (int)(threadIdx.x >> 8) : 0;
  const int tid = GROUPS == 2 ? (int)(threadIdx.x & 255) : (int)threadIdx.x;   // thread within the group
  const int warp = tid >> 5, q = warp >> 2;   // q: part of the row
  const int r = ((warp & 3) << 5) | (tid & 31);
  const uint32_t lane_addr = (uint32_t)((warp & 3) << 21);
  uint64_t* mbar;
  uint32_t tbase;
  constexpr uint32_t MISC = GROUPS == 2 ? T::MISC_Q2 : T::MISC_Q;
  setup_cta<N>(smem, MISC, GROUPS * T::TCOLS_QUERY, mbar, tbase);
  mbar += g;
  tbase += (uint32_t)(g * T::TCOLS_QUERY);
  constexpr uint32_t WOFF = GROUPS == 2 ? 0u : T::WOFF_Q, BOFF = GROUPS == 2 ? T::WBYTES : T::BOFF_Q;
  stage_weights_tc<N>(a.params, smem, WOFF, BOFF);
  if (GROUPS == 2) {   // weights staged by all 512 threads before either group's first MMA
    tc::fence_proxy_async();
    __syncthreads();
  }
  const uint32_t gbase = GROUPS == 2 ? T::QG0 + (uint32_t)g * T::QGB : 0u;
  auto qsync = [&]() {
    if (GROUPS == 2) tc::named_sync(1u + (uint32_t)g, 256u);
    else __syncthreads();
  };
  // The head's exchanges (softmax max / sums, lobe choice, sampled direction)
  // are between the TPR threads of one row only: warps w and w + 4 -- a
  // 64-thread named barrier per warp pair instead of the whole CTA.
  static_assert(TPR == 2, "pair barrier assumes 2 threads per row");
  auto psync = [&]() { tc::named_sync(3u + 4u * (uint32_t)g + (uint32_t)(warp & 3), 64u); };
  auto handoff = [&]() {
    tc::fence_proxy_async();
    tc::fence_before_sync();
    qsync();
  };
  const float4* tab = reinterpret_cast<const float4*>(a.params + N::N_MLP);
  const float* bias = reinterpret_cast<const float*>(smem + BOFF);
  float* red = reinterpret_cast<float*>(smem + (GROUPS == 2 ? gbase + T::QB + 2u * (W / 8) * CH : T::RED_Q));
  // slots 0..2: per-part partials; omega (3 floats) at 3 TPR R; slot 4 after it
  auto RS = [&](int slot, int qq) -> float& {
    return red[((slot < 3 ? slot * TPR : 3 * TPR + 3) + qq) * R + r];
  };
  const int64_t n = a.n;
  const int64_t ntiles = (n + R - 1) / R;
  uint32_t phase = 0;
  const uint32_t xbuf[2] = {sb + gbase + T::QA, sb + gbase + T::QB};
  const uint32_t xlo[2] = {(uint32_t)(T::QAF / 8) * CH, (uint32_t)(W / 8) * CH};
  // this thread's row, prefetched: the sample index two tiles ahead, the raw
  // position one tile ahead (issued while the current tile's first MMA runs;
  // normalised at use so nothing waits on the loads before the next tile)
  struct RowIn {
    int64_t i;
    bool valid;
    float x, y, z;
  };
  auto load_idx = [&](int64_t tl, int64_t& i, bool& v) {
    const int64_t slot = tl * R + r;                   // processing slot (spatially binned order)
    v = slot < n;
    i = v ? (a.perm ? (int64_t)__ldg(a.perm + slot) : slot) : 0;   // sample index
  };
  auto load_row = [&](int64_t i, bool v, RowIn& o) {
    o.valid = v;
    o.i = i;
    o.x = o.y = o.z = 0.0f;
    if (v && !a.feat_in) { o.x = __ldg(a.px + i); o.y = __ldg(a.py + i); o.z = __ldg(a.pz + i); }
  };
  RowIn nx_row;
  int64_t nx_i = 0;
  bool nx_v = false;
  const int64_t tile0 = (int64_t)blockIdx.x * GROUPS + g, tstep = (int64_t)gridDim.x * GROUPS;
  if (tile0 < ntiles) {
    load_idx(tile0, nx_i, nx_v);
    load_row(nx_i, nx_v, nx_row);
    if (tile0 + tstep < ntiles) load_idx(tile0 + tstep, nx_i, nx_v);
  }
  int qt = 0;
#ifdef NPM_QUERY_STAMPS
  const bool qstamp = a.dbg_clock && blockIdx.x == 0 && threadIdx.x == 0 && MODE == 0;
#define QSTAMP(idx) do { if (qstamp && qt < 64) a.dbg_clock[qt * 16 + (idx)] = clock64(); } while (0)
#else
#define QSTAMP(idx) do { } while (0)
#endif
  for (int64_t tile = tile0; tile < ntiles; tile += tstep, ++qt) {
    QSTAMP(0);
    const RowIn row = nx_row;
    const bool valid = row.valid;
    const int64_t i = row.i;
    const int64_t ic = i;
    // ---- encode (Eq. 13): levels [q LQ, (q+1) LQ) + conditioning -> buffer A
    {
      float g[GQ];
      if (valid && a.feat_in) {
#pragma unroll
        for (int j = 0; j < GQ; ++j) g[j] = __ldg(a.feat_in + (int64_t)(q * GQ + j) * n + i);
      } else if (valid) {
        const float ux = normalize_axis(row.x, a.grid.lo[0], a.grid.inv[0]);
        const float uy = normalize_axis(row.y, a.grid.lo[1], a.grid.inv[1]);
        const float uz = normalize_axis(row.z, a.grid.lo[2], a.grid.inv[2]);
#ifdef NPM_Q_PIPE   // level l + 1's loads issued before level l's blend
        LevelCorners lcn;
        float4 vn[8];
        level_corners(a.grid, q * LQ, ux, uy, uz, lcn);
#pragma unroll
        for (int c = 0; c < 8; ++c) vn[c] = __ldg(tab + a.grid.off[q * LQ] + lcn.idx[c]);
#endif
#pragma unroll
        for (int ll = 0; ll < LQ; ++ll) {
          const int l = q * LQ + ll;
#ifdef NPM_Q_PIPE
          float4 v[8];
          LevelCorners lc = lcn;
#pragma unroll
          for (int c = 0; c < 8; ++c) v[c] = vn[c];
          if (ll + 1 < LQ) {
            level_corners(a.grid, l + 1, ux, uy, uz, lcn);
#pragma unroll
            for (int c = 0; c < 8; ++c) vn[c] = __ldg(tab + a.grid.off[l + 1] + lcn.idx[c]);
          }
#else
          LevelCorners lc;
          level_corners(a.grid, l, ux, uy, uz, lc);
          // 8 single loads here: the binned query gathers are coherent already and
          // the paired form's wider registers cost more than it saves (B200: c2
          // query 269 -> 293 us with pairs, train 655 -> 641 us)
          const float4* t = tab + a.grid.off[l];
          float4 v[8];
#pragma unroll
          for (int c = 0; c < 8; ++c) v[c] = __ldg(t + lc.idx[c]);
#endif
          float4 gl = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            gl.x = fmaf(lc.w[c], v[c].x, gl.x); gl.y = fmaf(lc.w[c], v[c].y, gl.y);
            gl.z = fmaf(lc.w[c], v[c].z, gl.z); gl.w = fmaf(lc.w[c], v[c].w, gl.w);
          }
          g[4 * ll] = gl.x; g[4 * ll + 1] = gl.y; g[4 * ll + 2] = gl.z; g[4 * ll + 3] = gl.w;
        }
      } else {
#pragma unroll
        for (int j = 0; j < GQ; ++j) g[j] = 0.0f;
      }
      tc::store_feats<GQ>(xbuf[0], xbuf[0] + xlo[0], R, r, q * GQ, g);
      if constexpr (N::PRODUCT) {
        float e[16];
        // extra feature blocks: 0 SH(w_o) [32,48), 1 SH(n) [48,64), 2 roughness [64,80)
#pragma unroll
        for (int blk = 0; blk < 3; ++blk) {
          if (blk % TPR != q) continue;
#pragma unroll
          for (int j = 0; j < 16; ++j) e[j] = 0.0f;
          if (valid) {
            if (blk == 0) sh4(__ldg(a.wox + i), __ldg(a.woy + i), __ldg(a.woz + i), e);
            else if (blk == 1) sh4(__ldg(a.nx + i), __ldg(a.ny + i), __ldg(a.nz + i), e);
            else e[0] = __ldg(a.rough + i);
          }
          tc::store_feats<16>(xbuf[0], xbuf[0] + xlo[0], R, r, 32 + 16 * blk, e);
        }
      }
    }
    // ---- decoder
#pragma unroll
    for (int k = 0; k < NL - 1; ++k) {
      const int src = k & 1, dst = (k + 1) & 1;
      handoff();
      QSTAMP(1 + 2 * k);
      if (tid == 0) {
        tc::fence_after_sync();
        const uint32_t w = sb + WOFF + T::woff(k);
        issue_fwd(tbase, xbuf[src], xbuf[src] + xlo[src], w, w + T::wbytes(k), T::in_p(k), T::out(k));
        tc::mma_commit(mbar);
      }
      if (k == 0 && tile + tstep < ntiles) {
        load_row(nx_i, nx_v, nx_row);
        if (tile + 2 * tstep < ntiles) load_idx(tile + 2 * tstep, nx_i, nx_v);
      }
      wait_mma(mbar, phase);
      QSTAMP(2 + 2 * k);
      float h[WQ];
      tc::tmem_ldn<WQ>(tbase + lane_addr + (uint32_t)(q * WQ), h);
      tc::tmem_wait_ld();
      const float4* b4 = reinterpret_cast<const float4*>(bias + T::boff(k) / 4 + q * WQ);   // 16-byte aligned
#pragma unroll
      for (int j = 0; j < WQ / 4; ++j) {
        const float4 bb = b4[j];
        h[4 * j] = fmaxf(h[4 * j] + bb.x, 0.0f);
        h[4 * j + 1] = fmaxf(h[4 * j + 1] + bb.y, 0.0f);
        h[4 * j + 2] = fmaxf(h[4 * j + 2] + bb.z, 0.0f);
        h[4 * j + 3] = fmaxf(h[4 * j + 3] + bb.w, 0.0f);
      }
      tc::store_feats<WQ>(xbuf[dst], xbuf[dst] + xlo[dst], R, r, q * WQ, h);
      if (COMBINED && k == NL - 2 && a.alpha_w) {   // C-A34: this part's a . h_{L-1}
        float zp = 0.0f;
#pragma unroll
        for (int j = 0; j < WQ; ++j) zp = fmaf(__ldg(a.alpha_w + q * WQ + j), h[j], zp);
        red[(11 + q) * R + r] = zp;   // read after the next CTA / group barrier
      }
    }
    {
      constexpr int k = NL - 1, src = k & 1;
      handoff();
      if (tid == 0) {
        tc::fence_after_sync();
        const uint32_t w = sb + WOFF + T::woff(k);
        issue_fwd(tbase, xbuf[src], xbuf[src] + xlo[src], w, w + T::wbytes(k), T::in_p(k), T::out(k));
        tc::mma_commit(mbar);
      }
      wait_mma(mbar, phase);
      QSTAMP(6);
    }
    // ---- Table 1 on this quarter's lobes
    float lp[KQ], kp[KQ], tp[KQ], pp[KQ];
    tc::tmem_ldn<KQ>(tbase + lane_addr + (uint32_t)(q * KQ), lp);
    tc::tmem_ldn<KQ>(tbase + lane_addr + (uint32_t)(K + q * KQ), kp);
    tc::tmem_ldn<KQ>(tbase + lane_addr + (uint32_t)(2 * K + q * KQ), tp);
    tc::tmem_ldn<KQ>(tbase + lane_addr + (uint32_t)(3 * K + q * KQ), pp);
    tc::tmem_wait_ld();
    const float* b = bias + T::boff(NL - 1) / 4;
#pragma unroll
    for (int j = 0; j < KQ; ++j) {
      lp[j] += b[q * KQ + j]; kp[j] += b[K + q * KQ + j];
      tp[j] += b[2 * K + q * KQ + j]; pp[j] += b[3 * K + q * KQ + j];
    }
    if (a.raw && valid) {
#pragma unroll
      for (int j = 0; j < KQ; ++j) {
        const int l = q * KQ + j;
        a.raw[(int64_t)l * n + i] = lp[j];
        a.raw[(int64_t)(K + l) * n + i] = kp[j];
        a.raw[(int64_t)(2 * K + l) * n + i] = tp[j];
        a.raw[(int64_t)(3 * K + l) * n + i] = pp[j];
      }
    }
    float kap[KQ], mx[KQ], my[KQ], mz[KQ], nrm[KQ];
    float mloc = lp[0];
#pragma unroll
    for (int j = 0; j < KQ; ++j) {
      mloc = fmaxf(mloc, lp[j]);
      kap[j] = __expf(fminf(fmaxf(kp[j], a.log_kmin), a.log_kmax));
      float th, ph, st, ct, sp, cp;
      lobe_angles(tp[j], pp[j], kap[j], th, ph, st, ct, sp, cp);
      mx[j] = st * cp; my[j] = st * sp; mz[j] = ct;
      float em;
      nrm[j] = lobe_norm(kap[j], em);
    }
    if (COSPROD) {   // f-2: times the cosine lobe about n, renormalised via the logits
      const float nx = valid ? __ldg(a.bnx + ic) : 0.0f, ny = valid ? __ldg(a.bny + ic) : 0.0f,
                  nz = valid ? __ldg(a.bnz + ic) : 1.0f;
      mloc = -INFINITY;
#pragma unroll
      for (int j = 0; j < KQ; ++j) {
        lp[j] += vmf_product_inplace(mx[j], my[j], mz[j], kap[j], nx, ny, nz, a.kappa_c, a.log_c_kc);
        float em;
        nrm[j] = lobe_norm(fmaxf(kap[j], 1e-30f), em);
        mloc = fmaxf(mloc, lp[j]);
      }
    }
    if (valid && a.kappa) {
#pragma unroll
      for (int j = 0; j < KQ; ++j) a.kappa[(int64_t)(q * KQ + j) * n + i] = kap[j];
    }
    if (valid && a.mu) {
#pragma unroll
      for (int j = 0; j < KQ; ++j) {
        a.mu[(int64_t)(q * KQ + j) * n + i] = mx[j];
        a.mu[(int64_t)(K + q * KQ + j) * n + i] = my[j];
        a.mu[(int64_t)(2 * K + q * KQ + j) * n + i] = mz[j];
      }
    }
    RS(0, q) = mloc;
    psync();
    QSTAMP(7);
    float M = RS(0, 0);
#pragma unroll
    for (int qq = 1; qq < TPR; ++qq) M = fmaxf(M, RS(0, qq));
    float e[KQ], S = 0.0f, P = 0.0f;
    const bool want_pdf = a.pdf != nullptr;
    float qx = 0.f, qy = 0.f, qz = 0.f;
    if (want_pdf) { qx = __ldg(a.wx + ic); qy = __ldg(a.wy + ic); qz = __ldg(a.wz + ic); }
#pragma unroll
    for (int j = 0; j < KQ; ++j) {
      e[j] = __expf(lp[j] - M);
      S += e[j];
      if (want_pdf) P += e[j] * lobe_eval(nrm[j], kap[j], mx[j], my[j], mz[j], qx, qy, qz);
    }
    RS(1, q) = S;
    RS(2, q) = P;
    psync();
    QSTAMP(8);
    float B[TPR + 1];
    B[0] = 0.0f;
#pragma unroll
    for (int qq = 0; qq < TPR; ++qq) B[qq + 1] = B[qq] + RS(1, qq);
    const float invS = 1.0f / B[TPR];
    if (valid && a.lambda) {
#pragma unroll
      for (int j = 0; j < KQ; ++j) a.lambda[(int64_t)(q * KQ + j) * n + i] = e[j] * invS;
    }
    if (want_pdf && q == 0 && valid) {
      float Pt = 0.0f;
#pragma unroll
      for (int qq = 0; qq < TPR; ++qq) Pt += RS(2, qq);
      a.pdf[i] = Pt * invS;
    }
    if (a.do_sample) {
      float4 u;
      if (a.u) u = make_float4(__ldg(a.u + ic), __ldg(a.u + n + ic), __ldg(a.u + 2 * n + ic),
                               COMBINED ? __ldg(a.u + 3 * n + ic) : 1.0f);
      else u = philox_uniforms4(a.seed, (uint64_t)ic + a.offset);
      // f-1: BSDF with probability alpha (C-A25), else the guide
      // selection probability: the caller's alpha, or the learned alpha(x) (C-A34)
      float alpha = a.alpha;
      if (COMBINED && a.alpha_w) {
        float z = __ldg(a.alpha_w + W);
#pragma unroll
        for (int qq = 0; qq < TPR; ++qq) z += red[(11 + qq) * R + r];
        alpha = 1.0f / (1.0f + __expf(-z));
      }
      const bool use_bsdf = COMBINED && u.w < alpha;
      const bool before = u.x < B[q] * invS;                 // an earlier quarter owns u1
      const bool after = u.x >= B[q + 1] * invS && q < TPR - 1;   // a later part owns u1
      // the part owning u1 hands its chosen lobe (kappa, mu) to part 0, which
      // alone runs the sampler (one warp of the pair instead of both):
      // rows 0 / 1 (softmax maxima, dead after the second barrier) and 6 / 7
      if (!use_bsdf && !before && !after) {
        int sel = KQ - 1;
        float cum = B[q];
#pragma unroll
        for (int j = 0; j < KQ - 1; ++j) {
          cum += e[j];
          if (sel == KQ - 1 && u.x < cum * invS) sel = j;
        }
        float kk = kap[0], mmx = mx[0], mmy = my[0], mmz = mz[0];
#pragma unroll
        for (int j = 1; j < KQ; ++j)
          if (sel == j) { kk = kap[j]; mmx = mx[j]; mmy = my[j]; mmz = mz[j]; }
        red[r] = kk; red[R + r] = mmx; red[(3 * TPR) * R + r] = mmy; red[(3 * TPR + 1) * R + r] = mmz;
      }
      psync();
      if (q == 0) {
        float wx, wy, wz;
        if (use_bsdf) bsdf_sample(__ldg(a.bnx + ic), __ldg(a.bny + ic), __ldg(a.bnz + ic), u.x, u.y, wx, wy, wz);
        else lobe_sample(red[r], red[R + r], red[(3 * TPR) * R + r], red[(3 * TPR + 1) * R + r], u.y, u.z, wx, wy, wz);
        red[(3 * TPR) * R + r] = wx; red[(3 * TPR) * R + R + r] = wy; red[(3 * TPR) * R + 2 * R + r] = wz;
      }
      psync();
    QSTAMP(9);
      const float wx = red[(3 * TPR) * R + r], wy = red[(3 * TPR) * R + R + r], wz = red[(3 * TPR) * R + 2 * R + r];
      float P2 = 0.0f;
#pragma unroll
      for (int j = 0; j < KQ; ++j) P2 += e[j] * lobe_eval(nrm[j], kap[j], mx[j], my[j], mz[j], wx, wy, wz);
      RS(4, q) = P2;
      psync();
    QSTAMP(10);
      if (q == 0 && valid) {
        float Pt = 0.0f;
#pragma unroll
        for (int qq = 0; qq < TPR; ++qq) Pt += RS(4, qq);
        float V = Pt * invS, ox = wx, oy = wy, oz = wz, p = V;
        if (COMBINED) {
          const float nx = __ldg(a.bnx + ic), ny = __ldg(a.bny + ic), nz = __ldg(a.bnz + ic);
          int32_t t = use_bsdf ? 0 : 1;
          if (!use_bsdf && !(isfinite(V) && V >= kVFloor)) {   // guide pdf underflow (C-A26)
            bsdf_sample(nx, ny, nz, u.x, u.y, ox, oy, oz);
            p = bsdf_pdf(nx, ny, nz, ox, oy, oz);
            V = 0.0f;
            t = 2;
          } else {
            // one-sample balance heuristic p~ = alpha p_bsdf + (1 - alpha) V
            p = alpha * bsdf_pdf(nx, ny, nz, ox, oy, oz) + (1.0f - alpha) * V;
          }
          if (a.gpdf) a.gpdf[i] = V;
          if (a.tech) a.tech[i] = t;
        }
        a.sx[i] = ox; a.sy[i] = oy; a.sz[i] = oz;
        a.spdf[i] = p;
      }
    }
  }
#undef QSTAMP
  teardown_cta(tbase - (uint32_t)(g * T::TCOLS_QUERY), GROUPS * T::TCOLS_QUERY);
}

// ---------------------------------------------------------------------------
// Two-tile training kernel: a CTA (512 threads) runs two independent 64-sample
// tiles, one per 256-thread group g = warp / 8, so one group's MMA round trips
// and epilogues overlap the other's.  MMAs are M = 64 (cta_group::1): row r of
// an accumulator lives in TMEM lane 32 (r / 16) + r % 16; warp (quarter
// Q = warp % 4, h = (warp / 4) % 2) reads its 16 rows with tcgen05.ld
// 16x256b: thread t gets rows r0 = 16 Q + t / 4 and r0 + 8, column pairs
// 8 j + 2 (t % 4).  Ownership per thread (c = t % 4):
//   encode / scatter: row r0 + 8 (c & 1), levels h L/2 + 2 j + c / 2 (j < L/4)
//   hidden epilogues: both rows, columns [h W/2, (h+1) W/2) (pairs 2c)
//   Eq. 9 head:       row r0 + 8 h, lobes 8 jj + 2 c + {0,1} (4 threads of a
//                     row are adjacent lanes: softmax / mixture sums by shuffles)
// The weight-gradient accumulators (M = 128 over features, K = the 64 samples
// of a tile) are shared by both groups; zeroed once, always accumulated.
template <class N>
struct TC64 {
  using B = TC<N>;
  static constexpr int NL = N::NL, W = N::W, NOUT = N::NOUT, NIN = N::NIN;
  static constexpr int RT = 64;
  static constexpr uint32_t CHT = RT * 16;
  static constexpr int ZF = B::ZF, HF = B::HF;
  __host__ __device__ static constexpr uint32_t xfeat(int k) { return k == 0 ? ZF : HF; }
  __host__ __device__ static constexpr uint32_t xoff(int k) {
    return k == 0 ? 0u : 2u * (ZF / 8) * CHT + (uint32_t)(k - 1) * 2u * (HF / 8) * CHT;
  }
  static constexpr uint32_t DOFF = xoff(NL);
  static constexpr uint32_t DAOFF = DOFF + 2u * (NOUT / 8) * CHT;   // extra delta buffer (SEP)
  static constexpr uint32_t GB_NOSEP = DAOFF;
  static constexpr uint32_t GB_SEP = DAOFF + 2u * (W / 8) * CHT;
  // SEP: each backward batch commits dX_k before issuing dW_k, so the epilogue
  // (delta_{k-1}) runs under the dW_k MMAs; delta_{k-1} then needs a buffer that
  // dW_k does not read (neither X_k nor delta_k).  Measured on B200: c2 (173 KB)
  // 1 % faster; c5 (196 KB) 41 % slower -- the smaller L1 costs its
  // HBM-resident gathers more than the overlap gains.  Off above 180 KB.
  static constexpr bool SEP =
      2u * GB_SEP + B::WBYTES + B::BBYTES + 256u <= 180u * 1024u;
  static constexpr uint32_t GBYTES = SEP ? GB_SEP : GB_NOSEP;
  // buffer of delta_k (hi part; lo follows after dfeat(k) / 8 chunks):
  //   delta_{NL-1}: D_last.  SEP: alternately DA and X_{k+2} (free once dW_{k+1}
  //   completed).  !SEP: delta_k overwrites X_{k+1} (its ones chunk stays).
  __host__ __device__ static constexpr uint32_t dboff(int k) {
    return k == NL - 1 ? DOFF : (!SEP ? xoff(k + 1) : (((NL - 2 - k) % 2 == 0) ? DAOFF : xoff(k + 2)));
  }
  __host__ __device__ static constexpr uint32_t dfeat(int k) {
    return k == NL - 1 ? (uint32_t)NOUT : (!SEP ? xfeat(k + 1) : (((NL - 2 - k) % 2 == 0) ? (uint32_t)W : xfeat(k + 2)));
  }
  static constexpr uint32_t WOFF = 2u * GBYTES;
  static constexpr uint32_t BOFF = WOFF + B::WBYTES;
  static constexpr uint32_t MISC = (BOFF + B::BBYTES + 127u) & ~127u;
  // dW^T A operands read 16 feature chunks (M = 128) from a lo base
  __host__ __device__ static constexpr uint32_t overread(int k) {
    return GBYTES + xoff(k) + (xfeat(k) / 8) * CHT + 16u * CHT;
  }
  __host__ __device__ static constexpr uint32_t max_overread(int k) {
    return k < 0 ? 0u : (overread(k) > max_overread(k - 1) ? overread(k) : max_overread(k - 1));
  }
  static constexpr uint32_t SMEM_RAW = MISC + 64;
  static constexpr uint32_t SMEM = SMEM_RAW > max_overread(NL - 1) ? SMEM_RAW : max_overread(NL - 1);
  __host__ __device__ static constexpr int dwcol(int k) { return 128 + B::osum(k); }
  static constexpr int DWCOLS = dwcol(NL) - 128;
  static constexpr int TCOLS = 512;
};

template <int ROWS>
__device__ __forceinline__ void issue_fwd_r(uint32_t d, uint32_t xhi, uint32_t xlo, uint32_t whi, uint32_t wlo,
                                            int K, int out) {
  constexpr uint32_t CHR = ROWS * 16;
  const uint32_t idesc = tc::idesc_bf16(ROWS, out, false, false);
  const uint64_t ah = tc::sdesc(xhi, CHR, 128), al = tc::sdesc(xlo, CHR, 128);
  const uint64_t bh = tc::sdesc(whi, out * 16, 128), bl = tc::sdesc(wlo, out * 16, 128);
#pragma unroll
  for (int s = 0; s < K / 16; ++s) {
    const uint64_t xa = (uint64_t)(s * 2 * (int)CHR) >> 4, wa = (uint64_t)(s * 2 * out * 16) >> 4;
    mma3(d, ah + xa, al + xa, bh + wa, bl + wa, idesc, s > 0 ? 1u : 0u);
  }
}

template <int ROWS>
__device__ __forceinline__ void issue_dx_r(uint32_t d, uint32_t dhi, uint32_t dlo, uint32_t whi, uint32_t wlo,
                                           int out, int nin) {
  constexpr uint32_t CHR = ROWS * 16;
  const uint32_t idesc = tc::idesc_bf16(ROWS, nin, false, true);
  const uint64_t ah = tc::sdesc(dhi, CHR, 128), al = tc::sdesc(dlo, CHR, 128);
  const uint64_t bh = tc::sdesc(whi, 128, out * 16), bl = tc::sdesc(wlo, 128, out * 16);
#pragma unroll
  for (int s = 0; s < out / 16; ++s) {
    const uint64_t da = (uint64_t)(s * 2 * (int)CHR) >> 4, wa = (uint64_t)(s * 256) >> 4;
    mma3(d, ah + da, al + da, bh + wa, bl + wa, idesc, s > 0 ? 1u : 0u);
  }
}

// dW^T[128 feats x out] += X^T delta over the ROWS samples of a tile (always accumulates)
template <int ROWS>
__device__ __forceinline__ void issue_dw_r(uint32_t d, uint32_t xhi, uint32_t xlo, uint32_t dhi, uint32_t dlo,
                                           int out) {
  constexpr uint32_t CHR = ROWS * 16;
  const uint32_t idesc = tc::idesc_bf16(128, out, true, true);
  const uint64_t ah = tc::sdesc(xhi, 128, CHR), al = tc::sdesc(xlo, 128, CHR);
  const uint64_t bh = tc::sdesc(dhi, 128, CHR), bl = tc::sdesc(dlo, 128, CHR);
#pragma unroll
  for (int s = 0; s < ROWS / 16; ++s) {
    const uint64_t ra = (uint64_t)(s * 256) >> 4;
    mma3(d, ah + ra, al + ra, bh + ra, bl + ra, idesc, 1u);
  }
}

template <int V>
struct IC {
  static constexpr int value = V;
};
// f(IC<k>{}) for a k that is a constant after loop unrolling (the branches fold)
template <int NK, class F>
__device__ __forceinline__ void with_k(int k, F&& f) {
  if constexpr (NK > 0) {
    if (k == NK - 1) f(IC<NK - 1>{});
    else with_k<NK - 1>(k, f);
  }
}

template <class N>
__global__ void __launch_bounds__(512, 1) tc_train64_kernel(TrainArgs a) {
  using T = TC64<N>;
  using TB = TC<N>;
  constexpr int NL = N::NL, K = N::K, W = N::W, NOUT = N::NOUT, L = N::L;
  constexpr int RT = T::RT;
  constexpr uint32_t CHT = T::CHT;
  constexpr int WH = W / 2, XH = WH / 8;        // hidden cols per warp-pair half, 16dp reps
  constexpr int LJ = L / 4;                     // levels per thread (encode / scatter)
  constexpr int KJ = K / 8;                     // lobe groups of 8 per raw parameter block
  constexpr int KL = K / 4;                     // lobes per thread in the head
  static_assert(K % 8 == 0 && L % 4 == 0 && W % 16 == 0, "two-tile kernel shape");
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sb = tc::smem_u32(smem);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = warp >> 3, wq = warp & 3, h = (warp >> 2) & 1, c = lane & 3;
  const int gtid = tid & 255;
  const int r0 = 16 * wq + (lane >> 2);
  const int re = r0 + 8 * (c & 1);              // encode / scatter row
  const int rh = r0 + 8 * h;                    // head row
  const uint32_t qaddr = (uint32_t)(wq * 32) << 16;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + T::MISC);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + T::MISC + 32);
  if (tid == 0) {
    tc::mbar_init(mbar, 1);
    tc::mbar_init(mbar + 1, 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc(tslot, (uint32_t)T::TCOLS);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  // A 512-column allocation is the whole TMEM: its base is column 0, lane 0.
  // Using the constant (checked) keeps every MMA operand warp-uniform, so the
  // issue below compiles to uniform-datapath descriptor arithmetic with no
  // per-MMA R2UR/ELECT waterfall.
  static_assert(T::TCOLS == 512, "constant TMEM base needs the full allocation");
  constexpr uint32_t tbase = 0;
  if (*tslot != 0u) __trap();
  stage_weights_tc<N>(a.params, smem, T::WOFF, T::BOFF);
  // zero the shared dW^T accumulators (all later MMAs accumulate)
  for (int col = 16 * (warp >> 2); col < T::DWCOLS; col += 64)
    tc::tmem_zero16(tbase + qaddr + (uint32_t)(128 + col));
  tc::tmem_wait_st();
  const float4* tab = reinterpret_cast<const float4*>(a.params + N::N_MLP);
  float4* gtab = reinterpret_cast<float4*>(a.grads + N::N_MLP);
  const float* bias = reinterpret_cast<const float*>(smem + T::BOFF);
  uint64_t* gbar = mbar + g;
  // MMA issue for group G (compile-time): operand addresses are sb-relative
  // constants, i.e. uniform registers.
  auto issue_fwd_g = [&](auto G, auto KC) {
    constexpr int gg = decltype(G)::value, k = decltype(KC)::value;
    const uint32_t base = sb + (uint32_t)gg * T::GBYTES;
    const uint32_t xh = base + T::xoff(k), xl = xh + (T::xfeat(k) / 8) * CHT;
    const uint32_t w = sb + T::WOFF + TB::woff(k);
    issue_fwd_r<RT>(tbase + (uint32_t)(64 * gg), xh, xl, w, w + TB::wbytes(k), TB::in_p(k), TB::out(k));
    tc::mma_commit(mbar + gg);
  };
  auto issue_bwd_g = [&](auto G, auto KC) {
    constexpr int gg = decltype(G)::value, k = decltype(KC)::value;
    const uint32_t base = sb + (uint32_t)gg * T::GBYTES;
    const uint32_t xh = base + T::xoff(k), xl = xh + (T::xfeat(k) / 8) * CHT;
    const uint32_t dh = base + T::dboff(k), dl = dh + (T::dfeat(k) / 8) * CHT;
    const uint32_t w = sb + T::WOFF + TB::woff(k);
    issue_dx_r<RT>(tbase + (uint32_t)(64 * gg), dh, dl, w, w + TB::wbytes(k), TB::out(k), k > 0 ? W : N::NGRID);
    // SEP: the epilogue waits for dX_k only; dW_k completes before the next
    // commit (dX_{k-1}) fires, which is all a later overwrite needs.  k = 0
    // commits both: the next tile's encode rewrites X_0.
    if (T::SEP && k > 0) tc::mma_commit(mbar + gg);
    issue_dw_r<RT>(tbase + (uint32_t)T::dwcol(k), xh, xl, dh, dl, TB::out(k));
    if (!(T::SEP && k > 0)) tc::mma_commit(mbar + gg);
  };
  const uint32_t gsb = sb + (uint32_t)g * T::GBYTES;
  uint32_t xhi[NL], xlo[NL];
#pragma unroll
  for (int k = 0; k < NL; ++k) {
    xhi[k] = gsb + T::xoff(k);
    xlo[k] = xhi[k] + (T::xfeat(k) / 8) * CHT;
  }
  const uint32_t dlast_hi = gsb + T::DOFF, dlast_lo = dlast_hi + (NOUT / 8) * CHT;
  // constant "ones" features (bias rows of dW^T): X_0 at NIN (radiance), X_k at W
  if (gtid < RT) {
    const float e1[8] = {1.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f}, e0[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if constexpr (!N::PRODUCT) {
#pragma unroll
      for (int f = N::NGRID; f < T::ZF; f += 8) tc::store_chunk(xhi[0], xlo[0], RT, gtid, f / 8, f == N::NGRID ? e1 : e0);
    }
#pragma unroll
    for (int k = 1; k < NL; ++k) tc::store_chunk(xhi[k], xlo[k], RT, gtid, W / 8, e1);
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();

  const int64_t n = a.n;
  const int64_t ntiles = (n + RT - 1) / RT;
  uint32_t phase = 0;
  double loss = 0.0;
  unsigned c_used = 0, c_zero = 0, c_drop = 0;
  auto gsync = [&]() { tc::named_sync(1u + (uint32_t)g, 256u); };
  // All warps of the group poll the MMA mbarrier.  Measured on B200 (same-box
  // A/B): polling by one warp + a named barrier, or try_wait with a suspend
  // hint, were 0.6-2 % slower than plain polling despite its issue slots.
  auto gwait = [&]() {
    tc::mbar_wait(gbar, phase);
    phase ^= 1u;
    tc::fence_after_sync();
  };
  auto handoff = [&]() {
    tc::fence_proxy_async();
    tc::fence_before_sync();
    gsync();
  };
  struct TileIn {
    int64_t i;
    bool valid;
    float ux, uy, uz;
    float gf[4 * LJ];
  };
  // Next-tile encode.  SPREAD: positions loaded under the last forward MMA
  // (before the head) and level j's gathers issued under backward batch
  // gstep(j); else all of it under the last backward batch.  Measured on B200:
  // spreading helps the product shape (c4 train 4.11 -> 3.87 ms, more MMA
  // latency to cover) and costs c2 / c5 2-3 % (their gathers are throughput-
  // bound on L1TEX, so moving them only lengthens the other phases).
  constexpr bool SPREAD = N::PRODUCT;
  auto load_pos = [&](int64_t tl, TileIn& t) {
    const int64_t slot = tl * RT + re;
    t.valid = slot < n;
    t.i = t.valid ? (a.perm ? (int64_t)__ldg(a.perm + slot) : slot) : 0;
    t.ux = t.uy = t.uz = 0.f;
    if (t.valid) {
      t.ux = normalize_axis(__ldg(a.px + t.i), a.grid.lo[0], a.grid.inv[0]);
      t.uy = normalize_axis(__ldg(a.py + t.i), a.grid.lo[1], a.grid.inv[1]);
      t.uz = normalize_axis(__ldg(a.pz + t.i), a.grid.lo[2], a.grid.inv[2]);
    }
  };
  auto gather_lv = [&](TileIn& t, int j) {
    float4 gl = make_float4(0.f, 0.f, 0.f, 0.f);
    if (t.valid) {
      const int l = h * (L / 2) + 2 * j + (c >> 1);
      LevelCorners lc;
      level_corners(a.grid, l, t.ux, t.uy, t.uz, lc);
      gl = gather_level(tab, a.grid.off[l], lc);
    }
    t.gf[4 * j] = gl.x; t.gf[4 * j + 1] = gl.y; t.gf[4 * j + 2] = gl.z; t.gf[4 * j + 3] = gl.w;
  };
  auto load_tile = [&](int64_t tl, TileIn& t) {
    load_pos(tl, t);
#pragma unroll
    for (int j = 0; j < LJ; ++j) gather_lv(t, j);
  };
  const int64_t first_tile = (int64_t)blockIdx.x * 2 + g;
  const int64_t tstride = (int64_t)gridDim.x * 2;
  TileIn cur;
  if (first_tile < ntiles) load_tile(first_tile, cur);
  int tile_no = 0;
  const bool stamp = (a.debug & 4) && blockIdx.x == 0 && gtid == 0 && g == 0;
#define NPM_STAMP64(idx) \
  do { if (stamp && tile_no < 64) a.dbg_clock[tile_no * 16 + (idx)] = clock64(); } while (0)
  for (int64_t tile = first_tile; tile < ntiles; tile += tstride) {
    NPM_STAMP64(0);
    const bool evalid = cur.valid;
    const float ux = cur.ux, uy = cur.uy, uz = cur.uz;
    // head row inputs (consumed after the forward MMAs)
    const int64_t hslot = tile * RT + rh;
    const bool hvalid = hslot < n;
    const int64_t ih = hvalid ? (a.perm ? (int64_t)__ldg(a.perm + hslot) : hslot) : 0;
    const float h_wx = __ldg(a.wx + ih), h_wy = __ldg(a.wy + ih), h_wz = __ldg(a.wz + ih);
    const float h_t0 = __ldg(a.target + ih);
    const float h_t1 = a.channels == 3 ? __ldg(a.target + a.target_stride + ih) : 0.f;
    const float h_t2 = a.channels == 3 ? __ldg(a.target + 2 * a.target_stride + ih) : 0.f;
    const float h_p = __ldg(a.spdf + ih);
    uint32_t mask[NL];
    // ---- encode stores: this thread's levels of row re
#pragma unroll
    for (int j = 0; j < LJ; ++j) {
      const int l = h * (L / 2) + 2 * j + (c >> 1);
      tc::store_feats<4>(xhi[0], xlo[0], RT, re, 4 * l, cur.gf + 4 * j);
    }
    if constexpr (N::PRODUCT) {
      // per row: SH(w_o) [32,48) by (h0, c0/c1), SH(n) [48,64) by (h0, c2/c3),
      // roughness + ones [64,80) by (h1, c0/c1)
      const int64_t ie = cur.i;
      float e[16];
      const int blk = h == 0 ? (c >> 1) : (c < 2 ? 2 : 3);
      if (blk < 3) {
#pragma unroll
        for (int j = 0; j < 16; ++j) e[j] = 0.0f;
        if (blk == 0 && evalid) sh4(__ldg(a.wox + ie), __ldg(a.woy + ie), __ldg(a.woz + ie), e);
        if (blk == 1 && evalid) sh4(__ldg(a.nx + ie), __ldg(a.ny + ie), __ldg(a.nz + ie), e);
        if (blk == 2) {
          e[0] = evalid ? __ldg(a.rough + ie) : 0.0f;
          e[1] = 1.0f;   // feature NIN = 65: ones (bias row of dW_0^T)
        }
        tc::store_feats<16>(xhi[0], xlo[0], RT, re, 32 + 16 * blk, e);
      }
    }
    // ---- forward
    const bool has_next = tile + tstride < ntiles;
    TileIn nxt;
    nxt.valid = false;
#pragma unroll
    for (int k = 0; k < NL; ++k) {
      handoff();
      NPM_STAMP64(1 + 2 * k);
      if (gtid == 0) {
        tc::fence_after_sync();
        with_k<NL>(k, [&](auto KC) {
          if (g == 0) issue_fwd_g(IC<0>{}, KC);
          else issue_fwd_g(IC<1>{}, KC);
        });
      }
      if (SPREAD && k == NL - 1 && has_next) load_pos(tile + tstride, nxt);
      gwait();
      NPM_STAMP64(2 + 2 * k);
      const float* b = bias + TB::boff(k) / 4;
      if (k < NL - 1) {
        float v[4 * XH];
        tc::tmem_ld16dp<XH>(tbase + qaddr + (uint32_t)(64 * g + WH * h), v);
        tc::tmem_wait_ld();
        uint32_t mk = 0;
        float2 bj[XH];   // loaded before the stores (their asm memory clobbers force reloads)
#pragma unroll
        for (int j = 0; j < XH; ++j) bj[j] = *reinterpret_cast<const float2*>(b + WH * h + 8 * j + 2 * c);
#pragma unroll
        for (int j = 0; j < XH; ++j) {
#pragma unroll
          for (int half = 0; half < 2; ++half) {
            const int col = WH * h + 8 * j + 2 * c;
            const int idx = 2 * half + 4 * j;
            const float2 bb = bj[j];
            const float y0 = fmaxf(v[idx] + bb.x, 0.0f), y1 = fmaxf(v[idx + 1] + bb.y, 0.0f);
            mk |= (y0 > 0.0f ? 1u : 0u) << (idx);
            mk |= (y1 > 0.0f ? 1u : 0u) << (idx + 1);
            tc::store_pair(xhi[k + 1], xlo[k + 1], RT, r0 + 8 * half, col, y0, y1);
          }
        }
        mask[k + 1] = mk;
      } else {
        // ---- Eq. 9 head (C-O12, C-O13): row rh, lobes 8 jj + 2 c + w
        float v[2 * NOUT / 8 * 2];   // 16x256b x(NOUT/8): both row halves
        tc::tmem_ld16dp<NOUT / 8>(tbase + qaddr + (uint32_t)(64 * g), v);
        tc::tmem_wait_ld();
        float lp[KL], kp[KL], tp[KL], pp[KL];
#pragma unroll
        for (int jj = 0; jj < KJ; ++jj) {
#pragma unroll
          for (int w = 0; w < 2; ++w) {
            const int m = 2 * jj + w, lobe = 8 * jj + 2 * c + w;
            // row half h selects registers w or w + 2 (a select, not a dynamic
            // index: that would put v in local memory)
            auto pick = [&](int blk) { return h ? v[w + 2 + 4 * (blk * KJ + jj)] : v[w + 4 * (blk * KJ + jj)]; };
            lp[m] = pick(0) + b[lobe];
            kp[m] = pick(1) + b[K + lobe];
            tp[m] = pick(2) + b[2 * K + lobe];
            pp[m] = pick(3) + b[3 * K + lobe];
          }
        }
        float t = h_t0;
        bool all_zero = t == 0.0f;
        if (a.channels == 3) {
          all_zero = all_zero && h_t1 == 0.0f && h_t2 == 0.0f;
          t = 0.2126f * t + 0.7152f * h_t1 + 0.0722f * h_t2;
        }
        const float p = h_p;
        const float ratio = t / p;
        const bool drop = hvalid && (!isfinite(ratio) || !isfinite(p) || !(p > 0.0f));
        const bool zero = hvalid && !drop && all_zero;
        const bool use = hvalid && !drop && !zero;
        const float s = use ? (float)(-(double)ratio * a.inv_n_global) : 0.0f;
        const float wx = h_wx, wy = h_wy, wz = h_wz;
        float kap[KL], mx[KL], my[KL], mz[KL], th[KL], ph[KL], vv[KL], sth[KL], cth[KL], sph[KL], cph[KL];
        float emk[KL];
        float mloc = lp[0];
#pragma unroll
        for (int m = 0; m < KL; ++m) {
          mloc = fmaxf(mloc, lp[m]);
          kap[m] = __expf(fminf(fmaxf(kp[m], a.log_kmin), a.log_kmax));
          lobe_angles<false>(tp[m], pp[m], kap[m], th[m], ph[m], sth[m], cth[m], sph[m], cph[m]);
          mx[m] = sth[m] * cph[m]; my[m] = sth[m] * sph[m]; mz[m] = cth[m];
          const float nrm = lobe_norm_fast(kap[m], emk[m]);
          vv[m] = lobe_eval(nrm, kap[m], mx[m], my[m], mz[m], wx, wy, wz);
        }
        // the 4 threads of a row are lanes 4i..4i+3: reduce with xor 1, 2
        mloc = fmaxf(mloc, __shfl_xor_sync(0xffffffffu, mloc, 1));
        mloc = fmaxf(mloc, __shfl_xor_sync(0xffffffffu, mloc, 2));
        float e[KL], S = 0.0f, P = 0.0f;
#pragma unroll
        for (int m = 0; m < KL; ++m) {
          e[m] = __expf(lp[m] - mloc);
          S += e[m];
          P += e[m] * vv[m];
        }
        S += __shfl_xor_sync(0xffffffffu, S, 1);
        S += __shfl_xor_sync(0xffffffffu, S, 2);
        P += __shfl_xor_sync(0xffffffffu, P, 1);
        P += __shfl_xor_sync(0xffffffffu, P, 2);
        const float invS = 1.0f / S;
        const float Vb = fmaxf(P * invS, kVFloor);
        const float invV = 1.0f / Vb;
        // f-4 (C-A31): chi^2 scales Eq. 9's record weight by D^ / V
        const float chi = a.divergence ? (use ? t * invV : 0.0f) : 1.0f;   // t may be NaN on dropped records
        const float sd = s * chi;
#pragma unroll
        for (int jj = 0; jj < KJ; ++jj) {
          float dl[2], dk[2], dt[2], dp[2];
#pragma unroll
          for (int w = 0; w < 2; ++w) {
            const int m = 2 * jj + w;
            const float lam = e[m] * invS;
            const float gam = lam * vv[m] * invV;
            dl[w] = sd * (gam - lam);
            const float dx = mx[m] - wx, dy = my[m] - wy, dz = mz[m] - wz;
            const float d2 = dx * dx + dy * dy + dz * dz;
            // 2 kappa e^{-2 kappa} / (1 - e^{-2 kappa}) with em = 1 - e^{-2 kappa}
            const float dkk = sd * gam * (1.0f - kap[m] * 0.5f * d2 - __fdividef(2.0f * kap[m] * (1.0f - emk[m]), emk[m]));
            dk[w] = (kp[m] < a.log_kmin || kp[m] > a.log_kmax) ? 0.0f : dkk;
            const float wdth = kPi * (cth[m] * cph[m] * wx + cth[m] * sph[m] * wy - sth[m] * wz);
            const float wdph = kTwoPi * (-sth[m] * sph[m] * wx + sth[m] * cph[m] * wy);
            const float sgk = sd * gam * kap[m];
            dt[w] = sgk * wdth * th[m] * (1.0f - th[m]);
            dp[w] = sgk * wdph * ph[m] * (1.0f - ph[m]);
          }
          const int f = 8 * jj + 2 * c;
          tc::store_pair(dlast_hi, dlast_lo, RT, rh, f, dl[0], dl[1]);
          tc::store_pair(dlast_hi, dlast_lo, RT, rh, K + f, dk[0], dk[1]);
          tc::store_pair(dlast_hi, dlast_lo, RT, rh, 2 * K + f, dt[0], dt[1]);
          tc::store_pair(dlast_hi, dlast_lo, RT, rh, 3 * K + f, dp[0], dp[1]);
        }
        if (c == 0) {
          c_drop += drop; c_zero += zero;
          if (use) {
            loss += a.divergence ? -(double)sd : (double)s * (double)logf(Vb);   // chi^2: (D^/p~)(D^/V)/N
            c_used += 1;
          }
        }
      }
    }
    // ---- backward
    uint32_t dhi = dlast_hi, dlo = dlast_lo;
#pragma unroll
    for (int k = NL - 1; k >= 0; --k) {
      handoff();
      NPM_STAMP64(1 + 2 * NL + 2 * (NL - 1 - k));
      if (gtid == 0) {
        tc::fence_after_sync();
        with_k<NL>(k, [&](auto KC) {
          if (g == 0) issue_bwd_g(IC<0>{}, KC);
          else issue_bwd_g(IC<1>{}, KC);
        });
      }
      if (SPREAD && has_next) {
#pragma unroll
        for (int j = 0; j < LJ; ++j)
          if ((NL - 1 - j > 0 ? NL - 1 - j : 0) == k) gather_lv(nxt, j);   // gstep(j)
      }
      if (!SPREAD && k == 0 && has_next) load_tile(tile + tstride, nxt);
      gwait();
      NPM_STAMP64(2 + 2 * NL + 2 * (NL - 1 - k));
      if (k > 0) {
        float v[4 * XH];
        tc::tmem_ld16dp<XH>(tbase + qaddr + (uint32_t)(64 * g + WH * h), v);
        tc::tmem_wait_ld();
        const uint32_t mk = mask[k];
        dhi = gsb + T::dboff(k - 1);
        dlo = dhi + (T::dfeat(k - 1) / 8) * CHT;
#pragma unroll
        for (int j = 0; j < XH; ++j) {
#pragma unroll
          for (int half = 0; half < 2; ++half) {
            const int col = WH * h + 8 * j + 2 * c;
            const int idx = 2 * half + 4 * j;
            const float d0 = ((mk >> idx) & 1u) ? v[idx] : 0.0f;
            const float d1 = ((mk >> (idx + 1)) & 1u) ? v[idx + 1] : 0.0f;
            tc::store_pair(dhi, dlo, RT, r0 + 8 * half, col, d0, d1);
          }
        }
      } else {
        // dz: warp half h holds grid features [2 L h, 2 L (h+1)); pair lanes c, c^1
        // exchange so each holds the 4 features of level h L/2 + 2 j + c/2 of row re
        float v[4 * LJ];
        tc::tmem_ld16dp<LJ>(tbase + qaddr + (uint32_t)(64 * g + 2 * L * h), v);
        tc::tmem_wait_ld();
        const bool odd = c & 1;
#pragma unroll
        for (int j = 0; j < LJ; ++j) {
          const float s0 = odd ? v[4 * j + 0] : v[4 * j + 2];   // the partner's row
          const float s1 = odd ? v[4 * j + 1] : v[4 * j + 3];
          const float r0v = __shfl_xor_sync(0xffffffffu, s0, 1);
          const float r1v = __shfl_xor_sync(0xffffffffu, s1, 1);
          float gq[4];
          if (!odd) { gq[0] = v[4 * j]; gq[1] = v[4 * j + 1]; gq[2] = r0v; gq[3] = r1v; }
          else { gq[0] = r0v; gq[1] = r1v; gq[2] = v[4 * j + 2]; gq[3] = v[4 * j + 3]; }
          const int lsc = h * (L / 2) + 2 * j + (c >> 1);
          // measurement knobs (NPM_DEBUG): bit 3 skips the two coarsest levels' scatter, bit 4 the two finest
          const bool dbg_skip = ((a.debug & 8) && lsc < 2) || ((a.debug & 16) && lsc >= L - 2);
          if (evalid && !(a.debug & 1) && !dbg_skip &&
              (gq[0] != 0.0f || gq[1] != 0.0f || gq[2] != 0.0f || gq[3] != 0.0f)) {
            const int l = lsc;
            LevelCorners lc;
            level_corners(a.grid, l, ux, uy, uz, lc);
            float4* tg = ((a.priv_mask >> l) & 1u)
                             ? a.priv + (int64_t)blockIdx.x * a.priv_stride + a.priv_off[l]
                             : gtab + a.grid.off[l];
#pragma unroll
            for (int cc = 0; cc < 8; ++cc) {
              const float w = lc.w[cc];
              atomicAdd(tg + lc.idx[cc], make_float4(w * gq[0], w * gq[1], w * gq[2], w * gq[3]));
            }
          }
        }
      }
    }
    NPM_STAMP64(15);
    ++tile_no;
    cur = nxt;
  }
  // ---- flush dW^T / db (M = 128 layout: lane = input feature; quarter = warp / 4)
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  {
    const int q = warp >> 2, r = ((warp & 3) << 5) | lane;
    const uint32_t lane_addr = (uint32_t)((warp & 3) << 21);
#pragma unroll
    for (int k = 0; k < NL; ++k) {
      constexpr int MAXO = (NOUT > W ? NOUT : W) / 4;
      float vv[MAXO];
      const int out = TB::out(k), in = TB::in(k), oq = out / 4;
      if (out == NOUT) tc::tmem_ldn<NOUT / 4>(tbase + lane_addr + (uint32_t)(T::dwcol(k) + q * (NOUT / 4)), vv);
      else tc::tmem_ldn<W / 4>(tbase + lane_addr + (uint32_t)(T::dwcol(k) + q * (W / 4)), vv);
      tc::tmem_wait_ld();
      if (r < in) {
        float* gp = a.grads + N::gw_off(k) + r;
        for (int o = 0; o < oq; ++o) atomicAdd(gp + (q * oq + o) * in, vv[o]);
      } else if (r == in) {
        float* gp = a.grads + N::gb_off(k);
        for (int o = 0; o < oq; ++o) atomicAdd(gp + q * oq + o, vv[o]);
      }
    }
  }
  loss = warp_sum_d(loss);
  c_used = warp_sum_u(c_used); c_zero = warp_sum_u(c_zero); c_drop = warp_sum_u(c_drop);
  if (lane == 0) {
    atomicAdd(a.stats, loss);
    atomicAdd(a.counters + 0, (unsigned long long)c_used);
    atomicAdd(a.counters + 1, (unsigned long long)c_zero);
    atomicAdd(a.counters + 2, (unsigned long long)c_drop);
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  if (warp == 0) tc::tmem_dealloc(tbase, (uint32_t)T::TCOLS);
}

#include "npm_train_ws.cuh"
#include "npm_query_ws.cuh"

template <class N>
struct TcLaunch {
  static int query(const QueryArgs& a, int sms, cudaStream_t st) {
    using T = TC<N>;
    if constexpr ((!N::PRODUCT && N::K == 8) || (N::PRODUCT && N::K == 16)) {
      // warp-specialised kernel for sample / pdf and combined-MIS calls (npm_query_ws.cuh)
      if (a.qws && !a.feat_in && !a.raw && !a.lambda && !a.kappa && !a.mu &&
          (!N::PRODUCT || (!a.combined && !a.cos_product))) {
        auto go = [&](auto MC, auto GC) -> int {
          constexpr int MODE = decltype(MC)::value, G = decltype(GC)::value;
          using Q = qws::QW<N, MODE, G>;
          if (Q::MP == 4) {   // the setmaxnreg split assumes the launch allocation (a hang otherwise)
            static int regs = -1;
            if (regs < 0) {
              cudaFuncAttributes fa;
              regs = cudaFuncGetAttributes(&fa, qws::query_ws_kernel<N, MODE, G>) == cudaSuccess ? fa.numRegs : 0;
            }
            if (regs != Q::LAUNCH_REGS) return -1;
          }
          cudaFuncSetAttribute(qws::query_ws_kernel<N, MODE, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)Q::SMEM);
          const int64_t ntiles = (a.n + Q::R - 1) / Q::R;
          const int blocks = (int)(ntiles < (int64_t)sms ? ntiles : (int64_t)sms);
          qws::query_ws_kernel<N, MODE, G><<<blocks, Q::THREADS, Q::SMEM, st>>>(a);
          return 1;
        };
        using G1 = std::integral_constant<int, 1>;
        using G2 = std::integral_constant<int, 2>;
        // chain groups: the plain call takes the model's choice (qws_groups);
        // the product shape always one, the f-1 / f-2 calls two
        if constexpr (N::PRODUCT) return go(std::integral_constant<int, 0>{}, G1{});
        else return a.combined ? go(std::integral_constant<int, 1>{}, G2{})
                               : a.cos_product ? go(std::integral_constant<int, 2>{}, G2{})
                                               : a.qws_groups == 1 ? go(std::integral_constant<int, 0>{}, G1{})
                                                                   : go(std::integral_constant<int, 0>{}, G2{});
      }
    }
    // 2 threads per sample row, 256-thread CTAs, two CTAs per SM (their MMA
    // waits interleave); ~104 KB smem each.
    constexpr int TPR = 2;
    const int64_t ntiles = (a.n + R - 1) / R;
    if (a.query_groups == 2) {   // one CTA per SM, two tile groups over one weight copy
      auto kern = a.combined ? tc_query_kernel<N, TPR, 1, 2> : a.cos_product ? tc_query_kernel<N, TPR, 2, 2>
                                                                             : tc_query_kernel<N, TPR, 0, 2>;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)T::SMEM_QUERY2);
      const int64_t pairs = (ntiles + 1) / 2;
      const int blocks = (int)(pairs < (int64_t)sms ? pairs : (int64_t)sms);
      kern<<<blocks, 2 * TPR * R, T::SMEM_QUERY2, st>>>(a);
      return 1;
    }
    auto kern = a.combined ? tc_query_kernel<N, TPR, 1, 1> : a.cos_product ? tc_query_kernel<N, TPR, 2, 1>
                                                                           : tc_query_kernel<N, TPR, 0, 1>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)T::SMEM_QUERY);
    const int per_sm = (int)((228u * 1024u) / (T::SMEM_QUERY + 1024u)) >= 2 ? 2 : 1;
    const int64_t cap = (int64_t)sms * per_sm;
    const int blocks = (int)(ntiles < cap ? ntiles : cap);
    kern<<<blocks, TPR * R, T::SMEM_QUERY, st>>>(a);
    return 1;
  }
  static int train(const TrainArgs& a, int sms, cudaStream_t st) {
    if constexpr ((!N::PRODUCT && N::K == 8) || (N::PRODUCT && N::K == 16 && N::L == 8)) {
      if (a.ws) {   // warp-specialised kernel (npm_train_ws.cuh)
        if (!a.wimg || a.wimg_bytes < ws::WS<N>::WIMG) return -1;
        if (a.alpha_w && (!a.alpha_g || !a.bsdf_pdf)) return -1;
        ws::prep_wimg_kernel<N><<<8, 256, 0, st>>>(a.params, a.wimg);
        auto go = [&](auto AHC, auto VAC) {
          constexpr bool AH = decltype(AHC)::value, VA = decltype(VAC)::value;
          using T = ws::WS<N, AH, VA>;
          cudaFuncSetAttribute(ws::train_ws_kernel<N, AH, VA>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)T::SMEM);
          const int64_t ntiles = (a.n + T::R - 1) / T::R;
          const int blocks = (int)(ntiles < (int64_t)sms ? ntiles : (int64_t)sms);
          ws::train_ws_kernel<N, AH, VA><<<blocks, T::THREADS, T::SMEM, st>>>(a);
        };
        if (a.alpha_w && a.divergence == 2) return -1;   // one of the two per launch
        if constexpr (N::PRODUCT) {   // (the product shape: Eq. 9 / chi^2 only)
          if (a.alpha_w || a.divergence == 2) return -1;
          go(std::false_type{}, std::false_type{});
        } else {
          if (a.alpha_w) go(std::true_type{}, std::false_type{});
          else if (a.divergence == 2) go(std::false_type{}, std::true_type{});
          else go(std::false_type{}, std::false_type{});
        }
        return 2;
      }
    }
    // the C-A34 head and the variance-aware target (C-A35) are trained by the
    // warp-specialised kernel only
    if (a.alpha_w || a.divergence == 2) return -1;
    // two 64-sample tiles per CTA (tc_train64_kernel)
    using T64 = TC64<N>;
    cudaFuncSetAttribute(tc_train64_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)T64::SMEM);
    const int64_t pairs = (a.n + 2 * T64::RT - 1) / (2 * T64::RT);
    const int blocks = (int)(pairs < (int64_t)sms ? pairs : (int64_t)sms);
    tc_train64_kernel<N><<<blocks, 512, T64::SMEM, st>>>(a);
    return 1;
  }
};

}  // namespace tck
}  // namespace npm
