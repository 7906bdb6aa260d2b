// npm_train_ws.cuh -- warp-specialised fused training kernel (round 2).
// Included from npm_tc_kernels.cuh (namespace npm::tck).
//
// One persistent CTA per SM, 128-sample tiles (MMA M = 128, TMEM lane r =
// tile row r), three roles on warps (every role fits ptxas' 128 registers per
// thread of a 512-thread CTA without spills, so no setmaxnreg):
//
//   warps 0-7   CHAIN: the two threads of row r are warps w and w + 4 (lane
//       r % 32, w = r / 32), each owning half of the columns, lobes and
//       levels.  Thread 0 issues the tcgen05 MMAs; all 256 run the epilogues
//       (bias, ReLU, split-bf16 into smem), the Eq. 9 head (P:210-216,
//       C-O12/C-O13; softmax and mixture sums exchanged through smem) and the
//       backward epilogues (C-O14), and hand dz (the grid part of dL/dz) to
//       the scatter warps through smem.
//   warps 8-15  MEMORY: thread (part, row) with part = which half of the L
//       levels.  Iteration k: for tile k normalise x (C-O1), find the 8
//       corners per level (Eq. 13, C-O3/C-O4), gather and blend them (C-O5),
//       write X0 (split bf16, chunk-major) into an X0 stage and the head inputs
//       into a row-data stage; then for tile k - 1 scatter
//       dE_l[idx_c] += w_c dz_l (C-O15) with red.global.add.v4.f32 from the dz
//       stage the chain filled.
//
// The roles hand tiles over through mbarrier rings (x0 full/empty, dz
// full/empty), so a tile's gathers, its MMA chain and the previous tile's
// scatter run concurrently instead of in sequence (r01: one 256-thread group
// per tile did all three in turn).  The split-bf16 weight image (built once per
// launch by prep_wimg_kernel) is staged into smem with one cp.async.bulk (TMA
// bulk copy, completion through an mbarrier transaction count).
#pragma once

namespace ws {

#ifndef NPM_WS_PAIRS
#define NPM_WS_PAIRS true
#endif

template <class N, bool AH = false, bool VA = false>
struct WS {
  using B = TC<N>;
  static constexpr int NL = N::NL, W = N::W, NOUT = N::NOUT, NIN = N::NIN, L = N::L, K = N::K, NG = N::NGRID;
  static constexpr int R = 128;              // rows per tile = MMA M
  static constexpr uint32_t CHR = R * 16;    // bytes of one 8-feature chunk of a tile
  static constexpr int ZF = B::ZF, HF = B::HF, KIN = B::KIN;
  // radiance K = 8, or the product shape (K = 16, 8 levels; X0 = grid | SH4(w_o) |
  // SH4(n) | roughness, ones at NIN = 65 written per tile by the memory warps)
  static_assert((N::PRODUCT ? (K == 16 && L == 8 && ZF == 80 && !AH && !VA) : K == 8) && L % 2 == 0 &&
                W % 32 == 0, "warp-specialised kernel shape");
  static constexpr int TPR = 2;   // chain threads per row (B200 c2: 2 -> 520 us, 4 -> 561 us without the scatter)
  static constexpr int CHAIN_THREADS = TPR * R, MEM_THREADS = 256, THREADS = CHAIN_THREADS + MEM_THREADS;
  static constexpr int GATHER_THREADS = MEM_THREADS, SCATTER_THREADS = MEM_THREADS;
  static_assert(L % TPR == 0 && (L / 2) % 2 == 0 && K % TPR == 0 && (W / TPR) % 16 == 0, "quarters");
  // ---- smem map
  static constexpr uint32_t WIMG = B::WBYTES + B::BBYTES;   // weight image, bulk-copied
  static_assert(WIMG % 16 == 0, "bulk copy size");
  static constexpr uint32_t a1k(uint32_t x) { return (x + 1023u) & ~1023u; }
  static constexpr uint32_t X0_BYTES = 2u * (ZF / 8) * CHR;
  static constexpr uint32_t XH_BYTES = 2u * (HF / 8) * CHR;
  // AH (C-A34 head trained): delta_{NL-1} gets one more chunk whose first
  // column holds dM2/dz, and dW_{NL-1}'s MMA runs XD = 16 columns wider (M = 128
  // needs N % 16 == 0) so it also yields the head's gradient.  Only column NOUT
  // is read back: the MMA's second extra chunk reads whatever follows (the lo
  // half's first chunk / the X0 stage) into columns that are never used.
  static constexpr int XC = AH ? 8 : 0, XD = AH ? 16 : 0;
  static constexpr uint32_t D_BYTES = 2u * ((NOUT + XC) / 8) * CHR;
  static constexpr uint32_t AH_BYTES = AH ? 4u * (W + 4) : 0u;
  // VA (f-4 variance-aware target, C-A35): every lobe's (kappa, mu, e) of the
  // row for the pairwise terms of int V^2, [5 K][R] f32
  static constexpr uint32_t VX_BYTES = VA ? 5u * K * R * 4u : 0u;
  // row data [RDF][R] f32: slots 3 valid | 4-6 w_i | 7-9 target | 10 pdf |
  // 11 p_bsdf (AH).  It also carries the head's exchange between the row's two
  // threads (no separate buffer: the 164 KB carve-out leaves L1 92 KB -- the
  // gathers run ~6 % slower per 32 KB less L1): slots 0/1 the softmax max of
  // thread h (written before the first pair barrier, no other reader), slots
  // 4+2h / 5+2h its sums (written after that barrier, when both threads have
  // read the row's inputs); AH: the logit parts in slots 2 / 12.
  static constexpr int RDF = AH ? 13 : 11;
  static constexpr uint32_t RD_BYTES = RDF * R * 4;
  static constexpr uint32_t DZ_BYTES = (uint32_t)L * R * 16;   // [L][R] float4
  static constexpr uint32_t OFF_X1 = a1k(WIMG);
  __host__ __device__ static constexpr uint32_t xhoff(int k) { return OFF_X1 + (uint32_t)(k - 1) * XH_BYTES; }
  static constexpr uint32_t OFF_D = OFF_X1 + (uint32_t)(NL - 1) * XH_BYTES;
  static constexpr uint32_t OFF_X0 = OFF_D + D_BYTES;
  // X0 stages.  One: with two (gathers a full tile ahead) the memory warps'
  // extra in-flight loads slowed the chain more than the overlap gained
  // (B200 c2, same box: S0 = 2 545 us, S0 = 1 525 us); the 2-stage protocol
  // stays selectable for measurement (-DNPM_WS_S0=2).
#ifdef NPM_WS_S0   // measurement override
  static constexpr int S0 = NPM_WS_S0;
#else
  static constexpr int S0 = 1;
#endif
  static_assert(S0 == 1 || S0 == 2, "X0 stages");
  // delta_{NL-1} in D; delta_k (k < NL-1) over X_{k+1} (its ones chunk stays).
  // (Measured on B200 c2: a separate delta buffer letting each backward
  // epilogue run under the dW MMAs did not shorten the backward phases.)
  __host__ __device__ static constexpr uint32_t dboff(int k) { return k == NL - 1 ? OFF_D : xhoff(k + 1); }
  __host__ __device__ static constexpr uint32_t dfeat(int k) { return k == NL - 1 ? (uint32_t)(NOUT + XC) : (uint32_t)HF; }
  static constexpr uint32_t OFF_RD = OFF_X0 + (uint32_t)S0 * X0_BYTES;
  static constexpr uint32_t OFF_DZ = OFF_RD + (uint32_t)S0 * RD_BYTES;
  // C-A34 selection head: its parameters (a [W], c)
  static constexpr uint32_t OFF_AH = (OFF_DZ + DZ_BYTES + 15u) & ~15u;
  static constexpr uint32_t OFF_VX = OFF_AH + AH_BYTES;
  static constexpr uint32_t OFF_BAR = OFF_VX + VX_BYTES;
  // mbarriers: [0] weights, [1] mma, [2] dz full, [3] dz empty, [4..4+S0) x0 full, [4+S0..4+2 S0) x0 empty,
  // [4+2 S0] head start (the scatter of tile k-1 waits for tile k's head)
  static constexpr int NBAR = 6 + 2 * S0;   // + [5 + 2 S0]: the backward dW^T batches (second issuer)
  static constexpr uint32_t OFF_TSLOT = OFF_BAR + 8u * NBAR;
#ifndef NPM_WS_SMEM_PAD   // measurement knob: extra dynamic smem (a smaller L1 carve-out)
#define NPM_WS_SMEM_PAD 0
#endif
  static constexpr uint32_t SMEM_RAW = OFF_TSLOT + 16u + NPM_WS_SMEM_PAD;
  // dW^T MMAs read M_k / 8 feature chunks from a lo base (M_k = 64 or 128):
  // the rows past X_k's features are garbage rows of dW^T (ignored) but the
  // reads must stay inside the allocation
  __host__ __device__ static constexpr int dwm(int k) { return (k == 0 ? ZF : HF) <= 64 ? 64 : 128; }
  __host__ __device__ static constexpr uint32_t overread(int k) {
    return (k == 0 ? OFF_X0 + (uint32_t)(S0 - 1) * X0_BYTES + (ZF / 8) * CHR : xhoff(k) + (HF / 8) * CHR) +
           (uint32_t)(dwm(k) / 8) * CHR;
  }
  __host__ __device__ static constexpr uint32_t max_overread(int k) {
    return k < 0 ? 0u : (overread(k) > max_overread(k - 1) ? overread(k) : max_overread(k - 1));
  }
  static constexpr uint32_t SMEM = SMEM_RAW > max_overread(NL - 1) ? SMEM_RAW : max_overread(NL - 1);
  static_assert(SMEM <= 227u * 1024u, "warp-specialised kernel smem");
  // ---- TMEM columns: forward / dX accumulator, dz, dW^T accumulators
  static constexpr int C_ACC = 0, C_DZ = 64;
  static_assert(W <= 64 && NOUT <= 64 && NG <= 64, "accumulator columns");
  __host__ __device__ static constexpr int dwcol(int k) { return 128 + B::osum(k); }
  static_assert(128 + N::osum(NL) + XD <= 512, "TMEM columns");
  static constexpr int TCOLS = 512;
};

// mbarrier wait that traps instead of hanging (a legitimate wait here is
// microseconds; 2^28 polls means a protocol bug).  An iteration count, not
// clock64: the clock reads and 64-bit compares of every poll were issue slots
// taken from the chain warps (ncu r02s: polling was ~26 % of issued instructions).
__device__ __forceinline__ void mbar_wait_t(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0, it = 0;
  while (true) {
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P;\n\t}\n"
        : "=r"(ok) : "r"(tc::smem_u32(bar)), "r"(parity) : "memory");
    if (ok) return;
    if (++it > (1u << 28)) __trap();
  }
}

// the same for warps with nothing else to do: try_wait with a suspend-time
// hint -- the warp sleeps in the instruction until the phase completes (or
// the hint expires) instead of spinning on issue slots the chain needs
__device__ __forceinline__ void mbar_wait_idle(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0, it = 0;
  while (true) {
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, P;\n\t}\n"
        : "=r"(ok) : "r"(tc::smem_u32(bar)), "r"(parity), "r"(100000u) : "memory");
    if (ok) return;
    if (++it > (1u << 24)) __trap();
  }
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(tc::smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(tc::smem_u32(bar)), "r"(bytes)
               : "memory");
}
// TMA bulk copy global -> shared, completion counted on `bar` (UBLKCP)
__device__ __forceinline__ void bulk_g2s(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(tc::smem_u32(sdst)), "l"(gsrc), "r"(bytes), "r"(tc::smem_u32(bar)) : "memory");
}

// dW^T[M feats x out] += X^T[M feats x ROWS] delta[ROWS x out]: both MN-major,
// M = 64 or 128 (the X_k feature chunks read), K = the ROWS samples.
template <int ROWS, int M>
__device__ __forceinline__ void issue_dw_m(uint32_t d, uint32_t xhi, uint32_t xlo, uint32_t dhi, uint32_t dlo,
                                           int out) {
  constexpr uint32_t CHR = ROWS * 16;
  const uint32_t idesc = tc::idesc_bf16(M, out, true, true);
  const uint64_t ah = tc::sdesc(xhi, 128, CHR), al = tc::sdesc(xlo, 128, CHR);
  const uint64_t bh = tc::sdesc(dhi, 128, CHR), bl = tc::sdesc(dlo, 128, CHR);
#pragma unroll
  for (int s = 0; s < ROWS / 16; ++s) {
    const uint64_t ra = (uint64_t)(s * 256) >> 4;
    mma3(d, ah + ra, al + ra, bh + ra, bl + ra, idesc, 1u);
  }
}

// Split-bf16 weight image in the smem layout of stage_weights_tc (chunk-major,
// hi then lo per layer) + fp32 biases: built once per launch from the live
// parameters, then bulk-copied by every CTA.
template <class N>
__global__ void __launch_bounds__(256) prep_wimg_kernel(const float* __restrict__ g, uint8_t* __restrict__ img) {
  using T = TC<N>;
#pragma unroll
  for (int k = 0; k < N::NL; ++k) {
    const int in = T::in(k), inp = T::in_p(k), out = T::out(k);
    const float* gw = g + N::gw_off(k);
    uint8_t* hi = img + T::woff(k);
    uint8_t* lo = hi + T::wbytes(k);
    const int cnt = out * (inp / 8);
    for (int e = (int)(blockIdx.x * blockDim.x + threadIdx.x); e < cnt; e += (int)(gridDim.x * blockDim.x)) {
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
      *reinterpret_cast<uint4*>(hi + off) = make_uint4(h[0], h[1], h[2], h[3]);
      *reinterpret_cast<uint4*>(lo + off) = make_uint4(l[0], l[1], l[2], l[3]);
    }
    float* sb = reinterpret_cast<float*>(img + T::WBYTES + T::boff(k));
    for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < out; o += gridDim.x * blockDim.x)
      sb[o] = __ldg(g + N::gb_off(k) + o);
  }
}

// AH: the C-A34 selection head is trained (a learn_alpha model); VA: the
// variance-aware target (divergence 2, C-A35).  Separate instantiations so the
// plain kernel carries none of their code.
template <class N, bool AH, bool VA>
__global__ void __launch_bounds__(WS<N, AH, VA>::THREADS, 1) train_ws_kernel(TrainArgs a) {
  using T = WS<N, AH, VA>;
  using TB = TC<N>;
  constexpr int NL = N::NL, K = N::K, W = N::W, NOUT = N::NOUT, L = N::L, NG = N::NGRID, NIN = N::NIN;
  constexpr int R = T::R;
  constexpr uint32_t CHR = T::CHR;
  constexpr int S0 = T::S0;
  constexpr int TPR = T::TPR;
  constexpr int WH = W / TPR, KH = K / TPR, LH = L / TPR;   // per chain thread: its share of columns / lobes / levels
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sb = tc::smem_u32(smem);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + T::OFF_BAR);
  uint64_t* bar_w = bars + 0;
  uint64_t* bar_mma = bars + 1;
  uint64_t* bar_dzf = bars + 2;
  uint64_t* bar_dze = bars + 3;
  uint64_t* bar_hs = bars + 4 + 2 * S0;
  uint64_t* bar_mma2 = bars + 5 + 2 * S0;
  uint64_t* bar_x0f = bars + 4;
  uint64_t* bar_x0e = bars + 4 + S0;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + T::OFF_TSLOT);
  if (tid == 0) {
    tc::mbar_init(bar_w, 1);
    tc::mbar_init(bar_mma, 1);
    tc::mbar_init(bar_mma2, 1);   // the dW^T issuer (thread 128)
    tc::mbar_init(bar_dzf, T::CHAIN_THREADS);
    tc::mbar_init(bar_dze, T::SCATTER_THREADS);
    tc::mbar_init(bar_hs, 1);
    for (int s = 0; s < S0; ++s) {
      tc::mbar_init(bar_x0f + s, T::GATHER_THREADS);
      tc::mbar_init(bar_x0e + s, 1);
    }
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc(tslot, (uint32_t)T::TCOLS);
  // constant "ones" chunks (bias rows of dW^T): X0 stages at NIN, X_k at W
  if (tid < R) {
    const float e1[8] = {1.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f}, e0[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int s = 0; s < S0; ++s) {
      const uint32_t xh = sb + T::OFF_X0 + (uint32_t)s * T::X0_BYTES, xl = xh + (T::ZF / 8) * CHR;
      // (product: NIN = 65 shares chunk 8 with the roughness -- the memory warps
      // write that chunk every tile; only the zero chunk 9 is constant)
      constexpr int F0 = N::PRODUCT ? (NIN + 7) / 8 * 8 : NIN;
#pragma unroll
      for (int f = F0; f < T::ZF; f += 8) tc::store_chunk(xh, xl, R, tid, f / 8, f == NIN ? e1 : e0);
    }
#pragma unroll
    for (int k = 1; k < NL; ++k) {
      const uint32_t xh = sb + T::xhoff(k), xl = xh + (T::HF / 8) * CHR;
      tc::store_chunk(xh, xl, R, tid, W / 8, e1);
    }
  }
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  // the whole TMEM: base column 0, lane 0 (checked); keeps MMA operands uniform
  static_assert(T::TCOLS == 512, "constant TMEM base needs the full allocation");
  constexpr uint32_t tbase = 0;
  if (*tslot != 0u) __trap();
  if (tid == 0) {   // weight image: one TMA bulk copy
    mbar_expect_tx(bar_w, T::WIMG);
    bulk_g2s(smem, a.wimg, T::WIMG, bar_w);
  }
  const int64_t n = a.n;
  const int64_t ntiles = (n + R - 1) / R;
  const int64_t tstride = gridDim.x;
  const float4* tab = reinterpret_cast<const float4*>(a.params + N::N_MLP);

  if (warp < 4 * TPR) {
    // =========================== CHAIN =====================================
    // thread (h, r): row r = 32 (warp % 4) + lane (= TMEM lane), part h = warp / 4
    // of the columns (epilogues), lobes (head) and levels (dz).  The TPR
    // threads of a row are warps w % 4 + 4 h: they exchange through smem
    // behind a named barrier of those 4 warps (2 + w % 4).
    const int h = warp >> 2;
    const int r = ((warp & 3) << 5) | lane;
    const uint32_t lad = (uint32_t)((warp & 3) * 32) << 16;   // this warp's TMEM lane field
    // zero the dW^T accumulators (all later MMAs accumulate); halves by column
    for (int col = 16 * h; col < N::osum(NL) + T::XD; col += 16 * TPR) tc::tmem_zero16(tbase + lad + (uint32_t)(128 + col));
    tc::tmem_wait_st();
    mbar_wait_t(bar_w, 0);
    const float* bias = reinterpret_cast<const float*>(smem + TB::WBYTES);
    static_assert(TPR == 2, "the head exchange uses row-data slots of two threads");
    // C-A34 selection head (AH): its parameters in smem
    constexpr bool ahead = AH;
    float* ah_s = reinterpret_cast<float*>(smem + T::OFF_AH);
    if (ahead) {
      for (int j = tid; j < W + 1; j += T::CHAIN_THREADS) ah_s[j] = __ldg(a.alpha_w + j);
      tc::named_sync(1u, (uint32_t)T::CHAIN_THREADS);
    }
    const uint32_t wsb = sb;   // weight image at smem offset 0
    uint32_t phase = 0;
    uint32_t phase2 = 0;   // bar_mma2 (the dW^T batches)
    double loss = 0.0;
    unsigned c_used = 0, c_zero = 0, c_drop = 0;
    auto handoff = [&]() {
      tc::fence_proxy_async();
      tc::fence_before_sync();
      tc::named_sync(1u, (uint32_t)T::CHAIN_THREADS);
    };
    auto psync = [&]() { tc::named_sync(2u + (uint32_t)(warp & 3), 32u * TPR); };
    auto wait_mma = [&]() {
      tc::mbar_wait(bar_mma, phase);   // (a suspend hint here: +2 % on B200 c2)
      phase ^= 1u;
      tc::fence_after_sync();
    };
    // previous tile's dz -> dz stage (run while the next tile's first MMA
    // executes); the memory warps keep the rows' positions in registers
    auto dz_epilogue = [&](int kk) {
      float v[NG / TPR];
      tc::tmem_ldn<NG / TPR>(tbase + lad + (uint32_t)(T::C_DZ + h * (NG / TPR)), v);
      tc::tmem_wait_ld();
      mbar_wait_t(bar_dze, (uint32_t)((kk & 1) ^ 1));
      float4* dz = reinterpret_cast<float4*>(smem + T::OFF_DZ);
#pragma unroll
      for (int l = 0; l < LH; ++l)
        dz[(h * LH + l) * R + r] = make_float4(v[4 * l], v[4 * l + 1], v[4 * l + 2], v[4 * l + 3]);
      mbar_arrive(bar_dzf);
    };
    const bool stamp = (a.debug & 4) && blockIdx.x == 0 && tid == 0;
    int kt = 0;
#define NPM_WS_STAMP(idx) \
  do { if (stamp && kt < 64) a.dbg_clock[kt * 16 + (idx)] = clock64(); } while (0)
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += tstride, ++kt) {
      const int s = kt % S0;
      const uint32_t ph0 = (uint32_t)((kt / S0) & 1);
      const uint32_t x0h = sb + T::OFF_X0 + (uint32_t)s * T::X0_BYTES, x0l = x0h + (T::ZF / 8) * CHR;
      NPM_WS_STAMP(0);
      mbar_wait_t(bar_x0f + s, ph0);
      NPM_WS_STAMP(1);
      tc::fence_after_sync();
      if (tid == 0) {
        issue_fwd_r<R>(tbase + T::C_ACC, x0h, x0l, wsb + TB::woff(0), wsb + TB::woff(0) + TB::wbytes(0),
                       TB::in_p(0), TB::out(0));
        tc::mma_commit(bar_mma);
      }
      // this row's head inputs are read from the row-data stage at the head
      // (the stage is refilled only after bwd_0 completes): no registers held
      // across the forward epilogues (they spilled there)
      float* rd = reinterpret_cast<float*>(smem + T::OFF_RD + (uint32_t)s * T::RD_BYTES);
      if (kt > 0) dz_epilogue(kt - 1);
      NPM_WS_STAMP(2);
      // ---- forward
#pragma unroll
      for (int k = 0; k < NL; ++k) {
        if (k > 0) {
          handoff();
          if (tid == 0) {
            tc::fence_after_sync();
            const uint32_t xh = sb + T::xhoff(k), xl = xh + (T::HF / 8) * CHR;
            const uint32_t w = wsb + TB::woff(k);
            issue_fwd_r<R>(tbase + T::C_ACC, xh, xl, w, w + TB::wbytes(k), TB::in_p(k), TB::out(k));
            tc::mma_commit(bar_mma);
          }
        }
        wait_mma();
        NPM_WS_STAMP(3 + 2 * k);
        const float* b = bias + TB::boff(k) / 4;
        if (k < NL - 1) {
          const uint32_t xh = sb + T::xhoff(k + 1), xl = xh + (T::HF / 8) * CHR;
          float zpart = 0.0f;   // C-A34: this thread's part of a . h_{L-1}
#pragma unroll
          for (int c16 = 0; c16 < WH; c16 += 16) {   // 16 columns at a time (register pressure)
            float v[16];
            tc::tmem_ldn<16>(tbase + lad + (uint32_t)(T::C_ACC + h * WH + c16), v);
            tc::tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              v[j] = fmaxf(v[j] + b[h * WH + c16 + j], 0.0f);
              if (k == NL - 2 && ahead) zpart = fmaf(ah_s[h * WH + c16 + j], v[j], zpart);
            }
            tc::store_chunk(xh, xl, R, r, h * (WH / 8) + c16 / 8, v);
            tc::store_chunk(xh, xl, R, r, h * (WH / 8) + c16 / 8 + 1, v + 8);
          }
          if (k == NL - 2 && ahead) rd[(h == 0 ? 2 : 12) * R + r] = zpart;   // read after the head's first exchange
        } else {
          if (tid == 0) mbar_arrive(bar_hs);   // the memory warps may scatter now
          // ---- Eq. 9 head (C-O12, C-O13): row r, lobes [h K/2, (h+1) K/2)
          float lp[KH], kp[KH], tp[KH], pp[KH];
          tc::tmem_ldn<KH>(tbase + lad + (uint32_t)(T::C_ACC + h * KH), lp);
          tc::tmem_ldn<KH>(tbase + lad + (uint32_t)(T::C_ACC + K + h * KH), kp);
          tc::tmem_ldn<KH>(tbase + lad + (uint32_t)(T::C_ACC + 2 * K + h * KH), tp);
          tc::tmem_ldn<KH>(tbase + lad + (uint32_t)(T::C_ACC + 3 * K + h * KH), pp);
          tc::tmem_wait_ld();
          NPM_WS_STAMP(10);
#pragma unroll
          for (int m = 0; m < KH; ++m) {
            lp[m] += b[h * KH + m];
            kp[m] += b[K + h * KH + m];
            tp[m] += b[2 * K + h * KH + m];
            pp[m] += b[3 * K + h * KH + m];
          }
          const bool hvalid = rd[3 * R + r] != 0.0f;
          const float h_wx = rd[4 * R + r], h_wy = rd[5 * R + r], h_wz = rd[6 * R + r];
          float t = rd[7 * R + r];
          bool all_zero = t == 0.0f;
          if (a.channels == 3) {
            const float h_t1 = rd[8 * R + r], h_t2 = rd[9 * R + r];
            all_zero = all_zero && h_t1 == 0.0f && h_t2 == 0.0f;
            t = 0.2126f * t + 0.7152f * h_t1 + 0.0722f * h_t2;
          }
          const float p = rd[10 * R + r];
          const float ratio = t / p;
          const bool drop = hvalid && (!isfinite(ratio) || !isfinite(p) || !(p > 0.0f));
          const bool zero = hvalid && !drop && all_zero;
          const bool use = hvalid && !drop && !zero;
          const float s_ = use ? (float)(-(double)ratio * a.inv_n_global) : 0.0f;
          const float wx = h_wx, wy = h_wy, wz = h_wz;
          float kap[KH], mx[KH], my[KH], mz[KH], th[KH], ph[KH], vv[KH], sth[KH], cth[KH], sph[KH], cph[KH],
              emk[KH];
          float mloc = lp[0];
#pragma unroll
          for (int m = 0; m < KH; ++m) {
            mloc = fmaxf(mloc, lp[m]);
            kap[m] = __expf(fminf(fmaxf(kp[m], a.log_kmin), a.log_kmax));
            lobe_angles<false>(tp[m], pp[m], kap[m], th[m], ph[m], sth[m], cth[m], sph[m], cph[m]);
            mx[m] = sth[m] * cph[m]; my[m] = sth[m] * sph[m]; mz[m] = cth[m];
            const float nrm = lobe_norm_fast(kap[m], emk[m]);
            vv[m] = lobe_eval(nrm, kap[m], mx[m], my[m], mz[m], wx, wy, wz);
          }
          // softmax normaliser / mixture sum across the row's two threads in ONE
          // exchange: each part's sums relative to its own maximum m_h, rescaled
          // by e^{m_h - M} after the barrier (M = max(m_0, m_1))
          NPM_WS_STAMP(12);
          float e[KH], S = 0.0f, P = 0.0f;
#pragma unroll
          for (int m = 0; m < KH; ++m) {
            e[m] = __expf(lp[m] - mloc);
            S += e[m];
            P += e[m] * vv[m];
          }
          rd[h * R + r] = mloc;
          rd[(4 + 2 * h) * R + r] = S;
          rd[(5 + 2 * h) * R + r] = P;
          float* vx = reinterpret_cast<float*>(smem + T::OFF_VX);
          if constexpr (VA) {   // this part's lobes for the pairwise terms (read after the barrier)
#pragma unroll
            for (int m = 0; m < KH; ++m) {
              const int j = h * KH + m;
              vx[(5 * j) * R + r] = kap[m];
              vx[(5 * j + 1) * R + r] = mx[m];
              vx[(5 * j + 2) * R + r] = my[m];
              vx[(5 * j + 3) * R + r] = mz[m];
              vx[(5 * j + 4) * R + r] = e[m];   // relative to m_h (rescaled by the reader)
            }
          }
          psync();
          NPM_WS_STAMP(14);
          const float m0 = rd[r], m1 = rd[R + r], Mx = fmaxf(m0, m1);
          const float c0 = __expf(m0 - Mx), c1 = __expf(m1 - Mx);
          // the same association order on every thread of the row: parts 0, 1
          const float St = rd[4 * R + r] * c0 + rd[6 * R + r] * c1, Pt = rd[5 * R + r] * c0 + rd[7 * R + r] * c1;
          {
            const float ch = h ? c1 : c0;
#pragma unroll
            for (int m = 0; m < KH; ++m) e[m] *= ch;   // now e^{l - M}
          }
          const float invS = 1.0f / St;
          const float Vb = fmaxf(Pt * invS, kVFloor);
          const float invV = 1.0f / Vb;
          // f-4 (C-A31): chi^2 scales Eq. 9's record weight by D^ / V
          const float chi = a.divergence == 1 ? (use ? t * invV : 0.0f) : 1.0f;
          // f-4 (C-A35): the variance-aware target weighs -2 log V by a = D^^2 / p~
          const float a_n = use ? ratio * t : 0.0f;
          const float sd = VA ? (use ? (float)(-2.0 * (double)a_n * a.inv_n_global) : 0.0f) : s_ * chi;
          const float wzn = VA && use ? (float)((double)a_n * a.inv_n_global) : 0.0f;
          // d log Z / d (lambda', kappa', theta', phi') of this part's lobes, Z = int V^2
          float zl[KH], zk[KH], zt[KH], zp[KH];
          float logZ = 0.0f;
          if constexpr (VA) {
            // pairwise closed form (C-A35): I_ij = C_i C_j / C(r_ij) e^{r_ij - k_i - k_j}
            // = C_i C_j 2 pi (1 - e^{-2r}) / r e^{r - k_i - k_j} with
            // r - k_i - k_j = -k_i k_j |mu_i - mu_j|^2 / (r + k_i + k_j) (no cancellation);
            // Langevin(r) / r from the same 1 - e^{-2r} (series below r = 1/2)
            auto cnorm = [](float k) {   // C(k) 2 pi = k / (1 - e^{-2k}), -> 1/2 at 0
              const float kk = fmaxf(k, 1e-30f);
              return __fdividef(kk, one_minus_exp_neg(2.0f * kk));
            };
            auto lox_from = [](float x, float om, float inv_x) {   // (coth x - 1/x) / x, om = 1 - e^{-2x}
              const float x2 = x * x;
              const float ser = 0.33333334f - x2 * (0.022222223f - x2 * (0.0021164022f - x2 * 0.00021164022f));
              return x < 0.5f ? ser : (__fdividef(2.0f, om) - 1.0f - inv_x) * inv_x;
            };
            float A[KH], Bk[KH], Bx[KH], By[KH], Bz[KH], Ck[KH];
#pragma unroll
            for (int m = 0; m < KH; ++m) {
              A[m] = Bk[m] = Bx[m] = By[m] = Bz[m] = 0.0f;
              Ck[m] = cnorm(kap[m]) * 0.15915494f;   // C(k_i) 2 pi * C(k_j) 2 pi / (2 pi)
            }
            // the other part's 4 lobes against this thread's 4 (16 pairs), then the
            // own part's 10 unordered pairs once each (I_ij = I_ji: the pair core is
            // symmetric, only the e-weights and the accumulators differ; B200 c2
            // 833 -> 766 us against all 32 ordered pairs per thread)
            // the pair core, symmetric in (i, j): S = C_i C_j / (2 pi) 2 pi (1 - e^{-2r}) / r e^{r - k_i - k_j}
            auto pair_core = [&](float ki, float ix, float iy, float iz, float kj, float jx, float jy, float jz,
                                 float cij, float& S, float& lx, float& d2) {
              const float dx = ix - jx, dy = iy - jy, dz = iz - jz;
              d2 = dx * dx + dy * dy + dz * dz;
              const float sk = ki + kj, pk = ki * kj;
              const float rr = fmaxf(sqrtf(fmaxf(sk * sk - pk * d2, 0.0f)), 1e-30f);
              const float ex = -__fdividef(pk * d2, rr + sk);
              const float om = one_minus_exp_neg(2.0f * rr);
              const float inv_r = __fdividef(1.0f, rr);
              S = cij * om * inv_r * __expf(ex);
              lx = lox_from(rr, om, inv_r);
            };
            float cn[KH];
#pragma unroll
            for (int m = 0; m < KH; ++m) cn[m] = cnorm(kap[m]);
#pragma unroll 2
            for (int jj = 0; jj < KH; ++jj) {
              const int j = (1 - h) * KH + jj;
              const float kj = vx[(5 * j) * R + r], jx = vx[(5 * j + 1) * R + r], jy = vx[(5 * j + 2) * R + r],
                          jz = vx[(5 * j + 3) * R + r], ej = vx[(5 * j + 4) * R + r] * (h ? c0 : c1);
              const float Cj = ej * cnorm(kj);
#pragma unroll
              for (int m = 0; m < KH; ++m) {
                float S, lx, d2;
                pair_core(kap[m], mx[m], my[m], mz[m], kj, jx, jy, jz, Ck[m] * Cj, S, lx, d2);
                A[m] += S;
                const float q = S * lx;
                Bk[m] += q * (kap[m] + kj * (1.0f - 0.5f * d2));
                Bx[m] += q * kj * jx; By[m] += q * kj * jy; Bz[m] += q * kj * jz;
              }
            }
#pragma unroll
            for (int m = 0; m < KH; ++m) {
#pragma unroll
              for (int m2 = m; m2 < KH; ++m2) {
                float S, lx, d2;
                pair_core(kap[m], mx[m], my[m], mz[m], kap[m2], mx[m2], my[m2], mz[m2], Ck[m] * cn[m2], S, lx, d2);
                const float sl = S * lx;
                A[m] += e[m2] * S;
                const float q = e[m2] * sl;
                Bk[m] += q * (kap[m] + kap[m2] * (1.0f - 0.5f * d2));
                Bx[m] += q * kap[m2] * mx[m2]; By[m] += q * kap[m2] * my[m2]; Bz[m] += q * kap[m2] * mz[m2];
                if (m2 != m) {
                  A[m2] += e[m] * S;
                  const float q2 = e[m] * sl;
                  Bk[m2] += q2 * (kap[m2] + kap[m] * (1.0f - 0.5f * d2));
                  Bx[m2] += q2 * kap[m] * mx[m]; By[m2] += q2 * kap[m] * my[m]; Bz[m2] += q2 * kap[m] * mz[m];
                }
              }
            }
            float Zh = 0.0f;
#pragma unroll
            for (int m = 0; m < KH; ++m) Zh += e[m] * A[m];
            rd[(2 + h) * R + r] = Zh;   // rows 2 / 3 (unused in this mode / the validity flag, read before the barrier)
            psync();
            const float Zs = 0.0f + rd[2 * R + r] + rd[3 * R + r];   // sum_ij e_i e_j I_ij = Z S^2
            const float invZs = 1.0f / Zs;
            logZ = __logf(Zs * invS * invS);
#pragma unroll
            for (int m = 0; m < KH; ++m) {
              const float gi = e[m] * A[m] * invZs;            // sum_j G_ij
              const float lam = e[m] * invS;
              const float f = 2.0f * e[m] * invZs;
              zl[m] = 2.0f * (gi - lam);
              const float omk = one_minus_exp_neg(2.0f * kap[m]), ik = __fdividef(1.0f, kap[m]);
              const float dkz = -2.0f * kap[m] * lox_from(kap[m], omk, ik) * gi + f * Bk[m];
              zk[m] = (kp[m] < a.log_kmin || kp[m] > a.log_kmax) ? 0.0f : kap[m] * dkz;
              const float gx = f * kap[m] * Bx[m], gy = f * kap[m] * By[m], gz = f * kap[m] * Bz[m];
              zt[m] = kPi * (cth[m] * cph[m] * gx + cth[m] * sph[m] * gy - sth[m] * gz) * th[m] * (1.0f - th[m]);
              zp[m] = kTwoPi * (-sth[m] * sph[m] * gx + sth[m] * cph[m] * gy) * ph[m] * (1.0f - ph[m]);
            }
          }
          float dl[KH], dk[KH], dt[KH], dp[KH];
#pragma unroll
          for (int m = 0; m < KH; ++m) {
            const float lam = e[m] * invS;
            const float gam = lam * vv[m] * invV;
            dl[m] = sd * (gam - lam);
            if constexpr (VA) dl[m] += wzn * zl[m];
            const float dx = mx[m] - wx, dy = my[m] - wy, dz = mz[m] - wz;
            const float d2 = dx * dx + dy * dy + dz * dz;
            // 2 kappa e^{-2 kappa} / (1 - e^{-2 kappa}) with em = 1 - e^{-2 kappa}
            const float dkk = sd * gam * (1.0f - kap[m] * 0.5f * d2 - __fdividef(2.0f * kap[m] * (1.0f - emk[m]), emk[m]));
            dk[m] = (kp[m] < a.log_kmin || kp[m] > a.log_kmax) ? 0.0f : dkk;   // C-A8
            if constexpr (VA) dk[m] += wzn * zk[m];
            const float wdth = kPi * (cth[m] * cph[m] * wx + cth[m] * sph[m] * wy - sth[m] * wz);
            const float wdph = kTwoPi * (-sth[m] * sph[m] * wx + sth[m] * cph[m] * wy);
            const float sgk = sd * gam * kap[m];
            dt[m] = sgk * wdth * th[m] * (1.0f - th[m]);
            dp[m] = sgk * wdph * ph[m] * (1.0f - ph[m]);
            if constexpr (VA) { dt[m] += wzn * zt[m]; dp[m] += wzn * zp[m]; }
          }
          const uint32_t dh = sb + T::OFF_D, dlo = dh + (T::dfeat(NL - 1) / 8) * CHR;
          tc::store_feats<KH>(dh, dlo, R, r, h * KH, dl);
          tc::store_feats<KH>(dh, dlo, R, r, K + h * KH, dk);
          tc::store_feats<KH>(dh, dlo, R, r, 2 * K + h * KH, dt);
          tc::store_feats<KH>(dh, dlo, R, r, 3 * K + h * KH, dp);
          if (ahead) {
            // ---- C-A34: second-moment gradient of the selection head.  Logit
            // z = c + a . h_{L-1} (parts of both threads, the same order on each);
            // dM2/dz = -(1/N) D^2 (p_b - V) alpha (1 - alpha) / (p~_alpha^2 p~_s)
            float z = ah_s[W];
            z += rd[2 * R + r];
            z += rd[12 * R + r];
            const float al = 1.0f / (1.0f + __expf(-z));
            const float pb = rd[11 * R + r];
            const float Vm = Pt * invS;                  // V(w_i), not floored (C-A34)
            const float pa = al * pb + (1.0f - al) * Vm;
            const bool aok = use && isfinite(pb) && pb >= 0.0f && pa > 0.0f;
            const float q1 = aok ? t / pa : 0.0f;
            const float gz = aok ? (float)(-(double)(q1 * q1 * (pb - Vm) * al * (1.0f - al) / p) * a.inv_n_global)
                                 : 0.0f;
            // dM2/d(a, c) = sum_rows gz (h_{L-1}, 1): gz goes to delta_{NL-1}'s
            // column NOUT (the rest of the XD extra columns zero), so the dW_{NL-1}
            // MMA (X_{NL-1}^T delta, ones chunk included) accumulates it in TMEM
            if (h == 0) {
              float gzc[8] = {gz, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
              tc::store_chunk(dh, dlo, R, r, NOUT / 8, gzc);
            }
          }
          if (h == 0) {
            c_drop += drop; c_zero += zero;
            if (use) {
              if constexpr (VA) loss += (double)wzn * (-2.0 * (double)logf(Vb) + (double)logZ);
              else loss += a.divergence ? -(double)sd : (double)s_ * (double)logf(Vb);   // chi^2: (D^/p~)(D^/V)/N
              c_used += 1;
            }
          }
        }
        NPM_WS_STAMP(4 + 2 * k);
      }
      // ---- backward: k = NL-1 .. 0; delta_k in D (k = NL-1) or over X_{k+1}
#pragma unroll
      for (int k = NL - 1; k >= 0; --k) {
        handoff();
        // dX by thread 0, dW^T by thread 128 (two issuers, two commits; B200 c2:
        // one issuer 514 us, this split 497 us; dW^T further split by output
        // column halves over a third issuer re-reads X^T: 540 us)
        if (tid == 0 || tid == 128) {
          tc::fence_after_sync();
          with_k<NL>(k, [&](auto KC) {
            constexpr int kk = decltype(KC)::value;
            const uint32_t dh = sb + T::dboff(kk), dl = dh + (T::dfeat(kk) / 8) * CHR;
            const uint32_t w = wsb + TB::woff(kk);
            const uint32_t xh = kk == 0 ? x0h : sb + T::xhoff(kk);
            const uint32_t xl = kk == 0 ? x0l : xh + (T::HF / 8) * CHR;
            if (tid == 0) {
              issue_dx_r<R>(tbase + (kk == 0 ? T::C_DZ : T::C_ACC), dh, dl, w, w + TB::wbytes(kk), TB::out(kk),
                            kk > 0 ? W : NG);
              tc::mma_commit(bar_mma);
            } else {
              issue_dw_m<R, T::dwm(kk)>(tbase + (uint32_t)T::dwcol(kk), xh, xl, dh, dl,
                                        TB::out(kk) + (kk == NL - 1 ? T::XD : 0));
              tc::mma_commit(bar_mma2);
              if (kk == 0) tc::mma_commit(bar_x0e + s);   // X0 stage free once dW_0 has read it
            }
          });
        }
        wait_mma();
        mbar_wait_t(bar_mma2, phase2);
        phase2 ^= 1u;
        tc::fence_after_sync();

        NPM_WS_STAMP(3 + 2 * NL + 2 * (NL - 1 - k));
        if (k > 0) {
          // delta_{k-1} = dX_k * ReLU'(X_k) -> over X_k (read by dW_k, complete)
          const uint32_t dh = sb + T::dboff(k - 1), dl = dh + (T::dfeat(k - 1) / 8) * CHR;
#pragma unroll
          for (int c16 = 0; c16 < WH; c16 += 16) {
            float v[16];
            tc::tmem_ldn<16>(tbase + lad + (uint32_t)(T::C_ACC + h * WH + c16), v);
            // ReLU'(X_k) from the stored X_k = hi + lo (>= 0): > 0 iff a half
            // is non-zero; read before this thread overwrites its own slots.
            // (Keeping the masks in registers from the forward epilogue made the
            // chain spill: B200 c2 575 -> 547 us.)
            uint4 xhi[2], xlo[2];
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const uint32_t off = (uint32_t)((h * (WH / 8) + c16 / 8 + q) * CHR + r * 16);
              asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(xhi[q].x), "=r"(xhi[q].y), "=r"(xhi[q].z),
                           "=r"(xhi[q].w) : "r"(sb + T::xhoff(k) + off));
              asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(xlo[q].x), "=r"(xlo[q].y), "=r"(xlo[q].z),
                           "=r"(xlo[q].w) : "r"(sb + T::xhoff(k) + (T::HF / 8) * CHR + off));
            }
            tc::tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const uint4& hh = xhi[j / 8];
              const uint4& ll = xlo[j / 8];
              const uint32_t wh = (&hh.x)[(j % 8) / 2], wl = (&ll.x)[(j % 8) / 2];
              const uint32_t sh = (j & 1) ? 16u : 0u;
              const bool pos = (((wh | wl) >> sh) & 0xFFFFu) != 0u;
              v[j] = pos ? v[j] : 0.0f;
            }
            tc::store_chunk(dh, dl, R, r, h * (WH / 8) + c16 / 8, v);
            tc::store_chunk(dh, dl, R, r, h * (WH / 8) + c16 / 8 + 1, v + 8);
          }
        }
      }
      NPM_WS_STAMP(15);
    }
#undef NPM_WS_STAMP
    if (kt > 0) dz_epilogue(kt - 1);
    // ---- flush dW^T / db: lane = input feature (M = 128) or 32 (f/16) + f%16
    // (M = 64); the two threads of a lane split the output columns
#pragma unroll
    for (int k = 0; k < NL; ++k) {
      constexpr int MAXO = (NOUT > W ? NOUT : W) / TPR;
      float vv[MAXO];
      const int out = TB::out(k), in = TB::in(k), oh = out / TPR;
      if (out == NOUT) tc::tmem_ldn<NOUT / TPR>(tbase + lad + (uint32_t)(T::dwcol(k) + h * (NOUT / TPR)), vv);
      else tc::tmem_ldn<W / TPR>(tbase + lad + (uint32_t)(T::dwcol(k) + h * (W / TPR)), vv);
      tc::tmem_wait_ld();
      int f = r;
      bool ok = true;
      with_k<NL>(k, [&](auto KC) {
        if (T::dwm(decltype(KC)::value) == 64) {
          f = 16 * (warp & 3) + (lane & 15);
          ok = lane < 16;
        }
      });
      if (ok && f < in) {
        float* gp = a.grads + N::gw_off(k) + f;
        for (int o = 0; o < oh; ++o) atomicAdd(gp + (h * oh + o) * in, vv[o]);
      } else if (ok && f == in) {
        float* gp = a.grads + N::gb_off(k) + h * oh;
        for (int o = 0; o < oh; ++o) atomicAdd(gp + o, vv[o]);
      }
    }
    if constexpr (AH) {   // C-A34: the head's gradient, column NOUT of dW^T_{NL-1} -> GRADS
      float gv[1];
      tc::tmem_ldn<1>(tbase + lad + (uint32_t)(T::dwcol(NL - 1) + NOUT), gv);
      tc::tmem_wait_ld();
      int f = r;
      bool ok = h == 0;
      if (T::dwm(NL - 1) == 64) {
        f = 16 * (warp & 3) + (lane & 15);
        ok = ok && lane < 16;
      }
      if (ok && f <= W) atomicAdd(a.alpha_g + f, gv[0]);   // f = W: the ones row, dM2/dc
    }
    loss = warp_sum_d(loss);
    c_used = warp_sum_u(c_used); c_zero = warp_sum_u(c_zero); c_drop = warp_sum_u(c_drop);
    if (lane == 0 && h == 0) {
      atomicAdd(a.stats, loss);
      atomicAdd(a.counters + 0, (unsigned long long)c_used);
      atomicAdd(a.counters + 1, (unsigned long long)c_zero);
      atomicAdd(a.counters + 2, (unsigned long long)c_drop);
    }
  } else {
    // =========================== MEMORY ====================================
    // thread (part, row): row = m % 128, part = m / 128 owns levels
    // [part L/2, (part+1) L/2).  Iteration k gathers tile k into X0 stage
    // k % S0, then scatters tile k - 1 from the dz stage: the chain computes
    // tile k while this role scatters k - 1, and tile k + 1's gathers follow.
    const int m = tid - T::CHAIN_THREADS;
    const int row = m & (R - 1), part = m >> 7;
    constexpr int LP = L / 2;
    float4* gtab = reinterpret_cast<float4*>(a.grads + N::N_MLP);
    const int kt_end = blockIdx.x < ntiles ? (int)((ntiles - blockIdx.x + tstride - 1) / tstride) : 0;
    // memory-role clock stamps: measurement builds only (-DNPM_WS_MEMSTAMPS;
    // the runtime check alone cost the production kernel ~3 %)
#ifdef NPM_WS_MEMSTAMPS
    const bool mstamp = (a.debug & 4) && blockIdx.x == 0 && m == 0;
#define NPM_WS_MSTAMP(kk, idx) \
  do { if (mstamp && (kk) < 64) a.dbg_clock[64 * 16 + (kk) * 16 + (idx)] = clock64(); } while (0)
#else
#define NPM_WS_MSTAMP(kk, idx) do { } while (0)
#endif
    float sux = 0.f, suy = 0.f, suz = 0.f;   // the row's position in the tile to scatter
    bool svalid = false;
    auto scatter = [&](int kd) {
      mbar_wait_idle(bar_dzf, (uint32_t)(kd & 1));
      NPM_WS_MSTAMP(kd + 1, 4);
      // the scatter's reductions contend with the chain's epilogue smem stores
      // for the LSU: start them once the chain reaches tile kd + 1's head
      // (ALU / MUFU work; B200 c2: 610 -> 575 us; starting at the first
      // backward MMA instead: 606 us); the last tile has no successor head
      if (kd + 1 < kt_end) mbar_wait_idle(bar_hs, (uint32_t)((kd + 1) & 1));
      NPM_WS_MSTAMP(kd + 1, 5);
      const float4* dz = reinterpret_cast<const float4*>(smem + T::OFF_DZ);
      const float ux = sux, uy = suy, uz = suz;
      const bool valid = svalid;
      float4 d[LP];
#pragma unroll
      for (int l = 0; l < LP; ++l) d[l] = dz[(part * LP + l) * R + row];
      mbar_arrive(bar_dze);
      if (!valid || (a.debug & 1)) return;
#pragma unroll
      for (int j = 0; j < LP; ++j) {
        const float4 gq = d[j];
        if (gq.x == 0.0f && gq.y == 0.0f && gq.z == 0.0f && gq.w == 0.0f) continue;
        const int l = part * LP + j;
        LevelCorners lc;
        level_corners(a.grid, l, ux, uy, uz, lc);
        float4* tg = ((a.priv_mask >> l) & 1u) ? a.priv + (int64_t)blockIdx.x * a.priv_stride + a.priv_off[l]
                                                 : gtab + a.grid.off[l];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const float w = lc.w[c];
          atomicAdd(tg + lc.idx[c], make_float4(w * gq.x, w * gq.y, w * gq.z, w * gq.w));
        }
      }
      NPM_WS_MSTAMP(kd + 1, 6);
    };
    int kt = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += tstride, ++kt) {
      const int s = kt % S0;
      const uint32_t ph0 = (uint32_t)((kt / S0) & 1);
      NPM_WS_MSTAMP(kt, 0);
      const int64_t slot = tile * R + row;
      const bool valid = slot < n;
      const int64_t i = valid ? (a.perm ? (int64_t)__ldg(a.perm + slot) : slot) : 0;
      float ux = 0.f, uy = 0.f, uz = 0.f;
      if (valid) {
        ux = normalize_axis(__ldg(a.px + i), a.grid.lo[0], a.grid.inv[0]);
        uy = normalize_axis(__ldg(a.py + i), a.grid.lo[1], a.grid.inv[1]);
        uz = normalize_axis(__ldg(a.pz + i), a.grid.lo[2], a.grid.inv[2]);
      }
      float hin[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 1.f, 0.f};
      if (part == 0 && valid) {
        hin[0] = __ldg(a.wx + i); hin[1] = __ldg(a.wy + i); hin[2] = __ldg(a.wz + i);
        hin[3] = __ldg(a.target + i);
        if (a.channels == 3) {
          hin[4] = __ldg(a.target + a.target_stride + i);
          hin[5] = __ldg(a.target + 2 * a.target_stride + i);
        }
        hin[6] = __ldg(a.spdf + i);
        if (AH) hin[7] = __ldg(a.bsdf_pdf + i);   // C-A34
      }
      // product conditioning (X0 features 32-64): part 0 w_o, part 1 n + roughness
      float cv[4] = {0.f, 0.f, 1.f, 0.f};
      if constexpr (N::PRODUCT) {
        if (valid) {
          if (part == 0) { cv[0] = __ldg(a.wox + i); cv[1] = __ldg(a.woy + i); cv[2] = __ldg(a.woz + i); }
          else { cv[0] = __ldg(a.nx + i); cv[1] = __ldg(a.ny + i); cv[2] = __ldg(a.nz + i); cv[3] = __ldg(a.rough + i); }
        }
      }
      const uint32_t xh = sb + T::OFF_X0 + (uint32_t)s * T::X0_BYTES, xl = xh + (T::ZF / 8) * CHR;
      // all of this thread's levels in registers, then wait for the stage
      float gf[4 * LP];
      // branch-free over the levels (an invalid row gathers at u = 0 and is
      // zeroed) so one level's loads can overlap the previous blend (B200 c2
      // train 523 -> 517 us)
#pragma unroll
      for (int q = 0; q < LP; ++q) {
        const int l = part * LP + q;
        LevelCorners lc;
        level_corners(a.grid, l, ux, uy, uz, lc);
        float4 gl = gather_level<NPM_WS_PAIRS>(tab, a.grid.off[l], lc);
#ifdef NPM_WS_MEMSTAMPS
        if (a.debug & 2) gl = make_float4(0.f, 0.f, 0.f, 0.f);   // NPM_DEBUG bit 1 (measurement builds)
#endif
        gf[4 * q] = valid ? gl.x : 0.0f; gf[4 * q + 1] = valid ? gl.y : 0.0f;
        gf[4 * q + 2] = valid ? gl.z : 0.0f; gf[4 * q + 3] = valid ? gl.w : 0.0f;
      }
      NPM_WS_MSTAMP(kt, 1);
      mbar_wait_idle(bar_x0e + s, ph0 ^ 1u);
      NPM_WS_MSTAMP(kt, 2);
#pragma unroll
      for (int j = 0; j < LP / 2; ++j) tc::store_chunk(xh, xl, R, row, part * (LP / 2) + j, gf + 8 * j);
      if constexpr (N::PRODUCT) {   // [32, 48) SH4(w_o) by part 0; [48, 64) SH4(n), [64, 72) roughness + ones by part 1
        float e16[16];
        if (valid) sh4(cv[0], cv[1], cv[2], e16);
        else {
#pragma unroll
          for (int j = 0; j < 16; ++j) e16[j] = 0.0f;
        }
        tc::store_chunk(xh, xl, R, row, 4 + 2 * part, e16);
        tc::store_chunk(xh, xl, R, row, 5 + 2 * part, e16 + 8);
        if (part == 1) {
          const float ro[8] = {valid ? cv[3] : 0.0f, 1.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
          tc::store_chunk(xh, xl, R, row, 8, ro);
        }
      }
      if (part == 0) {
        float* rd = reinterpret_cast<float*>(smem + T::OFF_RD + (uint32_t)s * T::RD_BYTES);
        rd[3 * R + row] = valid ? 1.0f : 0.0f;
#pragma unroll
        for (int q = 0; q < (AH ? 8 : 7); ++q) rd[(4 + q) * R + row] = hin[q];
      }
      tc::fence_proxy_async();
      mbar_arrive(bar_x0f + s);
      NPM_WS_MSTAMP(kt, 3);
      if (kt > 0) scatter(kt - 1);
      sux = ux; suy = uy; suz = uz; svalid = valid;
    }
    if (kt > 0) scatter(kt - 1);
#undef NPM_WS_MSTAMP
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  if (warp == 0) tc::tmem_dealloc(tbase, (uint32_t)T::TCOLS);
}

}  // namespace ws

