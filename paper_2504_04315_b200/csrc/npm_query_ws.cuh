// npm_query_ws.cuh -- warp-specialised fused query kernel for the radiance
// shapes with K = 8 lobes (c1, c2 / c3, c5): guide sampling (C-O10),
// the pdf at the sample and the pdf at a caller direction (Eq. 3 mixture,
// P:201-206), one persistent 768-thread CTA per SM.
//
//   warps 0-7, 8-15  CHAIN groups g = 0, 1: group g runs the CTA's tiles
//       kt = g, g + 2, ... (a tile = 128 rows = the MMA M; row r = TMEM lane
//       r, its two threads are warps w and w + 4 of the group, each owning
//       half the columns and lobes).  Per tile: the layer-0 MMA from the X0
//       stage (smem), then per layer the epilogue (bias, ReLU, split-bf16) and
//       the next MMA, whose A operand the epilogue writes straight into TMEM
//       (tcgen05.st; `tcgen05.mma ... [a_tmem]`), then the Table 1 head:
//       softmax, pdf at w_q, the lobe choice (C-A17), the Jakob sampler in the
//       Duff ONB and the pdf at the sample, the two threads of a row exchanging
//       their partial sums through smem behind a 64-thread pair barrier.  The
//       two groups interleave: one's MMA round trips and head overlap the
//       other's.
//   warps 16-23  MEMORY: thread (part, row), part = which half of the L grid
//       levels.  For every tile in order: normalise x (C-O1), the 8 corners
//       per level (Eq. 13, C-O3/C-O4), gather + blend (C-O5) into an X0 stage
//       (split bf16, chunk-major) and the row data (sample index, validity,
//       w_q, the three uniforms: caller's or Philox of the sample index,
//       C-A18) into its row-data stage; S stages, so the gathers run ahead of
//       the chains.
//
// mbarriers: x0f[s] (memory arrivals: stage filled), x0e[s] (the consuming
// group's arrivals after its layer-0 MMA completed and the row data is in
// registers: stage free), mma[g] (tcgen05.commit of group g).
// Used for plain sample / pdf calls (the variants with decode outputs, f-1,
// f-2 and the product shape keep the r01 kernel).
#pragma once

namespace qws {

// MP: memory parts (levels L / MP per thread).  2: 8 memory warps, every
// warp at 128 registers.  4 (measurement): 16 memory warps at 64 registers and
// the chain at 112 via setmaxnreg -- no faster (the chain is the bound).
// MODE 0: guide sampling / pdf; 1: combined BSDF / guide one-sample MIS (f-1);
// 2: the mixture times the cosine lobe about the normal (f-2)
template <class N, int MODE = 0, int G = 2>
struct QW {
  using B = TC<N>;
  static constexpr int NL = N::NL, W = N::W, NOUT = N::NOUT, NIN = N::NIN, L = N::L, K = N::K;
  static constexpr int R = 128;
  static constexpr uint32_t CHR = R * 16;
  static constexpr int KIN = B::KIN;
  // radiance shapes with K = 8; the product shape (K = 16, X0 = grid features
  // + SH4(w_o) + SH4(n) + roughness, padded to KIN = 80) for plain sample / pdf
  static_assert((N::PRODUCT ? (K == 16 && MODE == 0 && KIN == 80 && L == 8) : (K == 8 && KIN == NIN)) &&
                L % 4 == 0 && W % 16 == 0, "query_ws shape");
#ifdef NPM_QWS_MP   // measurement override (4: B200 c2 233 us vs 229 us with 2)
  static constexpr int MP = L >= 4 * NPM_QWS_MP ? NPM_QWS_MP : 2;
#else
  static constexpr int MP = 2;
#endif
  static_assert((L / MP) % 2 == 0, "two levels (8 features) per X0 chunk");
  // TPR: chain threads per row.  1: a thread runs all K lobes of its row (no
  // exchanges); 2: warps w and w + 4 of a group split the row's columns and
  // lobes and exchange softmax / mixture sums / the sample through smem
#ifdef NPM_QWS_TPR   // measurement override (1: B200 c2 232 us vs 210 us with 2)
  static constexpr int TPR = NPM_QWS_TPR;
#else
  static constexpr int TPR = 2;
#endif
  static_assert(TPR == 1 || TPR == 2, "threads per row");
  // G chain groups (chosen per model by the host, `QueryArgs::qws_groups`):
  // two for L2-resident radiance tables (one group's MMA round trips and head
  // overlap the other's: B200 c2 205 vs 232 us with one); one for the
  // product shape, whose 8-lobe head spills at the 80 registers of a
  // 768-thread CTA and runs without spills at the 128 of a 512-thread one
  // (c4 1.84 -> 1.59 ms), and for HBM-resident tables (c5 3.04 -> 2.34 ms)
  static_assert(G == 1 || G == 2, "chain groups");
  static constexpr int GROUPS = G;
  static constexpr int GROUP_THREADS = TPR * R, CHAIN_THREADS = GROUPS * GROUP_THREADS;
  static constexpr int MEM_THREADS = MP * R;
  // MP = 4 register split (setmaxnreg moves registers only within the CTA's
  // launch allocation): TPR 1: 256 x 112 + 512 x 64 = 768 x 80; TPR 2:
  // 512 x 80 + 512 x 48 = 1024 x 64
  static constexpr int THREADS = CHAIN_THREADS + MEM_THREADS;
  static constexpr int LAUNCH_REGS = (65536 / THREADS) & ~7;
  static constexpr int CHAIN_REGS = TPR == 2 ? 80 : 112, MEM_REGS = TPR == 2 ? 48 : 64;
  static_assert(MP != 4 || CHAIN_THREADS * CHAIN_REGS + MEM_THREADS * MEM_REGS <= THREADS * LAUNCH_REGS, "regs");
  // row data [RDF][R]: 0 sample index (bits) | 1 valid | 2-4 w_q | 5-7 u | MODE 1: 8 u_sel;
  // MODE 1, 2: 9-11 normal
  static constexpr int RDF = MODE >= 1 ? 12 : 8;
  static constexpr uint32_t X0_BYTES = 2u * (KIN / 8) * CHR;
  // hidden-activation buffers: used only by the smem-A measurement variant
  // (NPM_QWS_SMEMA); with the A operand in TMEM they stay allocated as a gap
  // between the weights and the X0 stages -- the compact layout measured
  // slower on B200 (c2 212 vs 206 us, c5 3164 vs 3032 us; a pad at the end of
  // the layout instead: 212 us), cause not identified
  // (one-group layouts drop the gap: c4 query 1.59 -> 1.47 ms -- the layout
  // then fits the 164 KB carve-out -- and c5 2.34 -> 2.29 ms)
#if defined(NPM_QWS_SMEMA)
  static constexpr uint32_t H_BYTES = 2u * (W / 8) * CHR;
#else
  static constexpr uint32_t H_BYTES = G == 1 ? 0u : 2u * (W / 8) * CHR;
#endif
  static constexpr uint32_t RD_BYTES = RDF * R * 4;
  static constexpr uint32_t a1k(uint32_t x) { return (x + 1023u) & ~1023u; }
  static constexpr uint32_t OFF_W = 0, OFF_B = B::WBYTES;
  static constexpr uint32_t OFF_H = a1k(B::WBYTES + B::BBYTES);
  // TPR = 2 head exchange per group [RED_ROWS][R] f32: 0-1 max, 2-3 sums,
  // 4-5 pdf at w_q, 6-8 the sample, 9-10 pdf at the sample (part h in row +h)
  static constexpr int RED_ROWS = TPR == 2 ? (MODE == 1 ? 13 : 11) : 0;   // MODE 1: 11-12 logit parts (C-A34)
  static constexpr uint32_t RED_BYTES = (uint32_t)RED_ROWS * R * 4u;
  static constexpr uint32_t OFF_RED = OFF_H + GROUPS * H_BYTES;
  static constexpr uint32_t OFF_X0 = a1k(OFF_RED + GROUPS * RED_BYTES);
  // stages: 3 where the layout stays under the 164 KB carve-out (L1 for the gathers)
  static constexpr int S = OFF_X0 + 3u * (X0_BYTES + RD_BYTES) + 1024u <= 164u * 1024u ? 3 : 2;
  static constexpr uint32_t OFF_RD = OFF_X0 + (uint32_t)S * X0_BYTES;
  static constexpr uint32_t OFF_BAR = OFF_RD + (uint32_t)S * RD_BYTES;
  static constexpr int NBAR = 2 * S + GROUPS;
  static constexpr uint32_t OFF_TSLOT = OFF_BAR + 8u * NBAR;
  static constexpr uint32_t SMEM = OFF_TSLOT + 16u;
  static_assert(SMEM <= 227u * 1024u, "query_ws smem");
  static constexpr int TCOLS = 512;   // whole TMEM, base 0; group g: columns [64 g, 64 g + 64)
  static_assert(W <= 64 && NOUT <= 64, "accumulator columns");
};

template <class N, int MODE, int G>
__global__ void __launch_bounds__(QW<N, MODE, G>::THREADS, 1) query_ws_kernel(QueryArgs a) {
  using T = QW<N, MODE, G>;
  constexpr bool COMBINED = MODE == 1, COSPROD = MODE == 2;
  using TB = TC<N>;
  constexpr int NL = N::NL, K = N::K, W = N::W, L = N::L, KIN = T::KIN;
  constexpr int R = T::R, S = T::S;
  constexpr uint32_t CHR = T::CHR;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sb = tc::smem_u32(smem);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + T::OFF_BAR);
  uint64_t* bar_x0f = bars;
  uint64_t* bar_x0e = bars + S;
  uint64_t* bar_mma = bars + 2 * S;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + T::OFF_TSLOT);
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      tc::mbar_init(bar_x0f + s, T::MEM_THREADS);
      tc::mbar_init(bar_x0e + s, T::GROUP_THREADS);
    }
    for (int g = 0; g < T::GROUPS; ++g) tc::mbar_init(bar_mma + g, 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc(tslot, (uint32_t)T::TCOLS);
  stage_weights_tc<N>(a.params, smem, T::OFF_W, T::OFF_B);
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  if (*tslot != 0u) __trap();   // constant TMEM base 0 (the whole allocation)
  const int64_t n = a.n;
  const int64_t ntiles = (n + R - 1) / R, tstride = gridDim.x;
  const bool want_pdf = a.pdf != nullptr;

  constexpr int TPR = T::TPR;
  if (warp < T::CHAIN_THREADS / 32) {
    // =========================== CHAIN =====================================
    if constexpr (T::MP == 4) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" :: "n"(T::CHAIN_REGS));
    const int g = warp / (4 * TPR);
    const int gt = tid - g * T::GROUP_THREADS;                    // thread in group
    const int h = (warp >> 2) & (TPR - 1);                        // part of the row
    const int r = ((warp & 3) << 5) | lane;                       // row = TMEM lane
    constexpr int WQ = W / TPR, KQ = K / TPR;
    float* red = reinterpret_cast<float*>(smem + T::OFF_RED + (uint32_t)g * T::RED_BYTES);
    auto psync = [&]() { tc::named_sync(3u + 4u * (uint32_t)g + (uint32_t)(warp & 3), 64u); };
    const uint32_t lad = (uint32_t)((warp & 3) * 32) << 16;       // TMEM lane field
    const uint32_t tacc = (uint32_t)(64 * g);
#ifdef NPM_QWS_SMEMA
    const uint32_t hh = sb + T::OFF_H + (uint32_t)g * T::H_BYTES, hl = hh + (W / 8) * CHR;
#endif
#ifndef NPM_QWS_SMEMA
    // A operand of the hidden layers in TMEM: hi at columns 256 + 64 g, lo 32 further
    const uint32_t tah = (uint32_t)(256 + 64 * g), tal = tah + (uint32_t)(W / 2);
    static_assert(W / 2 <= 32, "A columns per group");
#endif
    const float* bias = reinterpret_cast<const float*>(smem + T::OFF_B);
    uint64_t* bmma = bar_mma + g;
    uint32_t phase = 0;
    auto handoff = [&]() {
      tc::fence_proxy_async();
      tc::fence_before_sync();
      tc::named_sync(1u + (uint32_t)g, (uint32_t)T::GROUP_THREADS);
    };
    auto wait_mma = [&]() {
      ws::mbar_wait_t(bmma, phase);
      phase ^= 1u;
      tc::fence_after_sync();
    };
#ifdef NPM_QWS_STAMPS   // measurement builds: phase stamps of CTA 0, group 0, row 0
    const bool stamp = a.dbg_clock && blockIdx.x == 0 && g == 0 && gt == 0;
#define QWS_STAMP(idx) do { if (stamp && kt / 2 < 64) a.dbg_clock[(kt / 2) * 16 + (idx)] = clock64(); } while (0)
#else
#define QWS_STAMP(idx) do { } while (0)
#endif
    int kt = g;
    for (int64_t tile = blockIdx.x + (int64_t)g * tstride; tile < ntiles; tile += T::GROUPS * tstride, kt += T::GROUPS) {
      QWS_STAMP(0);
      const int s = kt % S;
      const uint32_t x0h = sb + T::OFF_X0 + (uint32_t)s * T::X0_BYTES, x0l = x0h + (KIN / 8) * CHR;
      ws::mbar_wait_t(bar_x0f + s, (uint32_t)((kt / S) & 1));
      QWS_STAMP(1);
      tc::fence_after_sync();
      if (gt == 0) {
        const uint32_t w = sb + T::OFF_W + TB::woff(0);
        issue_fwd(tacc, x0h, x0l, w, w + TB::wbytes(0), KIN, TB::out(0));
        tc::mma_commit(bmma);
      }
      const float* rd = reinterpret_cast<const float*>(smem + T::OFF_RD + (uint32_t)s * T::RD_BYTES);
      const int64_t i = (int64_t)__float_as_uint(rd[r]);
      const bool valid = rd[R + r] != 0.0f;
      const float qx = rd[2 * R + r], qy = rd[3 * R + r], qz = rd[4 * R + r];
      const float u1 = rd[5 * R + r], u2 = rd[6 * R + r], u3 = rd[7 * R + r];
      float u4 = 1.0f, bnx = 0.0f, bny = 0.0f, bnz = 1.0f;
      if constexpr (COMBINED) u4 = rd[8 * R + r];
      if constexpr (COMBINED || COSPROD) { bnx = rd[9 * R + r]; bny = rd[10 * R + r]; bnz = rd[11 * R + r]; }
      wait_mma();
      QWS_STAMP(2);
      ws::mbar_arrive(bar_x0e + s);   // X0 read by the MMA, row data in registers
      // ---- hidden layers: epilogue of layer k, MMA of layer k + 1
#pragma unroll
      for (int k = 0; k < NL - 1; ++k) {
        const float* b = bias + TB::boff(k) / 4;
        // this part's WQ columns in flight at once (one TMEM round trip)
        float v[WQ];
#pragma unroll
        for (int c16 = 0; c16 < WQ; c16 += 16) tc::tmem_ldn<16>(lad + tacc + (uint32_t)(h * WQ + c16), v + c16);
        tc::tmem_wait_ld();
        const float4* b4 = reinterpret_cast<const float4*>(b + h * WQ);
#pragma unroll
        for (int j = 0; j < WQ / 4; ++j) {
          const float4 bb = b4[j];
          v[4 * j] = fmaxf(v[4 * j] + bb.x, 0.0f);
          v[4 * j + 1] = fmaxf(v[4 * j + 1] + bb.y, 0.0f);
          v[4 * j + 2] = fmaxf(v[4 * j + 2] + bb.z, 0.0f);
          v[4 * j + 3] = fmaxf(v[4 * j + 3] + bb.w, 0.0f);
        }
        if (COMBINED && k == NL - 2 && a.alpha_w) {   // C-A34: this part's a . h_{L-1}
          float zp = 0.0f;
#pragma unroll
          for (int j = 0; j < WQ; ++j) zp = fmaf(__ldg(a.alpha_w + h * WQ + j), v[j], zp);
          red[(11 + h) * R + r] = zp;   // read after the next group barrier
        }
#ifndef NPM_QWS_SMEMA
        // the next layer's A operand straight into tensor memory (split-bf16 hi /
        // lo, two features per column): no smem round trip, no proxy fence
        {
          uint32_t ph[WQ / 2], pl[WQ / 2];
#pragma unroll
          for (int q = 0; q < WQ / 2; ++q) tc::split_pack(v[2 * q], v[2 * q + 1], ph[q], pl[q]);
          if constexpr (WQ / 2 >= 16) {
#pragma unroll
            for (int c = 0; c < WQ / 2; c += 16) {
              tc::tmem_st16(lad + tah + (uint32_t)(h * (WQ / 2) + c), ph + c);
              tc::tmem_st16(lad + tal + (uint32_t)(h * (WQ / 2) + c), pl + c);
            }
          } else {
            static_assert(WQ / 2 == 8, "columns per row part");
            tc::tmem_st8(lad + tah + (uint32_t)(h * 8), ph);
            tc::tmem_st8(lad + tal + (uint32_t)(h * 8), pl);
          }
          tc::tmem_wait_st();
          tc::fence_before_sync();
          tc::named_sync(1u + (uint32_t)g, (uint32_t)T::GROUP_THREADS);
        }
        QWS_STAMP(3 + 2 * k);
        if (gt == 0) {
          tc::fence_after_sync();
          const uint32_t w = sb + T::OFF_W + TB::woff(k + 1);
          const int out = TB::out(k + 1);
          const uint32_t idesc = tc::idesc_bf16(R, out, false, false);
          const uint64_t bh = tc::sdesc(w, out * 16, 128), bl = tc::sdesc(w + TB::wbytes(k + 1), out * 16, 128);
#pragma unroll
          for (int ks = 0; ks < TB::in_p(k + 1) / 16; ++ks) {
            const uint64_t wa = (uint64_t)(ks * 2 * out * 16) >> 4;
            tc::mma_bf16_ts(tacc, tah + 8u * ks, bh + wa, idesc, ks > 0 ? 1u : 0u);
            tc::mma_bf16_ts(tacc, tah + 8u * ks, bl + wa, idesc, 1u);
            tc::mma_bf16_ts(tacc, tal + 8u * ks, bh + wa, idesc, 1u);
          }
          tc::mma_commit(bmma);
        }
#else
#pragma unroll
        for (int c8 = 0; c8 < WQ / 8; ++c8) tc::store_chunk(hh, hl, R, r, h * (WQ / 8) + c8, v + 8 * c8);
        handoff();
        QWS_STAMP(3 + 2 * k);
        if (gt == 0) {
          tc::fence_after_sync();
          const uint32_t w = sb + T::OFF_W + TB::woff(k + 1);
          issue_fwd(tacc, hh, hl, w, w + TB::wbytes(k + 1), TB::in_p(k + 1), TB::out(k + 1));
          tc::mma_commit(bmma);
        }
#endif
        wait_mma();
        QWS_STAMP(4 + 2 * k);
      }
      // ---- Table 1 head: lobes [h KQ, (h + 1) KQ) of this row
      float lp[KQ], kp[KQ], tp[KQ], pp[KQ];
      tc::tmem_ldn<KQ>(lad + tacc + (uint32_t)(h * KQ), lp);
      tc::tmem_ldn<KQ>(lad + tacc + (uint32_t)(K + h * KQ), kp);
      tc::tmem_ldn<KQ>(lad + tacc + (uint32_t)(2 * K + h * KQ), tp);
      tc::tmem_ldn<KQ>(lad + tacc + (uint32_t)(3 * K + h * KQ), pp);
      tc::tmem_wait_ld();
      // the group's next layer-0 MMA overwrites these columns: every thread's
      // read first
      tc::fence_before_sync();
      tc::named_sync(1u + (uint32_t)g, (uint32_t)T::GROUP_THREADS);
      QWS_STAMP(3 + 2 * (NL - 1));
#ifdef NPM_QWS_NOHEAD   // measurement variant: no Table 1 head
      if (valid) a.spdf[i] = lp[0] + kp[1] + tp[2] + pp[3] + qx + u1 + u2 + u3 + qy + qz;
      continue;
#endif
      const float* b = bias + TB::boff(NL - 1) / 4 + h * KQ;
      float kap[KQ], mx[KQ], my[KQ], mz[KQ], nrm[KQ];
      float M = -INFINITY;
      bool conc = false;
#pragma unroll
      for (int j = 0; j < KQ; ++j) {   // branch-free over the lobes (they interleave)
        lp[j] += b[j];
        tp[j] += b[2 * K + j];
        pp[j] += b[3 * K + j];
        M = fmaxf(M, lp[j]);
        kap[j] = __expf(fminf(fmaxf(kp[j] + b[K + j], a.log_kmin), a.log_kmax));
        float th, ph, st, ct, sp, cp;
        lobe_angles<false>(tp[j], pp[j], kap[j], th, ph, st, ct, sp, cp);
        mx[j] = st * cp; my[j] = st * sp; mz[j] = ct;
        float em;
        nrm[j] = lobe_norm_fast(kap[j], em);
        conc |= kap[j] > 1e3f;
      }
      // concentrated lobes: Table 1's angles precisely (lobe_angles<true>, C-A33),
      // only in warps that have one
      if (__any_sync(0xffffffffu, conc)) {
#pragma unroll
        for (int j = 0; j < KQ; ++j) {
          if (kap[j] > 1e3f) {
            float th, ph, st, ct, sp, cp;
            lobe_angles<true>(tp[j], pp[j], kap[j], th, ph, st, ct, sp, cp);
            mx[j] = st * cp; my[j] = st * sp; mz[j] = ct;
          }
        }
      }
      if constexpr (COSPROD) {   // f-2: times the cosine lobe about n, renormalised via the logits
        M = -INFINITY;
#pragma unroll
        for (int j = 0; j < KQ; ++j) {
          lp[j] += vmf_product_inplace(mx[j], my[j], mz[j], kap[j], bnx, bny, bnz, a.kappa_c, a.log_c_kc);
          float em;
          nrm[j] = lobe_norm(fmaxf(kap[j], 1e-30f), em);
          M = fmaxf(M, lp[j]);
        }
      }
      if constexpr (TPR == 2) {
        red[h * R + r] = M;
        psync();
        M = fmaxf(red[r], red[R + r]);
      }
      float e[KQ], Ssum = 0.0f, P = 0.0f;
#pragma unroll
      for (int j = 0; j < KQ; ++j) {
        e[j] = __expf(lp[j] - M);
        Ssum += e[j];
        if (want_pdf) P += e[j] * lobe_eval(nrm[j], kap[j], mx[j], my[j], mz[j], qx, qy, qz);
      }
      // part boundaries of the lobe CDF: B_h = sum of the earlier parts' e (C-A17)
      float Bh = 0.0f, Bn = Ssum, invS;
      if constexpr (TPR == 2) {
        red[(2 + h) * R + r] = Ssum;
        red[(4 + h) * R + r] = P;
        psync();
        const float S0 = red[2 * R + r], St = S0 + red[3 * R + r];
        invS = 1.0f / St;
        Bh = h ? S0 : 0.0f;
        Bn = h ? St : S0;
        P = red[4 * R + r] + red[5 * R + r];
      } else {
        invS = 1.0f / Ssum;
      }
      if (want_pdf && valid && h == 0) a.pdf[i] = P * invS;
      if (a.do_sample) {
        // i* = min{i : u1 < C_i}, C_i = sum_{j<=i} lambda_j; K-1 if none (C-A17):
        // the part whose range [B_h, B_h+1) holds u1 (the last part takes the rest)
        // f-1: BSDF with probability alpha (C-A25), else the guide; alpha the
        // caller's or the learned alpha(x) (C-A34)
        float alpha = a.alpha;
        if (COMBINED && a.alpha_w) {
          float z = __ldg(a.alpha_w + W);
#pragma unroll
          for (int qq = 0; qq < TPR; ++qq) z += red[(11 + qq) * R + r];
          alpha = 1.0f / (1.0f + __expf(-z));
        }
        const bool use_bsdf = COMBINED && u4 < alpha;
        const bool own = !use_bsdf && (TPR == 1 || (u1 >= Bh * invS && (u1 < Bn * invS || h == TPR - 1)));
        float wx = 0.f, wy = 0.f, wz = 0.f;
        if (COMBINED && use_bsdf && h == 0) {
          bsdf_sample(bnx, bny, bnz, u1, u2, wx, wy, wz);
          if constexpr (TPR == 2) { red[6 * R + r] = wx; red[7 * R + r] = wy; red[8 * R + r] = wz; }
        }
        if (own) {
          int sel = KQ - 1;
          float cum = Bh;
#pragma unroll
          for (int j = 0; j < KQ - 1; ++j) {
            cum += e[j];
            if (sel == KQ - 1 && u1 < cum * invS) sel = j;
          }
          float kk = kap[0], mmx = mx[0], mmy = my[0], mmz = mz[0];
#pragma unroll
          for (int j = 1; j < KQ; ++j)
            if (sel == j) { kk = kap[j]; mmx = mx[j]; mmy = my[j]; mmz = mz[j]; }
          lobe_sample(kk, mmx, mmy, mmz, u2, u3, wx, wy, wz);
          if constexpr (TPR == 2) { red[6 * R + r] = wx; red[7 * R + r] = wy; red[8 * R + r] = wz; }
        }
        if constexpr (TPR == 2) {
          psync();
          wx = red[6 * R + r]; wy = red[7 * R + r]; wz = red[8 * R + r];
        }
        float P2 = 0.0f;
#pragma unroll
        for (int j = 0; j < KQ; ++j) P2 += e[j] * lobe_eval(nrm[j], kap[j], mx[j], my[j], mz[j], wx, wy, wz);
        if constexpr (TPR == 2) {
          red[(9 + h) * R + r] = P2;
          psync();
          P2 = red[9 * R + r] + red[10 * R + r];
        }
        if (valid && h == 0) {
          if constexpr (COMBINED) {
            float V = P2 * invS, ox = wx, oy = wy, oz = wz, pc;
            int32_t tq = use_bsdf ? 0 : 1;
            if (!use_bsdf && !(isfinite(V) && V >= kVFloor)) {   // guide pdf underflow (C-A26)
              bsdf_sample(bnx, bny, bnz, u1, u2, ox, oy, oz);
              pc = bsdf_pdf(bnx, bny, bnz, ox, oy, oz);
              V = 0.0f;
              tq = 2;
            } else {
              // one-sample balance heuristic p~ = alpha p_bsdf + (1 - alpha) V
              pc = alpha * bsdf_pdf(bnx, bny, bnz, ox, oy, oz) + (1.0f - alpha) * V;
            }
            if (a.gpdf) a.gpdf[i] = V;
            if (a.tech) a.tech[i] = tq;
            a.sx[i] = ox; a.sy[i] = oy; a.sz[i] = oz;
            a.spdf[i] = pc;
          } else {
            a.sx[i] = wx; a.sy[i] = wy; a.sz[i] = wz;
            a.spdf[i] = P2 * invS;
          }
        }
      }
      QWS_STAMP(4 + 2 * (NL - 1));
    }
#undef QWS_STAMP
  } else {
    // =========================== MEMORY ====================================
    if constexpr (T::MP == 4) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" :: "n"(T::MEM_REGS));
    const int m = tid - T::CHAIN_THREADS;
    const int row = m & (R - 1), part = m >> 7;
    constexpr int LP = L / T::MP;
    const float4* tab = reinterpret_cast<const float4*>(a.params + N::N_MLP);
    // the row's sample index is loaded two tiles ahead and its raw position
    // one tile ahead, so the perm -> x -> corner-index chain of dependent
    // loads is off the gathers' path
    auto load_idx = [&](int64_t tl, int64_t& i, bool& v) {
      const int64_t slot = tl * R + row;
      v = slot < n;
      i = v ? (a.perm ? (int64_t)__ldg(a.perm + slot) : slot) : 0;
    };
    auto load_x = [&](int64_t i, bool v, float* x) {
      x[0] = x[1] = x[2] = 0.0f;
      if (v) { x[0] = __ldg(a.px + i); x[1] = __ldg(a.py + i); x[2] = __ldg(a.pz + i); }
    };
    int64_t i_n = 0, i_nn = 0;
    bool v_n = false, v_nn = false;
    float x_n[3];
    if (blockIdx.x < ntiles) load_idx(blockIdx.x, i_n, v_n);
    load_x(i_n, v_n, x_n);
    if (blockIdx.x + tstride < ntiles) load_idx(blockIdx.x + tstride, i_nn, v_nn);
#ifdef NPM_QWS_STAMPS
    const bool mstamp = a.dbg_clock && blockIdx.x == 0 && m == 0;
#define QWS_MSTAMP(idx) do { if (mstamp && kt < 64) a.dbg_clock[64 * 16 + kt * 16 + (idx)] = clock64(); } while (0)
#else
#define QWS_MSTAMP(idx) do { } while (0)
#endif
    int kt = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += tstride, ++kt) {
      QWS_MSTAMP(0);
      const int s = kt % S;
      const int64_t i = i_n;
      const bool valid = v_n;
      const float x0 = x_n[0], x1 = x_n[1], x2 = x_n[2];
      i_n = i_nn; v_n = v_nn;
      load_x(i_n, v_n, x_n);
      v_nn = false;
      if (tile + 2 * tstride < ntiles) load_idx(tile + 2 * tstride, i_nn, v_nn);
      float ux = 0.f, uy = 0.f, uz = 0.f;
      if (valid) {
        ux = normalize_axis(x0, a.grid.lo[0], a.grid.inv[0]);
        uy = normalize_axis(x1, a.grid.lo[1], a.grid.inv[1]);
        uz = normalize_axis(x2, a.grid.lo[2], a.grid.inv[2]);
      }
      // part 0: w_q (and the normal, MODE 1); part 1: the uniforms
      float ex[4] = {0.f, 0.f, 0.f, 1.f}, nn[3] = {0.f, 0.f, 1.f};
      float cv[4] = {0.f, 0.f, 1.f, 0.f};   // product conditioning: part 0 w_o, part 1 n + roughness
      if constexpr (N::PRODUCT) {
        if (valid) {
          if (part == 0) { cv[0] = __ldg(a.wox + i); cv[1] = __ldg(a.woy + i); cv[2] = __ldg(a.woz + i); }
          else { cv[0] = __ldg(a.nx + i); cv[1] = __ldg(a.ny + i); cv[2] = __ldg(a.nz + i); cv[3] = __ldg(a.rough + i); }
        }
      }
      if (part == 0) {
        if (want_pdf) { ex[0] = __ldg(a.wx + i); ex[1] = __ldg(a.wy + i); ex[2] = __ldg(a.wz + i); }
        if constexpr (COMBINED || COSPROD) {
          if (valid) { nn[0] = __ldg(a.bnx + i); nn[1] = __ldg(a.bny + i); nn[2] = __ldg(a.bnz + i); }
        }
      } else if (part == 1 && a.do_sample) {
        if (a.u) {
          ex[0] = __ldg(a.u + i); ex[1] = __ldg(a.u + n + i); ex[2] = __ldg(a.u + 2 * n + i);
          if constexpr (COMBINED) ex[3] = __ldg(a.u + 3 * n + i);
        } else {
          const float4 u = philox_uniforms4(a.seed, (uint64_t)i + a.offset);
          ex[0] = u.x; ex[1] = u.y; ex[2] = u.z; ex[3] = u.w;
        }
      }
      // branch-free over the levels (an invalid row gathers at the AABB corner
      // and is zeroed), so the compiler can overlap one level's loads with the
      // previous level's blend
      float gf[4 * LP];
#pragma unroll
      for (int q = 0; q < LP; ++q) {
        float4 gl = make_float4(0.f, 0.f, 0.f, 0.f);
#ifndef NPM_QWS_NOGATHER   // measurement variant: no grid gathers
        const int l = part * LP + q;
        LevelCorners lc;
        level_corners(a.grid, l, ux, uy, uz, lc);
        gl = gather_level<false>(tab, a.grid.off[l], lc);
#endif
        gf[4 * q] = valid ? gl.x : 0.0f; gf[4 * q + 1] = valid ? gl.y : 0.0f;
        gf[4 * q + 2] = valid ? gl.z : 0.0f; gf[4 * q + 3] = valid ? gl.w : 0.0f;
      }
      QWS_MSTAMP(1);
      ws::mbar_wait_idle(bar_x0e + s, (uint32_t)(((kt / S) & 1) ^ 1));
      QWS_MSTAMP(2);
      const uint32_t xh = sb + T::OFF_X0 + (uint32_t)s * T::X0_BYTES, xl = xh + (KIN / 8) * CHR;
#pragma unroll
      for (int j = 0; j < LP / 2; ++j) tc::store_chunk(xh, xl, R, row, part * (LP / 2) + j, gf + 8 * j);
      if constexpr (N::PRODUCT) {   // [32, 48) SH4(w_o) by part 0; [48, 64) SH4(n), [64, 80) roughness by part 1
        float e16[16];
        if (valid) sh4(cv[0], cv[1], cv[2], e16);
        else {
#pragma unroll
          for (int j = 0; j < 16; ++j) e16[j] = 0.0f;
        }
        tc::store_chunk(xh, xl, R, row, 4 + 2 * part, e16);
        tc::store_chunk(xh, xl, R, row, 5 + 2 * part, e16 + 8);
        if (part == 1) {
          float ro[8] = {valid ? cv[3] : 0.0f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
          const float z8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
          tc::store_chunk(xh, xl, R, row, 8, ro);
          tc::store_chunk(xh, xl, R, row, 9, z8);
        }
      }
      float* rd = reinterpret_cast<float*>(smem + T::OFF_RD + (uint32_t)s * T::RD_BYTES);
      if (part == 0) {
        rd[row] = __uint_as_float((uint32_t)i);
        rd[R + row] = valid ? 1.0f : 0.0f;
        rd[2 * R + row] = ex[0]; rd[3 * R + row] = ex[1]; rd[4 * R + row] = ex[2];
        if constexpr (COMBINED || COSPROD) { rd[9 * R + row] = nn[0]; rd[10 * R + row] = nn[1]; rd[11 * R + row] = nn[2]; }
      } else if (part == 1) {
        rd[5 * R + row] = ex[0]; rd[6 * R + row] = ex[1]; rd[7 * R + row] = ex[2];
        if constexpr (COMBINED) rd[8 * R + row] = ex[3];
      }
      tc::fence_proxy_async();
      ws::mbar_arrive(bar_x0f + s);
      QWS_MSTAMP(3);
    }
#undef QWS_MSTAMP
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  if (warp == 0) tc::tmem_dealloc(*tslot, (uint32_t)T::TCOLS);
}

}  // namespace qws
