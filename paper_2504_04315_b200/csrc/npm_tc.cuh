// npm_tc.cuh -- sm_100a tensor-core primitives (tcgen05 / TMEM / mbarrier)
// used by the fused decoder kernels.  Inline PTX only.
//
// Operand layout ("chunk-major", SWIZZLE_NONE canonical UMMA layout): a tile
// X[r][f] of R rows and F features in bf16 is stored as F/8 chunks, chunk j
// holding the 16-byte 8-feature slice of every row:  byte(r, f) =
// (f/8) * R*16 + r*16 + (f%8)*2.  The same bytes serve as
//   * a K-major operand (rows = M or N, features = K):  LBO = R*16 (K step),
//     SBO = 128 (8-row step);
//   * an MN-major operand (features = M or N, rows = K): SBO = R*16 (8-feature
//     step), LBO = 128 (8-row K step).
// so activations are written once (16-byte row stores, conflict free) and read
// by the forward MMA (K-major) and by the weight-gradient MMA (MN-major).
#pragma once
#include <cstdint>
#include <cuda_bf16.h>

namespace npm {
namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// UMMA shared-memory matrix descriptor, SWIZZLE_NONE, version 1 (sm_100).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1u << 46;
  return d;
}

// Instruction descriptor, kind::f16: A, B bf16; D fp32; dense.
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, bool a_mn, bool b_mn) {
  return (1u << 4)                        // D format F32
         | (1u << 7)                      // A format BF16
         | (1u << 10)                     // B format BF16
         | ((a_mn ? 1u : 0u) << 15)       // A major (0 = K, 1 = MN)
         | ((b_mn ? 1u : 0u) << 16)       // B major
         | ((uint32_t)(N >> 3) << 17)     // N >> 3
         | ((uint32_t)(M >> 4) << 24);    // M >> 4
}

// D[tmem] (+)= A[smem] * B[smem]^T, issued by one thread.
__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n"
      :: "r"(d_tmem), "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

// Arrive on an mbarrier when all previously issued MMAs of this thread completed.
__device__ __forceinline__ void mma_commit(uint64_t* mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
               :: "r"(smem_u32(mbar)) : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(mbar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* mbar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "NPM_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra NPM_WAIT_%=;\n\t}\n"
      :: "r"(smem_u32(mbar)), "r"(parity) : "memory");
}

// Same wait with a suspend-time hint: the thread sleeps in the try_wait until
// the phase completes (or ~1 ms passes) instead of re-polling.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* mbar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "NPM_WAITS_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1, %2;\n\t"
      "@!P bra NPM_WAITS_%=;\n\t}\n"
      :: "r"(smem_u32(mbar)), "r"(parity), "r"(1000000u) : "memory");
}

// TMEM allocation: executed by one full warp; writes the base address to smem.
__device__ __forceinline__ void tmem_alloc(uint32_t* dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
               :: "r"(smem_u32(dst)), "r"(ncols) : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(taddr), "r"(ncols) : "memory");
}

__device__ __forceinline__ void fence_before_sync() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after_sync() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// Generic-proxy smem writes -> visible to the tensor core (async proxy).
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// 32 lanes x 16 consecutive fp32 columns: thread i of the warp gets lane
// (32*(warp%4) + i) of the TMEM tile, columns [col, col+16).
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
template <int NC>
__device__ __forceinline__ void tmem_ldn(uint32_t taddr, float* v) {
  static_assert(NC == 1 || NC == 2 || NC == 4 || NC == 8 || NC == 16 || NC % 16 == 0, "columns");
  if constexpr (NC % 16 == 0 && NC > 16) {
#pragma unroll
    for (int c = 0; c < NC; c += 16) tmem_ld16(taddr + (uint32_t)c, v + c);
  } else if constexpr (NC == 16) {
    tmem_ld16(taddr, v);
  } else if constexpr (NC == 8) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
  } else if constexpr (NC == 4) {
    uint32_t r[4];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = __uint_as_float(r[i]);
  } else if constexpr (NC == 2) {
    uint32_t r[2];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];" : "=r"(r[0]), "=r"(r[1]) : "r"(taddr));
    v[0] = __uint_as_float(r[0]);
    v[1] = __uint_as_float(r[1]);
  } else {
    uint32_t r0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r0) : "r"(taddr));
    v[0] = __uint_as_float(r0);
  }
}

// 16 lanes x (8 X) fp32 columns ("16x256b.xX"): thread t of the warp gets
// lanes {t/4, t/4 + 8} (relative to the address lane) and, in repetition j,
// columns 8j + 2(t%4) + {0, 1}.  Register order: v[w + 2 half + 4 j].
template <int X>
__device__ __forceinline__ void tmem_ld16dp(uint32_t taddr, float* v) {
  static_assert(X == 1 || X == 2 || X == 4 || X == 8, "x");
  uint32_t r[4 * X];
  if constexpr (X == 1) {
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(taddr));
  } else if constexpr (X == 2) {
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
  } else if constexpr (X == 4) {
    asm volatile(
        "tcgen05.ld.sync.aligned.16x256b.x4.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
  } else {
    asm volatile(
        "tcgen05.ld.sync.aligned.16x256b.x8.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
  }
#pragma unroll
  for (int i = 0; i < 4 * X; ++i) v[i] = __uint_as_float(r[i]);
}

// Zero 16 fp32 columns of this warp's 32 TMEM lanes.
__device__ __forceinline__ void tmem_zero16(uint32_t taddr) {
  const uint32_t z = 0u;
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" :: "r"(taddr), "r"(z) : "memory");
}
// D[tmem] (+)= A[tmem] B[smem] (the .kind::f16 form with A in tensor memory:
// M = 128 rows = lanes, K = 16 bf16 per MMA packed two per 32-bit column)
__device__ __forceinline__ void mma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n"
      :: "r"(d_tmem), "r"(a_tmem), "l"(b), "r"(idesc), "r"(accumulate));
}
// 16 consecutive 32-bit columns of this warp's 32 lanes
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
      :: "r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
         "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
               :: "r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// Named barrier over `count` threads (id 1..15; id 0 is __syncthreads).
__device__ __forceinline__ void named_sync(uint32_t id, uint32_t count) {
  asm volatile("bar.sync %0, %1;" :: "r"(id), "r"(count) : "memory");
}

__device__ __forceinline__ void split_pack(float a, float b, uint32_t& hi, uint32_t& lo);

// Store one bf16 pair (features f, f+1 of a row), split hi/lo, chunk-major.
__device__ __forceinline__ void store_pair(uint32_t hi_base, uint32_t lo_base, int rows, int row, int f, float a,
                                           float b) {
  uint32_t h, l;
  split_pack(a, b, h, l);
  const uint32_t off = (uint32_t)((f / 8) * rows * 16 + row * 16 + (f % 8) * 2);
  asm volatile("st.shared.b32 [%0], %1;" :: "r"(hi_base + off), "r"(h) : "memory");
  asm volatile("st.shared.b32 [%0], %1;" :: "r"(lo_base + off), "r"(l) : "memory");
}

__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Split-bf16: x = hi + lo with hi = bf16(x), lo = bf16(x - hi); packs two
// consecutive features (even feature in the low half).  (Measured on B200, c2
// train: forming hi by integer rounding to spare the conversion pipe was
// 7 % slower than the two cvt instructions.)
__device__ __forceinline__ void split_pack(float a, float b, uint32_t& hi, uint32_t& lo) {
  // cvt.rn.bf16x2.f32 d, x, y puts x in the upper half: 6 instructions per pair
  // (cvt, shift, and-mask, 2 subtractions, cvt)
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(hi) : "f"(b), "f"(a));
  const float ha = __uint_as_float(hi << 16), hb = __uint_as_float(hi & 0xffff0000u);
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(lo) : "f"(b - hb), "f"(a - ha));
}

__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" :: "r"(addr), "r"(a), "r"(b), "r"(c), "r"(d)
               : "memory");
}

// Write features [8j, 8j+8) of one row (split hi/lo) into chunk-major tiles.
__device__ __forceinline__ void store_chunk(uint32_t hi_base, uint32_t lo_base, int rows, int row, int j,
                                            const float* v8) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) split_pack(v8[2 * q], v8[2 * q + 1], h[q], l[q]);
  const uint32_t off = (uint32_t)(j * rows * 16 + row * 16);
  st_shared_v4(hi_base + off, h[0], h[1], h[2], h[3]);
  st_shared_v4(lo_base + off, l[0], l[1], l[2], l[3]);
}

// Write CNT consecutive features [f0, f0 + CNT) of one row (split hi/lo);
// CNT in {2, 4, 8k}; f0 aligned to min(CNT, 8).
template <int CNT>
__device__ __forceinline__ void store_feats(uint32_t hi_base, uint32_t lo_base, int rows, int row, int f0,
                                            const float* v) {
  if constexpr (CNT >= 8) {
#pragma unroll
    for (int j = 0; j < CNT / 8; ++j) store_chunk(hi_base, lo_base, rows, row, f0 / 8 + j, v + 8 * j);
  } else {
    uint32_t h[CNT / 2], l[CNT / 2];
#pragma unroll
    for (int q = 0; q < CNT / 2; ++q) split_pack(v[2 * q], v[2 * q + 1], h[q], l[q]);
    const uint32_t off = (uint32_t)((f0 / 8) * rows * 16 + row * 16 + (f0 % 8) * 2);
    if constexpr (CNT == 4) {
      asm volatile("st.shared.v2.b32 [%0], {%1, %2};" :: "r"(hi_base + off), "r"(h[0]), "r"(h[1]) : "memory");
      asm volatile("st.shared.v2.b32 [%0], {%1, %2};" :: "r"(lo_base + off), "r"(l[0]), "r"(l[1]) : "memory");
    } else {
      asm volatile("st.shared.b32 [%0], %1;" :: "r"(hi_base + off), "r"(h[0]) : "memory");
      asm volatile("st.shared.b32 [%0], %1;" :: "r"(lo_base + off), "r"(l[0]) : "memory");
    }
  }
}

}  // namespace tc
}  // namespace npm
