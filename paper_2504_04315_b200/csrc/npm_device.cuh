// npm_device.cuh -- device building blocks of the NPM hot path (sm_100a).
//
// Citations: P:n = PAPER.md line n (equation / section named); C-xx = reading
// in DESIGN.md.  Nothing here is shared with oracle/ (independent code).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace npm {

constexpr int kMaxLevels = 16;
constexpr int kMaxLobes = 16;
constexpr float kPi = 3.14159265358979323846f;
constexpr float kTwoPi = 6.28318530717958647692f;
constexpr float kUMax = (float)(1.0 - 1e-6);  // S:163 clamp, C-O1
constexpr float kVFloor = 1e-30f;             // S:125, C-O13

// Grid embedding descriptor (Eq. 13; C-A3/C-A4).
struct GridDesc {
  int L;
  uint32_t hashed_mask;        // bit l set: level l uses the spatial hash (C-A4)
  int res[kMaxLevels];         // D_l lattice points per axis
  float resm1f[kMaxLevels];    // fl32(D_l - 1) (C-O3), precomputed: no I2F in the kernels
  int cellmax[kMaxLevels];     // D_l - 2 (largest cell index; 0 if D_l = 2)
  float cellmaxf[kMaxLevels];  // (float)cellmax
  uint32_t tsize[kMaxLevels];  // entries in level l (D^3 or T)
  int64_t off[kMaxLevels];     // first entry of level l (entries of F = 4 floats)
  float lo[3], inv[3];         // AABB min, fl32(1/(hi - lo)) (C-O1)
};

// ---------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al. SC'11), C-O11.
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) { k.x += W0; k.y += W1; }
    const uint32_t hi0 = __umulhi(M0, c.x), lo0 = M0 * c.x;
    const uint32_t hi1 = __umulhi(M1, c.z), lo1 = M1 * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
  }
  return c;
}

// u_j = (out_j >> 8) * 2^-24, counter = (lo32(i+offset), hi32(i+offset), 0, 0).
__device__ __forceinline__ float3 philox_uniforms(uint64_t seed, uint64_t ctr) {
  const uint4 o = philox4x32_10(make_uint4((uint32_t)ctr, (uint32_t)(ctr >> 32), 0u, 0u),
                                make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
  const float s = 5.9604644775390625e-08f;  // 2^-24
  return make_float3((float)(o.x >> 8) * s, (float)(o.y >> 8) * s, (float)(o.z >> 8) * s);
}

// The same counter's fourth output as a fourth uniform (C-A25: the technique
// selector of combined BSDF/guide sampling).
__device__ __forceinline__ float4 philox_uniforms4(uint64_t seed, uint64_t ctr) {
  const uint4 o = philox4x32_10(make_uint4((uint32_t)ctr, (uint32_t)(ctr >> 32), 0u, 0u),
                                make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
  const float s = 5.9604644775390625e-08f;  // 2^-24
  return make_float4((float)(o.x >> 8) * s, (float)(o.y >> 8) * s, (float)(o.z >> 8) * s, (float)(o.w >> 8) * s);
}

// ---------------------------------------------------------------------------
// Pinned fp32 cell-index sequence (C-O1, C-O3; C-A1): no FMA contraction.
__device__ __forceinline__ float normalize_axis(float x, float lo, float inv) {
  const float u = __fmul_rn(__fsub_rn(x, lo), inv);
  return fminf(fmaxf(u, 0.0f), kUMax);
}

// s = fl32(u * fl32(D - 1)), i = floor(s) clamped to [0, D - 2], f = s - i.
// floor without the conversion (XU) pipe, which the heads' MUFU work and the
// split-bf16 packs also need: for 0 <= s < 2^22, RD(s + 1.5 * 2^23) =
// 1.5 * 2^23 + floor(s) exactly (the ulp there is 1), so the integer is the
// difference of the bit patterns and floor(s) = t - 1.5 * 2^23 (exact).
// Bit-identical to floorf / (int) / (float) (u >= 0 after the clamp of C-O1);
// measured on B200 c2 train: neutral to -0.6 %.
__device__ __forceinline__ void cell_axis(float u, float dm1, int hi, float hif, int& i, float& f) {
  const float s = __fmul_rn(u, dm1);
  const float t = __fadd_rd(s, 12582912.0f);
  int ii = __float_as_int(t) - 0x4B400000;
  float fl = __fsub_rn(t, 12582912.0f);
  if (ii > hi) { ii = hi; fl = hif; }
  i = ii;
  f = __fsub_rn(s, fl);
}

// Corner entry index (C-O4): dense Px + D(Py + D Pz); hashed (C-A4 convention,
// not in the paper) (Px*1 ^ Py*2654435761 ^ Pz*805459861) & (T - 1).
__device__ __forceinline__ uint32_t corner_index(uint32_t px, uint32_t py, uint32_t pz, int d,
                                                 uint32_t tsize, bool hashed) {
  if (!hashed) return px + (uint32_t)d * (py + (uint32_t)d * pz);
  return (px ^ (py * 2654435761u) ^ (pz * 805459861u)) & (tsize - 1u);
}

// The 8 corners + trilinear weights of level l (Eq. 13 "eight corners",
// trilinear per C-A2), corner c = cx + 2 cy + 4 cz.
struct LevelCorners {
  uint32_t idx[8];
  float w[8];
};

__device__ __forceinline__ void level_corners(const GridDesc& g, int l, float ux, float uy, float uz,
                                              LevelCorners& lc) {
  const int d = g.res[l];
  const float dm1 = g.resm1f[l], hif = g.cellmaxf[l];
  const int hi = g.cellmax[l];
  int ix, iy, iz;
  float fx, fy, fz;
  cell_axis(ux, dm1, hi, hif, ix, fx);
  cell_axis(uy, dm1, hi, hif, iy, fy);
  cell_axis(uz, dm1, hi, hif, iz, fz);
  const bool hashed = (g.hashed_mask >> l) & 1u;
  const float gx0 = 1.0f - fx, gy0 = 1.0f - fy, gz0 = 1.0f - fz;
  // w_c = (gx * gy) * gz, the same product order as corner-by-corner
  const float wxy[4] = {gx0 * gy0, fx * gy0, gx0 * fy, fx * fy};
  // Same integer results as corner_index() per corner, built incrementally:
  // dense  base + cx + D cy + D^2 cz;  hashed  (x ^ y P1 ^ z P2) with
  // (y + 1) P1 = y P1 + P1 (mod 2^32).
  uint32_t ox[2], oy[2], oz[2];
  if (!hashed) {
    const uint32_t ud = (uint32_t)d;
    const uint32_t base = (uint32_t)ix + ud * ((uint32_t)iy + ud * (uint32_t)iz);
    ox[0] = base; ox[1] = base + 1u;
    oy[0] = 0u; oy[1] = ud;
    oz[0] = 0u; oz[1] = ud * ud;
  } else {
    const uint32_t hy = (uint32_t)iy * 2654435761u, hz = (uint32_t)iz * 805459861u;
    ox[0] = (uint32_t)ix; ox[1] = (uint32_t)ix + 1u;
    oy[0] = hy; oy[1] = hy + 2654435761u;
    oz[0] = hz; oz[1] = hz + 805459861u;
  }
  const uint32_t mask = g.tsize[l] - 1u;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const int cx = c & 1, cy = (c >> 1) & 1, cz = (c >> 2) & 1;
    lc.idx[c] = hashed ? ((ox[cx] ^ oy[cy] ^ oz[cz]) & mask) : (ox[cx] + oy[cy] + oz[cz]);
    lc.w[c] = wxy[c & 3] * (cz ? fz : gz0);
  }
}

// Eq. 13 gather + trilinear blend of one level, fetching x-neighbour corners
// together.  Corners c and c + 1 (cx = 0, 1) are entries e and e + 1 (dense)
// or e and e ^ 1 (hashed, ix even: the x prime is 1).  A 32-byte load of the
// aligned entry pair {e & ~1, e | 1} (absolute index from the 32-B aligned
// table start) returns both whenever they share it -- one L1/L2 sector
// instead of two; otherwise the second corner is a separate 16-byte load.
// Same products and summation order as the 8-load form (bit-identical).
// Requires: tab 32-B aligned and readable one entry past the last (the model
// pads its parameter buffers).
__device__ __forceinline__ void ld_pair(const float4* p, float4& lo, float4& hi) {
  asm("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=f"(lo.x), "=f"(lo.y), "=f"(lo.z), "=f"(lo.w), "=f"(hi.x), "=f"(hi.y), "=f"(hi.z), "=f"(hi.w)
      : "l"(p));
}
// the same 32-byte load allocating in L1 (coherent, binned query gathers)
__device__ __forceinline__ void ld_pair_l1(const float4* p, float4& lo, float4& hi) {
  asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=f"(lo.x), "=f"(lo.y), "=f"(lo.z), "=f"(lo.w), "=f"(hi.x), "=f"(hi.y), "=f"(hi.z), "=f"(hi.w)
      : "l"(p));
}

// The 32-byte pair loads bypass L1 allocation (the training gathers hit L1
// 8.9 % of the time): B200, c2 train 646 -> 630 us, c5 5.34 -> 5.04 ms.  The
// single second-corner loads keep allocating (no_allocate there: c5 +7 %).
// PAIRS = false: eight plain 16-byte loads (the warp-specialised training
// kernel's memory warps: fewer ALU / select instructions next to the chain;
// B200 c2 -1.4 %).
template <bool PAIRS = true, bool L1A = false>
__device__ __forceinline__ float4 gather_level(const float4* __restrict__ tab, uint32_t off, const LevelCorners& lc) {
  float4 v[8];
  if constexpr (!PAIRS) {
#pragma unroll
    for (int c = 0; c < 8; ++c) v[c] = __ldg(tab + off + lc.idx[c]);
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      a0 = fmaf(lc.w[c], v[c].x, a0); a1 = fmaf(lc.w[c], v[c].y, a1);
      a2 = fmaf(lc.w[c], v[c].z, a2); a3 = fmaf(lc.w[c], v[c].w, a3);
    }
    return make_float4(a0, a1, a2, a3);
  }
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const uint32_t e0 = off + lc.idx[2 * p], e1 = off + lc.idx[2 * p + 1];
    float4 lo, hi;
    if constexpr (L1A) ld_pair_l1(tab + (e0 & ~1u), lo, hi);
    else ld_pair(tab + (e0 & ~1u), lo, hi);
    v[2 * p] = (e0 & 1u) ? hi : lo;
    if ((e0 ^ e1) == 1u) v[2 * p + 1] = (e1 & 1u) ? hi : lo;
    else v[2 * p + 1] = __ldg(tab + e1);
  }
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    a0 = fmaf(lc.w[c], v[c].x, a0); a1 = fmaf(lc.w[c], v[c].y, a1);
    a2 = fmaf(lc.w[c], v[c].z, a2); a3 = fmaf(lc.w[c], v[c].w, a3);
  }
  return make_float4(a0, a1, a2, a3);
}

// ---------------------------------------------------------------------------
// Real orthonormal SH, 4 bands, l-major / m ascending, no Condon-Shortley
// phase (C-A20, C-O6).  Cartesian polynomial forms.
__device__ __forceinline__ void sh4(float x, float y, float z, float* o) {
  const float xx = x * x, yy = y * y, zz = z * z;
  o[0] = 0.28209479177387814f;
  o[1] = 0.48860251190291992f * y;
  o[2] = 0.48860251190291992f * z;
  o[3] = 0.48860251190291992f * x;
  o[4] = 1.0925484305920792f * x * y;
  o[5] = 1.0925484305920792f * y * z;
  o[6] = 0.31539156525252005f * (3.0f * zz - 1.0f);
  o[7] = 1.0925484305920792f * x * z;
  o[8] = 0.54627421529603959f * (xx - yy);
  o[9] = 0.59004358992664352f * y * (3.0f * xx - yy);
  o[10] = 2.8906114426405538f * x * y * z;
  o[11] = 0.45704579946446572f * y * (5.0f * zz - 1.0f);
  o[12] = 0.3731763325901154f * z * (5.0f * zz - 3.0f);
  o[13] = 0.45704579946446572f * x * (5.0f * zz - 1.0f);
  o[14] = 1.4453057213202769f * z * (xx - yy);
  o[15] = 0.59004358992664352f * x * (xx - 3.0f * yy);
}

// ---------------------------------------------------------------------------
// Table 1 mappings, C-O8: raw block layout [l' | k' | t' | p'] (C-A6).
template <int K>
struct Mixture {
  float lam[K], kap[K], mx[K], my[K], mz[K];
};

template <int K>
__device__ __forceinline__ void activate(const float* raw, float log_kmin, float log_kmax, Mixture<K>& m) {
  float mx = raw[0];
#pragma unroll
  for (int i = 1; i < K; ++i) mx = fmaxf(mx, raw[i]);
  float sum = 0.0f;
#pragma unroll
  for (int i = 0; i < K; ++i) { m.lam[i] = expf(raw[i] - mx); sum += m.lam[i]; }
  const float inv = 1.0f / sum;
#pragma unroll
  for (int i = 0; i < K; ++i) {
    m.lam[i] *= inv;
    m.kap[i] = expf(fminf(fmaxf(raw[K + i], log_kmin), log_kmax));
    const float th = 1.0f / (1.0f + expf(-raw[2 * K + i]));
    const float ph = 1.0f / (1.0f + expf(-raw[3 * K + i]));
    float st, ct, sp, cp;
    sincospif(th, &st, &ct);          // sin(pi theta), cos(pi theta)
    sincospif(2.0f * ph, &sp, &cp);   // sin(2 pi phi), cos(2 pi phi)
    m.mx[i] = st * cp;                // C-A7: polar angle from +z, azimuth from +x
    m.my[i] = st * sp;
    m.mz[i] = ct;
  }
}

// Fast-path math for the fused kernels' heads (MUFU ex2 / sin / cos / rcp):
// relative errors ~1e-6, far inside the parity tolerances (params 1e-4, pdf
// 1e-3 rel, gradient 2e-3 rel-L2).  The conditioning-sensitive pieces (the
// expm1 of the vMF normalisation, the sampler's log1p / expm1) stay precise.
__device__ __forceinline__ float fast_sigmoid(float x) { return __fdividef(1.0f, 1.0f + __expf(-x)); }

// Table 1 angles of one lobe: theta = sigma(t'), phi = sigma(p') and the
// sines / cosines of pi theta, 2 pi phi.  MUFU fast math by default; for a
// concentrated lobe (kappa > 1e3) they are re-evaluated precisely (IEEE expf
// and division, sincospif): the relative sensitivity of the lobe's pdf to its
// mean is kappa |mu - w| (DESIGN C-A33), so the ~1e-6 error of the fast path
// would exceed the 1e-3 pdf tolerance at kappa ~ 1e5.  The training heads use
// PRECISE = false: the gradient tolerance is rel-L2 and the branch cost the
// c2 train kernel 2.7 % (B200 A/B).
template <bool PRECISE = true>
__device__ __forceinline__ void lobe_angles(float tp, float pp, float kap, float& th, float& ph, float& sth,
                                            float& cth, float& sph, float& cph) {
  th = fast_sigmoid(tp);
  ph = fast_sigmoid(pp);
  __sincosf(kPi * th, &sth, &cth);
  __sincosf(kTwoPi * ph, &sph, &cph);
  if (PRECISE && kap > 1e3f) {
    th = 1.0f / (1.0f + expf(-tp));
    ph = 1.0f / (1.0f + expf(-pp));
    sincospif(th, &sth, &cth);
    sincospif(2.0f * ph, &sph, &cph);
  }
}
// kappa / (2 pi (1 - e^{-2 kappa})) with em = -expm1(-2 kappa) returned for reuse
// 1 - e^{-x} for x >= 0 without the branches of expm1f: an 8-term Taylor
// polynomial below x = 0.7 (truncation < 1.2e-7 relative) and MUFU ex2 above
// (where 1 - e^{-x} >= 0.5, so its ~1e-7 absolute error stays relative).
__device__ __forceinline__ float one_minus_exp_neg(float x) {
  const float p =
      x * (1.0f - x * (0.5f - x * (1.6666667e-1f - x * (4.1666668e-2f - x * (8.3333338e-3f -
      x * (1.3888889e-3f - x * (1.9841270e-4f - x * 2.4801587e-5f)))))));
  return x < 0.7f ? p : 1.0f - __expf(-x);
}

__device__ __forceinline__ float lobe_norm(float kap, float& em) {
  em = -expm1f(-2.0f * kap);   // (the branch form of vmf_log_c: +0.9 % c2 query, B200 A/B)
  return __fdividef(kap, kTwoPi * em);
}
// Branch-free variant for the training head (B200: c2 train -0.7 %; in the
// query kernel it cost +3 % through register allocation, so it stays there).
__device__ __forceinline__ float lobe_norm_fast(float kap, float& em) {
  em = one_minus_exp_neg(2.0f * kap);
  return __fdividef(kap, kTwoPi * em);
}
__device__ __forceinline__ float lobe_eval(float norm, float kap, float mx, float my, float mz, float wx, float wy,
                                           float wz) {
  const float dx = mx - wx, dy = my - wy, dz = mz - wz;
  return norm * __expf(-0.5f * kap * (dx * dx + dy * dy + dz * dz));
}

// Stable Eq. 3 (C-O9): kappa / (2 pi (1 - e^{-2 kappa})) exp(-kappa |mu - w|^2 / 2).
__device__ __forceinline__ float lobe_pdf(float kap, float mx, float my, float mz, float wx, float wy, float wz) {
  const float dx = mx - wx, dy = my - wy, dz = mz - wz;
  const float d2 = dx * dx + dy * dy + dz * dz;
  return kap / (kTwoPi * (-expm1f(-2.0f * kap))) * expf(-0.5f * kap * d2);
}

template <int K>
__device__ __forceinline__ float mixture_pdf(const Mixture<K>& m, float wx, float wy, float wz) {
  float v = 0.0f;
#pragma unroll
  for (int i = 0; i < K; ++i) v += m.lam[i] * lobe_pdf(m.kap[i], m.mx[i], m.my[i], m.mz[i], wx, wy, wz);
  return v;
}

__device__ __forceinline__ void lobe_sample(float kap, float mux, float muy, float muz, float u2, float u3,
                                            float& wx, float& wy, float& wz);

// Jakob 2012 stable vMF inversion in the Duff et al. ONB (C-O10).
template <int K>
__device__ __forceinline__ void mixture_sample(const Mixture<K>& m, float u1, float u2, float u3,
                                               float& wx, float& wy, float& wz) {
  // i* = min{i : u1 < C_i}, C_i = sum_{j<=i} lambda_j; K-1 if none (C-A17)
  int sel = K - 1;
  bool found = false;
  float cdf = 0.0f;
#pragma unroll
  for (int i = 0; i < K; ++i) {
    cdf += m.lam[i];
    if (!found && u1 < cdf) { sel = i; found = true; }
  }
  float kap = m.kap[0], mux = m.mx[0], muy = m.my[0], muz = m.mz[0];
#pragma unroll
  for (int i = 1; i < K; ++i)
    if (sel == i) { kap = m.kap[i]; mux = m.mx[i]; muy = m.my[i]; muz = m.mz[i]; }
  lobe_sample(kap, mux, muy, muz, u2, u3, wx, wy, wz);
}

// One vMF lobe sampled from (u2, u3): Jakob 2012 inversion of the cosine to
// mu + azimuth 2 pi u3 in the Duff et al. ONB (C-O10).
__device__ __forceinline__ void lobe_sample(float kap, float mux, float muy, float muz, float u2, float u3,
                                            float& wx, float& wy, float& wz) {
  // delta = -log(u2 + (1 - u2) e^{-2 kappa}) / kappa  (Jakob 2012, C-O10), evaluated in fp32
  // in whichever of two equal forms is well conditioned: log1p of
  // x = (1 - u2) expm1(-2 kappa) while 1 + x >= 1/2, else log of 1 + x formed
  // directly as u2 + (1 - u2) e^{-2 kappa} (keeps full precision when u2 -> 0).
  const float x = (1.0f - u2) * expm1f(-2.0f * kap);
  const float lg = x > -0.5f ? log1pf(x) : logf(u2 + (1.0f - u2) * expf(-2.0f * kap));
  const float delta = fminf(-lg / kap, 2.0f);
  // 2 - delta = log1p(u2 expm1(2 kappa)) / kappa, the same quantity evaluated so
  // that it stays accurate where delta -> 2 (u2 -> 0): r = sqrt(delta (2 - delta))
  // has an infinite derivative there.  expm1(2 kappa) overflows only for
  // kappa > ~44, where delta is near 2 only at u2 = 0 (then 2 - delta = 0).
  const float e2k = expm1f(2.0f * kap);
  const float eps = isfinite(e2k) ? fminf(log1pf(u2 * e2k) / kap, 2.0f) : 2.0f - delta;
  const float w = 1.0f - delta;
  const float r = sqrtf(fmaxf(delta * eps, 0.0f));
  const float s = copysignf(1.0f, muz);
  const float a = -1.0f / (s + muz);
  const float b = mux * muy * a;
  const float t1x = 1.0f + s * mux * mux * a, t1y = s * b, t1z = -s * mux;
  const float t2x = b, t2y = s + muy * muy * a, t2z = -muy;
  float sp, cp;
  sincospif(2.0f * u3, &sp, &cp);
  wx = w * mux + r * (cp * t1x + sp * t2x);
  wy = w * muy + r * (cp * t1y + sp * t2y);
  wz = w * muz + r * (cp * t1z + sp * t2z);
}

// log C(kappa), C(kappa) = kappa / (2 pi (1 - e^{-2 kappa})) the vMF normaliser
// of the stable form (C-O9); C(0) = 1 / (4 pi) (C-A28).
__device__ __forceinline__ float vmf_log_c(float k) {
  // 1 - e^{-2k}: precise expm1 only where it matters (small k); MUFU elsewhere
  const float em = k < 0.35f ? -expm1f(-2.0f * k) : 1.0f - __expf(-2.0f * k);
  const float r = k > 0.0f ? __fdividef(k, em) : 0.5f;
  return __logf(r) - 1.8378770664093453f;   // log(2 pi)
}

// Closed-form product of lobe (mu, kappa) with (n, kc) (f-2):
// kappa_p mu_p = kappa mu + kc n; returns log of the scale s in
// v v_c = s v(. | mu_p, kappa_p) and overwrites (mu, kappa) with the product.
__device__ __forceinline__ float vmf_product_inplace(float& mx, float& my, float& mz, float& kap, float nx, float ny,
                                                     float nz, float kc, float log_c_kc) {
  const float sx = kap * mx + kc * nx, sy = kap * my + kc * ny, sz = kap * mz + kc * nz;
  const float kp = sqrtf(sx * sx + sy * sy + sz * sz);
  const float ls = vmf_log_c(kap) + log_c_kc - vmf_log_c(kp) + (kp - kap - kc);
  if (kp > 0.0f) {
    const float inv = 1.0f / kp;
    mx = sx * inv; my = sy * inv; mz = sz * inv;
  } else {
    mx = nx; my = ny; mz = nz;   // uniform product (C-A28)
  }
  kap = fmaxf(kp, 1e-30f);   // keeps the sampler's -log(.)/kappa finite at kappa_p = 0
  return ls;
}

// BSDF stand-in (C-A24, f-1): Lambertian about the unit shading normal n.
// pdf max(n.w, 0) / pi; cosine-weighted sample r = sqrt(u1), phi = 2 pi u2,
// local (r cos phi, r sin phi, sqrt(1 - u1)) in the Duff ONB of n.
__device__ __forceinline__ float bsdf_pdf(float nx, float ny, float nz, float wx, float wy, float wz) {
  return fmaxf(nx * wx + ny * wy + nz * wz, 0.0f) * 0.31830988618379067f;
}

__device__ __forceinline__ void bsdf_sample(float nx, float ny, float nz, float u1, float u2, float& wx, float& wy,
                                            float& wz) {
  const float r = sqrtf(u1), lz = sqrtf(fmaxf(1.0f - u1, 0.0f));
  float sp, cp;
  sincospif(2.0f * u2, &sp, &cp);
  const float s = copysignf(1.0f, nz);
  const float a = -1.0f / (s + nz);
  const float b = nx * ny * a;
  const float t1x = 1.0f + s * nx * nx * a, t1y = s * b, t1z = -s * nx;
  const float t2x = b, t2y = s + ny * ny * a, t2z = -ny;
  const float lx = r * cp, ly = r * sp;
  wx = lx * t1x + ly * t2x + lz * nx;
  wy = lx * t1y + ly * t2y + lz * ny;
  wz = lx * t1z + ly * t2z + lz * nz;
}

// Eq. 9 head (C-O13): d loss / d raw for one record, multiplied by s.
// Returns log max(V, 1e-30).
template <int K>
__device__ __forceinline__ float grad_head(const float* raw, float log_kmin, float log_kmax,
                                           float wx, float wy, float wz, float s, float* draw) {
  Mixture<K> m;
  activate<K>(raw, log_kmin, log_kmax, m);
  float v[K];
  float V = 0.0f;
#pragma unroll
  for (int i = 0; i < K; ++i) {
    v[i] = lobe_pdf(m.kap[i], m.mx[i], m.my[i], m.mz[i], wx, wy, wz);
    V += m.lam[i] * v[i];
  }
  const float Vb = fmaxf(V, kVFloor);
  const float invV = 1.0f / Vb;
#pragma unroll
  for (int i = 0; i < K; ++i) {
    const float gam = m.lam[i] * v[i] * invV;
    draw[i] = s * (gam - m.lam[i]);
    const float kap = m.kap[i];
    const float kr = raw[K + i];
    const float dx = m.mx[i] - wx, dy = m.my[i] - wy, dz = m.mz[i] - wz;
    const float d2 = dx * dx + dy * dy + dz * dz;
    const float em = -expm1f(-2.0f * kap);
    float dk = s * gam * (1.0f - kap * 0.5f * d2 - 2.0f * kap * expf(-2.0f * kap) / em);
    draw[K + i] = (kr < log_kmin || kr > log_kmax) ? 0.0f : dk;
    const float th = 1.0f / (1.0f + expf(-raw[2 * K + i]));
    const float ph = 1.0f / (1.0f + expf(-raw[3 * K + i]));
    float st, ct, sp, cp;
    sincospif(th, &st, &ct);
    sincospif(2.0f * ph, &sp, &cp);
    const float wdth = kPi * (ct * cp * wx + ct * sp * wy - st * wz);
    const float wdph = kTwoPi * (-st * sp * wx + st * cp * wy);
    const float sgk = s * gam * kap;
    draw[2 * K + i] = sgk * wdth * th * (1.0f - th);
    draw[3 * K + i] = sgk * wdph * ph * (1.0f - ph);
  }
  return logf(Vb);
}

}  // namespace npm
