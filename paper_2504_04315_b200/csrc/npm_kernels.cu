// npm_kernels.cu -- shape-independent kernels (encode-only, Adam + EMA,
// initialisation) and the decoder-shape dispatch over the per-shape
// translation units npm_net_*.cu.
#include "npm_kernels_impl.cuh"
#include <type_traits>

namespace npm {
namespace detail {
// EMA blend (C-O18) with a pinned operation order, shared by adam_kernel and
// ema_kernel so the ZeRO-1 schedule (Adam on a shard, EMA after the gather)
// reproduces the fused update bit for bit.
__device__ __forceinline__ float ema_blend(float d, float e, float p) {
  return __fmaf_rn(d, e, __fmul_rn(1.0f - d, p));
}

// Adam + EMA (C-O17, C-O18); zeroes the gradient buffer.
__global__ void __launch_bounds__(256) adam_kernel(AdamArgs a) {
  // float4 per thread; n_mlp and n_total are multiples of 4, so a vector is
  // entirely MLP or entirely grid.  Untouched grid vectors (all g == 0) read
  // only g, p, e and write only e.
  double gn = 0.0;
  unsigned nf = 0;
  const int64_t n4 = a.n_total / 4;
  // the five buffers never alias; g, p, e are loaded before any store (one
  // HBM round trip per vector; m, v only for touched vectors)
  float4* __restrict__ g4 = reinterpret_cast<float4*>(a.g);
  float4* __restrict__ p4 = reinterpret_cast<float4*>(a.p);
  float4* __restrict__ m4 = reinterpret_cast<float4*>(a.m);
  float4* __restrict__ v4 = reinterpret_cast<float4*>(a.v);
  float4* __restrict__ e4 = reinterpret_cast<float4*>(a.e);
  auto body = [&](int64_t j, const float4 gv, const float4 pv, const float4 ev) {
    float g[4] = {gv.x, gv.y, gv.z, gv.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (!isfinite(g[q])) { g[q] = 0.0f; nf += 1; }
      gn += (double)g[q] * (double)g[q];
    }
    const bool grid = 4 * j >= a.n_mlp && 4 * j < a.grid_end;
    const bool any = g[0] != 0.0f || g[1] != 0.0f || g[2] != 0.0f || g[3] != 0.0f;
    float p[4] = {pv.x, pv.y, pv.z, pv.w};
    if (!grid || any) {
      const float4 mv = m4[j], vv = v4[j];   // (evict-first hints on m, v: c5 925 -> 1190 us)
      float m[4] = {mv.x, mv.y, mv.z, mv.w}, v[4] = {vv.x, vv.y, vv.z, vv.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (grid && g[q] == 0.0f) continue;     // untouched grid entry
        m[q] = a.beta1 * m[q] + (1.0f - a.beta1) * g[q];
        v[q] = a.beta2 * v[q] + (1.0f - a.beta2) * g[q] * g[q];
        p[q] = p[q] - a.lr * (m[q] * a.c1) / (sqrtf(v[q] * a.c2) + a.eps);
      }
      m4[j] = make_float4(m[0], m[1], m[2], m[3]);
      v4[j] = make_float4(v[0], v[1], v[2], v[3]);
      p4[j] = make_float4(p[0], p[1], p[2], p[3]);
      g4[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    } else if (gv.x != 0.0f || gv.y != 0.0f || gv.z != 0.0f || gv.w != 0.0f) {
      g4[j] = make_float4(0.f, 0.f, 0.f, 0.f);   // non-finite entries zeroed
    }
    if (a.ema)
      __stcs(e4 + j, make_float4(ema_blend(a.decay, ev.x, p[0]), ema_blend(a.decay, ev.y, p[1]),
                                 ema_blend(a.decay, ev.z, p[2]), ema_blend(a.decay, ev.w, p[3])));
  };
  // one float4 per thread per iteration (measured on B200: two per iteration
  // with all loads hoisted was slower, c5 925 -> 1180 us)
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n4; j += (int64_t)gridDim.x * blockDim.x)
    body(j, g4[j], p4[j], a.ema ? __ldcs(e4 + j) : make_float4(0.f, 0.f, 0.f, 0.f));
  // block reduction, then one atomic per block: per-warp double atomics on
  // one address serialise at its L2 slice (~19 k per c2 step)
  __shared__ double sgn[8];
  __shared__ unsigned snf[8];
  gn = warp_sum_d(gn);
  nf = warp_sum_u(nf);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { sgn[w] = gn; snf[w] = nf; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    unsigned u = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) { t += sgn[i]; u += snf[i]; }
    atomicAdd(a.gnorm, t);
    if (u) atomicAdd(a.nonfinite, (unsigned long long)u);
  }
}

// Training-record unwind (f-1): <L_i(x_v)> = L_e[v] + f_s cos / p~ at v + 1 times
// <L_i(x_{v+1})>, backward along each path; a successor
// with p~ <= 0 or non-finite ends the path (C-A27); v >= depth -> 0.
// D^ = <L_i> (radiance) or f_s <L_i> cos (product, Eq. 12).  Thread per path;
// every [.][v][n] access is coalesced over paths.  For D <= MAXD a path's
// cos / pdf and then each channel's le / fs are loaded into registers before
// the (sequential) recurrence, so the loads of all vertices are in flight at
// once (a path batch has few threads: n = records / D).  128-thread CTAs,
// >= 7 per SM (<= 72 registers): a c2 frame (115,200 8-vertex paths) runs as
// one wave of one path per thread (the all-channels-at-once form took 255
// registers for MAXD = 8: one CTA per SM, three grid-stride rounds, 26.6 us).
template <int MAXD>
__global__ void __launch_bounds__(128, 7) unwind_kernel(UnwindArgs a) {
  const int64_t n = a.n;
  const int D = a.max_depth, C = a.channels;
  const float* __restrict__ le = a.le;
  const float* __restrict__ fs = a.fs;
  const float* __restrict__ cosv = a.cosv;
  const float* __restrict__ pdf = a.pdf;
  float* __restrict__ out = a.target;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    const int d = min(max(__ldg(a.depth + p), 0), D);
    // the path's cos / pdf, then one channel at a time (its le / fs loads all
    // in flight; 2 x MAXD + 2 x MAXD values in registers instead of 8 x MAXD)
    float cs[MAXD], pd[MAXD];
#pragma unroll
    for (int v = 0; v < MAXD; ++v) {
      const int64_t at = (int64_t)v * n + p;
      const bool in = v < d;
      cs[v] = in ? __ldg(cosv + at) : 0.0f;
      pd[v] = in ? __ldg(pdf + at) : 0.0f;
    }
#pragma unroll 1
    for (int c = 0; c < C; ++c) {
      float L[MAXD], F[MAXD];
#pragma unroll
      for (int v = 0; v < MAXD; ++v) {
        const int64_t at = (int64_t)c * D * n + (int64_t)v * n + p;
        const bool in = v < d;
        L[v] = in ? __ldg(le + at) : 0.0f;
        F[v] = in ? __ldg(fs + at) : 0.0f;
      }
      float li = 0.0f;
#pragma unroll
      for (int v = MAXD - 1; v >= 0; --v) {
        if (v >= D) continue;
        const int vn = v + 1 < MAXD ? v + 1 : v;
        const float q = v + 1 < MAXD ? pd[vn] : 0.0f;   // p~ at the successor
        const bool cont = v + 1 < d && isfinite(q) && q > 0.0f;
        float acc = L[v];
        if (cont) acc += __fdiv_rn(F[vn] * cs[vn], q) * li;
        li = v < d ? acc : 0.0f;
        out[(int64_t)c * D * n + (int64_t)v * n + p] = a.product ? F[v] * li * cs[v] : li;
      }
    }
  }
}

// Same recurrence for long paths (D > 32), one vertex at a time.
__global__ void __launch_bounds__(256) unwind_long_kernel(UnwindArgs a) {
  const int64_t n = a.n;
  const int D = a.max_depth, C = a.channels;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    const int d = min(max(__ldg(a.depth + p), 0), D);
    float li[3] = {0.f, 0.f, 0.f};
    for (int v = D - 1; v >= 0; --v) {
      const int64_t at = (int64_t)v * n + p;
      if (v >= d) {
        for (int c = 0; c < C; ++c) a.target[(int64_t)c * D * n + at] = 0.0f;
        continue;
      }
      const float q = v + 1 < d ? __ldg(a.pdf + at + n) : 0.0f;
      const bool cont = isfinite(q) && q > 0.0f;
      const float cs = cont ? __ldg(a.cosv + at + n) : 0.0f;
      for (int c = 0; c < C; ++c) {
        const int64_t ca = (int64_t)c * D * n + at;
        float acc = __ldg(a.le + ca);
        if (cont) acc += __fdiv_rn(__ldg(a.fs + ca + n) * cs, q) * li[c];   // (f_s cos) / p~ * Li
        li[c] = acc;
        a.target[ca] = a.product ? __ldg(a.fs + ca) * acc * __ldg(a.cosv + at) : acc;
      }
    }
  }
}

// Initialisation (C-A21): Xavier-uniform weights, zero biases, features
// U(-1e-2, 1e-2); uniforms from Philox keyed by the init seed.
__global__ void init_kernel(float* p, int64_t n_mlp, int64_t n_total, uint64_t seed, int nl, int4 dims_in,
                            int4 dims_out) {
  const int ins[3] = {dims_in.x, dims_in.y, dims_in.z};
  const int outs[3] = {dims_out.x, dims_out.y, dims_out.z};
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n_total; j += (int64_t)gridDim.x * blockDim.x) {
    const float u = philox_uniforms(seed, (uint64_t)j).x;
    if (j >= n_mlp) { p[j] = (2.0f * u - 1.0f) * 1e-2f; continue; }
    int64_t off = 0;
    float val = 0.0f;
    for (int k = 0; k < nl; ++k) {
      const int64_t nw = (int64_t)ins[k] * outs[k];
      if (j < off + nw) { const float lim = sqrtf(6.0f / (ins[k] + outs[k])); val = (2.0f * u - 1.0f) * lim; break; }
      off += nw;
      if (j < off + outs[k]) { val = 0.0f; break; }
      off += outs[k];
    }
    p[j] = val;
  }
}

}  // namespace detail

using namespace detail;

// Per-shape entry points, defined in npm_net_*.cu.
#define NPM_DECLARE_NET(TAG)                                                         \
  int net_smem_##TAG();                                                             \
  int net_query_tc_##TAG(const QueryArgs&, int, cudaStream_t);                     \
  int net_train_tc_##TAG(const TrainArgs&, int, cudaStream_t);
NPM_DECLARE_NET(c1)
NPM_DECLARE_NET(c2)
NPM_DECLARE_NET(c5)
NPM_DECLARE_NET(p16)
#undef NPM_DECLARE_NET

namespace {
enum Op { kSmem, kQueryTc, kTrainTc };

template <class Args>
int call(const NetShape& s, Op op, const Args* a, int sms, cudaStream_t st) {
#define NPM_CASE(TAG, NIN, W, NL, NOUT, PROD)                                                          \
  if (s.n_in == NIN && s.width == W && s.n_layers == NL && s.n_out == NOUT && s.product == PROD) {     \
    if constexpr (std::is_same<Args, QueryArgs>::value) {                                              \
      if (op == kQueryTc) return net_query_tc_##TAG(*a, sms, st);                                      \
    } else if constexpr (std::is_same<Args, TrainArgs>::value) {                                       \
      if (op == kTrainTc) return net_train_tc_##TAG(*a, sms, st);                                      \
    }                                                                                                  \
    if (op == kSmem) return net_smem_##TAG();                                                          \
    return -1;                                                                                         \
  }
  NPM_CASE(c1, 16, 32, 2, 32, false)
  NPM_CASE(c2, 32, 64, 3, 32, false)
  NPM_CASE(c5, 64, 64, 3, 32, false)
  NPM_CASE(p16, 65, 64, 3, 64, true)
#undef NPM_CASE
  return -1;
}
}  // namespace

bool shape_supported(const NetShape& s) { return call<int>(s, kSmem, nullptr, 0, 0) > 0; }
size_t weight_smem_bytes(const NetShape& s) {
  const int r = call<int>(s, kSmem, nullptr, 0, 0);
  return r < 0 ? 0 : (size_t)r;
}

int launch_query_tc(const NetShape& s, const QueryArgs& a, int sms, cudaStream_t st) {
  if (a.n == 0) return 0;
  return call(s, kQueryTc, &a, sms, st);
}
int launch_train_tc(const NetShape& s, const TrainArgs& a, int sms, cudaStream_t st) {
  if (a.n == 0) return 0;
  return call(s, kTrainTc, &a, sms, st);
}

int launch_encode(int L, const QueryArgs& a, int sms, cudaStream_t st) {
  if (a.n == 0) return 0;
  const int64_t need = (a.n + kThreads - 1) / kThreads;
  const int blocks = (int)(need < (int64_t)sms * 16 ? need : (int64_t)sms * 16);
  switch (L) {
#define NPM_L(LL) case LL: encode_kernel<LL><<<blocks, kThreads, 0, st>>>(a); return 1;
    NPM_L(1) NPM_L(2) NPM_L(3) NPM_L(4) NPM_L(5) NPM_L(6) NPM_L(7) NPM_L(8)
    NPM_L(9) NPM_L(10) NPM_L(11) NPM_L(12) NPM_L(13) NPM_L(14) NPM_L(15) NPM_L(16)
#undef NPM_L
    default: return -1;
  }
}

// thread (e, s): entry e, copies b = s, s + S, ... (all loads in flight),
// then one v4 reduction into the gradient; copies re-zeroed in the same pass
constexpr int kFoldSlices = 8;
__global__ void __launch_bounds__(256) fold_priv_kernel(FoldArgs a) {
  const int64_t total = a.priv_stride * kFoldSlices;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = t / kFoldSlices;
    const int sl = (int)(t % kFoldSlices);
    float4* __restrict__ base = a.priv + e;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    constexpr int U = 8;
    for (int b0 = sl; b0 < a.ctas; b0 += U * kFoldSlices) {
      float4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int b = b0 + u * kFoldSlices;
        v[u] = b < a.ctas ? base[(int64_t)b * a.priv_stride] : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int b = b0 + u * kFoldSlices;
        if (b < a.ctas) base[(int64_t)b * a.priv_stride] = make_float4(0.f, 0.f, 0.f, 0.f);
        acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w;
      }
    }
    int l = 0;
    while (l + 1 < a.nlev && e >= a.lev_priv_off[l + 1]) ++l;
    float4* g = reinterpret_cast<float4*>(a.grads) + a.lev_grid_off[l] + (e - a.lev_priv_off[l]);
    atomicAdd(g, acc);
  }
}

int launch_fold_priv(const FoldArgs& a, int sms, cudaStream_t st) {
  if (a.priv_stride == 0) return 0;
  const int64_t need = (a.priv_stride * kFoldSlices + 255) / 256;
  const int blocks = (int)(need < (int64_t)sms * 8 ? need : (int64_t)sms * 8);
  fold_priv_kernel<<<blocks, 256, 0, st>>>(a);
  return 1;
}

int launch_unwind(const UnwindArgs& a, int sms, cudaStream_t st) {
  if (a.n == 0 || a.max_depth == 0) return 0;
  if (a.max_depth > 16) {
    const int64_t need = (a.n + 255) / 256;
    const int blocks = (int)(need < (int64_t)sms * 8 ? need : (int64_t)sms * 8);
    unwind_long_kernel<<<blocks, 256, 0, st>>>(a);
    return 1;
  }
  const int64_t need = (a.n + 127) / 128;
  const int blocks = (int)(need < (int64_t)sms * 7 ? need : (int64_t)sms * 7);   // one wave
  if (a.max_depth <= 4) unwind_kernel<4><<<blocks, 128, 0, st>>>(a);
  else if (a.max_depth <= 8) unwind_kernel<8><<<blocks, 128, 0, st>>>(a);
  else unwind_kernel<16><<<blocks, 128, 0, st>>>(a);
  return 1;
}

// EMA e <- d e + (1 - d) p (C-O18) over n floats (n % 4 == 0), float4 per thread.
__global__ void __launch_bounds__(256) ema_kernel(float4* __restrict__ e, const float4* __restrict__ p, int64_t n4,
                                                  float d) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n4; j += (int64_t)gridDim.x * blockDim.x) {
    const float4 ev = __ldcs(e + j), pv = p[j];
    __stcs(e + j, make_float4(ema_blend(d, ev.x, pv.x), ema_blend(d, ev.y, pv.y), ema_blend(d, ev.z, pv.z),
                              ema_blend(d, ev.w, pv.w)));
  }
}

int launch_ema(float* e, const float* p, int64_t n, float decay, int sms, cudaStream_t st) {
  if (n <= 0) return 0;
  const int64_t need = (n / 4 + 255) / 256;
  const int blocks = (int)(need < (int64_t)sms * 16 ? need : (int64_t)sms * 16);
  ema_kernel<<<blocks, 256, 0, st>>>(reinterpret_cast<float4*>(e), reinterpret_cast<const float4*>(p), n / 4, decay);
  return 1;
}

int launch_adam(const AdamArgs& a, int sms, cudaStream_t st) {
  if (a.n_total <= 0) return 0;
  const int64_t need = (a.n_total / 4 + 255) / 256;
  const int blocks = (int)(need < (int64_t)sms * 16 ? need : (int64_t)sms * 16);
  adam_kernel<<<blocks, 256, 0, st>>>(a);
  return 1;
}

int launch_init_params(float* p, int64_t n_mlp, int64_t n_total, const NetShape& s, uint64_t seed,
                       cudaStream_t st) {
  int4 din = make_int4(s.n_in, s.width, s.width, 0);
  int4 dout = make_int4(s.width, s.n_layers == 2 ? s.n_out : s.width, s.n_out, 0);
  init_kernel<<<592, 256, 0, st>>>(p, n_mlp, n_total, seed, s.n_layers, din, dout);
  return 1;
}

}  // namespace npm
