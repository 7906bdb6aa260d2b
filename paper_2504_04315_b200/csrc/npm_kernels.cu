// npm_kernels.cu -- shape-independent kernels (encode-only, Adam + EMA,
// initialisation) and the decoder-shape dispatch over the per-shape
// translation units npm_net_*.cu.
#include "npm_kernels_impl.cuh"
#include <type_traits>

namespace npm {
namespace detail {
// Adam + EMA (C-O17, C-O18); zeroes the gradient buffer.
__global__ void __launch_bounds__(256) adam_kernel(AdamArgs a) {
  // float4 per thread; n_mlp and n_total are multiples of 4, so a vector is
  // entirely MLP or entirely grid.  Untouched grid vectors (all g == 0) read
  // only g, p, e and write only e.
  double gn = 0.0;
  unsigned nf = 0;
  const int64_t n4 = a.n_total / 4;
  float4* g4 = reinterpret_cast<float4*>(a.g);
  float4* p4 = reinterpret_cast<float4*>(a.p);
  float4* m4 = reinterpret_cast<float4*>(a.m);
  float4* v4 = reinterpret_cast<float4*>(a.v);
  float4* e4 = reinterpret_cast<float4*>(a.e);
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n4; j += (int64_t)gridDim.x * blockDim.x) {
    float4 gv = g4[j];
    float g[4] = {gv.x, gv.y, gv.z, gv.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (!isfinite(g[q])) { g[q] = 0.0f; nf += 1; }
      gn += (double)g[q] * (double)g[q];
    }
    const bool grid = 4 * j >= a.n_mlp;
    const bool any = g[0] != 0.0f || g[1] != 0.0f || g[2] != 0.0f || g[3] != 0.0f;
    float4 pv = p4[j];
    float p[4] = {pv.x, pv.y, pv.z, pv.w};
    if (!grid || any) {
      const float4 mv = m4[j], vv = v4[j];
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
    const float4 ev = e4[j];
    e4[j] = make_float4(a.decay * ev.x + (1.0f - a.decay) * p[0], a.decay * ev.y + (1.0f - a.decay) * p[1],
                        a.decay * ev.z + (1.0f - a.decay) * p[2], a.decay * ev.w + (1.0f - a.decay) * p[3]);
  }
  gn = warp_sum_d(gn);
  nf = warp_sum_u(nf);
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(a.gnorm, gn);
    if (nf) atomicAdd(a.nonfinite, (unsigned long long)nf);
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
  int net_query_##TAG(const QueryArgs&, int, cudaStream_t);                        \
  int net_train_fwd_##TAG(const TrainArgs&, int, cudaStream_t);                    \
  int net_train_bwd_##TAG(const TrainArgs&, int, cudaStream_t);                    \
  int net_dw_##TAG(const TrainArgs&, int, cudaStream_t);                           \
  int net_smem_##TAG();                                                             \
  int net_query_tc_##TAG(const QueryArgs&, int, cudaStream_t);                     \
  int net_train_tc_##TAG(const TrainArgs&, int, cudaStream_t);
NPM_DECLARE_NET(c1)
NPM_DECLARE_NET(c2)
NPM_DECLARE_NET(c5)
NPM_DECLARE_NET(p16)
#undef NPM_DECLARE_NET

namespace {
enum Op { kQuery, kTrainFwd, kTrainBwd, kDw, kSmem, kQueryTc, kTrainTc };

template <class Args>
int call(const NetShape& s, Op op, const Args* a, int sms, cudaStream_t st) {
#define NPM_CASE(TAG, NIN, W, NL, NOUT, PROD)                                                          \
  if (s.n_in == NIN && s.width == W && s.n_layers == NL && s.n_out == NOUT && s.product == PROD) {     \
    if constexpr (std::is_same<Args, QueryArgs>::value) {                                              \
      if (op == kQuery) return net_query_##TAG(*a, sms, st);                                           \
      if (op == kQueryTc) return net_query_tc_##TAG(*a, sms, st);                                      \
    } else if constexpr (std::is_same<Args, TrainArgs>::value) {                                       \
      if (op == kTrainFwd) return net_train_fwd_##TAG(*a, sms, st);                                    \
      if (op == kTrainBwd) return net_train_bwd_##TAG(*a, sms, st);                                    \
      if (op == kDw) return net_dw_##TAG(*a, sms, st);                                                 \
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

int launch_query(const NetShape& s, const QueryArgs& a, int sms, cudaStream_t st) {
  if (a.n == 0) return 0;
  return call(s, kQuery, &a, sms, st);
}
int launch_query_tc(const NetShape& s, const QueryArgs& a, int sms, cudaStream_t st) {
  if (a.n == 0) return 0;
  return call(s, kQueryTc, &a, sms, st);
}
int launch_train_tc(const NetShape& s, const TrainArgs& a, int sms, cudaStream_t st) {
  if (a.n == 0) return 0;
  return call(s, kTrainTc, &a, sms, st);
}
int launch_train_forward(const NetShape& s, const TrainArgs& a, int sms, cudaStream_t st) {
  if (a.n == 0) return 0;
  return call(s, kTrainFwd, &a, sms, st);
}
int launch_train_backward(const NetShape& s, const TrainArgs& a, int sms, cudaStream_t st) {
  if (a.n == 0) return 0;
  return call(s, kTrainBwd, &a, sms, st);
}
int launch_weight_grads(const NetShape& s, const TrainArgs& a, int sms, cudaStream_t st) {
  if (a.n == 0) return 0;
  return call(s, kDw, &a, sms, st);
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

int launch_adam(const AdamArgs& a, int sms, cudaStream_t st) {
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
