// npm_kernels.cuh -- launch interface between the C ABI (npm_capi.cu) and the
// sm_100a kernels.  Internal header: not part of the public ABI.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "npm_device.cuh"

namespace npm {

// Decoder shape (C-A5): n_in -> width (x n_layers-1) -> 4K.
struct NetShape {
  int n_in, width, n_layers, n_out;  // n_out = 4K
  bool product;
};

struct QueryArgs {
  int64_t n;
  const uint32_t* perm;     // optional processing order (spatial binning); NULL = identity
  const float *px, *py, *pz, *wox, *woy, *woz, *nx, *ny, *nz, *rough;
  const float* params;      // live or EMA flat parameter buffer
  GridDesc grid;
  float log_kmin, log_kmax;
  // encode-only outputs
  float* feat;              // [L*F][n]
  uint32_t* dbg_idx;        // [L][8][n]
  float* dbg_w;             // [L][8][n]
  // decode
  const float* feat_in;     // optional [L*F][n] input instead of G(x)
  float *raw, *lambda, *kappa, *mu;
  // pdf at caller directions
  const float *wx, *wy, *wz;
  float* pdf;
  // sampling
  int do_sample;
  const float* u;           // [3][n] or NULL -> Philox
  uint64_t seed, offset;
  float *sx, *sy, *sz, *spdf;
  // combined BSDF / guide sampling (f-1; C-A24..C-A26): u is [4][n] then
  int combined;
  float alpha;                        // BSDF selection probability
  const float *bnx, *bny, *bnz;       // unit shading normals (BSDF stand-in)
  float* gpdf;                        // V(w) at the returned direction (0 on fallback), optional
  int32_t* tech;                      // 0 BSDF, 1 guide, 2 fallback; optional
  // cosine-lobe product (f-2, C-A28/C-A29): the decoded mixture times
  // v(. | n, kappa_c), renormalised, before sampling / pdf; normals in bnx..
  int cos_product;
  float kappa_c, log_c_kc;            // kappa_c and log C(kappa_c) (host-computed)
  int query_groups;                   // 1: two 256-thread CTAs per SM; 2: one CTA, two groups (NPM_QUERY_GROUPS)
  long long* dbg_clock;               // measurement builds (-DNPM_QUERY_STAMPS): [64 tiles][16] stamps of CTA 0
  const float* alpha_w;               // C-A34 selection head (a [W], c) of `params`, or NULL: use `alpha`
  int qws;                            // warp-specialised kernel for plain sample / pdf calls (NPM_QUERY_WS)
  int qws_groups;                     // its chain groups for plain calls: 1 or 2 (NPM_QWS_GROUPS)
};

struct TrainArgs {
  int64_t n;
  const uint32_t* perm;     // optional processing order (spatial binning); NULL = identity
  const float *px, *py, *pz, *wox, *woy, *woz, *nx, *ny, *nz, *rough;
  const float *wx, *wy, *wz;
  const float* target;      // [C][target_stride] (channel c at target + c * target_stride)
  int64_t target_stride;    // = n unless the batch is a slice of a longer one (micro-steps)
  int divergence;           // 0 KL (Eq. 9), 1 Pearson chi^2 (f-4): record scale times D^ / V
  int channels;
  const float* spdf;        // p~
  double inv_n_global;
  const float* params;
  float* grads;
  GridDesc grid;
  float log_kmin, log_kmax;
  int debug;                // measurement knob (NPM_DEBUG): bit0 skip scatter, bit1 skip gathers,
                            // bit2 record per-phase clock64 stamps of CTA 0 into dbg_clock
  long long* dbg_clock;     // [64 tiles][16 stamps] (debug only)
  // Privatised coarse levels: levels in priv_mask scatter into the CTA's own
  // copy (priv + blockIdx.x * priv_stride + priv_off[l] entries) instead of
  // the shared gradient: every sample touches 8 of their few entries, and all
  // SMs' reductions on the same L2 lines serialise.  fold_priv adds the copies.
  float4* priv;
  uint32_t priv_mask;
  // split-bf16 weight image scratch (prep_wimg_kernel -> TMA bulk copy), and
  // the kernel choice: 1 = warp-specialised kernel where the shape has one
  uint8_t* wimg;
  uint32_t wimg_bytes;
  int ws;
  // C-A34 selection head (learn_alpha): its parameters / gradient (a [W], c)
  // and the records' BSDF pdf; alpha_w == NULL: no head
  const float* alpha_w;
  float* alpha_g;
  const float* bsdf_pdf;
  int64_t priv_stride;
  int64_t priv_off[16];
  double* stats;            // [0] loss, [1] unused, then int counters as double
  unsigned long long* counters;  // [0] used, [1] zero, [2] dropped
};

struct AdamArgs {
  int64_t n_mlp, n_total;   // of the range processed (a shard: n_mlp relative to its start)
  int64_t grid_end;         // grid entries are [n_mlp, grid_end) of the range (the C-A34 head follows)
  float *p, *g, *m, *v, *e;
  float lr, beta1, beta2, eps, decay, c1, c2;  // c1 = 1/(1-b1^t), c2 = 1/(1-b2^t)
  int ema;                  // 1: EMA in the same pass; 0: Adam only (ZeRO-1 shard, EMA after the all-gather)
  double* gnorm;
  unsigned long long* nonfinite;
};
// EMA over the whole parameter vector (C-O18), after a sharded Adam step.
int launch_ema(float* e, const float* p, int64_t n, float decay, int num_sms, cudaStream_t st);

bool shape_supported(const NetShape& s);
size_t weight_smem_bytes(const NetShape& s);

// Every launcher returns the number of kernels launched (>= 1) or -1 on error.
int launch_encode(int L, const QueryArgs& a, int num_sms, cudaStream_t st);  // a.params = grid section
int launch_adam(const AdamArgs& a, int num_sms, cudaStream_t st);

// Adds the per-CTA private copies of the privatised levels into the gradient
// (entry e of privatised block: grads[n_mlp + 4 goff(e) + f]) and re-zeroes them.
struct FoldArgs {
  float4* priv;
  int64_t priv_stride;      // entries per CTA copy
  int ctas;
  float* grads;             // + n_mlp: grid section
  int nlev;
  int64_t lev_priv_off[16], lev_grid_off[16], lev_entries[16];
};
int launch_fold_priv(const FoldArgs& a, int num_sms, cudaStream_t st);

// Training-record unwind (f-1, C-A27): one thread per path.
struct UnwindArgs {
  const float *le, *fs;     // [C][D][n]
  const float *cosv, *pdf;  // [D][n]
  const int32_t* depth;     // [n]
  float* target;            // [C][D][n]
  int channels, max_depth, product;
  int64_t n;
};
int launch_unwind(const UnwindArgs& a, int num_sms, cudaStream_t st);
// Fused tcgen05/TMEM decoder paths (npm_tc_kernels.cuh).
int launch_query_tc(const NetShape& s, const QueryArgs& a, int num_sms, cudaStream_t st);
int launch_train_tc(const NetShape& s, const TrainArgs& a, int num_sms, cudaStream_t st);
int launch_init_params(float* p, int64_t n_mlp, int64_t n_total, const NetShape& s, uint64_t seed,
                       cudaStream_t st);

}  // namespace npm

namespace npm {
// Spatial binning (npm_bin.cu): a counting sort of the samples by the Morton
// code of their cell in a 16^3 grid over the AABB, so that the 32 samples of a
// warp are spatially clustered and their grid gathers / scatter-adds touch
// few cache lines.  perm[t] = original index of the t-th processed sample.
#ifdef NPM_BIN_BITS   // measurement override (bins = 2^bits Morton cells; 12 = 16^3)
constexpr int kBinBits = NPM_BIN_BITS;
#else
constexpr int kBinBits = 12;
#endif
constexpr int64_t kSortChunk = 1 << 20;   // sort-chunk for L2-resident tables (npm_capi.cu)
int bin_hist_entries(int64_t n, int64_t sort_chunk);   // histogram entries launch_bin needs
int launch_bin(const float* px, const float* py, const float* pz, int64_t n, int64_t sort_chunk, bool refine,
               const GridDesc& g,
               uint32_t* keys, uint32_t* hist, uint32_t* perm, int num_sms, cudaStream_t st);
}  // namespace npm
