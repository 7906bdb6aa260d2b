/*
 * npm.h -- C ABI of the B200-native Neural Parametric Mixtures hot path.
 *
 * Paper: Dong, Wang, Li, "Neural Parametric Mixtures for Path Guiding",
 * arXiv 2504.04315.  Citations: P:n = line n of the paper's LaTeX source
 * with the section / equation named; C-xx = the reading recorded in
 * DESIGN.md ("Readings of the paper").
 *
 * The library evaluates and trains
 *
 *     NPM(x | Phi) = Theta_hat(x)                 (Eq. 6,  P:152-154)
 *     NPM_product(x, w_o | Phi) = Theta_hat(x, w_o) (Eq. 11)
 *     MLP(G(x | Phi_E) | Phi_M) = Theta_hat(x)    (Eq. 14)
 *
 * with G the multi-resolution grid embedding (Eq. 13), Theta_hat a
 * K-lobe vMF mixture (Eq. 3/4) after the Table 1 mappings
 * (P:166-179), trained with the Monte Carlo KL gradient (Eq. 9)
 * back-propagated through decoder and grid into Adam + EMA.
 *
 * ---------------------------------------------------------------------------
 * Conventions common to every call
 *   - Batches are structure-of-arrays ("structure-of-arrays (SoA) memory
 *     layout"): one float32 array per component, length n.
 *   - POINTERS MAY BE HOST OR DEVICE.  The library inspects every array
 *     pointer (cudaPointerGetAttributes).  Device (or managed) pointers are used
 *     in place.  Host pointers (pinned or pageable) are staged through
 *     library-owned device scratch: inputs copied host->device, outputs
 *     device->host, all on `stream`; the call then returns only after the
 *     output copies completed (pageable) or after they were enqueued (pinned
 *     host memory, still ordered on `stream`: synchronise `stream` before
 *     reading them).  Device pointers never cause a host synchronisation
 *     except where a host out-parameter (stats) is requested.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *     stream).  All work is enqueued on it, in call order.
 *   - Ownership: every array is caller-owned; outputs must not alias inputs.
 *     The model owns parameters, gradients, Adam moments, EMA shadow and
 *     scratch.
 *   - Errors: a bad argument returns NPM_ERR_INVALID with nothing enqueued; a
 *     CUDA failure returns NPM_ERR_CUDA (the model may then be unusable).
 *     npm_last_error() gives a thread-local message.  n == 0 is a no-op
 *     returning NPM_OK.  Data problems are NOT errors (see npm_train_step).
 *   - Concurrency: queries (encode/decode/pdf/sample) only read the model and
 *     may run concurrently with each other; a training call must not overlap
 *     queries on the same model (training happens between render waves).
 *     Batches of >= 65,536 samples are processed in a spatially binned order
 *     whose permutation lives in per-model scratch: a binning pass on one
 *     stream waits (cudaStreamWaitEvent) for the kernel that consumed the
 *     previous permutation, so device-pointer queries on different streams
 *     stay correct (their binned parts serialise on the GPU).
 *     Calls with HOST pointers stage through the model's scratch: issued on
 *     different streams, the caller must order them (one stream, or events).
 *   - Host batches: when every array of npm_sample / npm_accumulate_grads /
 *     npm_train_step is a host pointer and n >= 131,072, the call runs in
 *     NPM_PIPE_CHUNKS chunks (default 3) whose host<->device copies (two
 *     internal copy streams) overlap the kernels of the neighbouring chunks;
 *     results equal the device path (NPM_PIPELINE=0 disables).
 *
 * Supported configurations (validated by npm_create; the decoder kernels are
 * compiled per shape): n_features = 4 and
 *   radiance, L = 4, K = 8,  2 affine layers of width 32  (n_in 16)  [c1]
 *   radiance, L = 8, K = 8,  3 affine layers of width 64  (n_in 32)  [c2, c3]
 *   radiance, L = 16, K = 8, 3 affine layers of width 64  (n_in 64)  [c5]
 *   product,  L = 8, K = 16, 3 affine layers of width 64  (n_in 65)  [c4]
 * with any D_1 < D_L, log2_hashmap, AABB.  Anything else -> NPM_ERR_INVALID.
 */
#ifndef NPM_H
#define NPM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NPM_VERSION 1

typedef struct npm_model npm_model; /* opaque */

typedef enum {
  NPM_OK = 0,
  NPM_ERR_INVALID = 1, /* bad config / argument; nothing was enqueued */
  NPM_ERR_CUDA = 2,    /* CUDA runtime failure */
  NPM_ERR_NCCL = 3,    /* collective failure (multi-GPU) */
  NPM_ERR_OOM = 4,     /* device allocation failed */
  NPM_ERR_STATE = 5    /* call not valid in the model's current state */
} npm_status;

typedef enum { NPM_RADIANCE = 0, NPM_PRODUCT = 1 } npm_mode;

/* Parameter-sized buffers, all in the same flat float32 layout:
 * the decoder's affine layers in order, each W[out][in] row-major then b[out];
 * then the grid levels coarsest first, each [entries][F] (entry index as in
 * npm_encode_debug). Total length n_mlp + n_grid (npm_param_count). */
typedef enum {
  NPM_BUF_PARAMS = 0, /* live trainable parameters Phi = Phi_M u Phi_E (Eq. 14) */
  NPM_BUF_GRADS = 1,  /* gradient accumulator (sum over records, already / N_global) */
  NPM_BUF_ADAM_M = 2, /* Adam first moment */
  NPM_BUF_ADAM_V = 3, /* Adam second moment */
  NPM_BUF_EMA = 4     /* EMA shadow used by queries with use_ema = 1 */
} npm_buffer;

typedef struct {
  int32_t mode;              /* npm_mode; PRODUCT conditions on w_o, n, roughness (§4.3) */
  int32_t n_lobes;           /* K vMF components (K = 8) */
  int32_t n_levels;          /* L grid levels (L = 8) */
  int32_t n_features;        /* F features per lattice point (F = 4) */
  int32_t base_res;          /* D_1 lattice points per axis (8) */
  int32_t max_res;           /* D_L (86); D_l = ceil(D_1 b^(l-1) - 1e-9), C-A3 */
  int32_t log2_hashmap;      /* T = 2^log2_hashmap entries cap per level; levels with
                                D^3 > T are spatially hashed (C-A4); 0 = all dense */
  int32_t mlp_linear_layers; /* affine layers incl. output ("3 linear layers") */
  int32_t mlp_width;         /* hidden width (64) */
  int32_t sh_bands;          /* SH bands for w_o and n in product mode (C-A20: 4) */
  float aabb_lo[3], aabb_hi[3]; /* scene bounds mapped onto the grids (C-O1) */
  float lr;                  /* Adam learning rate (0.005) */
  float beta1, beta2, adam_eps; /* 0.9, 0.999, 1e-8 (C-A14) */
  float ema_decay;           /* 0.99 (C-A15) */
  float kappa_min, kappa_max;/* clamp of kappa = exp(kappa') (C-A8): 1e-5, 1e5 */
  uint64_t init_seed;        /* parameter initialisation seed (C-A21) */
  int32_t divergence;        /* training objective: 0 = KL (Eq. 8/9), 1 = Pearson chi^2
                                (f-4; "other divergence metrics", C-A31), 2 = the
                                variance-aware target (f-4; "(2) the improved
                                variance-aware target distribution ... could be learned",
                                reading C-A35): KL from the normalised second moment of the
                                estimate to V^2 / int V^2, per record (D^^2/p~/N)(-2 log V +
                                log int V^2), so that V ~ sqrt(E[D^^2]); radiance shapes
                                with K = 8, exclusive with learn_alpha */
  int32_t learn_alpha;       /* 1: learn the BSDF selection probability (f-4'; "(1) the
                                BSDF selection probability could also be learned by our
                                network", reading C-A34): alpha(x) = sigmoid(a . h_{L-1} + c),
                                a logistic-linear head on the last hidden layer, its W + 1
                                parameters (zero-initialised: alpha = 1/2, the paper's fixed
                                choice) stored AFTER the grid, zero-padded to a multiple of 4.
                                Trained on the second moment of the one-sample MIS estimator
                                (needs npm_query.bsdf_pdf in training calls); used by
                                npm_combined_sample in place of its alpha argument.  Radiance
                                mode only; the model then always uses the warp-specialised
                                training kernel. */
} npm_config;

/* One SoA queue of shading points. px/py/pz: world-space x.
 * wox.., nx.., rough: product mode only (w_o unit outgoing direction, n unit
 * normal, roughness in [0,1]); ignored (may be NULL) in radiance mode.
 * bsdf_pdf: training calls of a learn_alpha model only -- the BSDF sampling
 * pdf p_bsdf(w_i) of each record's direction (C-A34); ignored otherwise. */
typedef struct {
  int64_t n;
  const float *px, *py, *pz;
  const float *wox, *woy, *woz;
  const float *nx, *ny, *nz;
  const float *rough;
  const float *bsdf_pdf;
} npm_query;

/* Training statistics of one step. loss_proxy = sum_n s_n log max(V_n,
 * 1e-30) with s_n = -(D^_n / p~_n) / N_global: the Theta-dependent part of the
 * Eq. 8 estimate. */
typedef struct {
  double loss_proxy;
  double grad_norm_sq;        /* ||g||^2 of the (reduced) gradient, finite entries */
  int64_t n_used;             /* records with finite, non-zero D^/p~ */
  int64_t n_zero_target;      /* records with D^ = 0 (zero gradient) */
  int64_t n_dropped;          /* non-finite D^ or p~ <= 0 / non-finite */
  int64_t n_nonfinite_grad;   /* gradient entries zeroed before Adam */
} npm_step_stats;

/* Defaults of the paper's model + readings C-A3..C-A15. */
void npm_default_config(npm_config* cfg);

/* Validate cfg, allocate all model state on `cuda_device`, initialise
 * parameters (features U(-1e-2, 1e-2), Xavier-uniform weights, zero biases;
 * C-A21), Adam moments 0, EMA := params, step t = 0.  Synchronous. */
npm_status npm_create(const npm_config* cfg, int cuda_device, npm_model** out);
npm_status npm_destroy(npm_model* model);

/* n_mlp = sum over layers of out*in + out; n_grid = F * sum_l entries_l. */
npm_status npm_param_count(const npm_model* model, int64_t* n_grid, int64_t* n_mlp);
/* Per-level lattice resolution D_l and table entries (min(D^3, T)). */
npm_status npm_level_info(const npm_model* model, int32_t* res, int64_t* entries);

/* Copy a whole parameter-sized buffer out of / into the model (count must be
 * n_mlp + n_grid). Used for checkpoints and for parity (identical params on
 * both sides). src/dst host or device. */
npm_status npm_get_buffer(npm_model* model, npm_buffer which, float* dst, int64_t count, void* stream);
npm_status npm_set_buffer(npm_model* model, npm_buffer which, const float* src, int64_t count, void* stream);
/* Adam step counter t (bias correction uses the global t, C-A14). */
npm_status npm_get_step(const npm_model* model, int64_t* t);
npm_status npm_set_step(npm_model* model, int64_t t);

/* Eq. 13: feat = G(x) as [L*F][n] (feature-major SoA, level-major,
 * coarsest level first, C-O5). use_ema selects the EMA shadow. */
npm_status npm_encode(npm_model* model, const npm_query* q, int use_ema, float* feat, void* stream);

/* Parity/debug view of Eq. 13: the 8 corner entry indices per level
 * (uint32 [L][8][n]; corner c = cx + 2cy + 4cz; dense index Px + D(Py + D Pz),
 * hashed levels (Px ^ Py*2654435761 ^ Pz*805459861) & (T-1), C-O4) and the
 * trilinear weights (float [L][8][n]). The cell index is the pinned fp32
 * sequence C-O1/C-O3 (bit-exact with the oracle). Either output may be NULL. */
npm_status npm_encode_debug(npm_model* model, const npm_query* q, uint32_t* idx, float* w, void* stream);

/* Eq. 14 + Table 1. feat: optional [L*F][n] encoding to decode instead of
 * G(x) (radiance mode only; NULL = encode internally). Outputs (each may be
 * NULL): raw [4K][n] in the block layout [lambda' | kappa' | theta' | phi']
 * (C-A6); lambda [K][n]; kappa [K][n]; mu [3][K][n] (C-A7 convention). */
npm_status npm_decode(npm_model* model, const npm_query* q, const float* feat, int use_ema,
                      float* raw, float* lambda, float* kappa, float* mu, void* stream);

/* Eq. 4 mixture pdf V(w | Theta_hat(x)) at caller unit directions w. */
npm_status npm_pdf(npm_model* model, const npm_query* q, const float* wix, const float* wiy,
                   const float* wiz, int use_ema, float* pdf, void* stream);

/* Guided direction sampled from V(. | Theta_hat(x)) with the numerically
 * stable vMF inversion (Jakob 2012; C-O10) and the FULL mixture pdf at
 * it. u: [3][n] uniforms in [0,1) or NULL => Philox4x32-10 with key = seed,
 * counter = (i + offset) (C-O11). Optional fused query: if qx/qy/qz/pdf_q are
 * all non-NULL, V is also evaluated at the caller directions q for the same
 * x (one encode + decode serves both: the "pdf + sample" query). */
npm_status npm_sample(npm_model* model, const npm_query* q, const float* u, uint64_t seed,
                      uint64_t offset, int use_ema, float* wix, float* wiy, float* wiz,
                      float* pdf, const float* qx, const float* qy, const float* qz,
                      float* pdf_q, void* stream);

/* f-2, cosine-lobe product ("the cosine term could be approximated with
 * a constant vMF lobe"; "closed-form product"): the decoded mixture is
 * multiplied by v(. | n, kappa_c) and renormalised -- per lobe
 * kappa_p mu_p = kappa mu + kappa_c n, weight lambda s / sum(lambda s) with
 * s = C(kappa) C(kappa_c) / C(kappa_p) exp(kappa_p - kappa - kappa_c),
 * C(k) = k / (2 pi (1 - e^{-2k})), C(0) = 1/(4 pi) (C-A28) -- then sampled and
 * evaluated exactly as npm_sample (same u / Philox convention, optional fused
 * pdf at qx/qy/qz).  nx/ny/nz: unit shading normals [n].  kappa_c in [0, 1e5]
 * (C-A29 least-squares fit to the clamped cosine: 2.1438).  Optional outputs
 * of the product mixture: lambda, kappa [K][n], mu [3][K][n].  Needs the
 * tensor-core path. */
npm_status npm_sample_cosine_product(npm_model* model, const npm_query* q, const float* nx, const float* ny,
                                     const float* nz, float kappa_c, const float* u, uint64_t seed, uint64_t offset,
                                     int use_ema, float* wix, float* wiy, float* wiz, float* pdf, const float* qx,
                                     const float* qy, const float* qz, float* pdf_q, float* lambda, float* kappa,
                                     float* mu, void* stream);

/* f-1, guided one-sample MIS ("a combination of the BSDF importance
 * sampling and guiding distribution"; P:425 BSDF selection probability 50 %;
 * SPEC S:339-347).  Per query: u_sel < alpha -> BSDF sample, else a guide
 * sample exactly as npm_sample; pdf = p~ = alpha p_bsdf(w) + (1 - alpha) V(w)
 * (balance heuristic, the divisor to store in the training record).  BSDF
 * stand-in (C-A24): Lambertian about the unit normals nx/ny/nz [n],
 * p_bsdf = max(n.w, 0)/pi, cosine-sampled from (u1, u2) in the Duff ONB of n.
 * u: [4][n] = (u1, u2, u3, u_sel) or NULL -> Philox4x32-10 (C-O11; u_sel =
 * out3, C-A25).  If the guide branch is taken and V(w) < 1e-30 or non-finite
 * (C-A26), the record falls back to the BSDF sample with pdf = p_bsdf.
 * Outputs [n]: wix/wiy/wiz, pdf (p~); optional guide_pdf (V(w); 0 on
 * fallback) and technique (int32: 0 BSDF, 1 guide, 2 fallback).
 * alpha in [0, 1] else NPM_ERR_INVALID; needs the tensor-core path. */
npm_status npm_combined_sample(npm_model* model, const npm_query* q, const float* nx, const float* ny,
                               const float* nz, float alpha, const float* u, uint64_t seed, uint64_t offset,
                               int use_ema, float* wix, float* wiy, float* wiz, float* pdf, float* guide_pdf,
                               int32_t* technique, void* stream);

/* f-1, training-record construction ("collect MC radiance estimates
 * along each traced path"): backward unwind per path
 *   <L_i(x_v)> = le[v] + fs[v+1] cos[v+1] / pdf[v+1] * <L_i(x_{v+1})>
 * for v < depth, where le[v] is the radiance arriving at vertex v along its
 * sampled ray (emitted by the vertex it hit), fs/cos/pdf the BSDF value,
 * |cos theta_i| and p~ of vertex v's sampled direction.  A successor with
 * p~ <= 0 or non-finite ends the path (C-A27); v >= depth gives 0.
 * target = <L_i> (product = 0) or fs[v] <L_i> cos[v] (product = 1, Eq. 12).
 * Layouts (n = n_paths, D = max_depth, C = channels in {1, 3}):
 * le, fs, target [C][D][n]; cos_theta, pdf [D][n]; depth int32 [n] -- i.e.
 * target is directly the [C][D*n] target of npm_train_step over D*n records.
 * Uses the model only for its stream staging (host or device pointers). */
npm_status npm_unwind_records(npm_model* model, const float* le, const float* fs, const float* cos_theta,
                              const float* pdf, const int32_t* depth, int channels, int max_depth, int64_t n_paths,
                              int product, float* target, void* stream);

/* f-3, micro-step training on a frame's record stream ("split them
 * into mini-batches for training. The optimization step is performed for
 * each spp"; 2^18 samples per batch).  The n records of q (and wi,
 * target [C][n], sample_pdf) are cut into consecutive micro-batches of
 * micro_batch records (the last may be shorter); each is one full
 * optimisation step: Eq. 9 with 1/N = that micro-batch's size, back
 * propagation, Adam + EMA.  Equivalent to npm_train_step on each slice in
 * order; single-GPU (the data-parallel form loops accumulate / allreduce /
 * optimizer per micro-step in dp.py).  per_step: optional host array of
 * ceil(n / micro_batch) stats (one host sync per micro-step when given).
 * micro_batch <= 0 -> NPM_ERR_INVALID. */
npm_status npm_train_stream(npm_model* model, const npm_query* q, const float* wix, const float* wiy,
                            const float* wiz, const float* target, int target_channels, const float* sample_pdf,
                            int64_t micro_batch, npm_step_stats* per_step, void* stream);

/* One optimisation step ("optimization step is performed for each spp"):
 * Eq. 9 gradient over the batch, back propagation through decoder and grid
 * (P:216), [allreduce if a communicator is attached], Adam + EMA.
 * Records: directions wi (unit), target = D^ as [C][n] with C = 1 or 3 (RGB
 * reduced by luminance, C-A11), sample_pdf = p~ the direction was drawn from
 * (stop-gradient, C-A12). n_global = records across all ranks (the 1/N of
 * Eq. 9, C-A13); pass n on one GPU. Data problems are not errors: D^ = 0 gives
 * no gradient; non-finite D^ or p~ <= 0 drops the record (still counted in N);
 * non-finite gradient entries are zeroed; V is floored at 1e-30. stats may be
 * NULL (no host synchronisation); otherwise the call synchronises `stream`. */
npm_status npm_train_step(npm_model* model, const npm_query* q, const float* wix, const float* wiy,
                          const float* wiz, const float* target, int target_channels,
                          const float* sample_pdf, int64_t n_global, npm_step_stats* stats,
                          void* stream);

/* Split form: npm_train_step == npm_accumulate_grads + npm_optimizer_step.
 * accumulate_grads ADDS the batch's gradient into NPM_BUF_GRADS (no update);
 * optimizer_step [allreduces GRADS,] applies Adam + EMA at t := t + 1 and
 * zeroes GRADS. */
npm_status npm_accumulate_grads(npm_model* model, const npm_query* q, const float* wix,
                                const float* wiy, const float* wiz, const float* target,
                                int target_channels, const float* sample_pdf, int64_t n_global,
                                npm_step_stats* stats, void* stream);
npm_status npm_optimizer_step(npm_model* model, npm_step_stats* stats, void* stream);

/* One frame of the hot path in one call: npm_sample over the query batch q
 * (same arguments, including the optional fused pdf at caller directions),
 * then npm_accumulate_grads over the records tq, then npm_optimizer_step
 * (with the attached communicator's exchange).  Results equal the three
 * calls.  When every array is a host pointer, q->n == tq->n (one record per
 * queried vertex, the paper's per-frame stream) and n >= 131,072, both
 * phases' host<->device copies run in ONE chunked pipeline: chunk j's query
 * and training inputs move together and chunk j's kernels (queries, then the
 * records' gradient) run while chunk j+1 uploads and chunk j-1's outputs
 * download -- one pipeline fill and one drain per frame instead of two.
 * stats as npm_train_step (NULL: no host synchronisation). */
npm_status npm_frame_step(npm_model* model, const npm_query* q, const float* u, uint64_t seed, uint64_t offset,
                          int use_ema, float* wix, float* wiy, float* wiz, float* pdf, const float* qx,
                          const float* qy, const float* qz, float* pdf_q, const npm_query* tq, const float* twx,
                          const float* twy, const float* twz, const float* target, int target_channels,
                          const float* sample_pdf, int64_t n_global, npm_step_stats* stats, void* stream);

/* Multi-GPU (A11): rank 0 calls npm_get_unique_id and shares
 * the 128-byte id with the other ranks (e.g. over the torch process group);
 * every rank then attaches a communicator with npm_comm_init (one process per
 * GPU, `model` on that GPU).  From then on npm_optimizer_step and
 * npm_train_step / npm_train_stream sum GRADS over the ranks (ncclAllReduce
 * on the call's stream) before Adam + EMA, so replicas stay identical; each
 * rank passes n_global = the records of all ranks (1/N scaling, C-A13).
 * NCCL is resolved at run time (libnccl.so.2); without it these return
 * NPM_ERR_NCCL.  A second npm_comm_init on a model -> NPM_ERR_STATE. */
npm_status npm_get_unique_id(uint8_t out[128]);
npm_status npm_comm_init(npm_model* model, int rank, int world, const uint8_t uid[128]);

/* The exchange schedule of the attached communicator:
 *   NPM_EXCHANGE_ALLREDUCE (default): ncclAllReduce(GRADS), then Adam + EMA
 *     on every rank over the whole vector;
 *   NPM_EXCHANGE_ZERO1: ncclReduceScatter(GRADS) -> Adam on this rank's
 *     shard (npm_shard_range) -> ncclAllGather(PARAMS) -> EMA over the whole
 *     (replicated) vector on every rank.  Same update as ALLREDUCE (the EMA
 *     needs no exchange: it is elementwise in the gathered parameters); each
 *     rank reads / writes the Adam moments of 1/P of the parameters.
 * Bad mode -> NPM_ERR_INVALID. */
typedef enum { NPM_EXCHANGE_ALLREDUCE = 0, NPM_EXCHANGE_ZERO1 = 1 } npm_exchange;
npm_status npm_set_exchange(npm_model* model, int mode);

/* ZeRO-1 building blocks, for a caller that runs the collectives on its own
 * process group (paper_2504_04315_b200/dp.py with zero1=True):
 *   npm_shard_range: rank's shard of the flat parameter vector, [*begin,
 *     *begin + *count), *chunk = ceil(n_total / world / 4) * 4 floats per rank;
 *     world * chunk <= n_total + 264, and every buffer is allocated (zero-
 *     padded) to that size, so a reduce-scatter / all-gather may view
 *     world * chunk floats from the buffer's start.  1 <= world <= 64.
 *   npm_optimizer_step_shard: t := t + 1, Adam over the shard (GRADS there
 *     must already hold the reduced gradient), then GRADS := 0 everywhere;
 *     stats (optional, synchronises) hold the shard's grad_norm_sq and
 *     n_nonfinite_grad.  No EMA: call npm_ema_update after gathering PARAMS.
 *   npm_ema_update: EMA <- d EMA + (1 - d) PARAMS over the whole vector (C-O18).
 * Bad rank / world -> NPM_ERR_INVALID. */
npm_status npm_shard_range(const npm_model* model, int rank, int world, int64_t* begin, int64_t* count,
                           int64_t* chunk);
npm_status npm_optimizer_step_shard(npm_model* model, int rank, int world, npm_step_stats* stats, void* stream);
npm_status npm_ema_update(npm_model* model, void* stream);

/* Asynchronous form of the statistics read: enqueues on `stream` the copy of
 * the last training step's statistics (loss proxy, gradient norm, record
 * counters; as npm_train_step's stats) into `out`, which should be pinned
 * host memory; valid once `stream` has synchronised.  Lets a caller read
 * every step's loss without a host synchronisation per step. */
npm_status npm_step_stats_async(npm_model* model, npm_step_stats* out, void* stream);

/* Raw device pointer of a model buffer (for zero-copy collectives by the
 * caller's process group). */
npm_status npm_buffer_device_ptr(npm_model* model, npm_buffer which, float** ptr, int64_t* count);

/* Number of library kernels launched on this model since creation (the
 * bench's gpu_launches evidence). */
int64_t npm_launch_count(const npm_model* model);

/* Kernel timing: when enabled, every library kernel launch is bracketed by
 * CUDA events recorded on its launch stream (used by bench.py for the
 * per-kernel roofline). Kinds are 0 .. npm_profile_kinds()-1; npm_profile_read
 * synchronises on the recorded events and returns the kind's name, launches
 * and total device milliseconds since the last reset. */
int npm_profile_kinds(void);
npm_status npm_profile_enable(npm_model* model, int enable);
npm_status npm_profile_reset(npm_model* model);
npm_status npm_profile_read(npm_model* model, int kind, const char** name, int64_t* launches,
                            double* total_ms);

/* Measurement probe ("a measured L2 random-gather peak"), not
 * part of the method.  Times `reps` launches of a kernel that, for each of
 * n_samples samples, makes 8*levels uniformly random float4 accesses into a
 * table of table_entries float4 (16 B) entries: kind 0 = gathers (ld.global.nc
 * .v4), kind 1 = scatter-adds (red.global.add.v4.f32).  With a c2-sized table
 * (636,927 entries, 10.2 MB) the table is L2-resident, which is the ceiling
 * for the fused kernels' grid accesses; with c5's (632 MB) it is HBM-bound.
 * Allocates and frees its own device memory on cuda_device; synchronous.
 * levels must be even and > 0; table_entries in [1, 2^32).  Writes the mean
 * milliseconds per launch to *ms_per_rep.  Errors: NPM_ERR_INVALID for bad
 * arguments, NPM_ERR_CUDA (npm_last_error unset) for CUDA failures. */
npm_status npm_probe_grid_access(int cuda_device, int64_t table_entries, int64_t n_samples, int levels,
                                 int kind, int reps, double* ms_per_rep);

/* sizeof(npm_config), sizeof(npm_query), sizeof(npm_step_stats) as compiled
 * into the library (bindings check their struct mirrors against these). */
void npm_abi_sizes(int32_t* config, int32_t* query, int32_t* stats);

const char* npm_last_error(void);
int npm_version(void);

#ifdef __cplusplus
}
#endif
#endif /* NPM_H */
