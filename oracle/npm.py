"""The NPM model: encode -> decode -> Table 1 -> pdf / sample, and one
optimisation step (Fig. 2 stages (1)-(5); §4.1-4.3, §5).

TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py.

  NPM(x | Phi) = Theta_hat(x)                                  (Eq. 6)
  NPM_product(x, w_o | Phi) = Theta_hat(x, w_o)                (Eq. 11)
  MLP(G(x | Phi_E) | Phi_M) = Theta_hat(x)                     (Eq. 14)

Parameter layout (flat, the C-ABI's NPM_BUF_* layout): the MLP affine layers in
order, each W [out][in] row-major followed by b [out]; then the grid levels
coarsest first, each [entries][F].

Product mode (C-O6): z = [G(x), SH4(w_o), SH4(n), roughness].
RGB targets are reduced by luminance 0.2126/0.7152/0.0722 (C-A11).
"""
from dataclasses import dataclass, field
import numpy as np

from . import grid, mlp, sh, vmf, adam, variance

RADIANCE, PRODUCT = 0, 1
KL, CHI2 = 0, 1   # training divergence (f-4; "Other divergence metrics are also available")
VARIANCE_AWARE = 2   # f-4: KL to the second moment, V^2 / int V^2 (reading C-A35; oracle/variance.py)
LUMA = np.array([0.2126, 0.7152, 0.0722])


@dataclass
class Config:
    mode: int = RADIANCE
    n_lobes: int = 8
    n_levels: int = 8
    n_features: int = 4
    base_res: int = 8
    max_res: int = 86
    log2_hashmap: int = 18
    mlp_linear_layers: int = 3
    mlp_width: int = 64
    sh_bands: int = 4
    aabb_lo: tuple = (-1.0, -1.0, -1.0)
    aabb_hi: tuple = (1.0, 1.0, 1.0)
    lr: float = 5e-3
    beta1: float = 0.9
    beta2: float = 0.999
    adam_eps: float = 1e-8
    ema_decay: float = 0.99
    kappa_min: float = 1e-5
    kappa_max: float = 1e5
    divergence: int = KL
    learn_alpha: int = 0   # f-4' (C-A34): the BSDF selection-probability head

    @property
    def resolutions(self):
        return grid.level_resolutions(self.base_res, self.max_res, self.n_levels)

    @property
    def table_sizes(self):
        return grid.level_table_sizes(self.resolutions, self.log2_hashmap)

    @property
    def n_in(self):
        n = self.n_levels * self.n_features
        if self.mode == PRODUCT:
            n += 2 * self.sh_bands ** 2 + 1
        return n

    @property
    def layer_dims(self):
        dims = [self.n_in] + [self.mlp_width] * (self.mlp_linear_layers - 1) + [4 * self.n_lobes]
        return list(zip(dims[:-1], dims[1:]))

    @property
    def n_mlp(self):
        return sum(o * i + o for i, o in self.layer_dims)

    @property
    def n_grid(self):
        return sum(self.table_sizes) * self.n_features

    @property
    def n_alpha(self):
        """C-A34: selection head a [W], c, zero-padded to a multiple of 4."""
        return (self.mlp_width + 1 + 3) // 4 * 4 if self.learn_alpha else 0

    @property
    def n_total(self):
        return self.n_mlp + self.n_grid + self.n_alpha


def unpack(cfg, flat):
    """Flat parameter vector -> (layers [(W, b)], tables [[size_l, F]])."""
    layers, off = [], 0
    for i, o in cfg.layer_dims:
        w = flat[off:off + o * i].reshape(o, i); off += o * i
        b = flat[off:off + o]; off += o
        layers.append((w, b))
    tables = []
    for s in cfg.table_sizes:
        tables.append(flat[off:off + s * cfg.n_features].reshape(s, cfg.n_features))
        off += s * cfg.n_features
    return layers, tables


def pack(cfg, layers, tables, alpha_grad=None):
    parts = []
    for w, b in layers:
        parts += [w.ravel(), b.ravel()]
    parts += [t.ravel() for t in tables]
    if cfg.n_alpha:
        parts.append(np.zeros(cfg.n_alpha) if alpha_grad is None else alpha_grad)
    return np.concatenate(parts)


def alpha_head(cfg, flat):
    """C-A34: (a [W], c) of the selection head, stored after the grid."""
    off = cfg.n_mlp + cfg.n_grid
    return flat[off:off + cfg.mlp_width], flat[off + cfg.mlp_width]


def grid_mask(cfg):
    m = np.zeros(cfg.n_total, bool)
    m[cfg.n_mlp:cfg.n_mlp + cfg.n_grid] = True
    return m


def encode(cfg, flat, x):
    """Eq. 13 -> G [L*F, n] (float64)."""
    _, tables = unpack(cfg, flat)
    return grid.encode(x, cfg.aabb_lo, cfg.aabb_hi, cfg.resolutions, cfg.table_sizes,
                       cfg.log2_hashmap, tables)


def network_input(cfg, flat, q):
    """z = G(x) (radiance) or [G, SH(w_o), SH(n), roughness] (product)."""
    g = encode(cfg, flat, q['x'])
    if cfg.mode != PRODUCT:
        return g
    return np.concatenate([g, sh.sh_encode(q['wo'], cfg.sh_bands), sh.sh_encode(q['n'], cfg.sh_bands),
                           np.asarray(q['rough'], np.float64)[None, :]], axis=0)


def decode(cfg, flat, q):
    """Eq. 14 + Table 1: returns (raw [4K, n], activated mixture dict)."""
    layers, _ = unpack(cfg, flat)
    raw, _, _ = mlp.forward(layers, network_input(cfg, flat, q))
    return raw, vmf.activate(raw, cfg.n_lobes, cfg.kappa_min, cfg.kappa_max)


def selection_probability(cfg, flat, q):
    """C-A34 ("the BSDF selection probability could also be learned by
    our network"): alpha(x) = sigmoid(a . h_{L-1} + c), a logistic-linear
    read-out of the decoder's last hidden layer.  Returns alpha [n]."""
    layers, _ = unpack(cfg, flat)
    _, _, inputs = mlp.forward(layers, network_input(cfg, flat, q))
    a, c = alpha_head(cfg, flat)
    return 1.0 / (1.0 + np.exp(-(a @ inputs[-1] + c)))


def alpha_second_moment_grad(cfg, flat, q, wi, t, sample_pdf, bsdf_pdf, used, n_global):
    """C-A34: gradient of the MC second moment of the one-sample MIS estimator,
        M2 = (1/N) sum_n D^_n^2 / (p~_alpha(w_n) p~_s(w_n)),
        p~_alpha = alpha p_bsdf + (1 - alpha) V     (P:208's combination),
    with respect to the head (a, c): for the logit z = a . h + c,
        dM2/dz_n = -(1/N) D^_n^2 (p_bsdf - V) alpha (1 - alpha) / (p~_alpha^2 p~_s)
    (V and h stop-gradient: the mixture keeps Eq. 9).  Records outside `used`
    (dropped / zero target, C-O12), or with non-finite p_bsdf < 0 or
    p~_alpha = 0, contribute 0.  Returns (grad [W + 1], M2 estimate)."""
    layers, _ = unpack(cfg, flat)
    raw, _, inputs = mlp.forward(layers, network_input(cfg, flat, q))
    h = inputs[-1]
    a, c = alpha_head(cfg, flat)
    alpha = 1.0 / (1.0 + np.exp(-(a @ h + c)))
    v = vmf.mixture_pdf(np.asarray(wi, np.float64), vmf.activate(raw, cfg.n_lobes, cfg.kappa_min, cfg.kappa_max))
    pb = np.asarray(bsdf_pdf, np.float64)
    ps = np.asarray(sample_pdf, np.float64)
    pa = alpha * pb + (1.0 - alpha) * v
    ok = used & np.isfinite(pb) & (pb >= 0) & (pa > 0)
    tt = np.where(ok, t, 0.0)
    pa_s = np.where(ok, pa, 1.0)
    ps_s = np.where(ok, ps, 1.0)
    gz = np.where(ok, -(tt * tt) * (pb - v) * alpha * (1.0 - alpha) / (pa_s * pa_s * ps_s), 0.0) / n_global
    m2 = float(np.sum(np.where(ok, tt * tt / (pa_s * ps_s), 0.0)) / n_global)
    return np.concatenate([h @ gz, [gz.sum()]]), m2


def pdf(cfg, flat, q, w):
    """Eq. 4 at caller directions w [3, n]."""
    _, act = decode(cfg, flat, q)
    return vmf.mixture_pdf(np.asarray(w, np.float64), act)


def sample(cfg, flat, q, u):
    """C-O10 with caller uniforms u [3, n] -> (omega [3,n], V(omega) [n], lobe)."""
    _, act = decode(cfg, flat, q)
    return vmf.sample(act, np.asarray(u, np.float64), cfg.n_lobes)


def scalar_target(target):
    t = np.asarray(target, np.float64)
    if t.ndim == 1:
        return t
    if t.shape[0] == 1:
        return t[0]
    return (LUMA[:, None] * t).sum(axis=0)


def gradient(cfg, flat, q, wi, target, sample_pdf, n_global, bsdf_pdf=None):
    """Eq. 9 + back propagation: the flat gradient of
    l = sum_n s_n log max(V_n, 1e-30), s_n = -(D^_n/p~_n)/N_global, with respect
    to every parameter, plus step statistics."""
    layers, _ = unpack(cfg, flat)
    z = network_input(cfg, flat, q)
    raw, pres, inputs = mlp.forward(layers, z)
    wi = np.asarray(wi, np.float64)
    tgt = np.asarray(target, np.float64)
    is_zero = (tgt == 0).all(axis=0) if tgt.ndim == 2 else (tgt == 0)
    t = scalar_target(target)
    s, dropped, zero = vmf.record_scale(t, np.asarray(sample_pdf, np.float64), n_global, is_zero)
    if cfg.divergence == CHI2:
        # f-4 (C-A31): Pearson chi^2, D_chi2 = int D^2 / V - 1, MC estimate
        # (1/N) sum (D^/p~) D^ / V; its gradient is -(1/N) sum (D^/p~)(D^/V) grad log V,
        # i.e. Eq. 9's head with the record scale s multiplied by D^ / V
        vbar = np.maximum(vmf.mixture_pdf(wi, vmf.activate(raw, cfg.n_lobes, cfg.kappa_min, cfg.kappa_max)),
                          vmf.V_FLOOR)
        tt = np.where(dropped | zero, 0.0, t)
        chi = tt / vbar
        s_chi = s * chi
        draw, _ = vmf.grad_head(raw, wi, s_chi, cfg.n_lobes, cfg.kappa_min, cfg.kappa_max)
        mgrads, dz = mlp.backward(layers, pres, inputs, draw)
        gl = cfg.n_levels * cfg.n_features
        ggrads = grid.scatter_grad(q['x'], cfg.aabb_lo, cfg.aabb_hi, cfg.resolutions, cfg.table_sizes,
                                   dz[:gl], cfg.n_features)
        stats = dict(loss_proxy=float((-s * chi).sum()), n_used=int((~dropped & ~zero).sum()),
                     n_zero_target=int(zero.sum()), n_dropped=int(dropped.sum()))
        return pack(cfg, mgrads, ggrads, _alpha_block(cfg, flat, q, wi, t, sample_pdf, bsdf_pdf,
                                                      ~dropped & ~zero, n_global, stats)), stats
    if cfg.divergence == VARIANCE_AWARE:
        # f-4 (C-A35): l_n = (a_n / N)(-2 log V(w_n) + log int V^2), a_n = D^_n^2 / p~_n
        draw, proxy = variance.variance_aware_head(raw, wi, t, np.asarray(sample_pdf, np.float64), n_global,
                                                   dropped, zero, cfg.n_lobes, cfg.kappa_min, cfg.kappa_max)
        mgrads, dz = mlp.backward(layers, pres, inputs, draw)
        gl = cfg.n_levels * cfg.n_features
        ggrads = grid.scatter_grad(q['x'], cfg.aabb_lo, cfg.aabb_hi, cfg.resolutions, cfg.table_sizes,
                                   dz[:gl], cfg.n_features)
        stats = dict(loss_proxy=proxy, n_used=int((~dropped & ~zero).sum()),
                     n_zero_target=int(zero.sum()), n_dropped=int(dropped.sum()))
        return pack(cfg, mgrads, ggrads, _alpha_block(cfg, flat, q, wi, t, sample_pdf, bsdf_pdf,
                                                      ~dropped & ~zero, n_global, stats)), stats
    draw, logv = vmf.grad_head(raw, wi, s, cfg.n_lobes, cfg.kappa_min, cfg.kappa_max)
    mgrads, dz = mlp.backward(layers, pres, inputs, draw)
    gl = cfg.n_levels * cfg.n_features
    ggrads = grid.scatter_grad(q['x'], cfg.aabb_lo, cfg.aabb_hi, cfg.resolutions, cfg.table_sizes,
                               dz[:gl], cfg.n_features)
    stats = dict(loss_proxy=float((s * logv).sum()), n_used=int((~dropped & ~zero).sum()),
                 n_zero_target=int(zero.sum()), n_dropped=int(dropped.sum()))
    g = pack(cfg, mgrads, ggrads, _alpha_block(cfg, flat, q, wi, t, sample_pdf, bsdf_pdf, ~dropped & ~zero,
                                               n_global, stats))
    return g, stats


def _alpha_block(cfg, flat, q, wi, t, sample_pdf, bsdf_pdf, used, n_global, stats):
    """The selection head's slice of the gradient (zero-padded to n_alpha)."""
    if not cfg.learn_alpha:
        return None
    if bsdf_pdf is None:
        raise ValueError("learn_alpha needs the BSDF pdf of every record")
    ga, m2 = alpha_second_moment_grad(cfg, flat, q, wi, t, sample_pdf, bsdf_pdf, used, n_global)
    stats["alpha_m2"] = m2
    out = np.zeros(cfg.n_alpha)
    out[:ga.size] = ga
    return out


@dataclass
class State:
    cfg: Config
    params: np.ndarray
    m: np.ndarray = None
    v: np.ndarray = None
    ema: np.ndarray = None
    t: int = 0

    def __post_init__(self):
        n = self.params.size
        self.m = np.zeros(n) if self.m is None else self.m
        self.v = np.zeros(n) if self.v is None else self.v
        self.ema = self.params.copy() if self.ema is None else self.ema


def optimizer_step(state, g):
    """C-O17 + C-O18 at t := t + 1.  Returns n_nonfinite."""
    c = state.cfg
    state.t += 1
    state.params, state.m, state.v, state.ema, nnf = adam.adam_ema_step(
        state.params, g, state.m, state.v, state.ema, state.t, grid_mask(c),
        c.lr, c.beta1, c.beta2, c.adam_eps, c.ema_decay)
    return nnf


def train_step(state, q, wi, target, sample_pdf, n_global=None, bsdf_pdf=None):
    n = np.asarray(q['x']).shape[1]
    g, stats = gradient(state.cfg, state.params, q, wi, target, sample_pdf, n if n_global is None else n_global,
                        bsdf_pdf)
    stats['grad_norm_sq'] = float(np.sum(np.where(np.isfinite(g), g, 0.0) ** 2))
    stats['n_nonfinite_grad'] = optimizer_step(state, g)
    return g, stats


def train_stream(state, q, wi, target, sample_pdf, micro_batch):
    """f-3 ("split them into mini-batches for training. The optimization
    step is performed for each spp"; P:482 2^18 per batch): one train_step per
    consecutive micro-batch, 1/N = the micro-batch size.  Returns the list of
    per-step (gradient, stats)."""
    n = np.asarray(q['x']).shape[1]
    out = []
    for a in range(0, n, micro_batch):
        b = min(a + micro_batch, n)
        sl = lambda v: np.asarray(v)[..., a:b]
        qs = {k: sl(v) for k, v in q.items()}
        out.append(train_step(state, qs, sl(wi), sl(target), sl(sample_pdf), b - a))
    return out
