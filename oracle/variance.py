"""Variance-aware target ("(2) the improved
variance-aware target distribution [Rath et al. 2020] could be learned to
account for the variance within the noisy MC estimates").  Test
infrastructure only -- see oracle/__init__.py.

Reading C-A35: the variance-aware guide is proportional to the
square root of the second moment of the incident estimate,
    p_va(w) ~ sqrt(E[D^(w)^2]),
and is learned by fitting the squared, renormalised mixture to the
normalised second moment,
    min_Theta  KL(p2 || V^2 / Z),   p2 = E[D^^2] / int E[D^^2],   Z = int V^2 dw,
so that at the optimum V^2 ~ E[D^^2], i.e. V ~ sqrt(E[D^^2]).  With records
w_n ~ p~ and weights a_n = D^_n^2 / p~_n the per-record loss is
    l_n = (a_n / N) (-2 log V(w_n) + log Z(x_n)),
whose expectation is int E[D^^2] times the KL gradient (the same role Eq. 9's
D^/p~ plays for the first moment).  Z has a closed form for vMF
mixtures (products of lobes; v = C(k) e^{k (mu.w - 1)}):
    Z = sum_ij lambda_i lambda_j I_ij,
    I_ij = int v_i v_j = C(k_i) C(k_j) / C(r_ij) e^{r_ij - k_i - k_j},   r_ij = |k_i mu_i + k_j mu_j|,
    C(k) = k / (2 pi (1 - e^{-2k})),  C(0) = 1/(4 pi).
With the Langevin function Lg(x) = coth x - 1/x (= 1 - d log C/dk; Lg(x)/x -> 1/3
at 0), G_ij = lambda_i lambda_j I_ij / Z and g_i = sum_j G_ij:
    d log Z / d lambda'_i = 2 (g_i - lambda_i)
    d log Z / d kappa_i   = 2 sum_j G_ij (-Lg(k_i) + Lg(r_ij)/r_ij (k_i + k_j mu_i.mu_j))
    d log Z / d mu_i      = 2 sum_j G_ij Lg(r_ij)/r_ij k_i k_j mu_j            (tangent part)
chained through Table 1 as in Eq. 9's head (kappa' clamped: 0)."""
import numpy as np

from . import vmf
from .product import log_c


def langevin_over_x(x):
    """Lg(x) / x = (coth x - 1/x) / x; 1/3 - x^2/45 below 1e-3."""
    x = np.asarray(x, np.float64)
    small = x < 1e-3
    xs = np.where(small, 1.0, x)
    big = (1.0 + 2.0 / np.expm1(np.minimum(2.0 * xs, 700.0)) - 1.0 / xs) / xs
    return np.where(small, 1.0 / 3.0 - x * x / 45.0, big)


def pair_terms(act):
    """Per record, all lobe pairs: I_ij [K, K, n], r_ij, mu_i.mu_j."""
    kap, mu = act['kappa'], act['mu']
    c = np.einsum('ain,ajn->ijn', mu, mu)
    r2 = kap[:, None, :] ** 2 + kap[None, :, :] ** 2 + 2 * kap[:, None, :] * kap[None, :, :] * c
    r = np.sqrt(np.maximum(r2, 0.0))
    log_i = log_c(kap)[:, None, :] + log_c(kap)[None, :, :] - log_c(r) + r - kap[:, None, :] - kap[None, :, :]
    return np.exp(log_i), r, c


def log_z(act):
    """log int V^2 dw per record (closed form)."""
    lam = act['lam']
    i_ij, _, _ = pair_terms(act)
    return np.log(np.einsum('in,jn,ijn->n', lam, lam, i_ij))


def grad_log_z(raw, k, kappa_min=vmf.KAPPA_MIN, kappa_max=vmf.KAPPA_MAX):
    """d log Z / d raw [4K, n] (C-A6 layout) and log Z [n]."""
    act = vmf.activate(raw, k, kappa_min, kappa_max)
    lam, kap, th, ph, mu = act['lam'], act['kappa'], act['theta'], act['phi'], act['mu']
    i_ij, r, c = pair_terms(act)
    zz = np.einsum('in,jn,ijn->n', lam, lam, i_ij)
    g_ij = lam[:, None, :] * lam[None, :, :] * i_ij / zz
    g_i = g_ij.sum(axis=1)
    lrx = langevin_over_x(r)                                                  # Lg(r) / r
    lk = kap * langevin_over_x(kap)                                           # Lg(k)
    dk = 2 * (g_ij * (-lk[:, None, :] + lrx * (kap[:, None, :] + kap[None, :, :] * c))).sum(axis=1)
    coef = 2 * g_ij * lrx * kap[:, None, :] * kap[None, :, :]                 # [i, j, n]
    dmu = np.einsum('ijn,ajn->ain', coef, mu)                                 # [3, K, n]
    dlam = 2 * (g_i - lam)
    dkap = np.where(act['clamped'], 0.0, dk * kap)
    pt, pp2 = np.pi * th, 2 * np.pi * ph
    dmu_dth = np.pi * np.stack([np.cos(pt) * np.cos(pp2), np.cos(pt) * np.sin(pp2), -np.sin(pt)])
    dmu_dph = 2 * np.pi * np.stack([-np.sin(pt) * np.sin(pp2), np.sin(pt) * np.cos(pp2), np.zeros_like(pt)])
    dth = (dmu * dmu_dth).sum(axis=0) * th * (1 - th)
    dph = (dmu * dmu_dph).sum(axis=0) * ph * (1 - ph)
    return np.concatenate([dlam, dkap, dth, dph], axis=0), np.log(zz)


def record_weight(target, sample_pdf, dropped, zero):
    """a_n = D^_n^2 / p~_n (0 for dropped / zero-target records, C-O12)."""
    t = np.where(dropped | zero, 0.0, target)
    ps = np.where(dropped | zero, 1.0, sample_pdf)
    return t * t / ps


def variance_aware_head(raw, wi, target, sample_pdf, n_global, dropped, zero, k,
                        kappa_min=vmf.KAPPA_MIN, kappa_max=vmf.KAPPA_MAX):
    """Per-record gradient of l_n = (a_n/N)(-2 log V(w_n) + log Z) w.r.t. the raw
    outputs, and the loss proxy sum_n l_n."""
    a = record_weight(target, sample_pdf, dropped, zero)
    draw, logv = vmf.grad_head(raw, wi, -2.0 * a / n_global, k, kappa_min, kappa_max)
    dz, logz = grad_log_z(raw, k, kappa_min, kappa_max)
    draw = draw + (a / n_global)[None, :] * dz
    return draw, float(((a / n_global) * (-2.0 * logv + logz)).sum())
