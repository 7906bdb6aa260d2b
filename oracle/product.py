"""vMF products and the cosine-lobe factorisation of NPM-product (SURVEY 8(f)
f-2).  Test infrastructure only -- see oracle/__init__.py.

P:129: vMF mixtures have a "closed-form product".  P:244: in the product
variant "the cosine term could be approximated with a constant vMF lobe",
leaving NPM the rest of the integrand; the guide is then the normalised
product of the decoded mixture with that lobe about the shading normal.

  v(w | mu, kappa) = C(kappa) exp(kappa (mu.w - 1)),  C(kappa) = kappa / (2 pi (1 - e^{-2 kappa}))
  v_a v_b = C_a C_b exp(kappa_a mu_a.w + kappa_b mu_b.w - kappa_a - kappa_b)
          = [C_a C_b / C_p exp(kappa_p - kappa_a - kappa_b)] v(w | mu_p, kappa_p),
  kappa_p mu_p = kappa_a mu_a + kappa_b mu_b

so the product of a mixture sum_i lambda_i v_i with a lobe v_c is the mixture
with lobes (mu_p,i, kappa_p,i) and weights lambda_i s_i / sum_j lambda_j s_j,
s_i the bracket above (log_scale = log s).

Readings:
  C-A28  kappa_p = 0 (antipodal lobes of equal kappa): the product is uniform;
         mu_p := mu_b, C(0) := 1 / (4 pi).
  C-A29  The cosine lobe: mu = n, kappa_c and its amplitude fitted by least
         squares to the clamped cosine max(n.w, 0) over the sphere
         (fit_cosine_lobe; "fitted offline by least-squares").
"""
import math

import numpy as np
from scipy import optimize

from . import vmf


def log_c(kappa):
    """log C(kappa), C(kappa) = kappa / (2 pi (1 - e^{-2 kappa})); C(0) = 1/(4 pi)."""
    k = np.asarray(kappa, np.float64)
    with np.errstate(divide='ignore', invalid='ignore'):
        r = np.where(k > 0, k / -np.expm1(-2 * np.where(k > 0, k, 1.0)), 0.5)
    return np.log(r) - math.log(2 * math.pi)


def vmf_product(mu_a, k_a, mu_b, k_b):
    """Closed-form product of two vMF lobes.  mu: [3, ...]; k: [...].
    Returns (mu_p, k_p, log_scale) with v_a v_b = exp(log_scale) v(. | mu_p, k_p)."""
    s = k_a[None] * mu_a + k_b[None] * mu_b
    k_p = np.sqrt((s ** 2).sum(axis=0))
    with np.errstate(divide='ignore', invalid='ignore'):
        mu_p = np.where(k_p[None] > 0, s / np.where(k_p > 0, k_p, 1.0)[None], mu_b * np.ones_like(s))
    log_scale = log_c(k_a) + log_c(k_b) - log_c(k_p) + k_p - k_a - k_b
    return mu_p, k_p, log_scale


def cosine_product(act, n, kappa_c):
    """The decoded mixture (vmf.activate dict) times the cosine lobe
    v(. | n, kappa_c), renormalised.  n: [3, m].  Returns an activated-mixture
    dict (lam, kappa, mu) of the product."""
    K = act['kappa'].shape[0]
    nb = np.repeat(np.asarray(n, np.float64)[:, None, :], K, axis=1)
    kc = np.full(act['kappa'].shape, float(kappa_c))
    mu_p, k_p, ls = vmf_product(act['mu'], act['kappa'], nb, kc)
    logw = np.log(act['lam']) + ls
    w = np.exp(logw - logw.max(axis=0, keepdims=True))
    return dict(lam=w / w.sum(axis=0, keepdims=True), kappa=k_p, mu=mu_p)


def fit_cosine_lobe():
    """C-A29: (kappa_c, amplitude a) minimising the L2 distance over the sphere
    between max(t, 0) and a exp(kappa (t - 1)), t = n.w (the integral over the
    azimuth is 2 pi; over t by Gauss-Legendre on [-1, 0] and [0, 1])."""
    x, wq = np.polynomial.legendre.leggauss(200)
    t = np.concatenate([(x - 1) / 2, (x + 1) / 2])
    w = np.concatenate([wq / 2, wq / 2]) * 2 * np.pi
    f = np.maximum(t, 0.0)

    def err(kappa):
        g = np.exp(kappa * (t - 1))
        a = (w * f * g).sum() / (w * g * g).sum()     # optimal amplitude for this kappa
        return (w * (f - a * g) ** 2).sum()

    r = optimize.minimize_scalar(err, bounds=(0.1, 20.0), method='bounded', options=dict(xatol=1e-10))
    g = np.exp(r.x * (t - 1))
    return float(r.x), float((w * f * g).sum() / (w * g * g).sum())


def product_sample(act, n, kappa_c, u, k):
    """Guided sample from the cosine-product mixture (C-O10 on the product
    lobes) and its pdf.  Returns (w [3, m], pdf [m], product act)."""
    pa = cosine_product(act, n, kappa_c)
    w, pdf, _ = vmf.sample(pa, np.asarray(u, np.float64), k)
    return w, pdf, pa
