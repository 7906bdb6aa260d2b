"""vMF mixture: Table 1 mappings, Eq. 3/4 pdf, Jakob sampling, Eq. 9 head.

TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py.

  v(w | mu, kappa) = kappa / (4 pi sinh kappa) exp(kappa mu^T w)     (Eq. 3)
  V(w | Theta) = sum_i lambda_i v(w | mu_i, kappa_i)                  (Eq. 4)
  kappa = exp(kappa'), lambda = softmax(lambda'), theta = 1/(1+e^-theta')
                                                                     (Table 1)
  grad_Theta D_KL ~= -(1/N) sum_j D(w_j) grad V(w_j) / (p~(w_j) V(w_j))  (Eq. 9)

Readings: C-A6 raw layout [lambda'(K) | kappa'(K) | theta'(K) | phi'(K)];
C-A7 mu = (sin pi theta cos 2 pi phi, sin pi theta sin 2 pi phi, cos pi theta);
C-A8 kappa' clamped to [ln 1e-5, ln 1e5] with zero gradient outside;
C-O9 stable pdf form kappa/(2 pi (-expm1(-2 kappa))) exp(-kappa |mu - w|^2 / 2);
C-O10 Jakob 2012 stable inverse CDF in the Duff et al. ONB;
C-O12/13 the per-record Eq. 9 head, V floored at 1e-30.
"""
import math
import numpy as np

KAPPA_MIN = 1e-5
KAPPA_MAX = 1e5
V_FLOOR = 1e-30


def activate(raw, k, kappa_min=KAPPA_MIN, kappa_max=KAPPA_MAX):
    """Table 1 mappings (C-O8).  raw: [4K, n].  Returns dict with
    lam [K,n], kappa [K,n], theta, phi [K,n], mu [3,K,n], clamped [K,n]."""
    lp, kp, tp, pp = raw[0:k], raw[k:2 * k], raw[2 * k:3 * k], raw[3 * k:4 * k]
    e = np.exp(lp - lp.max(axis=0, keepdims=True))
    lam = e / e.sum(axis=0, keepdims=True)
    lo, hi = math.log(kappa_min), math.log(kappa_max)
    kappa = np.exp(np.clip(kp, lo, hi))
    clamped = (kp < lo) | (kp > hi)
    theta = 1.0 / (1.0 + np.exp(-tp))
    phi = 1.0 / (1.0 + np.exp(-pp))
    mu = np.stack([np.sin(np.pi * theta) * np.cos(2 * np.pi * phi),
                   np.sin(np.pi * theta) * np.sin(2 * np.pi * phi),
                   np.cos(np.pi * theta)])
    return dict(lam=lam, kappa=kappa, theta=theta, phi=phi, mu=mu, clamped=clamped)


def vmf_pdf_eq3(w, mu, kappa):
    """Eq. 3 exactly as printed (overflows for kappa > ~700; pins only)."""
    return kappa / (4 * np.pi * np.sinh(kappa)) * np.exp(kappa * np.einsum('a...,a...->...', mu, w))


def lobe_pdf(w, mu, kappa):
    """C-O9 stable form of Eq. 3: 1 - mu.w = |mu - w|^2 / 2 for unit vectors.
    w: [3, n]; mu: [3, K, n]; kappa: [K, n] -> [K, n]."""
    d2 = ((mu - w[:, None, :]) ** 2).sum(axis=0)
    return kappa / (2 * np.pi * (-np.expm1(-2 * kappa))) * np.exp(-kappa * 0.5 * d2)


def mixture_pdf(w, act):
    """Eq. 4: V = sum_i lambda_i v_i.  Returns [n]."""
    return (act['lam'] * lobe_pdf(w, act['mu'], act['kappa'])).sum(axis=0)


def duff_onb(mu):
    """Duff et al. 2017 branchless ONB around unit mu: [3,n] -> (t1, t2)."""
    s = np.copysign(1.0, mu[2])
    a = -1.0 / (s + mu[2])
    b = mu[0] * mu[1] * a
    t1 = np.stack([1 + s * mu[0] ** 2 * a, s * b, -s * mu[0]])
    t2 = np.stack([b, s + mu[1] ** 2 * a, -mu[1]])
    return t1, t2


def sample(act, u, k):
    """C-O10: lobe i* = min{i : u1 < C_i} (K-1 if none), C_i = sum_{j<=i} lambda_j;
    delta = min(-log1p((1-u2) expm1(-2 kappa)) / kappa, 2); w = 1 - delta;
    r = sqrt(max(delta (2 - delta), 0)); omega = w mu + r (cos 2 pi u3 t1 + sin 2 pi u3 t2).
    Returns (omega [3,n], V(omega) [n], lobe [n])."""
    n = u.shape[1]
    cdf = np.cumsum(act['lam'], axis=0)                     # [K, n]
    below = u[0][None, :] < cdf
    lobe = np.where(below.any(axis=0), below.argmax(axis=0), k - 1)
    cols = np.arange(n)
    kap = act['kappa'][lobe, cols]
    mu = act['mu'][:, lobe, cols]                           # [3, n]
    delta = np.minimum(-np.log1p((1 - u[1]) * np.expm1(-2 * kap)) / kap, 2.0)
    wz = 1.0 - delta
    r = np.sqrt(np.maximum(delta * (2.0 - delta), 0.0))
    t1, t2 = duff_onb(mu)
    c, s = np.cos(2 * np.pi * u[2]), np.sin(2 * np.pi * u[2])
    omega = wz[None, :] * mu + r[None, :] * (c[None, :] * t1 + s[None, :] * t2)
    return omega, mixture_pdf(omega, act), lobe


def record_scale(target, sample_pdf, n_global, is_zero=None):
    """C-O12: a = D^/p~; the record is dropped (a := 0) if a is non-finite or
    p~ <= 0 or p~ is non-finite; s = -a / N_global (N counts every record,
    C-A13).  ``is_zero``: the D^ = 0 decision (for RGB targets: every channel
    is 0, C-A11); default target == 0.
    Returns (s [n], dropped bool [n], zero_target bool [n])."""
    with np.errstate(divide='ignore', invalid='ignore'):
        a = target / sample_pdf
    dropped = ~np.isfinite(a) | ~np.isfinite(sample_pdf) | (sample_pdf <= 0)
    a = np.where(dropped, 0.0, a)
    zero = (~dropped) & ((target == 0) if is_zero is None else is_zero)
    return -a / n_global, dropped, zero


def grad_head(raw, w, s, k, kappa_min=KAPPA_MIN, kappa_max=KAPPA_MAX):
    """Eq. 9 per-record gradient w.r.t. the raw outputs (C-O13), already
    multiplied by the record scale s = -(D^/p~)/N:
      d/dlambda'_k = s (gamma_k - lambda_k),   gamma_i = lambda_i v_i / max(V, 1e-30)
      d/dkappa'_i  = s gamma_i (1 - kappa_i |mu_i - w|^2/2 - 2 kappa_i e^{-2 kappa_i} / (-expm1(-2 kappa_i)))
                     (0 where kappa' is clamped)
      d/dtheta'_i  = s gamma_i kappa_i (w . dmu/dtheta) theta (1 - theta)
      d/dphi'_i    = s gamma_i kappa_i (w . dmu/dphi)   phi (1 - phi)
    Returns (draw [4K, n], log V_floor [n])."""
    act = activate(raw, k, kappa_min, kappa_max)
    lam, kap, th, ph, mu = act['lam'], act['kappa'], act['theta'], act['phi'], act['mu']
    v = lobe_pdf(w, mu, kap)
    vbar = np.maximum((lam * v).sum(axis=0), V_FLOOR)
    gamma = lam * v / vbar
    d2 = ((mu - w[:, None, :]) ** 2).sum(axis=0)
    em = -np.expm1(-2 * kap)
    dlam = s * (gamma - lam)
    dkap = s * gamma * (1.0 - kap * 0.5 * d2 - 2 * kap * np.exp(-2 * kap) / em)
    dkap = np.where(act['clamped'], 0.0, dkap)
    pt, pp2 = np.pi * th, 2 * np.pi * ph
    dmu_dth = np.pi * np.stack([np.cos(pt) * np.cos(pp2), np.cos(pt) * np.sin(pp2), -np.sin(pt)])
    dmu_dph = 2 * np.pi * np.stack([-np.sin(pt) * np.sin(pp2), np.sin(pt) * np.cos(pp2), np.zeros_like(pt)])
    wdth = np.einsum('akn,an->kn', dmu_dth, w)
    wdph = np.einsum('akn,an->kn', dmu_dph, w)
    dth = s * gamma * kap * wdth * th * (1 - th)
    dph = s * gamma * kap * wdph * ph * (1 - ph)
    return np.concatenate([dlam, dkap, dth, dph], axis=0), np.log(vbar)
