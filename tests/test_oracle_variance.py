"""Pins for the variance-aware target (f-4, reading C-A35;
oracle/variance.py): V is trained so that V^2 / int V^2 matches the normalised
second moment of the estimate, per record l_n = (a_n/N)(-2 log V + log Z),
a_n = D^_n^2 / p~_n, Z = int V^2.

* Z's closed form (pairwise vMF products) against sphere quadrature of
  V^2, incl. the kappa -> 0 limit 1/(4 pi) and antipodal equal lobes (r = 0);
* d log Z / d raw against central finite differences of the closed form
  (clamped kappa' gives 0);
* the expected per-record gradient (sphere quadrature over records drawn from
  p~) equals int f^2 times the gradient of KL(f^2/int f^2 || V^2/Z) computed by
  quadrature and finite differences -- a dropped normaliser term, a missing
  factor 2 or a first-moment weight fails it -- and vanishes when f = V (V^2 is
  then proportional to the second moment);
* end to end through the decoder and the grid: central FD of the loss proxy
  assembled from the forward functions (radiance + product).
"""
import numpy as np
import pytest

from oracle import npm, variance, vmf
from tests.test_oracle_npm import tiny_cfg, random_params, random_batch
from tests.test_oracle_vmf import sphere_quadrature, random_raw


def test_z_closed_form_matches_quadrature():
    rng = np.random.default_rng(1)
    w, qw = sphere_quadrature(300, 600)
    raw = random_raw(rng, 4, 6, kscale=1.0)
    raw[4:8, 0] = np.log([1e-5, 1e-4, 0.01, 0.3])      # near-uniform lobes
    raw[4:8, 1] = np.log([5.0, 20.0, 40.0, 2.0])        # concentrated lobes
    act = vmf.activate(raw, 4)
    z = np.exp(variance.log_z(act))
    for n in range(raw.shape[1]):
        one = {k: (v[..., n:n + 1] if k != 'mu' else v[:, :, n:n + 1]) for k, v in act.items()}
        vq = vmf.mixture_pdf(w, {k: np.repeat(v, w.shape[1], axis=-1) for k, v in one.items()})
        zq = float((qw * vq * vq).sum())
        assert abs(z[n] - zq) <= 1e-9 * zq, (n, z[n], zq)
    # one uniform lobe: Z = 1 / (4 pi); two antipodal lobes of equal kappa (r_ij = 0)
    a1 = vmf.activate(np.array([[0.0], [np.log(1e-5)], [0.0], [0.0]]), 1)
    assert abs(np.exp(variance.log_z(a1))[0] - 1 / (4 * np.pi)) <= 1e-6
    raw2 = np.array([[0.0], [0.0], [np.log(3.0)], [np.log(3.0)], [-30.0], [30.0], [0.0], [0.0]])
    a2 = vmf.activate(raw2, 2)
    assert abs(a2['mu'][2, 0, 0] + a2['mu'][2, 1, 0]) < 1e-9        # mu_1 = -mu_0
    vq = vmf.mixture_pdf(w, {k: np.repeat(v, w.shape[1], axis=-1) for k, v in a2.items()})
    assert abs(np.exp(variance.log_z(a2))[0] - (qw * vq * vq).sum()) <= 1e-9


def test_grad_log_z_vs_central_fd():
    rng = np.random.default_rng(2)
    k = 4
    raw = random_raw(rng, k, 5, kscale=1.2)
    raw[k + 1, 2] = np.log(1e-5) - 1.0      # clamped below
    raw[k + 2, 3] = np.log(1e5) + 1.0       # clamped above
    g, lz = variance.grad_log_z(raw, k)
    assert np.allclose(lz, variance.log_z(vmf.activate(raw, k)), rtol=0, atol=1e-12)
    h = 1e-6
    for c in range(4 * k):
        rp, rm = raw.copy(), raw.copy()
        rp[c] += h; rm[c] -= h
        fd = (variance.log_z(vmf.activate(rp, k)) - variance.log_z(vmf.activate(rm, k))) / (2 * h)
        assert np.all(np.abs(fd - g[c]) <= 1e-6 * np.maximum(1.0, np.abs(fd))), (c, fd, g[c])
    assert g[k + 1, 2] == 0.0 and g[k + 2, 3] == 0.0


def _quadrature_records(raw1, k, f_of_w, w, qw, ps):
    """Per-record gradients for records at every quadrature direction."""
    m = w.shape[1]
    raw = np.repeat(raw1, m, axis=1)
    t = f_of_w(w)
    dropped = np.zeros(m, bool)
    draw, _ = variance.variance_aware_head(raw, w, t, ps, 1.0, dropped, dropped, k)
    return draw, raw


def test_expected_gradient_is_the_kl_gradient_and_vanishes_at_the_optimum():
    rng = np.random.default_rng(3)
    k = 3
    raw1 = random_raw(rng, k, 1, kscale=0.6)
    w, qw = sphere_quadrature(200, 400)
    # records drawn from a positive p~ (mixture of uniform and a lobe about z)
    ps = 0.5 / (4 * np.pi) + 0.5 * 2.0 / (2 * np.pi * (1 - np.exp(-4.0))) * np.exp(2.0 * (w[2] - 1))
    f = lambda d: 0.3 + np.maximum(d[0] * 0.4 + d[1] * 0.2 + d[2] * 0.7, 0.0) ** 2   # a positive integrand
    draw, _ = _quadrature_records(raw1, k, f, w, qw, ps)
    mean = (draw * (qw * ps)[None, :]).sum(axis=1)          # E_{w ~ p~}[per-record gradient]

    def kl(r1):
        raw = np.repeat(r1, w.shape[1], axis=1)
        v = vmf.mixture_pdf(w, vmf.activate(raw, k))
        f2 = f(w) ** 2
        p2 = f2 / (qw * f2).sum()
        q2 = v * v / (qw * v * v).sum()
        return float((qw * p2 * np.log(p2 / q2)).sum())
    c = float((qw * f(w) ** 2).sum())
    h = 1e-5
    for j in range(4 * k):
        rp, rm = raw1.copy(), raw1.copy()
        rp[j] += h; rm[j] -= h
        fd = c * (kl(rp) - kl(rm)) / (2 * h)
        assert abs(mean[j] - fd) <= 1e-6 * max(1.0, abs(fd)), (j, mean[j], fd)
    assert np.abs(mean).max() > 1e-3                       # not trivially zero here
    # f = V: V^2 is proportional to the second moment -> zero expected gradient
    vfun = lambda d: vmf.mixture_pdf(d, vmf.activate(np.repeat(raw1, d.shape[1], axis=1), k))
    draw0, _ = _quadrature_records(raw1, k, vfun, w, qw, ps)
    mean0 = (draw0 * (qw * ps)[None, :]).sum(axis=1)
    assert np.abs(mean0).max() <= 1e-9 * np.abs(draw0).max(), np.abs(mean0).max()


def va_loss_from_forward(cfg, flat, q, wi, target, pdf, n_global):
    """sum_n (D^_n^2 / p~_n / N)(-2 log max(V_n, 1e-30) + log int V_n^2), Z by
    quadrature of the decoded mixture at each record (independent of the closed form)."""
    t = npm.scalar_target(target)
    v = np.maximum(npm.pdf(cfg, flat, q, wi), 1e-30)
    _, act = npm.decode(cfg, flat, q)
    w, qw = sphere_quadrature(120, 240)
    lz = np.empty(t.size)
    for n in range(t.size):
        one = {kk: np.repeat(vv[..., n:n + 1], w.shape[1], axis=-1) for kk, vv in act.items()}
        vq = vmf.mixture_pdf(w, one)
        lz[n] = np.log((qw * vq * vq).sum())
    a = t * t / pdf
    return float((a / n_global * (-2 * np.log(v) + lz)).sum())


@pytest.mark.parametrize("mode", [npm.RADIANCE, npm.PRODUCT])
def test_variance_aware_gradient_end_to_end_vs_fd(mode):
    cfg = tiny_cfg(mode)
    cfg.divergence = npm.VARIANCE_AWARE
    rng = np.random.default_rng(30 + mode)
    flat = random_params(cfg, rng)
    q, wi, tgt, pdf = random_batch(cfg, rng, 12)
    g, stats = npm.gradient(cfg, flat, q, wi, tgt, pdf, 12)
    L = lambda f: va_loss_from_forward(cfg, f, q, wi, tgt, pdf, 12)
    assert abs(stats['loss_proxy'] - L(flat)) <= 1e-8 * abs(L(flat))
    h = 1e-6
    idx = list(rng.choice(cfg.n_mlp, 12, replace=False)) + list(np.flatnonzero(g[cfg.n_mlp:] != 0)[:10] + cfg.n_mlp)
    for j in idx:
        fp, fm = flat.copy(), flat.copy()
        fp[j] += h; fm[j] -= h
        fd = (L(fp) - L(fm)) / (2 * h)
        assert abs(fd - g[j]) <= 1e-5 * max(abs(fd), 1e-3), (j, fd, g[j])


def test_dropped_and_zero_records_contribute_nothing():
    cfg = tiny_cfg()
    cfg.divergence = npm.VARIANCE_AWARE
    rng = np.random.default_rng(40)
    flat = random_params(cfg, rng)
    q, wi, tgt, pdf = random_batch(cfg, rng, 10)
    tgt[:, :4] = 0.0
    pdf[4:7] = np.array([0.0, np.nan, -1.0])
    g, st = npm.gradient(cfg, flat, q, wi, tgt, pdf, 10)
    keep = np.arange(7, 10)
    g2, _ = npm.gradient(cfg, flat, {kk: (v[..., keep] if np.ndim(v) else v) for kk, v in q.items()},
                         wi[:, keep], tgt[:, keep], pdf[keep], 10)
    assert np.allclose(g, g2, rtol=1e-12, atol=1e-15)
    assert st['n_zero_target'] == 4 and st['n_dropped'] == 3 and st['n_used'] == 3
