"""Pins for oracle/vmf.py: Table 1, Eq. 3/4,
Jakob sampling, Eq. 9 head."""
import math
import numpy as np
import pytest
from scipy import stats

from oracle import vmf


def sphere_quadrature(nz=400, nphi=800):
    """Gauss-Legendre in z = cos(theta) x uniform (periodic trapezoid) in phi."""
    z, wz = np.polynomial.legendre.leggauss(nz)
    phi = (np.arange(nphi) + 0.5) * 2 * np.pi / nphi
    Z, P = np.meshgrid(z, phi, indexing='ij')
    r = np.sqrt(1 - Z ** 2)
    w = np.stack([r * np.cos(P), r * np.sin(P), Z]).reshape(3, -1)
    weights = (wz[:, None] * np.full(nphi, 2 * np.pi / nphi)[None, :]).ravel()
    return w, weights


def random_raw(rng, k, n, kscale=1.5):
    raw = rng.normal(size=(4 * k, n))
    raw[k:2 * k] *= kscale
    return raw


def test_activate_zero_raw():
    # all raw zeros -> lambda = 1/K, kappa = 1, theta = phi = 1/2, mu = (-1, 0, 0)
    a = vmf.activate(np.zeros((32, 3)), 8)
    assert np.allclose(a['lam'], 1 / 8) and np.allclose(a['kappa'], 1.0)
    assert np.allclose(a['mu'][0], -1) and np.allclose(a['mu'][1:], 0, atol=1e-15)


def test_softmax_identity():
    # lambda' = (ln 2, 0), K = 2 -> (2/3, 1/3)
    raw = np.zeros((8, 1)); raw[0, 0] = math.log(2)
    a = vmf.activate(raw, 2)
    assert np.allclose(a['lam'][:, 0], [2 / 3, 1 / 3], atol=1e-15)


def test_activate_invariants_fuzz():
    rng = np.random.default_rng(0)
    a = vmf.activate(rng.normal(scale=5, size=(32, 10000)), 8)
    assert np.allclose(a['lam'].sum(axis=0), 1, atol=1e-12)
    assert np.allclose((a['mu'] ** 2).sum(axis=0), 1, atol=1e-12)
    assert (a['kappa'] >= 1e-5 * (1 - 1e-12)).all() and (a['kappa'] <= 1e5 * (1 + 1e-12)).all()


def test_pdf_closed_forms():
    w = np.array([[0.0], [0.0], [1.0]])
    mu = w[:, None, :]
    # kappa -> 0: uniform 1/(4 pi)
    assert np.isclose(vmf.lobe_pdf(w, mu, np.array([[1e-5]]))[0, 0], 1 / (4 * np.pi), rtol=1e-5)
    # w = mu, kappa = 1: e / (4 pi sinh 1) = 0.18406556...
    assert np.isclose(vmf.lobe_pdf(w, mu, np.array([[1.0]]))[0, 0], math.e / (4 * math.pi * math.sinh(1.0)), rtol=1e-14)
    assert abs(math.e / (4 * math.pi * math.sinh(1.0)) - 0.1840655) < 1e-7


def test_stable_form_equals_eq3():
    rng = np.random.default_rng(1)
    a = vmf.activate(random_raw(rng, 8, 200), 8)
    w = rng.normal(size=(3, 200)); w /= np.linalg.norm(w, axis=0)
    stable = vmf.lobe_pdf(w, a['mu'], a['kappa'])
    kap = np.minimum(a['kappa'], 300)     # Eq. 3 as printed overflows beyond ~700
    eq3 = vmf.vmf_pdf_eq3(w[:, None, :], a['mu'], kap)
    stable_c = vmf.lobe_pdf(w, a['mu'], kap)
    assert np.allclose(stable_c, eq3, rtol=1e-10)
    assert np.all(np.isfinite(stable))


@pytest.mark.parametrize("kappa", [0.01, 1.0, 10.0, 100.0])
def test_single_lobe_integrates_to_one(kappa):
    w, q = sphere_quadrature()
    mu = np.array([0.48, -0.6, 0.64]); mu /= np.linalg.norm(mu)
    v = vmf.lobe_pdf(w, np.repeat(mu[:, None, None], w.shape[1], axis=2), np.full((1, w.shape[1]), kappa))
    assert abs((v[0] * q).sum() - 1) < 1e-9


def test_mixture_integrates_to_one():
    rng = np.random.default_rng(2)
    w, q = sphere_quadrature()
    for _ in range(3):
        a = vmf.activate(random_raw(rng, 8, 1), 8)
        act = {k2: np.repeat(v, w.shape[1], axis=-1) for k2, v in a.items()}
        assert abs((vmf.mixture_pdf(w, act) * q).sum() - 1) < 1e-9


def test_duff_onb_orthonormal():
    rng = np.random.default_rng(3)
    mu = rng.normal(size=(3, 1000)); mu /= np.linalg.norm(mu, axis=0)
    mu[:, 0] = [0, 0, -1]; mu[:, 1] = [0, 0, 1]
    t1, t2 = vmf.duff_onb(mu)
    for a, b in [(t1, t1), (t2, t2)]:
        assert np.allclose((a * b).sum(0), 1, atol=1e-12)
    for a, b in [(t1, t2), (t1, mu), (t2, mu)]:
        assert np.allclose((a * b).sum(0), 0, atol=1e-12)


def lobe_act(mu, kappa, n):
    """A K=1 'mixture' with given lobe, shaped like activate() output."""
    return dict(lam=np.ones((1, n)), kappa=np.full((1, n), kappa), mu=np.repeat(mu[:, None, None], n, axis=2))


@pytest.mark.parametrize("kappa", [1e-5, 0.5, 5.0, 50.0, 900.0])
def test_sampler_cosine_cdf_ks(kappa):
    # closed-form CDF of t = mu.w: F(t) = (e^{kappa (t-1)} - e^{-2 kappa}) / (1 - e^{-2 kappa})
    rng = np.random.default_rng(4)
    n = 20000
    mu = np.array([0.2, 0.3, -0.9]); mu /= np.linalg.norm(mu)
    u = rng.uniform(size=(3, n))
    om, pdf, lobe = vmf.sample(lobe_act(mu, kappa, n), u, 1)
    assert np.allclose((om ** 2).sum(0), 1, atol=1e-9)
    t = mu @ om
    cdf = lambda tt: (np.exp(kappa * (np.minimum(tt, 1) - 1)) - np.exp(-2 * kappa)) / (-np.expm1(-2 * kappa))
    assert stats.kstest(t, cdf).pvalue > 1e-3
    # azimuth uniform around mu
    t1, t2 = vmf.duff_onb(mu[:, None])
    az = np.arctan2(t2[:, 0] @ om, t1[:, 0] @ om)
    assert stats.kstest((az + np.pi) / (2 * np.pi), 'uniform').pvalue > 1e-3


def test_sampler_u2_zero_guard():
    # C-O10: at u2 = 0 with large kappa, expm1(-2 kappa) = -1 -> log1p(-1) = -inf; min(., 2) guard
    om, pdf, _ = vmf.sample(lobe_act(np.array([0, 0, 1.0]), 50.0, 1), np.array([[0.5], [0.0], [0.3]]), 1)
    assert np.all(np.isfinite(om)) and np.isclose(om[2, 0], -1.0)


def test_concentration_and_uniform_limits():
    rng = np.random.default_rng(5)
    n = 100000
    mu = np.array([0, 1.0, 0])
    om, _, _ = vmf.sample(lobe_act(mu, 1e4, n), rng.uniform(size=(3, n)), 1)
    assert (mu @ om > 0.999).mean() >= 0.99
    om, _, _ = vmf.sample(lobe_act(mu, 1e-5, n), rng.uniform(size=(3, n)), 1)
    assert np.linalg.norm(om.mean(axis=1)) < 0.01


def test_mixture_sampler_chi_square_and_returned_pdf():
    rng = np.random.default_rng(6)
    k, n = 8, 200000
    a1 = vmf.activate(random_raw(rng, k, 1), k)
    act = {kk: np.repeat(v, n, axis=-1) for kk, v in a1.items()}
    om, pdf, lobe = vmf.sample(act, rng.uniform(size=(3, n)), k)
    assert np.allclose(pdf, vmf.mixture_pdf(om, act), rtol=1e-12)
    # 64 equal-area bins: 8 bands in z x 8 sectors in phi; expected mass by quadrature
    zb = np.clip(((om[2] + 1) / 2 * 8).astype(int), 0, 7)
    pb = np.clip(((np.arctan2(om[1], om[0]) + np.pi) / (2 * np.pi) * 8).astype(int), 0, 7)
    counts = np.bincount(zb * 8 + pb, minlength=64)
    w, q = sphere_quadrature(800, 1600)
    actq = {kk: np.repeat(v, w.shape[1], axis=-1) for kk, v in a1.items()}
    dens = vmf.mixture_pdf(w, actq) * q
    zq = np.clip(((w[2] + 1) / 2 * 8).astype(int), 0, 7)
    pq = np.clip(((np.arctan2(w[1], w[0]) + np.pi) / (2 * np.pi) * 8).astype(int), 0, 7)
    expected = np.bincount(zq * 8 + pq, weights=dens, minlength=64) * n
    keep = expected > 5
    chi2 = ((counts[keep] - expected[keep]) ** 2 / expected[keep]).sum()
    assert stats.chi2.sf(chi2, keep.sum() - 1) > 1e-3


def lossfn(raw, w, s, k):
    a = vmf.activate(raw, k)
    return s * np.log(np.maximum(vmf.mixture_pdf(w, a), 1e-30))


def test_grad_head_vs_central_fd():
    rng = np.random.default_rng(7)
    k, n = 8, 40
    raw = random_raw(rng, k, n)
    w = rng.normal(size=(3, n)); w /= np.linalg.norm(w, axis=0)
    s = rng.uniform(-2, -0.1, n)
    g, _ = vmf.grad_head(raw, w, s, k)
    h = 1e-5
    fd = np.zeros_like(raw)
    for j in range(4 * k):
        rp, rm = raw.copy(), raw.copy()
        rp[j] += h; rm[j] -= h
        fd[j] = (lossfn(rp, w, s, k) - lossfn(rm, w, s, k)) / (2 * h)
    assert np.abs(g - fd).max() <= 1e-6 * max(1.0, np.abs(fd).max())
    # softmax invariance: lambda' gradients sum to 0
    assert np.allclose(g[:k].sum(axis=0), 0, atol=1e-12)


def test_grad_head_stationary_at_mu():
    # single dominant lobe evaluated at w = mu: theta/phi gradients vanish
    k = 2
    raw = np.array([[8.0], [-8.0], [2.0], [0.0], [0.3], [-0.2], [1.1], [0.4]])
    a = vmf.activate(raw, k)
    w = a['mu'][:, 0, :]
    g, _ = vmf.grad_head(raw, w, np.array([-1.0]), k)
    assert abs(g[2 * k, 0]) < 1e-10 and abs(g[3 * k, 0]) < 1e-10


def test_clamped_kappa_has_zero_gradient():
    k = 1
    raw = np.array([[0.0], [20.0], [0.3], [0.1]])      # kappa' > ln 1e5 -> clamped
    w = np.array([[0.0], [0.0], [1.0]])
    g, _ = vmf.grad_head(raw, w, np.array([-1.0]), k)
    assert g[1, 0] == 0.0


def test_eq9_unbiased_when_target_equals_model():
    # With D = V and p~ uniform, E_w[grad] = -(1/4pi)^-1... = grad of int V = 0:
    # the quadrature-weighted Eq. 9 gradient vanishes ("unbiased").
    rng = np.random.default_rng(8)
    k = 8
    raw1 = random_raw(rng, k, 1, kscale=1.0)
    w, q = sphere_quadrature()
    raw = np.repeat(raw1, w.shape[1], axis=1)
    act = vmf.activate(raw, k)
    d = vmf.mixture_pdf(w, act)
    p_unif = 1 / (4 * np.pi)
    s = -(d / p_unif)
    g, _ = vmf.grad_head(raw, w, s, k)
    mean_grad = (g * (q * p_unif)[None, :]).sum(axis=1)
    assert np.abs(mean_grad).max() < 1e-10


def test_record_scale_drops_and_counts():
    t = np.array([1.0, 0.0, np.nan, 2.0, 1.0, np.inf])
    p = np.array([0.5, 0.5, 0.5, 0.0, -1.0, 1.0])
    s, dropped, zero = vmf.record_scale(t, p, 10)
    assert list(dropped) == [False, False, True, True, True, True]
    assert list(zero) == [False, True, False, False, False, False]
    assert s[0] == -0.2 and np.all(s[1:] == 0)
