"""Pins for oracle/product.py: the closed-form vMF product
("closed-form product") and the cosine-lobe factorisation of
NPM-product.  Pinned against the definition (pointwise product of the
two densities), special cases with known answers, normalisation by
quadrature, and optimality of the fitted cosine lobe."""
import math

import numpy as np

from oracle import product, vmf
from tests.test_oracle_vmf import random_raw, sphere_quadrature


def unit(rng, *shape):
    v = rng.normal(size=(3,) + shape)
    return v / np.linalg.norm(v, axis=0)


def lobe(w, mu, k):
    return vmf.lobe_pdf(w, mu[:, None, :], k[None, :])[0]


def test_product_pointwise_equals_product_of_densities():
    # exp(log_scale) v(w | product) = v(w | a) v(w | b) at random w
    rng = np.random.default_rng(0)
    m = 500
    mu_a, mu_b = unit(rng, m), unit(rng, m)
    k_a = np.exp(rng.uniform(-3, 4.5, m))
    k_b = np.exp(rng.uniform(-3, 4.5, m))
    mu_p, k_p, ls = product.vmf_product(mu_a, k_a, mu_b, k_b)
    for _ in range(5):
        w = unit(rng, m)
        lhs = np.exp(ls) * lobe(w, mu_p, k_p)
        rhs = lobe(w, mu_a, k_a) * lobe(w, mu_b, k_b)
        assert np.allclose(lhs, rhs, rtol=1e-10, atol=0)


def test_product_special_cases():
    rng = np.random.default_rng(1)
    mu, k = unit(rng, 4), np.array([0.5, 2.0, 30.0, 700.0])
    # kappa_b = 0: lobe a unchanged, log_scale = log(1 / 4 pi)
    mu_p, k_p, ls = product.vmf_product(mu, k, unit(rng, 4), np.zeros(4))
    assert np.allclose(mu_p, mu) and np.allclose(k_p, k) and np.allclose(ls, math.log(1 / (4 * math.pi)))
    # identical lobes -> (mu, 2 kappa)
    mu_p, k_p, _ = product.vmf_product(mu, k, mu, k)
    assert np.allclose(mu_p, mu) and np.allclose(k_p, 2 * k)
    # antipodal, equal kappa -> uniform (kappa_p = 0, C-A28); pointwise identity still holds
    kk = np.array([0.5, 2.0, 3.0, 1.0])
    mu_p, k_p, ls = product.vmf_product(mu, kk, -mu, kk)
    assert np.allclose(k_p, 0)
    w = unit(rng, 4)
    assert np.allclose(np.exp(ls) / (4 * math.pi), lobe(w, mu, kk) * lobe(w, -mu, kk), rtol=1e-10)


def test_log_c_limits():
    assert np.isclose(product.log_c(0.0), math.log(1 / (4 * math.pi)))
    for k in (1e-8, 1e-3, 1.0, 50.0, 1e4):
        assert np.isclose(product.log_c(k), math.log(k / (2 * math.pi * (1 - math.exp(-2 * k)))), rtol=1e-12)


def test_cosine_product_is_normalised_product():
    # the product mixture is V(w) v_c(w) / integral: normalised (quadrature),
    # and its ratio to V v_c is constant over the sphere
    rng = np.random.default_rng(2)
    act = vmf.activate(random_raw(rng, 8, 3, kscale=1.0), 8)
    n = unit(rng, 3)
    kc, _ = product.fit_cosine_lobe()
    pa = product.cosine_product(act, n, kc)
    assert np.allclose(pa['lam'].sum(axis=0), 1.0)
    w, qw = sphere_quadrature(300, 600)
    for j in range(3):
        one = lambda a: {k: v[..., j:j + 1].repeat(w.shape[1], axis=-1) for k, v in a.items() if k in ('lam', 'kappa', 'mu')}
        vp = vmf.mixture_pdf(w, one(pa))
        assert abs((vp * qw).sum() - 1.0) < 1e-6
        base = vmf.mixture_pdf(w, one(act)) * lobe(w, np.repeat(n[:, j:j + 1], w.shape[1], axis=1),
                                                       np.full(w.shape[1], kc))
        r = vp / base
        assert np.allclose(r, r[0], rtol=1e-9)


def test_cosine_lobe_fit_is_least_squares_optimal():
    # C-A29: the fitted (kappa, a) minimise the L2 error to max(t, 0) on the sphere
    kc, a = product.fit_cosine_lobe()
    x, wq = np.polynomial.legendre.leggauss(200)
    t = np.concatenate([(x - 1) / 2, (x + 1) / 2])
    wt = np.concatenate([wq / 2, wq / 2]) * 2 * np.pi
    f = np.maximum(t, 0)
    err = lambda k, amp: (wt * (f - amp * np.exp(k * (t - 1))) ** 2).sum()
    e0 = err(kc, a)
    for dk, da in ((1e-3, 0), (-1e-3, 0), (0, 1e-3), (0, -1e-3), (1e-2, 1e-2), (-1e-2, -1e-2)):
        assert e0 < err(kc + dk, a + da)
    assert 1.5 < kc < 3.0 and e0 / (wt * f * f).sum() < 0.05


def test_product_sample_pdf_is_product_mixture_pdf():
    rng = np.random.default_rng(3)
    m = 2000
    act = vmf.activate(random_raw(rng, 8, m), 8)
    n = unit(rng, m)
    u = rng.random((3, m))
    w, pdf, pa = product.product_sample(act, n, 2.0, u, 8)
    assert np.allclose(pdf, vmf.mixture_pdf(w, pa))
    assert np.allclose(np.linalg.norm(w, axis=0), 1)
