"""Pins for the learned BSDF selection probability (f-4'; "(1) the BSDF
selection probability could also be learned by our network"; reading C-A34):
alpha(x) = sigmoid(a . h_{L-1} + c), trained on the second moment of the
one-sample MIS estimator f / p~_alpha, p~_alpha = alpha p_bsdf + (1-alpha) V.

* central finite differences of the MC second-moment estimate in (a, c);
* the estimator's expectation: with the records' directions drawn from p~_s,
  the quadrature mean of the per-record head gradient equals
  alpha (1 - alpha) d/d alpha of the TRUE second moment int f^2 / p~_alpha
  (computed by sphere quadrature and a scalar derivative, independently of
  the oracle's gradient formula), and it vanishes at the alpha minimising
  that integral;
* special cases: p_bsdf = V gives 0, zero / dropped records give 0;
* the head is stop-gradient: the rest of the gradient equals learn_alpha = 0's.
"""
import numpy as np
from scipy import optimize

from oracle import npm, vmf, guide
from tests.test_oracle_npm import tiny_cfg, random_params, random_batch
from tests.test_oracle_vmf import sphere_quadrature


def alpha_cfg():
    c = tiny_cfg()
    c.learn_alpha = 1
    return c


def params_with_head(cfg, rng, scale=0.7):
    p = random_params(cfg, rng)
    head = np.zeros(cfg.n_alpha)
    head[:cfg.mlp_width + 1] = rng.normal(scale=scale, size=cfg.mlp_width + 1)
    return np.concatenate([p, head])


def batch(cfg, rng, n):
    q, wi, tgt, pdf = random_batch(cfg, rng, n)
    nrm = q["n"]
    pb = guide.bsdf_pdf(nrm, wi)
    return dict(x=q["x"]), wi, tgt, pdf, pb


def test_layout_and_grid_mask():
    cfg = alpha_cfg()
    assert cfg.n_alpha == 12 and cfg.n_total == cfg.n_mlp + cfg.n_grid + 12
    m = npm.grid_mask(cfg)
    assert m.size == cfg.n_total and m[cfg.n_mlp:cfg.n_mlp + cfg.n_grid].all()
    assert not m[:cfg.n_mlp].any() and not m[cfg.n_mlp + cfg.n_grid:].any()   # the head: always updated


def test_head_gradient_vs_central_fd():
    cfg = alpha_cfg()
    rng = np.random.default_rng(3)
    p = params_with_head(cfg, rng)
    q, wi, tgt, pdf, pb = batch(cfg, rng, 64)
    t = npm.scalar_target(tgt)
    used = np.ones(64, bool)
    g, _ = npm.alpha_second_moment_grad(cfg, p, q, wi, t, pdf, pb, used, 64)
    off = cfg.n_mlp + cfg.n_grid
    h = 1e-6
    for j in list(range(cfg.mlp_width)) + [cfg.mlp_width]:
        pp, pm = p.copy(), p.copy()
        pp[off + j] += h
        pm[off + j] -= h
        fp = npm.alpha_second_moment_grad(cfg, pp, q, wi, t, pdf, pb, used, 64)[1]
        fm = npm.alpha_second_moment_grad(cfg, pm, q, wi, t, pdf, pb, used, 64)[1]
        fd = (fp - fm) / (2 * h)
        assert abs(g[j] - fd) <= 1e-6 * max(1.0, abs(fd)), (j, g[j], fd)


def test_expected_gradient_is_the_derivative_of_the_true_second_moment():
    """One position x, directions over the sphere by quadrature.  With records
    drawn from p~_s (weight p~_s dw), the mean head gradient for the logit is
    alpha (1 - alpha) dM2/dalpha / N-normalisation, M2(alpha) = int f^2 / p~_alpha
    -- and 0 at the minimiser of M2."""
    cfg = alpha_cfg()
    rng = np.random.default_rng(5)
    p = params_with_head(cfg, rng)
    off = cfg.n_mlp + cfg.n_grid
    p[off:off + cfg.mlp_width] = 0.0          # constant alpha = sigmoid(c)
    w, qw = sphere_quadrature(200, 400)
    m = w.shape[1]
    x = np.tile(np.array([[0.2], [-0.3], [0.4]], np.float32), (1, m))
    nrm = np.tile(np.array([[0.0], [0.6], [0.8]]), (1, m))
    q = dict(x=x)
    _, act = npm.decode(cfg, p, q)
    v = vmf.mixture_pdf(w, act)
    pb = guide.bsdf_pdf(nrm, w)
    # integrand f: a smooth positive function of w (a D^ stand-in), and a
    # sampling pdf p~_s that the records came from (normalised, positive)
    f = 0.2 + np.maximum((w * np.array([[0.3], [0.5], [0.81]])).sum(0), 0.0) ** 3
    ps = 0.5 / (4 * np.pi) + 0.5 * pb
    used = np.ones(m, bool)

    def m2(alpha):
        return float(np.sum(qw * f * f / (alpha * pb + (1 - alpha) * v)))

    def mean_grad(c):
        pc = p.copy()
        pc[off + cfg.mlp_width] = c
        g, _ = npm.alpha_second_moment_grad(cfg, pc, q, w, f, ps, pb, used, 1.0)
        # g[-1] = sum_records g_z: re-weight the per-record terms by qw * ps
        alpha = 1 / (1 + np.exp(-c))
        pa = alpha * pb + (1 - alpha) * v
        gz = -(f * f) * (pb - v) * alpha * (1 - alpha) / (pa * pa * ps)
        assert np.isclose(g[-1], gz.sum(), rtol=1e-12)
        return float(np.sum(qw * ps * gz))

    for c in (-1.5, 0.0, 0.8):
        alpha = 1 / (1 + np.exp(-c))
        h = 1e-6
        dm2 = (m2(alpha + h) - m2(alpha - h)) / (2 * h)
        assert np.isclose(mean_grad(c), alpha * (1 - alpha) * dm2, rtol=1e-6, atol=1e-12)
    res = optimize.minimize_scalar(lambda z: m2(1 / (1 + np.exp(-z))), bounds=(-8, 8), method="bounded",
                                   options=dict(xatol=1e-10))
    assert abs(mean_grad(res.x)) <= 1e-6 * abs(mean_grad(res.x - 1.0))
    assert mean_grad(res.x - 1.0) < 0 < mean_grad(res.x + 1.0)   # descent moves towards the optimum


def test_special_cases_give_zero():
    cfg = alpha_cfg()
    rng = np.random.default_rng(7)
    p = params_with_head(cfg, rng)
    q, wi, tgt, pdf, pb = batch(cfg, rng, 32)
    t = npm.scalar_target(tgt)
    _, act = npm.decode(cfg, p, q)
    v = vmf.mixture_pdf(wi, act)
    g, _ = npm.alpha_second_moment_grad(cfg, p, q, wi, t, pdf, v, np.ones(32, bool), 32)   # p_bsdf = V
    assert np.all(np.abs(g) <= 1e-15)
    g, m2 = npm.alpha_second_moment_grad(cfg, p, q, wi, np.zeros(32), pdf, pb, np.ones(32, bool), 32)
    assert np.all(g == 0) and m2 == 0
    g, _ = npm.alpha_second_moment_grad(cfg, p, q, wi, t, pdf, pb, np.zeros(32, bool), 32)
    assert np.all(g == 0)


def test_head_is_stop_gradient_for_the_mixture():
    cfg = alpha_cfg()
    rng = np.random.default_rng(9)
    p = params_with_head(cfg, rng)
    q, wi, tgt, pdf, pb = batch(cfg, rng, 48)
    g, st = npm.gradient(cfg, p, q, wi, tgt, pdf, 48, bsdf_pdf=pb)
    c0 = tiny_cfg()
    g0, st0 = npm.gradient(c0, p[:c0.n_mlp + c0.n_grid], q, wi, tgt, pdf, 48)
    assert np.array_equal(g[:c0.n_mlp + c0.n_grid], g0) and st["loss_proxy"] == st0["loss_proxy"]
    ga, m2 = npm.alpha_second_moment_grad(cfg, p, q, wi, npm.scalar_target(tgt), pdf, pb, np.ones(48, bool), 48)
    assert np.allclose(g[c0.n_mlp + c0.n_grid:][:ga.size], ga, rtol=1e-12, atol=0) and st["alpha_m2"] == m2
    assert np.all(g[c0.n_mlp + c0.n_grid + ga.size:] == 0)


def test_combined_sample_with_a_per_record_alpha_is_unbiased():
    """P:208's one-sample MIS with alpha(x) per record: E[g / p~] = int g for
    g = 1 + a.w (4 pi), the same pin as f-1's with a varying alpha."""
    rng = np.random.default_rng(11)
    m = 400000
    raw = rng.normal(size=(4 * 3, 1)).repeat(m, axis=1)
    act = vmf.activate(raw, 3, 1e-5, 1e5)
    nrm = np.tile(np.array([[0.0], [0.0], [1.0]]), (1, m))
    alpha = rng.uniform(0.1, 0.9, m)
    u = rng.uniform(size=(4, m))
    w, pt, _, _ = guide.combined_sample(act, 3, nrm, alpha, u)
    g = 1.0 + (np.array([[0.3], [-0.2], [0.5]]) * w).sum(0)
    est = g / pt
    assert abs(est.mean() - 4 * np.pi) <= 4 * est.std() / np.sqrt(m)
