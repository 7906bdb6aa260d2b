"""End-to-end pins for oracle/npm.py: Eq. 9 + back propagation through the
decoder and the grid (Fig. 2 dashed lines P:187) checked against
central finite differences of the loss proxy assembled from the forward
functions (encode, MLP forward, Table 1, Eq. 4)."""
import numpy as np
import pytest

from oracle import npm, vmf


def tiny_cfg(mode=npm.RADIANCE):
    return npm.Config(mode=mode, n_lobes=3, n_levels=3, n_features=2, base_res=2, max_res=7,
                      log2_hashmap=6, mlp_linear_layers=3, mlp_width=8, sh_bands=2,
                      aabb_lo=(-1, -1, -1), aabb_hi=(1, 1, 1))


def random_params(cfg, rng):
    parts = []
    for i, o in cfg.layer_dims:
        parts += [rng.normal(size=o * i) * np.sqrt(2.0 / (i + o)), rng.normal(size=o) * 0.3]
    parts.append(rng.normal(scale=0.5, size=cfg.n_grid))
    return np.concatenate(parts)


def random_batch(cfg, rng, n):
    x = rng.uniform(-1, 1, (3, n)).astype(np.float32)
    def unit(m):
        w = rng.normal(size=(3, m)); return w / np.linalg.norm(w, axis=0)
    q = dict(x=x, wo=unit(n), n=unit(n), rough=rng.uniform(0.05, 1, n))
    return q, unit(n), rng.uniform(0.1, 2, (3, n)), rng.uniform(0.05, 0.5, n)


def loss_from_forward(cfg, flat, q, wi, target, pdf, n_global):
    s, _, _ = vmf.record_scale(npm.scalar_target(target), pdf, n_global)
    return float((s * np.log(np.maximum(npm.pdf(cfg, flat, q, wi), 1e-30))).sum())


@pytest.mark.parametrize("mode", [npm.RADIANCE, npm.PRODUCT])
def test_full_gradient_vs_fd(mode):
    cfg = tiny_cfg(mode)
    rng = np.random.default_rng(10 + mode)
    flat = random_params(cfg, rng)
    q, wi, tgt, pdf = random_batch(cfg, rng, 30)
    g, stats = npm.gradient(cfg, flat, q, wi, tgt, pdf, 30)
    assert np.isclose(stats['loss_proxy'], loss_from_forward(cfg, flat, q, wi, tgt, pdf, 30), rtol=1e-12)
    h = 1e-6
    idx = list(rng.choice(cfg.n_mlp, 25, replace=False)) + list(cfg.n_mlp + rng.choice(cfg.n_grid, 25, replace=False))
    # make sure touched grid entries are included
    idx += list(np.flatnonzero(g[cfg.n_mlp:] != 0)[:15] + cfg.n_mlp)
    for j in idx:
        fp, fm = flat.copy(), flat.copy()
        fp[j] += h; fm[j] -= h
        fd = (loss_from_forward(cfg, fp, q, wi, tgt, pdf, 30) - loss_from_forward(cfg, fm, q, wi, tgt, pdf, 30)) / (2 * h)
        assert abs(fd - g[j]) <= 1e-5 * max(abs(fd), 1e-3), (j, fd, g[j])


def test_zero_target_gives_zero_gradient_and_untouched_entries_zero():
    cfg = tiny_cfg()
    rng = np.random.default_rng(11)
    flat = random_params(cfg, rng)
    q, wi, tgt, pdf = random_batch(cfg, rng, 20)
    g, st = npm.gradient(cfg, flat, q, wi, np.zeros(20), pdf, 20)
    assert np.all(g == 0) and st['n_zero_target'] == 20
    # one record: grid gradient only at the <= 8 L corners it touches
    g1, _ = npm.gradient(cfg, flat, {k: (v[..., :1]) for k, v in q.items()}, wi[:, :1], tgt[:, :1], pdf[:1], 1)
    assert np.count_nonzero(g1[cfg.n_mlp:].reshape(-1, cfg.n_features).any(axis=1)) <= 8 * cfg.n_levels


def test_union_batch_equals_sum_of_shards():
    # C-A13 / C-O16: with the global 1/N scaling the DP gradient is a plain sum
    cfg = tiny_cfg()
    rng = np.random.default_rng(12)
    flat = random_params(cfg, rng)
    q, wi, tgt, pdf = random_batch(cfg, rng, 40)
    g, _ = npm.gradient(cfg, flat, q, wi, tgt, pdf, 40)
    sh = lambda a, s: a[..., s]
    ga, _ = npm.gradient(cfg, flat, {k: sh(v, slice(0, 17)) for k, v in q.items()}, wi[:, :17], tgt[:, :17], pdf[:17], 40)
    gb, _ = npm.gradient(cfg, flat, {k: sh(v, slice(17, 40)) for k, v in q.items()}, wi[:, 17:], tgt[:, 17:], pdf[17:], 40)
    assert np.allclose(g, ga + gb, rtol=1e-12, atol=1e-15)


def test_train_step_descends_on_repeated_batch():
    # S:363 descent sanity: the loss proxy decreases over steps on a fixed batch
    cfg = tiny_cfg()
    rng = np.random.default_rng(13)
    st = npm.State(cfg, random_params(cfg, rng) * 0.3)
    q, wi, tgt, pdf = random_batch(cfg, rng, 200)
    losses = [npm.train_step(st, q, wi, tgt, pdf)[1]['loss_proxy'] for _ in range(40)]
    assert losses[-1] < losses[0]
    assert st.t == 40


def test_param_layout_counts():
    c2 = npm.Config()
    assert c2.n_mlp == 8352 and c2.n_grid == 2547708
    c1 = npm.Config(n_levels=4, base_res=2, max_res=16, log2_hashmap=0, mlp_linear_layers=2, mlp_width=32)
    assert c1.resolutions == [2, 4, 8, 16] and c1.n_mlp == 1600 and c1.n_grid == 18720
    c4 = npm.Config(mode=npm.PRODUCT, n_lobes=16)
    assert c4.n_in == 65


def test_train_stream_is_a_sequence_of_slice_steps():
    # f-3 (P:298 one optimisation step per mini-batch; P:482 2^18 per batch):
    # micro = n reproduces train_step; micro < n is train_step on each
    # consecutive slice with 1/N = the slice size (last slice ragged)
    cfg = tiny_cfg()
    rng = np.random.default_rng(14)
    p0 = random_params(cfg, rng) * 0.3
    q, wi, tgt, pdf = random_batch(cfg, rng, 50)
    a, b = npm.State(cfg, p0.copy()), npm.State(cfg, p0.copy())
    npm.train_stream(a, q, wi, tgt, pdf, 50)
    npm.train_step(b, q, wi, tgt, pdf)
    assert np.array_equal(a.params, b.params) and a.t == b.t == 1
    c, d = npm.State(cfg, p0.copy()), npm.State(cfg, p0.copy())
    outs = npm.train_stream(c, q, wi, tgt, pdf, 20)
    assert c.t == 3 and len(outs) == 3
    for s0, s1 in ((0, 20), (20, 40), (40, 50)):
        sl = lambda v: v[..., s0:s1]
        g, st = npm.train_step(d, {k: sl(v) for k, v in q.items()}, sl(wi), sl(tgt), sl(pdf), s1 - s0)
    assert np.array_equal(c.params, d.params) and np.array_equal(c.ema, d.ema)
    # the micro-steps differ from one step over the union (not a reordering)
    assert not np.allclose(c.params, a.params)


def chi2_loss_from_forward(cfg, flat, q, wi, target, pdf, n_global):
    # f-4: the MC estimate of int D^2 / V ("other divergence metrics"),
    # (1/N) sum (D^/p~) D^ / max(V, 1e-30), written from the forward functions
    t = npm.scalar_target(target)
    v = np.maximum(npm.pdf(cfg, flat, q, wi), 1e-30)
    return float((t / pdf * t / v).sum() / n_global)


@pytest.mark.parametrize("mode", [npm.RADIANCE, npm.PRODUCT])
def test_chi2_gradient_vs_fd(mode):
    cfg = tiny_cfg(mode)
    cfg.divergence = npm.CHI2
    rng = np.random.default_rng(20 + mode)
    flat = random_params(cfg, rng)
    q, wi, tgt, pdf = random_batch(cfg, rng, 30)
    g, stats = npm.gradient(cfg, flat, q, wi, tgt, pdf, 30)
    assert np.isclose(stats['loss_proxy'], chi2_loss_from_forward(cfg, flat, q, wi, tgt, pdf, 30), rtol=1e-12)
    # the 1/V of chi^2 is more curved than log V: Richardson-extrapolated central FD
    L = lambda f: chi2_loss_from_forward(cfg, f, q, wi, tgt, pdf, 30)

    def cfd(j, h):
        fp, fm = flat.copy(), flat.copy()
        fp[j] += h; fm[j] -= h
        return (L(fp) - L(fm)) / (2 * h)
    idx = list(rng.choice(cfg.n_mlp, 25, replace=False)) + list(np.flatnonzero(g[cfg.n_mlp:] != 0)[:20] + cfg.n_mlp)
    for j in idx:
        fd = (4 * cfd(j, 5e-6) - cfd(j, 1e-5)) / 3
        assert abs(fd - g[j]) <= 1e-5 * max(abs(fd), 1e-3), (j, fd, g[j])


def test_chi2_gradient_unbiased_at_the_target():
    # with D = V (the target is the model itself) and p~ uniform, the expected
    # chi^2 gradient is -int D^2 grad V / V^2 = -grad int V = 0: the
    # quadrature-weighted mean of the per-record raw gradients vanishes
    from tests.test_oracle_vmf import sphere_quadrature, random_raw
    rng = np.random.default_rng(21)
    raw1 = random_raw(rng, 8, 1, kscale=0.7)
    w, qw = sphere_quadrature(300, 600)
    m = w.shape[1]
    raw = np.repeat(raw1, m, axis=1)
    act = vmf.activate(raw, 8)
    D = vmf.mixture_pdf(w, act)
    pdf = np.full(m, 1 / (4 * np.pi))
    s, _, _ = vmf.record_scale(D, pdf, 1.0)
    draw, _ = vmf.grad_head(raw, w, s * D / D, 8)   # s * D^/V with V = D
    mean = (draw * qw[None, :]).sum(axis=1) / (4 * np.pi)
    assert np.abs(mean).max() < 1e-9, np.abs(mean).max()
    # the KL head differs from it by the factor D^/V (here 1): sanity that the factor is applied
    draw_kl, _ = vmf.grad_head(raw, w, s, 8)
    assert np.allclose(draw, draw_kl)
