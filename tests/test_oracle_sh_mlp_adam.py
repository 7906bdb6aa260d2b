"""Pins for oracle/sh.py, oracle/mlp.py (Eq. 14),
oracle/adam.py."""
import math
import numpy as np

from oracle import sh, mlp, adam
from tests.test_oracle_vmf import sphere_quadrature


def unit(rng, n):
    w = rng.normal(size=(3, n))
    return w / np.linalg.norm(w, axis=0)


def test_sh_textbook_low_bands():
    rng = np.random.default_rng(0)
    w = unit(rng, 100)
    y = sh.sh_encode(w, 4)
    x, yy, z = w
    c1 = math.sqrt(3 / (4 * math.pi))
    assert np.allclose(y[0], 1 / (2 * math.sqrt(math.pi)))         # Y_0^0
    assert np.allclose(y[1], c1 * yy) and np.allclose(y[2], c1 * z) and np.allclose(y[3], c1 * x)
    assert np.allclose(y[6], 0.25 * math.sqrt(5 / math.pi) * (3 * z * z - 1))
    assert np.allclose(y[8], 0.25 * math.sqrt(15 / math.pi) * (x * x - yy * yy))
    assert np.allclose(y[9], 0.25 * math.sqrt(35 / (2 * math.pi)) * yy * (3 * x * x - yy * yy))


def test_sh_orthonormal_by_quadrature():
    w, q = sphere_quadrature(60, 120)
    y = sh.sh_encode(w, 4)
    gram = (y * q) @ y.T
    assert np.allclose(gram, np.eye(16), atol=1e-10)


def test_sh_parity():
    rng = np.random.default_rng(1)
    w = unit(rng, 50)
    y, ym = sh.sh_encode(w), sh.sh_encode(-w)
    for l in range(4):
        sl = slice(l * l, (l + 1) ** 2)
        assert np.allclose(ym[sl], (-1) ** l * y[sl], atol=1e-12)


def make_layers(rng, dims):
    return [(rng.normal(size=(o, i)) / math.sqrt(i), rng.normal(size=o) * 0.1) for i, o in dims]


def test_mlp_zero_weights_and_per_sample_loops():
    rng = np.random.default_rng(2)
    dims = [(5, 7), (7, 7), (7, 3)]
    z = rng.normal(size=(5, 4))
    zero = [(np.zeros((o, i)), np.zeros(o)) for i, o in dims]
    assert np.all(mlp.forward(zero, z)[0] == 0)
    layers = make_layers(rng, dims)
    out, _, _ = mlp.forward(layers, z)
    for n in range(4):                                                # scalar-loop brute force
        h = list(z[:, n])
        for k, (w, b) in enumerate(layers):
            h2 = [sum(w[o][i] * h[i] for i in range(len(h))) + b[o] for o in range(len(b))]
            h = [max(v, 0.0) for v in h2] if k < 2 else h2
        assert np.allclose(out[:, n], h, atol=1e-13)


def test_mlp_backward_fd():
    rng = np.random.default_rng(3)
    dims = [(6, 9), (9, 9), (9, 4)]
    layers = make_layers(rng, dims)
    z = rng.normal(size=(6, 5))
    dout = rng.normal(size=(4, 5))
    loss = lambda L, zz: (mlp.forward(L, zz)[0] * dout).sum()
    out, pres, inputs = mlp.forward(layers, z)
    grads, dz = mlp.backward(layers, pres, inputs, dout)
    h = 1e-6
    for k, (w, b) in enumerate(layers):
        for (i, j) in [(0, 0), (w.shape[0] - 1, w.shape[1] - 1), (1, 2)]:
            wp = [(ww.copy(), bb.copy()) for ww, bb in layers]; wm = [(ww.copy(), bb.copy()) for ww, bb in layers]
            wp[k][0][i, j] += h; wm[k][0][i, j] -= h
            fd = (loss(wp, z) - loss(wm, z)) / (2 * h)
            assert abs(fd - grads[k][0][i, j]) < 1e-6 * max(1, abs(fd))
        bp = [(ww.copy(), bb.copy()) for ww, bb in layers]; bm = [(ww.copy(), bb.copy()) for ww, bb in layers]
        bp[k][1][0] += h; bm[k][1][0] -= h
        assert abs((loss(bp, z) - loss(bm, z)) / (2 * h) - grads[k][1][0]) < 1e-6
    zp, zm = z.copy(), z.copy(); zp[2, 3] += h; zm[2, 3] -= h
    assert abs((loss(layers, zp) - loss(layers, zm)) / (2 * h) - dz[2, 3]) < 1e-6


def test_dead_relu_zero_grad():
    w1 = np.array([[1.0, 0.0], [0.0, 1.0]]); b1 = np.array([-100.0, 0.0])
    layers = [(w1, b1), (np.ones((1, 2)), np.zeros(1))]
    z = np.array([[0.5], [0.5]])
    out, pres, inputs = mlp.forward(layers, z)
    grads, _ = mlp.backward(layers, pres, inputs, np.ones((1, 1)))
    assert np.all(grads[0][0][0] == 0) and grads[0][1][0] == 0


def test_adam_first_step_identity():
    # first step with gradient g: delta = -lr g / (|g| + eps) exactly
    g = np.array([0.3, -2.0, 1e-3, 0.0, 5.0])
    is_grid = np.array([False, False, True, True, True])
    p0 = np.ones(5)
    p, m, v, e, nnf = adam.adam_ema_step(p0, g, np.zeros(5), np.zeros(5), p0.copy(), 1, is_grid)
    assert np.allclose(p - p0, -5e-3 * g / (np.abs(g) + 1e-8), rtol=1e-12, atol=0)
    assert p[3] == 1.0 and m[3] == 0 and v[3] == 0                  # zero grid grad skipped
    assert nnf == 0


def test_adam_zero_gradient_mlp_unchanged_and_nonfinite():
    p0 = np.arange(4.0)
    g = np.array([0.0, np.nan, np.inf, 0.0])
    p, m, v, e, nnf = adam.adam_ema_step(p0, g, np.zeros(4), np.zeros(4), p0.copy(), 1, np.zeros(4, bool))
    assert np.array_equal(p, p0) and nnf == 2


def test_adam_grid_skip_keeps_moments():
    p0, m0, v0 = np.ones(2), np.array([0.1, 0.1]), np.array([0.2, 0.2])
    p, m, v, _, _ = adam.adam_ema_step(p0, np.array([0.0, 0.0]), m0, v0, p0, 5, np.array([True, False]))
    assert p[0] == 1 and m[0] == 0.1 and v[0] == 0.2                 # grid: skipped
    assert p[1] != 1 and m[1] != 0.1                                  # MLP: always updated


def test_ema_closed_form():
    # after n steps from e0 = 0 with constant p: e = p (1 - d^n)
    p = np.array([2.0, -3.0])
    e = np.zeros(2); m = np.zeros(2); v = np.zeros(2); pp = p.copy()
    for t in range(1, 31):
        pp, m, v, e, _ = adam.adam_ema_step(pp, np.zeros(2), m, v, e, t, np.array([True, True]))
    assert np.allclose(e, p * (1 - 0.99 ** 30), rtol=1e-13)


def test_adam_convex_quadratic():
    # steps on a convex quadratic drive the gradient down
    a = np.array([1.0, 4.0, 0.5])
    p = np.array([1.0, -1.0, 0.7]); m = np.zeros(3); v = np.zeros(3); e = p.copy()
    for t in range(1, 2001):
        p, m, v, e, _ = adam.adam_ema_step(p, a * p, m, v, e, t, np.zeros(3, bool), lr=5e-3)
    assert np.abs(a * p).max() < 1e-2
