"""GPU parity for f-4' (SURVEY 8(f) "next"; "the BSDF selection
probability could also be learned by our network"; reading C-A34): the
selection head alpha(x) = sigmoid(a . h_{L-1} + c) of a learn_alpha model,
trained in the warp-specialised kernel on the second moment of the one-sample
MIS estimator, and used by npm_combined_sample in place of the fixed alpha.

Against the float64 oracle (oracle/npm.py alpha_second_moment_grad, gradient,
selection_probability; oracle/guide.py combined_sample):
* gradient rel-L2 2e-3, whole vector and per block INCLUDING the head's
  W + 1 entries (the mixture blocks must equal the learn_alpha = 0 gradient:
  the head is stop-gradient); the head's padding stays exactly 0;
* Adam + EMA from identical GRADS, abs 1e-6 + rel 1e-5, the head updated every
  step like the MLP (not under the grid's zero-gradient skip rule);
* the combined sample with the per-record learned alpha: technique exact
  away from |u_sel - alpha| < 1e-5 (C-A16-style decision boundary),
  directions abs 1e-4, pdfs rel 1e-3;
* a fresh model's head is 0 (alpha = 1/2, the paper's fixed choice)."""
import numpy as np
import pytest

from workloads import synth
from workloads.configs import CONFIGS
from tests.helpers import oracle_config, rel_l2

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2504_04315_b200 import npm  # noqa: E402
from oracle import npm as onpm, guide as oguide, adam as oadam  # noqa: E402
from tests.test_gpu_parity import grad_blocks, _boundary_mask  # noqa: E402

_CACHE = {}


def alpha_pair(name):
    if name not in _CACHE:
        ocfg = oracle_config(name)
        ocfg.learn_alpha = 1
        m = npm.Model(0, learn_alpha=1, **CONFIGS[name]["model"])
        assert m.n_alpha == ocfg.n_alpha and m.n_params == ocfg.n_total
        fresh = m.get(npm.BUF_PARAMS).cpu().numpy()[ocfg.n_mlp + ocfg.n_grid:]
        assert np.all(fresh == 0)
        p = synth.random_params(ocfg.layer_dims, ocfg.n_grid, ocfg.n_lobes, seed=7)
        head = np.zeros(ocfg.n_alpha, np.float32)
        rng = np.random.default_rng(8)
        head[:ocfg.mlp_width] = rng.normal(scale=1.0, size=ocfg.mlp_width)
        head[ocfg.mlp_width] = 0.1
        pf = np.concatenate([p.astype(np.float32), head])
        m.set(npm.BUF_PARAMS, pf)
        m.set(npm.BUF_EMA, pf)
        _CACHE[name] = (m, ocfg, pf.astype(np.float64))
    return _CACHE[name]


@pytest.mark.parametrize("name,n,rgb", [("c1", 4097, False), ("c2", 20000, True), ("c2", 131, False)])
def test_alpha_gradient_parity(name, n, rgb):
    m, ocfg, p = alpha_pair(name)
    b = synth.training_batch(n, seed=91, rgb=rgb, nan_rate=1e-3)
    pb = oguide.bsdf_pdf(b["nrm"].astype(np.float64), b["wi"].astype(np.float64))
    q = m.query(b["x"], bsdf_pdf=pb.astype(np.float32))
    m.set(npm.BUF_GRADS, np.zeros(m.n_params, np.float32))
    st = m.accumulate_grads(q, b["wi"], b["target"], b["pdf"], n_global=2 * n)
    g = m.get(npm.BUF_GRADS).cpu().numpy().astype(np.float64)
    og, ost = onpm.gradient(ocfg, p, dict(x=b["x"]), b["wi"].astype(np.float64), b["target"].astype(np.float64),
                            b["pdf"].astype(np.float64), 2 * n, bsdf_pdf=pb.astype(np.float32).astype(np.float64))
    assert rel_l2(g, og) <= 2e-3
    head = ocfg.n_mlp + ocfg.n_grid
    blocks = grad_blocks(ocfg) + [("alpha", head, head + ocfg.mlp_width + 1)]
    for kind, a, e in blocks:
        if np.linalg.norm(og[a:e]) > 0:
            assert rel_l2(g[a:e], og[a:e]) <= 2e-3, (kind, a, e, rel_l2(g[a:e], og[a:e]))
    assert np.linalg.norm(og[head:head + ocfg.mlp_width + 1]) > 0
    assert np.all(g[head + ocfg.mlp_width + 1:] == 0)
    for k in ("n_used", "n_zero_target", "n_dropped"):
        assert st[k] == ost[k], k
    m.set(npm.BUF_GRADS, np.zeros(m.n_params, np.float32))


def test_alpha_training_requires_bsdf_pdf():
    m, ocfg, p = alpha_pair("c1")
    b = synth.training_batch(256, seed=92)
    with pytest.raises(RuntimeError):
        m.accumulate_grads(m.query(b["x"]), b["wi"], b["target"], b["pdf"])


def test_alpha_adam_updates_the_head_every_step():
    m, ocfg, p = alpha_pair("c2")
    rng = np.random.default_rng(93)
    npar = m.n_params
    g = rng.normal(scale=1e-3, size=npar).astype(np.float32)
    g[ocfg.n_mlp:ocfg.n_mlp + ocfg.n_grid][rng.uniform(size=ocfg.n_grid) < 0.7] = 0.0
    head = ocfg.n_mlp + ocfg.n_grid
    g[head:head + 8] = 0.0                  # zero head gradients are still Adam steps
    mm = rng.normal(scale=1e-4, size=npar).astype(np.float32)
    vv = rng.uniform(0, 1e-6, npar).astype(np.float32)
    ee = (p + rng.normal(scale=1e-2, size=npar)).astype(np.float32)
    for which, val in ((npm.BUF_GRADS, g), (npm.BUF_ADAM_M, mm), (npm.BUF_ADAM_V, vv), (npm.BUF_EMA, ee)):
        m.set(which, val)
    m.step = 2
    m.optimizer_step()
    pp, m2, v2, e2 = oadam.adam_ema_step(p, g.astype(np.float64), mm.astype(np.float64), vv.astype(np.float64),
                                         ee.astype(np.float64), 3, onpm.grid_mask(ocfg))[:4]
    assert np.all(pp[head:head + 8] != p[head:head + 8])
    for which, ref in ((npm.BUF_PARAMS, pp), (npm.BUF_ADAM_M, m2), (npm.BUF_ADAM_V, v2), (npm.BUF_EMA, e2)):
        got = m.get(which).cpu().numpy().astype(np.float64)
        assert np.all(np.abs(got - ref) <= 1e-6 + 1e-5 * np.abs(ref)), which
    # restore
    m.set(npm.BUF_PARAMS, p.astype(np.float32)); m.set(npm.BUF_EMA, p.astype(np.float32))
    for which in (npm.BUF_ADAM_M, npm.BUF_ADAM_V):
        m.set(which, np.zeros(npar, np.float32))
    m.step = 0


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_combined_sample_with_learned_alpha(name):
    m, ocfg, p = alpha_pair(name)
    n = 6001
    b = synth.query_batch(n, seed=94)
    v = np.random.default_rng(95).normal(size=(3, n))
    nrm = (v / np.linalg.norm(v, axis=0)).astype(np.float32)
    u = np.random.default_rng(96).uniform(size=(4, n)).astype(np.float32)
    q = m.query(b["x"])
    # the fixed-alpha argument is ignored by a learn_alpha model
    res = [t.cpu().numpy() for t in m.combined_sample(q, nrm, 0.0, u=u)]
    res2 = [t.cpu().numpy() for t in m.combined_sample(q, nrm, 1.0, u=u)]
    for a, r in zip(res, res2):
        assert np.array_equal(a, r)
    wi, pdf, gpdf, tech = res
    alpha = onpm.selection_probability(ocfg, p, dict(x=b["x"]))
    assert alpha.std() > 0.08 and alpha.max() - alpha.min() > 0.3   # a non-trivial alpha(x)
    _, act = onpm.decode(ocfg, p, dict(x=b["x"]))
    ow, opdf, ov, otech = oguide.combined_sample(act, ocfg.n_lobes, nrm.astype(np.float64), alpha,
                                                 u.astype(np.float64))
    u64 = u.astype(np.float64)
    ok = np.abs(u64[3] - alpha) >= 1e-5
    ok &= ~((otech == oguide.GUIDE) & _boundary_mask(act, u64[0], ocfg.n_lobes))
    assert ok.mean() > 0.99
    assert np.array_equal(tech[ok], otech[ok])
    err = np.abs(wi - ow).max(axis=0)
    assert err[ok].max() <= 1e-4
    assert (np.abs(pdf[ok] - opdf[ok]) / opdf[ok]).max() <= 1e-3
    pos = ok & (ov > 0)
    assert (np.abs(gpdf[pos] - ov[pos]) / ov[pos]).max() <= 1e-3
    frac = (tech == oguide.BSDF).mean()
    assert abs(frac - alpha.mean()) < 0.03
