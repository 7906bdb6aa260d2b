"""GPU parity at BASELINE.json's full sizes, in the launch configuration
bench.py times, checked on sampled outputs the oracle computes one by one
(SURVEY §8(c)), plus size-independent properties of the training step:
c3 (8,388,608 records / queries, c2 model), c4 (4,194,304, product mode,
K = 16) and c5 (2^22 per GPU, 16 levels, 2^22-entry hashed levels)."""
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
from oracle import npm as onpm, vmf as ovmf, philox as ophilox  # noqa: E402


def make(name, seed=31):
    ocfg = oracle_config(name)
    m = npm.Model(0, **CONFIGS[name]["model"])
    p = synth.random_params(ocfg.layer_dims, ocfg.n_grid, ocfg.n_lobes, seed=seed)
    m.set(npm.BUF_PARAMS, p)
    m.set(npm.BUF_EMA, p)
    return m, ocfg, p


def gq(m, b):
    return m.query(b["x"], b.get("wo"), b.get("nrm"), b.get("rough"))


def sub(b, sel):
    return {k: np.ascontiguousarray(v[..., sel]) for k, v in b.items()}


def oq(b, product):
    q = dict(x=b["x"])
    if product:
        q.update(wo=b["wo"].astype(np.float64), n=b["nrm"].astype(np.float64), rough=b["rough"].astype(np.float64))
    return q


def boundary(act, u1, k):
    cdf = np.cumsum(act["lam"], axis=0)
    near = (np.abs(cdf - u1[None, :]) < 1e-5).any(axis=0)
    below = u1[None, :] < cdf
    lobe = np.where(below.any(axis=0), below.argmax(axis=0), k - 1)
    muz = act["mu"][2, lobe, np.arange(u1.size)]
    return near | (np.abs(muz) < 1e-5)


@pytest.mark.parametrize("name", ["c3", "c4", "c5"])
def test_full_size_query_sampled(name):
    m, ocfg, p = make(name)
    prod = ocfg.mode == onpm.PRODUCT
    n = CONFIGS[name]["n"]
    b = synth.query_batch(n, seed=41, product=prod)
    wi, pdf, pdf_q = (t.cpu().numpy() for t in m.sample(gq(m, b), seed=7, offset=3, wq=b["wq"], use_ema=True))
    assert np.all(np.isfinite(wi)) and np.all(pdf > 0) and np.all(pdf_q > 0)
    sel = np.concatenate([np.random.default_rng(2).choice(n, 2000, replace=False), [0, n - 1]])
    bs = sub(b, sel)
    _, act = onpm.decode(ocfg, p.astype(np.float64), oq(bs, prod))
    u = ophilox.sample_uniforms(n, 7, 3)[:, sel]
    ow, opdf, _ = ovmf.sample(act, u, ocfg.n_lobes)
    ok = ~boundary(act, u[0], ocfg.n_lobes)
    assert np.abs(wi[:, sel][:, ok] - ow[:, ok]).max() <= 1e-4
    assert (np.abs(pdf[sel][ok] - opdf[ok]) / opdf[ok]).max() <= 1e-3
    opq = ovmf.mixture_pdf(bs["wq"].astype(np.float64), act)
    assert (np.abs(pdf_q[sel] - opq) / opq).max() <= 1e-3


@pytest.mark.parametrize("name", ["c3", "c4", "c5"])
def test_full_size_train_properties_and_subset_parity(name):
    """Full-size step: counters partition the batch, the gradient is finite
    and linear in the batch (full = shard A + shard B); the c-config model is
    checked against the oracle on a subset of the same records."""
    m, ocfg, p = make(name)
    prod = ocfg.mode == onpm.PRODUCT
    n = CONFIGS[name]["n"]
    b = synth.training_batch(n, seed=43, product=prod, nan_rate=1e-6)
    st = m.accumulate_grads(gq(m, b), b["wi"], b["target"], b["pdf"], n_global=n)
    assert st["n_used"] + st["n_zero_target"] + st["n_dropped"] == n
    assert st["n_dropped"] >= 1 and np.isfinite(st["loss_proxy"])
    g = m.get(npm.BUF_GRADS).cpu().numpy().astype(np.float64)
    assert np.all(np.isfinite(g))
    m.set(npm.BUF_GRADS, np.zeros(m.n_params, np.float32))
    h = n // 2
    for lo, hi in ((0, h), (h, n)):
        bb = sub(b, slice(lo, hi))
        m.accumulate_grads(gq(m, bb), bb["wi"], bb["target"], bb["pdf"], n_global=n)
    g2 = m.get(npm.BUF_GRADS).cpu().numpy().astype(np.float64)
    assert rel_l2(g2, g) <= 1e-4            # fp32 atomic order only
    m.set(npm.BUF_GRADS, np.zeros(m.n_params, np.float32))
    # subset parity vs the oracle at this configuration's model shape
    sel = np.sort(np.random.default_rng(3).choice(n, 6000, replace=False))
    bs = sub(b, sel)
    stq = m.accumulate_grads(gq(m, bs), bs["wi"], bs["target"], bs["pdf"], n_global=n)
    gs = m.get(npm.BUF_GRADS).cpu().numpy().astype(np.float64)
    og, ost = onpm.gradient(ocfg, p.astype(np.float64), oq(bs, prod), bs["wi"].astype(np.float64),
                            bs["target"].astype(np.float64), bs["pdf"].astype(np.float64), n)
    assert rel_l2(gs, og) <= 2e-3
    assert abs(stq["loss_proxy"] - ost["loss_proxy"]) <= 1e-4 * abs(ost["loss_proxy"])
    m.set(npm.BUF_GRADS, np.zeros(m.n_params, np.float32))


def test_maximum_size_query_and_train():
    """Largest batch the configurations name for one step (c5: 2^25 samples per
    iteration) on ONE GPU, ragged (+3): 64-bit sample indices, tile counts and
    Philox counters past 2^25; sampled rows (incl. the last) against the oracle.
    Training at 2^24 + 5 records: counters partition the batch, gradient finite."""
    m, ocfg, p = make("c2")
    n = (1 << 25) + 3
    b = synth.query_batch(n, seed=51)
    off = (1 << 32) - 7                      # Philox counters cross 2^32
    wi, pdf, pdf_q = (t.cpu().numpy() for t in m.sample(gq(m, b), seed=9, offset=off, wq=b["wq"], use_ema=True))
    sel = np.concatenate([np.random.default_rng(5).choice(n, 1500, replace=False), [0, n - 2, n - 1]])
    bs = sub(b, sel)
    _, act = onpm.decode(ocfg, p.astype(np.float64), oq(bs, False))
    u = ophilox.sample_uniforms(n, 9, off)[:, sel]
    ow, opdf, _ = ovmf.sample(act, u, ocfg.n_lobes)
    ok = ~boundary(act, u[0], ocfg.n_lobes)
    assert np.abs(wi[:, sel][:, ok] - ow[:, ok]).max() <= 1e-4
    assert (np.abs(pdf[sel][ok] - opdf[ok]) / opdf[ok]).max() <= 1e-3
    opq = ovmf.mixture_pdf(bs["wq"].astype(np.float64), act)
    assert (np.abs(pdf_q[sel] - opq) / opq).max() <= 1e-3
    del b, wi, pdf, pdf_q
    nt = (1 << 24) + 5
    tb = synth.training_batch(nt, seed=52, nan_rate=1e-6)
    st = m.accumulate_grads(gq(m, tb), tb["wi"], tb["target"], tb["pdf"], n_global=nt)
    assert st["n_used"] + st["n_zero_target"] + st["n_dropped"] == nt
    g = m.get(npm.BUF_GRADS).cpu().numpy()
    assert np.all(np.isfinite(g)) and np.abs(g).max() > 0
    m.set(npm.BUF_GRADS, np.zeros(m.n_params, np.float32))
