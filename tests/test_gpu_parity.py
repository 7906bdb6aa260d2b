"""GPU parity: the CUDA path (through the C ABI) against the float64 oracle on
identical seeded inputs and parameters.  Tolerances (BASELINE north_star,
SURVEY §8(c)): cell indices bit-exact; features abs 1e-6; mixture parameters
abs 1e-4 (kappa rel 1e-4); pdf rel 1e-3; sampled directions abs 1e-4 away from
lobe-CDF boundaries; gradient rel-L2 2e-3 (whole vector and per block); loss
rel 1e-4; post-Adam state abs 1e-6 + rel 1e-5 from identical GRADS."""
import numpy as np
import pytest

from workloads import synth
from workloads.configs import CONFIGS
from tests.helpers import oracle_config, rel_l2

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2504_04315_b200 import npm  # noqa: E402  (loads libnpm.so; fails loudly if missing)
from oracle import npm as onpm, grid as ogrid, vmf as ovmf, philox as ophilox, adam as oadam  # noqa: E402


def make_pair(name, seed=7):
    ocfg = oracle_config(name)
    m = npm.Model(0, **CONFIGS[name]["model"])
    assert (m.n_mlp, m.n_grid) == (ocfg.n_mlp, ocfg.n_grid)
    p = synth.random_params(ocfg.layer_dims, ocfg.n_grid, ocfg.n_lobes, seed=seed)
    m.set(npm.BUF_PARAMS, p)
    m.set(npm.BUF_EMA, p)
    return m, ocfg, p.astype(np.float64)


def oq(b, product):
    q = dict(x=b["x"])
    if product:
        q.update(wo=b["wo"].astype(np.float64), n=b["nrm"].astype(np.float64), rough=b["rough"].astype(np.float64))
    return q


def gq(m, b):
    return m.query(b["x"], b.get("wo"), b.get("nrm"), b.get("rough"))


_CACHE = {}


def pair(name):
    if name not in _CACHE:
        _CACHE[name] = make_pair(name)
    return _CACHE[name]


@pytest.mark.parametrize("name,n", [("c1", 3001), ("c2", 5003), ("c5", 2001)])
def test_encode_indices_bit_exact_and_features(name, n):
    m, ocfg, p = pair(name)
    b = synth.query_batch(n, seed=11)
    # include AABB faces, corners and out-of-box points (clamp path)
    b["x"][:, :6] = np.array([[-1, 1, 1, -1.5, 2, 0.999999], [-1, 1, -1, 0, 3, -0.999999],
                              [-1, 1, 1, 0.5, -7, 1e-7]], np.float32)
    q = gq(m, b)
    idx, w = m.encode_debug(q)
    idx, w = idx.cpu().numpy().view(np.uint32), w.cpu().numpy()
    u = ogrid.normalize_position(b["x"], ocfg.aabb_lo, ocfg.aabb_hi)
    for l, (d, s) in enumerate(zip(ocfg.resolutions, ocfg.table_sizes)):
        oi, ow = ogrid.level_corners(u, d, s, s != d ** 3)
        assert np.array_equal(idx[l].astype(np.int64), oi), "level %d" % l
        assert np.abs(w[l] - ow).max() <= 1e-6
    feat = m.encode(q).cpu().numpy()
    ofeat = onpm.encode(ocfg, p, b["x"])
    assert np.abs(feat - ofeat).max() <= 1e-6 * max(1.0, np.abs(ofeat).max())


@pytest.mark.parametrize("name,n", [("c1", 4096), ("c2", 3000), ("c4", 2000), ("c5", 1500)])
def test_decode_mixture_parameters(name, n):
    m, ocfg, p = pair(name)
    prod = ocfg.mode == onpm.PRODUCT
    b = synth.query_batch(n, seed=12, product=prod)
    raw, lam, kap, mu = (t.cpu().numpy() for t in m.decode(gq(m, b)))
    oraw, act = onpm.decode(ocfg, p, oq(b, prod))
    assert np.abs(raw - oraw).max() <= 1e-4
    assert np.abs(lam - act["lam"]).max() <= 1e-4
    assert np.abs(mu - act["mu"]).max() <= 1e-4
    assert (np.abs(kap - act["kappa"]) / act["kappa"]).max() <= 1e-4


def test_decode_from_given_features_and_ema_switch():
    m, ocfg, p = pair("c2")
    b = synth.query_batch(1000, seed=13)
    feat = np.random.default_rng(0).normal(scale=0.5, size=(32, 1000)).astype(np.float32)
    raw = m.decode(gq(m, b), feat=feat)[0].cpu().numpy()
    layers, _ = onpm.unpack(ocfg, p)
    from oracle import mlp as omlp
    oraw = omlp.forward(layers, feat.astype(np.float64))[0]
    assert np.abs(raw - oraw).max() <= 1e-4
    # EMA shadow differs from live params -> use_ema selects it
    p2 = p * 0.5
    m.set(npm.BUF_EMA, p2.astype(np.float32))
    raw_e = m.decode(gq(m, b), use_ema=True)[0].cpu().numpy()
    assert np.abs(raw_e - onpm.decode(ocfg, p2, dict(x=b["x"]))[0]).max() <= 1e-4
    m.set(npm.BUF_EMA, p.astype(np.float32))


@pytest.mark.parametrize("name", ["c1", "c2", "c4"])
def test_pdf(name):
    m, ocfg, p = pair(name)
    prod = ocfg.mode == onpm.PRODUCT
    b = synth.query_batch(4000, seed=14, product=prod)
    pdf = m.pdf(gq(m, b), b["wq"]).cpu().numpy()
    opdf = onpm.pdf(ocfg, p, oq(b, prod), b["wq"])
    assert (np.abs(pdf - opdf) / opdf).max() <= 1e-3


def _boundary_mask(act, u1, k):
    """Records whose result is decided by a floating-point comparison that
    fp32 and fp64 may take differently (C-A16/C-A17): u1 within 1e-5 of a lobe
    CDF value (lobe choice), or the chosen lobe's mu_z within 1e-5 of 0 (the
    sign that picks the Duff ONB branch)."""
    cdf = np.cumsum(act["lam"], axis=0)
    near_cdf = (np.abs(cdf - u1[None, :]) < 1e-5).any(axis=0)
    below = u1[None, :] < cdf
    lobe = np.where(below.any(axis=0), below.argmax(axis=0), k - 1)
    muz = act["mu"][2, lobe, np.arange(u1.size)]
    return near_cdf | (np.abs(muz) < 1e-5)


@pytest.mark.parametrize("name", ["c1", "c2", "c4"])
def test_sample_with_caller_uniforms_and_fused_pdf(name):
    m, ocfg, p = pair(name)
    prod = ocfg.mode == onpm.PRODUCT
    n = 4000
    b = synth.query_batch(n, seed=15, product=prod)
    u = np.random.default_rng(3).uniform(size=(3, n)).astype(np.float32)
    u[1, :5] = 0.0                     # the u2 = 0 guard of C-O10
    wi, pdf, pdf_q = (t.cpu().numpy() for t in m.sample(gq(m, b), u=u, wq=b["wq"]))
    _, act = onpm.decode(ocfg, p, oq(b, prod))
    ow, opdf, _ = ovmf.sample(act, u.astype(np.float64), ocfg.n_lobes)
    ok = ~_boundary_mask(act, u[0].astype(np.float64), ocfg.n_lobes)
    assert ok.mean() > 0.99
    err = np.abs(wi - ow).max(axis=0)
    err[~ok] = 0
    j = int(err.argmax())
    assert err[j] <= 1e-4, dict(j=j, err=err[j], u=u[:, j], gpu=wi[:, j], ora=ow[:, j],
                                kappa=act["kappa"][:, j], lam=act["lam"][:, j])
    assert (np.abs(pdf[ok] - opdf[ok]) / opdf[ok]).max() <= 1e-3
    assert np.all(np.isfinite(wi)) and np.allclose((wi ** 2).sum(0), 1, atol=1e-5)
    opdf_q = ovmf.mixture_pdf(b["wq"].astype(np.float64), act)
    assert (np.abs(pdf_q - opdf_q) / opdf_q).max() <= 1e-3


@pytest.mark.parametrize("name,groups", [("c2", "1"), ("c5", "2")])
def test_query_ws_chain_groups_override(name, groups, monkeypatch):
    """query_ws_kernel's other chain-group count for a shape (the default is
    two for L2-resident radiance tables, one for HBM-resident ones and the
    product shape; NPM_QWS_GROUPS overrides at model creation), several tiles
    per CTA and a ragged tail, against the oracle."""
    monkeypatch.setenv("NPM_QWS_GROUPS", groups)
    m, ocfg, p = make_pair(name, seed=13)
    n = 4 * 128 * 148 + 45   # >= 65,536: the binned order bench.py times
    b = synth.query_batch(n, seed=16)
    u = np.random.default_rng(4).uniform(size=(3, n)).astype(np.float32)
    wi, pdf, pdf_q = (t.cpu().numpy() for t in m.sample(gq(m, b), u=u, wq=b["wq"]))
    sel = np.concatenate([np.random.default_rng(5).choice(n, 3000, replace=False), [0, n - 1]])
    _, act = onpm.decode(ocfg, p, dict(x=np.ascontiguousarray(b["x"][:, sel])))
    us = u[:, sel].astype(np.float64)
    ow, opdf, _ = ovmf.sample(act, us, ocfg.n_lobes)
    ok = ~_boundary_mask(act, us[0], ocfg.n_lobes)
    assert np.abs(wi[:, sel][:, ok] - ow[:, ok]).max() <= 1e-4
    assert (np.abs(pdf[sel][ok] - opdf[ok]) / opdf[ok]).max() <= 1e-3
    opq = ovmf.mixture_pdf(b["wq"][:, sel].astype(np.float64), act)
    assert (np.abs(pdf_q[sel] - opq) / opq).max() <= 1e-3


def test_philox_sampling_matches_oracle_generator():
    m, ocfg, p = pair("c2")
    n = 3000
    b = synth.query_batch(n, seed=16)
    seed, offset = 0x0123456789ABCDEF, 1 << 33
    q = gq(m, b)
    w_gen, pdf_gen = (t.cpu().numpy() for t in m.sample(q, seed=seed, offset=offset))
    u = ophilox.sample_uniforms(n, seed, offset).astype(np.float32)   # exact: 24-bit values
    w_u, pdf_u = (t.cpu().numpy() for t in m.sample(q, u=u))
    assert np.array_equal(w_gen, w_u) and np.array_equal(pdf_gen, pdf_u)


def grad_blocks(ocfg):
    blocks, off = [], 0
    for i, o in ocfg.layer_dims:
        blocks.append(("W", off, off + o * i)); off += o * i
        blocks.append(("b", off, off + o)); off += o
    for s in ocfg.table_sizes:
        blocks.append(("grid", off, off + s * ocfg.n_features)); off += s * ocfg.n_features
    return blocks


@pytest.mark.parametrize("name,n,rgb", [("c1", 4096, False), ("c2", 20000, True), ("c4", 6000, False)])
def test_train_gradient_and_stats(name, n, rgb):
    m, ocfg, p = pair(name)
    prod = ocfg.mode == onpm.PRODUCT
    b = synth.training_batch(n, seed=17, product=prod, rgb=rgb, nan_rate=1e-3)
    q = gq(m, b)
    st = m.accumulate_grads(q, b["wi"], b["target"], b["pdf"], n_global=2 * n)
    g = m.get(npm.BUF_GRADS).cpu().numpy().astype(np.float64)
    og, ost = onpm.gradient(ocfg, p, oq(b, prod), b["wi"].astype(np.float64), b["target"].astype(np.float64),
                            b["pdf"].astype(np.float64), 2 * n)
    assert rel_l2(g, og) <= 2e-3
    for kind, a, e in grad_blocks(ocfg):
        if np.linalg.norm(og[a:e]) > 0:
            assert rel_l2(g[a:e], og[a:e]) <= 2e-3, (kind, a, e)
    # untouched grid entries are exactly zero on both sides
    gz = og[ocfg.n_mlp:] == 0
    assert np.all(g[ocfg.n_mlp:][gz] == 0)
    assert abs(st["loss_proxy"] - ost["loss_proxy"]) <= 1e-4 * abs(ost["loss_proxy"])
    for k in ("n_used", "n_zero_target", "n_dropped"):
        assert st[k] == ost[k], k
    # clear GRADS for the next test (optimizer zeroes them)
    m.set(npm.BUF_GRADS, np.zeros(m.n_params, np.float32))


@pytest.mark.parametrize("train_ws", ["1", "0"])
def test_product_train_gradient_both_kernels(train_ws, monkeypatch):
    """The product shape (c4, K = 16) trains in the warp-specialised kernel by
    default; the r01 two-group kernel stays selectable (NPM_TRAIN_WS=0, read at
    model creation).  Both against the oracle at 2 tiles + a ragged tail."""
    monkeypatch.setenv("NPM_TRAIN_WS", train_ws)
    m, ocfg, p = make_pair("c4", seed=11)
    n = 2 * 128 * 148 + 77
    b = synth.training_batch(n, seed=19, product=True, rgb=True, nan_rate=1e-3)
    st = m.accumulate_grads(gq(m, b), b["wi"], b["target"], b["pdf"], n_global=n)
    g = m.get(npm.BUF_GRADS).cpu().numpy().astype(np.float64)
    og, ost = onpm.gradient(ocfg, p, oq(b, True), b["wi"].astype(np.float64), b["target"].astype(np.float64),
                            b["pdf"].astype(np.float64), n)
    assert rel_l2(g, og) <= 2e-3
    for kind, a, e in grad_blocks(ocfg):
        if np.linalg.norm(og[a:e]) > 0:
            assert rel_l2(g[a:e], og[a:e]) <= 2e-3, (kind, a, e)
    gz = og[ocfg.n_mlp:] == 0
    assert np.all(g[ocfg.n_mlp:][gz] == 0)
    assert abs(st["loss_proxy"] - ost["loss_proxy"]) <= 1e-4 * abs(ost["loss_proxy"])
    for k in ("n_used", "n_zero_target", "n_dropped"):
        assert st[k] == ost[k], k


def test_adam_ema_from_identical_grads():
    m, ocfg, p = pair("c2")
    rng = np.random.default_rng(5)
    npar = m.n_params
    g = rng.normal(scale=1e-3, size=npar).astype(np.float32)
    g[ocfg.n_mlp:][rng.uniform(size=npar - ocfg.n_mlp) < 0.7] = 0.0   # untouched grid entries
    g[3] = np.nan
    mm = rng.normal(scale=1e-4, size=npar).astype(np.float32)
    vv = rng.uniform(0, 1e-6, npar).astype(np.float32)
    ee = (p + rng.normal(scale=1e-2, size=npar)).astype(np.float32)
    for which, val in ((npm.BUF_GRADS, g), (npm.BUF_ADAM_M, mm), (npm.BUF_ADAM_V, vv), (npm.BUF_EMA, ee)):
        m.set(which, val)
    m.step = 4
    st = m.optimizer_step()
    pp, m2, v2, e2 = oadam.adam_ema_step(p, g.astype(np.float64), mm.astype(np.float64), vv.astype(np.float64),
                                         ee.astype(np.float64), 5, onpm.grid_mask(ocfg))[:4]
    for which, ref in ((npm.BUF_PARAMS, pp), (npm.BUF_ADAM_M, m2), (npm.BUF_ADAM_V, v2), (npm.BUF_EMA, e2)):
        got = m.get(which).cpu().numpy().astype(np.float64)
        assert np.all(np.abs(got - ref) <= 1e-6 + 1e-5 * np.abs(ref)), which
    assert st["n_nonfinite_grad"] == 1
    gf = np.where(np.isfinite(g), g, 0).astype(np.float64)
    assert abs(st["grad_norm_sq"] - (gf ** 2).sum()) <= 1e-4 * (gf ** 2).sum()
    assert np.all(m.get(npm.BUF_GRADS).cpu().numpy() == 0)
    assert m.step == 5
    # restore
    m.set(npm.BUF_PARAMS, p.astype(np.float32)); m.set(npm.BUF_EMA, p.astype(np.float32))
    for which in (npm.BUF_ADAM_M, npm.BUF_ADAM_V):
        m.set(which, np.zeros(npar, np.float32))
    m.step = 0


def test_train_step_equals_accumulate_plus_optimizer_and_descends():
    name = "c1"
    ocfg = oracle_config(name)
    b = synth.training_batch(4096, seed=18)
    ms = []
    for _ in range(2):
        mm = npm.Model(0, **CONFIGS[name]["model"])
        ms.append(mm)
    q0, q1 = gq(ms[0], b), gq(ms[1], b)
    s0 = ms[0].train_step(q0, b["wi"], b["target"], b["pdf"])
    ms[1].accumulate_grads(q1, b["wi"], b["target"], b["pdf"])
    ms[1].optimizer_step()
    assert rel_l2(ms[0].get().cpu().numpy(), ms[1].get().cpu().numpy()) < 1e-5
    losses = [s0["loss_proxy"]] + [ms[0].train_step(q0, b["wi"], b["target"], b["pdf"])["loss_proxy"]
                                   for _ in range(30)]
    assert losses[-1] < losses[0]


def test_edge_cases_empty_single_zero_targets_and_errors():
    m, ocfg, p = pair("c2")
    b = synth.training_batch(1, seed=19)
    q = gq(m, b)
    # n = 1
    pdf = m.pdf(q, b["wi"]).cpu().numpy()
    assert np.isclose(pdf[0], onpm.pdf(ocfg, p, dict(x=b["x"]), b["wi"])[0], rtol=1e-3)
    # n = 0 is a no-op
    e = np.zeros((3, 0), np.float32)
    q0 = m.query(e)
    assert m.pdf(q0, e).numel() == 0
    st = m.accumulate_grads(q0, e, np.zeros((1, 0), np.float32), np.zeros(0, np.float32), n_global=1)
    assert st["n_used"] == 0
    # all-zero targets -> zero gradient
    bz = synth.training_batch(3000, seed=20)
    st = m.accumulate_grads(gq(m, bz), bz["wi"], np.zeros((1, 3000), np.float32), bz["pdf"])
    assert st["n_zero_target"] == 3000 and st["loss_proxy"] == 0
    assert np.all(m.get(npm.BUF_GRADS).cpu().numpy() == 0)
    # invalid arguments fail without enqueuing work
    with pytest.raises(npm.NpmError):
        npm.npm_pdf(m.h, q, None, None, None, 0, None)
    with pytest.raises(npm.NpmError):
        npm.npm_train_step(m.h, q, *[torch.zeros(1, device="cuda")] * 4, 2, torch.ones(1, device="cuda"), 1)


def test_host_pointers_are_staged():
    m, ocfg, p = pair("c2")
    b = synth.query_batch(777, seed=21)
    x = np.ascontiguousarray(b["x"])
    q = npm.make_query(777, x[0], x[1], x[2])
    w = np.ascontiguousarray(b["wq"])
    out = np.zeros(777, np.float32)
    npm.npm_pdf(m.h, q, w[0], w[1], w[2], 0, out)          # pageable host in and out
    opdf = onpm.pdf(ocfg, p, dict(x=b["x"]), b["wq"])
    assert (np.abs(out - opdf) / opdf).max() <= 1e-3


def test_full_size_c2_sampled_parity():
    """BASELINE c2 at full size (921,600 queries / records) in the launch
    configuration bench.py times; outputs checked on a random sample that the
    oracle computes one by one."""
    m, ocfg, p = pair("c2")
    n = CONFIGS["c2"]["n"]
    b = synth.query_batch(n, seed=22)
    q = gq(m, b)
    wi, pdf, pdf_q = (t.cpu().numpy() for t in m.sample(q, seed=99, offset=0, wq=b["wq"]))
    sel = np.random.default_rng(1).choice(n, 3000, replace=False)
    sel = np.concatenate([sel, [0, n - 1]])
    bx = dict(x=np.ascontiguousarray(b["x"][:, sel]))
    _, act = onpm.decode(ocfg, p, bx)
    u = ophilox.sample_uniforms(n, 99, 0)[:, sel]
    ow, opdf, _ = ovmf.sample(act, u, ocfg.n_lobes)
    ok = ~_boundary_mask(act, u[0], ocfg.n_lobes)
    assert np.abs(wi[:, sel][:, ok] - ow[:, ok]).max() <= 1e-4
    assert (np.abs(pdf[sel][ok] - opdf[ok]) / opdf[ok]).max() <= 1e-3
    opq = ovmf.mixture_pdf(b["wq"][:, sel].astype(np.float64), act)
    assert (np.abs(pdf_q[sel] - opq) / opq).max() <= 1e-3
    # training at full size: per-sample-independent properties + loss vs oracle on the whole batch
    tb = synth.training_batch(n, seed=23)
    st = m.accumulate_grads(gq(m, tb), tb["wi"], tb["target"], tb["pdf"])
    g = m.get(npm.BUF_GRADS).cpu().numpy().astype(np.float64)
    assert np.all(np.isfinite(g))
    og, ost = onpm.gradient(ocfg, p, dict(x=tb["x"]), tb["wi"].astype(np.float64),
                            tb["target"].astype(np.float64), tb["pdf"].astype(np.float64), n)
    assert rel_l2(g, og) <= 2e-3
    assert abs(st["loss_proxy"] - ost["loss_proxy"]) <= 1e-4 * abs(ost["loss_proxy"])
    m.set(npm.BUF_GRADS, np.zeros(m.n_params, np.float32))
