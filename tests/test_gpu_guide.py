"""GPU parity for f-1: npm_combined_sample (one-sample MIS of
the BSDF stand-in and the guide) and
npm_unwind_records through the C ABI against oracle/guide.py.
Tolerances as for npm_sample (BASELINE north_star): directions abs 1e-4 away
from lobe-CDF / ONB-sign boundaries, pdfs rel 1e-3, technique exact; the
unwind is a short fp32 recurrence: rel 1e-5."""
import numpy as np
import pytest

from workloads import synth
from tests.helpers import oracle_config

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2504_04315_b200 import npm  # noqa: E402
from oracle import npm as onpm, guide as oguide, philox as ophilox  # noqa: E402
from tests.test_gpu_parity import pair, gq, oq, _boundary_mask  # noqa: E402


def unit_normals(n, seed):
    v = np.random.default_rng(seed).normal(size=(3, n))
    return (v / np.linalg.norm(v, axis=0)).astype(np.float32)


def check_combined(name, n, alpha, seed):
    m, ocfg, p = pair(name)
    prod = ocfg.mode == onpm.PRODUCT
    b = synth.query_batch(n, seed=seed, product=prod)
    nrm = unit_normals(n, seed + 1)
    u = np.random.default_rng(seed + 2).uniform(size=(4, n)).astype(np.float32)
    wi, pdf, gpdf, tech = (t.cpu().numpy() for t in m.combined_sample(gq(m, b), nrm, alpha, u=u))
    _, act = onpm.decode(ocfg, p, oq(b, prod))
    ow, opdf, ov, otech = oguide.combined_sample(act, ocfg.n_lobes, nrm.astype(np.float64), alpha, u.astype(np.float64))
    assert np.array_equal(tech, otech)
    guide_rec = otech == oguide.GUIDE
    ok = ~(guide_rec & _boundary_mask(act, u[0].astype(np.float64), ocfg.n_lobes))
    assert ok.mean() > 0.99
    err = np.abs(wi - ow).max(axis=0)
    err[~ok] = 0
    assert err.max() <= 1e-4, (int(err.argmax()), err.max())
    assert (np.abs(pdf[ok] - opdf[ok]) / opdf[ok]).max() <= 1e-3
    pos = ok & (ov > 0)
    assert (np.abs(gpdf[pos] - ov[pos]) / ov[pos]).max() <= 1e-3
    return tech


@pytest.mark.parametrize("name,alpha", [("c1", 0.5), ("c2", 0.5), ("c2", 0.2), ("c4", 0.5)])
def test_combined_sample_parity(name, alpha):
    tech = check_combined(name, 4099, alpha, 40)
    frac = (tech == oguide.BSDF).mean()
    assert abs(frac - alpha) < 0.05
    assert not (tech == oguide.FALLBACK).any()


def test_combined_sample_degenerate_alpha():
    t0 = check_combined("c2", 1000, 0.0, 50)
    assert (t0 == oguide.GUIDE).all()
    t1 = check_combined("c2", 1000, 1.0, 51)
    assert (t1 == oguide.BSDF).all()


def test_combined_sample_philox_is_four_uniform_stream():
    m, ocfg, p = pair("c2")
    n = 2000
    b = synth.query_batch(n, seed=52)
    nrm = unit_normals(n, 53)
    q = gq(m, b)
    seed, offset = 0xFEEDFACE12345, 77
    got = [t.cpu().numpy() for t in m.combined_sample(q, nrm, 0.5, seed=seed, offset=offset)]
    u = ophilox.sample_uniforms(n, seed, offset, count=4).astype(np.float32)   # exact 24-bit values
    ref = [t.cpu().numpy() for t in m.combined_sample(q, nrm, 0.5, u=u)]
    for a, r in zip(got, ref):
        assert np.array_equal(a, r)


def test_combined_sample_underflow_fallback():
    # non-finite parameters: every guide-branch record falls back (C-A26)
    name = "c1"
    m, ocfg, p = pair(name)
    n = 1000
    b = synth.query_batch(n, seed=54)
    nrm = unit_normals(n, 55)
    u = np.random.default_rng(56).uniform(size=(4, n)).astype(np.float32)
    bad = np.full(p.size, np.nan, np.float32)
    m.set(npm.BUF_EMA, bad)
    try:
        wi, pdf, gpdf, tech = (t.cpu().numpy() for t in m.combined_sample(gq(m, b), nrm, 0.5, u=u, use_ema=True))
    finally:
        m.set(npm.BUF_EMA, p.astype(np.float32))
    _, act = onpm.decode(ocfg, bad.astype(np.float64), oq(b, False))
    ow, opdf, ov, otech = oguide.combined_sample(act, ocfg.n_lobes, nrm.astype(np.float64), 0.5, u.astype(np.float64))
    assert np.array_equal(tech, otech)
    fb = otech == oguide.FALLBACK
    assert fb.sum() > 400
    assert np.abs(wi[:, fb] - ow[:, fb]).max() <= 1e-5
    pos = fb & (opdf > 1e-3)
    assert (np.abs(pdf[pos] - opdf[pos]) / opdf[pos]).max() <= 1e-5
    assert (gpdf[fb] == 0).all()


def test_combined_sample_errors_and_empty():
    m, _, _ = pair("c2")
    b = synth.query_batch(10, seed=57)
    q = gq(m, b)
    nrm = unit_normals(10, 58)
    with pytest.raises(npm.NpmError):
        m.combined_sample(q, nrm, 1.5)
    with pytest.raises(npm.NpmError):
        m.combined_sample(q, nrm, float("nan"))
    q0 = m.query(np.zeros((3, 0), np.float32))
    out = m.combined_sample(q0, np.zeros((3, 0), np.float32), 0.5)
    assert out[0].shape == (3, 0)


def random_paths(C, D, n, seed):
    rng = np.random.default_rng(seed)
    le = (rng.random((C, D, n)) * (rng.random((1, D, n)) < 0.3) * 4).astype(np.float32)
    fs = (rng.random((C, D, n)) / np.pi).astype(np.float32)
    cosv = rng.random((D, n)).astype(np.float32)
    pdf = (0.05 + rng.random((D, n))).astype(np.float32)
    pdf[rng.random((D, n)) < 0.01] = 0.0          # terminated successors (C-A27)
    depth = rng.integers(0, D + 1, size=n).astype(np.int32)
    depth[:4] = [0, 1, D, D - 1]
    return le, fs, cosv, pdf, depth


@pytest.mark.parametrize("C,D,n,product", [(3, 8, 10007, False), (3, 8, 10007, True), (1, 5, 3001, False),
                                           (1, 1, 17, True)])
def test_unwind_parity(C, D, n, product):
    m, _, _ = pair("c2")
    le, fs, cosv, pdf, depth = random_paths(C, D, n, 60 + D)
    got = m.unwind_records(le, fs, cosv, pdf, depth, product=product).cpu().numpy()
    ref = oguide.unwind_records(le, fs, cosv, pdf, depth, product=product)
    assert np.array_equal(got == 0, ref == 0)
    assert (np.abs(got - ref) <= 1e-5 * np.abs(ref) + 1e-30).all()


def test_unwind_host_pointers_and_train_feed():
    # host (numpy) inputs are staged; the output feeds npm_train_step as D*n records
    m, ocfg, p = pair("c2")
    C, D, n = 3, 4, 512
    le, fs, cosv, pdf, depth = random_paths(C, D, n, 70)
    target = np.zeros((C, D, n), np.float32)
    npm.npm_unwind_records(m.h, le, fs, cosv, pdf, depth, C, D, n, 0, target)
    torch.cuda.synchronize()
    assert np.allclose(target, oguide.unwind_records(le, fs, cosv, pdf, depth), rtol=1e-5, atol=0)
    x = synth.query_batch(D * n, seed=71)["x"]
    wi = unit_normals(D * n, 72)
    st = m.accumulate_grads(m.query(x), wi, target.reshape(C, D * n), pdf.reshape(D * n) + 0.1)
    assert st["n_used"] + st["n_zero_target"] + st["n_dropped"] == D * n
    m.set(npm.BUF_GRADS, np.zeros(p.size, np.float32))
