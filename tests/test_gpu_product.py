"""GPU parity for f-2: npm_sample_cosine_product -- the decoded
mixture times the cosine lobe v(. | n, kappa_c), renormalised
-- against oracle/product.py.  Tolerances as for npm_decode / npm_sample
(BASELINE north_star): lambda, mu abs 1e-4; kappa rel 1e-4; directions abs
1e-4 away from lobe-CDF / ONB-sign boundaries; pdfs rel 1e-3."""
import numpy as np
import pytest

from workloads import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2504_04315_b200 import npm  # noqa: E402
from oracle import npm as onpm, product as oproduct, vmf as ovmf  # noqa: E402
from tests.test_gpu_parity import pair, gq, oq, _boundary_mask  # noqa: E402

KAPPA_C = oproduct.fit_cosine_lobe()[0]


def unit_normals(n, seed):
    v = np.random.default_rng(seed).normal(size=(3, n))
    return (v / np.linalg.norm(v, axis=0)).astype(np.float32)


@pytest.mark.parametrize("name", ["c1", "c2", "c4"])
def test_cosine_product_parity(name):
    m, ocfg, p = pair(name)
    prod = ocfg.mode == onpm.PRODUCT
    n = 4001
    b = synth.query_batch(n, seed=80, product=prod)
    nrm = b["nrm"].astype(np.float32) if prod else unit_normals(n, 81)
    u = np.random.default_rng(82).uniform(size=(3, n)).astype(np.float32)
    wi, pdf, pdf_q, lam, kap, mu = (t.cpu().numpy() if t is not None else None for t in
                                    m.sample_cosine_product(gq(m, b), nrm, KAPPA_C, u=u, wq=b["wq"]))
    _, act = onpm.decode(ocfg, p, oq(b, prod))
    ow, opdf, pa = oproduct.product_sample(act, nrm.astype(np.float64), float(np.float32(KAPPA_C)),
                                           u.astype(np.float64), ocfg.n_lobes)
    assert np.abs(lam - pa["lam"]).max() <= 1e-4
    assert np.abs(mu - pa["mu"]).max() <= 1e-4
    assert (np.abs(kap - pa["kappa"]) / pa["kappa"]).max() <= 1e-4
    ok = ~_boundary_mask(pa, u[0].astype(np.float64), ocfg.n_lobes)
    assert ok.mean() > 0.99
    err = np.abs(wi - ow).max(axis=0)
    err[~ok] = 0
    assert err.max() <= 1e-4
    assert (np.abs(pdf[ok] - opdf[ok]) / opdf[ok]).max() <= 1e-3
    opq = ovmf.mixture_pdf(b["wq"].astype(np.float64), pa)
    assert (np.abs(pdf_q - opq) / opq).max() <= 1e-3


def test_zero_kappa_c_is_plain_sampling():
    # kappa_c = 0: the cosine lobe is uniform, the product is the mixture itself
    m, ocfg, p = pair("c2")
    n = 3000
    b = synth.query_batch(n, seed=83)
    u = np.random.default_rng(84).uniform(size=(3, n)).astype(np.float32)
    q = gq(m, b)
    wi0, pdf0 = (t.cpu().numpy() for t in m.sample(q, u=u))
    wi1, pdf1, _, lam, kap, mu = m.sample_cosine_product(q, unit_normals(n, 85), 0.0, u=u)
    _, lam_r, kap_r, mu_r = (t.cpu().numpy() for t in m.decode(q))
    assert np.abs(lam.cpu().numpy() - lam_r).max() <= 1e-6
    assert np.allclose(kap.cpu().numpy(), kap_r, rtol=1e-6)
    assert np.abs(wi1.cpu().numpy() - wi0).max() <= 1e-5
    assert np.allclose(pdf1.cpu().numpy(), pdf0, rtol=1e-5)


def test_cosine_product_errors():
    m, _, _ = pair("c2")
    b = synth.query_batch(8, seed=86)
    q = gq(m, b)
    with pytest.raises(npm.NpmError):
        m.sample_cosine_product(q, unit_normals(8, 87), -1.0)
