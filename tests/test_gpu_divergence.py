"""GPU parity for f-4: the Pearson chi^2 training divergence
("Other divergence metrics are also available following a similar
derivation"; reading C-A31) against oracle.npm.gradient with
divergence = CHI2.  Tolerances as for the KL gradient (BASELINE north_star):
rel-L2 2e-3 for the whole vector and per block, loss proxy rel 1e-4, record
counts exact."""
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
from oracle import npm as onpm  # noqa: E402
from tests.test_gpu_parity import gq, oq, grad_blocks  # noqa: E402


def chi2_pair(name, seed=31):
    model = dict(CONFIGS[name]["model"], divergence=1)
    ocfg = oracle_config(model)
    m = npm.Model(0, **model)
    p = synth.random_params(ocfg.layer_dims, ocfg.n_grid, ocfg.n_lobes, seed=seed)
    m.set(npm.BUF_PARAMS, p)
    m.set(npm.BUF_EMA, p)
    return m, ocfg, p.astype(np.float64)


@pytest.mark.parametrize("name,n,rgb", [("c1", 4096, False), ("c2", 20000, True), ("c4", 6000, False)])
def test_chi2_gradient_and_stats(name, n, rgb):
    m, ocfg, p = chi2_pair(name)
    assert ocfg.divergence == onpm.CHI2
    prod = ocfg.mode == onpm.PRODUCT
    b = synth.training_batch(n, seed=32, product=prod, rgb=rgb, nan_rate=1e-3)
    st = m.accumulate_grads(gq(m, b), b["wi"], b["target"], b["pdf"], n_global=n)
    g = m.get(npm.BUF_GRADS).cpu().numpy().astype(np.float64)
    og, ost = onpm.gradient(ocfg, p, oq(b, prod), b["wi"].astype(np.float64), b["target"].astype(np.float64),
                            b["pdf"].astype(np.float64), n)
    assert rel_l2(g, og) <= 2e-3
    for kind, a, e in grad_blocks(ocfg):
        if np.linalg.norm(og[a:e]) > 0:
            assert rel_l2(g[a:e], og[a:e]) <= 2e-3, (kind, a, e)
    assert abs(st["loss_proxy"] - ost["loss_proxy"]) <= 1e-4 * abs(ost["loss_proxy"])
    for k in ("n_used", "n_zero_target", "n_dropped"):
        assert st[k] == ost[k], k
    # the objective changes the gradient: chi^2 and KL differ on the same batch
    okl, _ = onpm.gradient(oracle_config(name), p, oq(b, prod), b["wi"].astype(np.float64),
                           b["target"].astype(np.float64), b["pdf"].astype(np.float64), n)
    assert rel_l2(og, okl) > 0.05


def test_chi2_training_descends():
    m, ocfg, p = chi2_pair("c1")
    b = synth.training_batch(4096, seed=33)
    q = gq(m, b)
    losses = [m.train_step(q, b["wi"], b["target"], b["pdf"])["loss_proxy"] for _ in range(30)]
    assert losses[-1] < losses[0]


def test_bad_divergence_rejected():
    with pytest.raises(npm.NpmError):
        npm.Model(0, **dict(CONFIGS["c1"]["model"], divergence=3))
