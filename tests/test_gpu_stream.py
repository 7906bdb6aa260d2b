"""GPU parity for f-3: npm_train_stream -- one optimisation step
per consecutive micro-batch of a frame's records -- against
oracle.npm.train_stream, and against npm_train_step on each slice.

The first micro-step starts from identical parameters: its loss proxy meets
the north_star tolerance (rel 1e-4).  Later micro-steps start from parameters
that already differ by the fp32 gradient-summation noise, which Adam's first
steps amplify for near-zero gradient elements ("Why post-Adam
parity must start from identical GRADS"): their losses are compared at rel
1e-3 and the parameters elementwise at abs 1e-5 + rel 1e-4 for >= 99 % of
elements (measured on B200, c1, 3 micro-steps: 99.4 %), every element within
the amplification bound 2 lr per step."""
import numpy as np
import pytest

from workloads import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2504_04315_b200 import npm  # noqa: E402
from oracle import npm as onpm  # noqa: E402
from tests.test_gpu_parity import make_pair, gq, oq  # noqa: E402


def batch(n, seed, rgb=False):
    return synth.training_batch(n, seed=seed, rgb=rgb)


@pytest.mark.parametrize("name,n,micro,rgb", [("c1", 2500, 1000, False), ("c2", 3000, 1024, True)])
def test_train_stream_vs_oracle(name, n, micro, rgb):
    m, ocfg, p = make_pair(name, seed=21)
    tb = batch(n, 22, rgb)
    stats = m.train_stream(gq(m, tb), tb["wi"], tb["target"], tb["pdf"], micro_batch=micro)
    st = onpm.State(ocfg, p.copy())
    ref = onpm.train_stream(st, oq(tb, False), tb["wi"].astype(np.float64), tb["target"].astype(np.float64),
                            tb["pdf"].astype(np.float64), micro)
    steps = (n + micro - 1) // micro
    assert len(stats) == len(ref) == steps
    for j, (a, (_, b)) in enumerate(zip(stats, ref)):
        for k in ("n_used", "n_zero_target", "n_dropped"):
            assert a[k] == b[k], (j, k)
        tol = 1e-4 if j == 0 else 1e-3
        assert abs(a["loss_proxy"] - b["loss_proxy"]) <= tol * abs(b["loss_proxy"]), j
    assert m.step == steps
    got = m.get(npm.BUF_PARAMS).cpu().numpy().astype(np.float64)
    d = np.abs(got - st.params)
    close = d <= 1e-5 + 1e-4 * np.abs(st.params)
    assert close.mean() >= 0.99, close.mean()
    assert d.max() <= 2 * ocfg.lr * steps, d.max()


def test_train_stream_equals_slice_steps_and_single_step():
    name, n, micro = "c2", 2600, 1000
    m1, ocfg, p = make_pair(name, seed=23)
    m2, _, _ = make_pair(name, seed=23)
    tb = batch(n, 24, rgb=True)
    s1 = m1.train_stream(gq(m1, tb), tb["wi"], tb["target"], tb["pdf"], micro_batch=micro)
    s2 = []
    for a in range(0, n, micro):
        b = min(a + micro, n)
        sl = lambda v: np.ascontiguousarray(v[..., a:b])
        s2.append(m2.train_step(m2.query(sl(tb["x"])), sl(tb["wi"]), sl(tb["target"]), sl(tb["pdf"])))
    for a, b in zip(s1, s2):
        assert a["n_used"] == b["n_used"] and a["n_zero_target"] == b["n_zero_target"]
        assert abs(a["loss_proxy"] - b["loss_proxy"]) <= 1e-3 * abs(b["loss_proxy"])
    assert m1.step == m2.step == 3
    # micro >= n is exactly one train_step
    m3, _, _ = make_pair(name, seed=23)
    m4, _, _ = make_pair(name, seed=23)
    a = m3.train_stream(gq(m3, tb), tb["wi"], tb["target"], tb["pdf"], micro_batch=n + 5)
    b = m4.train_step(gq(m4, tb), tb["wi"], tb["target"], tb["pdf"])
    assert len(a) == 1 and a[0]["n_used"] == b["n_used"]
    assert abs(a[0]["loss_proxy"] - b["loss_proxy"]) <= 1e-6 * abs(b["loss_proxy"])


def test_train_stream_errors():
    m, _, _ = make_pair("c1", seed=25)
    tb = batch(100, 26)
    with pytest.raises(npm.NpmError):
        m.train_stream(gq(m, tb), tb["wi"], tb["target"], tb["pdf"], micro_batch=0)


@pytest.mark.parametrize("divergence", [1, 2])
def test_train_stream_other_objectives_vs_oracle(divergence):
    """f-3 micro-steps under the f-4 objectives (chi^2, C-A31; variance-aware,
    C-A35): the same loss / count / parameter tolerances as above."""
    from workloads.configs import CONFIGS
    from tests.helpers import oracle_config
    model = dict(CONFIGS["c1"]["model"], divergence=divergence)
    ocfg = oracle_config(model)
    m = npm.Model(0, **model)
    p = synth.random_params(ocfg.layer_dims, ocfg.n_grid, ocfg.n_lobes, seed=25)
    m.set(npm.BUF_PARAMS, p)
    m.set(npm.BUF_EMA, p)
    n, micro = 2500, 1000
    tb = batch(n, 26)
    stats = m.train_stream(gq(m, tb), tb["wi"], tb["target"], tb["pdf"], micro_batch=micro)
    st = onpm.State(ocfg, p.astype(np.float64).copy())
    ref = onpm.train_stream(st, oq(tb, False), tb["wi"].astype(np.float64), tb["target"].astype(np.float64),
                            tb["pdf"].astype(np.float64), micro)
    assert len(stats) == len(ref) == 3
    for j, (a, (_, b)) in enumerate(zip(stats, ref)):
        for k in ("n_used", "n_zero_target", "n_dropped"):
            assert a[k] == b[k], (j, k)
        tol = 1e-4 if j == 0 else 1e-3
        assert abs(a["loss_proxy"] - b["loss_proxy"]) <= tol * abs(b["loss_proxy"]), j
    got = m.get(npm.BUF_PARAMS).cpu().numpy().astype(np.float64)
    d = np.abs(got - st.params)
    # the record weights D^/V (chi^2) and D^^2/p~ (variance-aware) are heavier-tailed
    # than Eq. 9's, so Adam's amplification of the first micro-step's fp32 noise
    # reaches more near-zero-gradient elements (B200, c1: chi^2 98.2 %)
    frac = (d <= 1e-5 + 1e-4 * np.abs(st.params)).mean()
    assert frac >= 0.95, frac
    assert d.max() <= 2 * ocfg.lr * 3, d.max()
    m.close()
