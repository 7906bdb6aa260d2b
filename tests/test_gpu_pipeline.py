"""Host-batch pipelining (npm_capi.cu HostPipe): when every array of a
npm_sample / npm_accumulate_grads / npm_train_step call is a host pointer and
n >= 131,072, the batch is processed in NPM_PIPE_CHUNKS (default 3) chunks with the host<->device copies
of neighbouring chunks overlapping the kernels.  The results must equal the
device-pointer path: sample outputs bit for bit (each query is independent of
the others), gradients up to fp32 summation order, statistics exactly."""
import numpy as np
import pytest

from workloads import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2504_04315_b200 import npm  # noqa: E402
from tests.helpers import rel_l2  # noqa: E402
from tests.test_gpu_parity import make_pair  # noqa: E402


@pytest.mark.parametrize("pinned", [True, False])
@pytest.mark.parametrize("philox", [True, False])
def test_pipelined_sample_equals_device_path(pinned, philox):
    m, _, _ = make_pair("c2", seed=41)
    n = 300007                                   # ragged last chunk
    b = synth.query_batch(n, seed=42)
    u = None if philox else np.random.default_rng(43).uniform(size=(3, n)).astype(np.float32)
    H = (lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()) if pinned else \
        (lambda a: torch.from_numpy(np.ascontiguousarray(a)))
    hx, hw = H(b["x"]), H(b["wq"])
    hu = H(u) if u is not None else None
    hq = npm.make_query(n, hx[0], hx[1], hx[2])
    hwi, hp, hpq = H(np.zeros((3, n), np.float32)), H(np.zeros(n, np.float32)), H(np.zeros(n, np.float32))
    npm.npm_sample(m.h, hq, hu, 99, 1234, 1, hwi[0], hwi[1], hwi[2], hp, hw[0], hw[1], hw[2], hpq)
    torch.cuda.synchronize()
    dq = m.query(b["x"])
    wi, pdf, pdf_q = (t.cpu().numpy() for t in m.sample(dq, u=u, seed=99, offset=1234, use_ema=True, wq=b["wq"]))
    assert np.array_equal(hwi.numpy(), wi) and np.array_equal(hp.numpy(), pdf) and np.array_equal(hpq.numpy(), pdf_q)


@pytest.mark.parametrize("rgb", [False, True])
def test_pipelined_accumulate_equals_device_path(rgb):
    m1, _, p = make_pair("c2", seed=44)
    m2, _, _ = make_pair("c2", seed=44)
    n = 262147
    tb = synth.training_batch(n, seed=45, rgb=rgb, nan_rate=1e-4)
    P = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    hx, hwi, ht, hp = P(tb["x"]), P(tb["wi"]), P(tb["target"]), P(tb["pdf"])
    hq = npm.make_query(n, hx[0], hx[1], hx[2])
    C = ht.shape[0] if ht.dim() == 2 else 1
    s1 = npm.npm_accumulate_grads(m1.h, hq, hwi[0], hwi[1], hwi[2], ht, C, hp, n, True)
    s2 = m2.accumulate_grads(m2.query(tb["x"]), tb["wi"], tb["target"], tb["pdf"], n_global=n)
    for k in ("n_used", "n_zero_target", "n_dropped"):
        assert s1[k] == s2[k], k
    assert abs(s1["loss_proxy"] - s2["loss_proxy"]) <= 1e-6 * abs(s2["loss_proxy"])
    g1 = m1.get(npm.BUF_GRADS).cpu().numpy().astype(np.float64)
    g2 = m2.get(npm.BUF_GRADS).cpu().numpy().astype(np.float64)
    assert rel_l2(g1, g2) <= 1e-5


def test_step_stats_async_equals_sync_read():
    import ctypes
    m, _, _ = make_pair("c2", seed=46)
    tb = synth.training_batch(5000, seed=47, nan_rate=1e-3)
    st = m.train_step(m.query(tb["x"]), tb["wi"], tb["target"], tb["pdf"])
    buf = torch.zeros(ctypes.sizeof(npm.npm_step_stats), dtype=torch.uint8).pin_memory()
    npm.npm_step_stats_async(m.h, buf.data_ptr())
    torch.cuda.synchronize()
    got = npm.npm_step_stats.from_buffer_copy(buf.numpy().tobytes()).as_dict()
    assert got == st


def test_native_nccl_communicator_single_rank():
    # npm_comm_init at world size 1: the allreduce inside npm_optimizer_step is
    # the identity, so the step equals the one without a communicator
    m1, _, _ = make_pair("c1", seed=48)
    m2, _, _ = make_pair("c1", seed=48)
    npm.npm_comm_init(m2.h, 0, 1, npm.npm_get_unique_id())
    with pytest.raises(npm.NpmError):
        npm.npm_comm_init(m2.h, 0, 1, npm.npm_get_unique_id())       # already attached
    with pytest.raises(npm.NpmError):
        npm.npm_comm_init(m1.h, 1, 1, npm.npm_get_unique_id())       # rank out of range
    tb = synth.training_batch(4096, seed=49)
    s1 = m1.train_step(m1.query(tb["x"]), tb["wi"], tb["target"], tb["pdf"])
    s2 = m2.train_step(m2.query(tb["x"]), tb["wi"], tb["target"], tb["pdf"])
    assert s1["n_used"] == s2["n_used"]
    assert abs(s1["loss_proxy"] - s2["loss_proxy"]) <= 1e-6 * abs(s1["loss_proxy"])
    p1 = m1.get(npm.BUF_PARAMS).cpu().numpy()
    p2 = m2.get(npm.BUF_PARAMS).cpu().numpy()
    assert np.abs(p1 - p2).max() <= 2 * 5e-3   # Adam amplification of fp32 atomic-order noise only
    assert (p1 == p2).mean() > 0.99


def test_binned_queries_on_two_streams_with_different_sizes():
    """the binning permutation is per-model scratch; two
    device-pointer queries of different sizes (both >= 65,536, so both binned)
    enqueued back to back on two streams must give exactly the results of the
    same queries run one after the other on one stream."""
    m, _, _ = make_pair("c2", seed=44)
    sizes = (300007, 70001)
    bs = [synth.query_batch(n, seed=45 + j) for j, n in enumerate(sizes)]
    ref = []
    for b in bs:
        q = m.query(b["x"])
        ref.append([t.cpu().numpy() for t in m.sample(q, seed=7, offset=0, wq=b["wq"])])
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    qs = [m.query(b["x"]) for b in bs]
    wqs = [torch.from_numpy(b["wq"]).cuda() for b in bs]
    torch.cuda.synchronize()
    outs = []
    for _ in range(3):                           # several rounds of interleaving
        for s, q, wq in zip(streams, qs, wqs):
            with torch.cuda.stream(s):
                outs.append((s, m.sample(q, seed=7, offset=0, wq=wq)))
    torch.cuda.synchronize()
    for j, (s, o) in enumerate(outs):
        got = [t.cpu().numpy() for t in o]
        for a, b in zip(got, ref[j % 2]):
            assert np.array_equal(a, b), j


@pytest.mark.parametrize("pipelined", [True, False])
def test_frame_step_equals_sample_then_train_step(pipelined):
    """npm_frame_step (one pipeline over a frame's queries and records) gives
    the query outputs of npm_sample bit for bit and the training step's
    statistics (loss proxy, record counts, gradient norm) of
    npm_accumulate_grads + npm_optimizer_step; the post-step parameters agree
    to the Adam amplification bound (2 lr) and mostly exactly."""
    n = 300007 if pipelined else 5003
    b = synth.query_batch(n, seed=51)
    tb = synth.training_batch(n, seed=52, rgb=True)
    H = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    res = []
    for fused in (True, False):
        m, _, _ = make_pair("c2", seed=50)
        hx, hw, tx, twi, ttg, tpd = H(b["x"]), H(b["wq"]), H(tb["x"]), H(tb["wi"]), H(tb["target"]), H(tb["pdf"])
        hq = npm.make_query(n, hx[0], hx[1], hx[2])
        ht = npm.make_query(n, tx[0], tx[1], tx[2])
        wi, pdf, pdfq = H(np.zeros((3, n), np.float32)), H(np.zeros(n, np.float32)), H(np.zeros(n, np.float32))
        if fused:
            st = npm.npm_frame_step(m.h, hq, None, 5, 77, 1, wi[0], wi[1], wi[2], pdf, hw[0], hw[1], hw[2], pdfq,
                                    ht, twi[0], twi[1], twi[2], ttg, 3, tpd, n)
        else:
            npm.npm_sample(m.h, hq, None, 5, 77, 1, wi[0], wi[1], wi[2], pdf, hw[0], hw[1], hw[2], pdfq)
            st = npm.npm_train_step(m.h, ht, twi[0], twi[1], twi[2], ttg, 3, tpd, n)
        torch.cuda.synchronize()
        res.append((wi.numpy().copy(), pdf.numpy().copy(), pdfq.numpy().copy(), st, m.get(npm.BUF_PARAMS).cpu().numpy()))
    (w0, p0, q0, s0, par0), (w1, p1, q1, s1, par1) = res
    assert np.array_equal(w0, w1) and np.array_equal(p0, p1) and np.array_equal(q0, q1)
    for k in ("n_used", "n_zero_target", "n_dropped", "n_nonfinite_grad"):
        assert s0[k] == s1[k], k
    assert abs(s0["loss_proxy"] - s1["loss_proxy"]) <= 1e-5 * abs(s1["loss_proxy"])
    assert abs(s0["grad_norm_sq"] - s1["grad_norm_sq"]) <= 1e-3 * s1["grad_norm_sq"]
    d = np.abs(par0.astype(np.float64) - par1)
    assert d.max() <= 2 * 5e-3 + 1e-6 and (d == 0).mean() > 0.9


@pytest.mark.parametrize("kind", ["learn_alpha", "variance_aware"])
def test_frame_step_with_the_f4_objectives(kind):
    """npm_frame_step from pinned host buffers on a learn_alpha model (records
    carry p_bsdf, staged path: C-A34) and a variance-aware model (divergence
    2, C-A35): the same statistics and parameters as npm_sample +
    npm_train_step on the same host buffers."""
    from workloads.configs import CONFIGS
    from oracle import guide as oguide
    n = 300007   # >= 2 pipeline chunks (the variance-aware model takes the pipelined path)
    b = synth.query_batch(n, seed=53)
    tb = synth.training_batch(n, seed=54)
    pb = oguide.bsdf_pdf(tb["nrm"].astype(np.float64), tb["wi"].astype(np.float64)).astype(np.float32)
    H = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    kw = dict(learn_alpha=1) if kind == "learn_alpha" else dict(divergence=2)
    res = []
    for fused in (True, False):
        m = npm.Model(0, **dict(CONFIGS["c2"]["model"], **kw))
        hx, hw, tx, twi, ttg, tpd, hpb = (H(b["x"]), H(b["wq"]), H(tb["x"]), H(tb["wi"]), H(tb["target"]),
                                          H(tb["pdf"]), H(pb))
        hq = npm.make_query(n, hx[0], hx[1], hx[2])
        ht = npm.make_query(n, tx[0], tx[1], tx[2], bsdf_pdf=hpb if kind == "learn_alpha" else None)
        wi, pdf, pdfq = H(np.zeros((3, n), np.float32)), H(np.zeros(n, np.float32)), H(np.zeros(n, np.float32))
        if fused:
            st = npm.npm_frame_step(m.h, hq, None, 5, 77, 1, wi[0], wi[1], wi[2], pdf, hw[0], hw[1], hw[2], pdfq,
                                    ht, twi[0], twi[1], twi[2], ttg, 1, tpd, n)
        else:
            npm.npm_sample(m.h, hq, None, 5, 77, 1, wi[0], wi[1], wi[2], pdf, hw[0], hw[1], hw[2], pdfq)
            st = npm.npm_train_step(m.h, ht, twi[0], twi[1], twi[2], ttg, 1, tpd, n)
        torch.cuda.synchronize()
        res.append((wi.numpy().copy(), st, m.get(npm.BUF_PARAMS).cpu().numpy()))
        m.close()
    (w0, s0, par0), (w1, s1, par1) = res
    assert np.array_equal(w0, w1)
    for k in ("n_used", "n_zero_target", "n_dropped", "n_nonfinite_grad"):
        assert s0[k] == s1[k], k
    assert abs(s0["loss_proxy"] - s1["loss_proxy"]) <= 1e-5 * abs(s1["loss_proxy"])
    d = np.abs(par0.astype(np.float64) - par1)
    assert d.max() <= 2 * 5e-3 + 1e-6 and (d == 0).mean() > 0.9
    if kind == "learn_alpha":   # the selection head moved away from 0 in both
        head = par0[-((CONFIGS["c2"]["model"].get("mlp_width", 64) + 1 + 3) // 4 * 4):]
        assert np.abs(head).max() > 0
