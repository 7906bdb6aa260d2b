"""Pins for oracle/guide.py: one-sample MIS of the BSDF
stand-in and the guide and the training-record
unwind.  Each pin is something other than the oracle's
own formula: closed-form distributions, quadrature, the unbiasedness of the
combined estimator against a closed-form integral, a hand-computed path
(tests/golden/unwind_3vertex.txt) and the suffix-sum form of the unwind."""
import os

import numpy as np
from scipy import stats

from oracle import guide, philox, vmf
from tests.test_oracle_vmf import random_raw, sphere_quadrature

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def random_normals(rng, m):
    n = rng.normal(size=(3, m))
    return n / np.linalg.norm(n, axis=0)


def test_bsdf_pdf_normalised():
    # C-A24: integral over the sphere of max(n.w, 0)/pi = 1 (quadrature)
    w, qw = sphere_quadrature(200, 400)
    for n in (np.array([0.0, 0.0, 1.0]), np.array([0.6, -0.0, 0.8]), np.array([-0.48, 0.6, -0.64])):
        p = guide.bsdf_pdf(np.repeat(n[:, None], w.shape[1], axis=1), w)
        assert abs((p * qw).sum() - 1.0) < 1e-4   # kink at n.w = 0 limits the quadrature


def test_bsdf_sample_is_cosine_distributed():
    # cosine-weighted hemisphere: t = n.w has cdf t^2 on [0, 1]; azimuth uniform
    rng = np.random.default_rng(1)
    m = 200000
    n = random_normals(rng, m)
    u = rng.random((2, m))
    w = guide.bsdf_sample(n, u[0], u[1])
    assert np.allclose(np.linalg.norm(w, axis=0), 1.0, atol=1e-12)
    t = (n * w).sum(axis=0)
    assert (t >= -1e-12).all()
    assert stats.kstest(t, lambda x: np.clip(x, 0, 1) ** 2).pvalue > 1e-3
    # closed form: t = sqrt(1 - u1) exactly
    assert np.allclose(t, np.sqrt(1 - u[0]), atol=1e-12)


def test_alpha_one_is_pure_bsdf():
    rng = np.random.default_rng(2)
    m = 4000
    act = vmf.activate(random_raw(rng, 8, m), 8)
    n = random_normals(rng, m)
    u = rng.random((4, m))
    w, p, v, tech = guide.combined_sample(act, 8, n, 1.0, u)
    assert (tech == guide.BSDF).all()
    assert np.allclose(w, guide.bsdf_sample(n, u[0], u[1]))
    assert np.allclose(p, guide.bsdf_pdf(n, w))


def test_alpha_zero_is_pure_guide():
    rng = np.random.default_rng(3)
    m = 4000
    act = vmf.activate(random_raw(rng, 8, m), 8)
    n = random_normals(rng, m)
    u = rng.random((4, m))
    w, p, v, tech = guide.combined_sample(act, 8, n, 0.0, u)
    wg, vg, _ = vmf.sample(act, u[:3], 8)
    assert (tech == guide.GUIDE).all()
    assert np.allclose(w, wg) and np.allclose(p, vg) and np.allclose(v, vg)


def test_combined_estimator_unbiased():
    # The balance-heuristic pdf must be the density the samples are drawn
    # from: E[g(w)/p~(w)] = integral of g = 4 pi for g(w) = 1 + a.w (closed
    # form: the linear term integrates to 0).  A p~ that omits either term of
    # the mixture (or weights it wrongly) is biased by O(1) here.
    rng = np.random.default_rng(4)
    m = 400000
    raw = np.repeat(random_raw(rng, 8, 1, kscale=0.8), m, axis=1)
    act = vmf.activate(raw, 8)
    n = np.repeat(random_normals(rng, 1), m, axis=1)
    a = np.array([0.3, -0.5, 0.7])
    for alpha in (0.5, 0.25):
        u = rng.random((4, m))
        w, p, _, _ = guide.combined_sample(act, 8, n, alpha, u)
        est = (1.0 + a @ w) / p
        se = est.std() / np.sqrt(m)
        assert abs(est.mean() - 4 * np.pi) < 4 * se, (alpha, est.mean(), se)


def test_pdf_symmetric_in_branch():
    # the pdf returned depends only on w, not on the branch that drew it
    rng = np.random.default_rng(5)
    m = 2000
    act = vmf.activate(random_raw(rng, 8, m), 8)
    n = random_normals(rng, m)
    u = rng.random((4, m))
    w, p, v, tech = guide.combined_sample(act, 8, n, 0.5, u)
    assert set(np.unique(tech)) == {guide.BSDF, guide.GUIDE}
    assert np.allclose(p, 0.5 * np.maximum((n * w).sum(axis=0), 0) / np.pi + 0.5 * vmf.mixture_pdf(w, act))


def test_underflow_falls_back_to_bsdf():
    # C-A26: a non-finite guide (NaN raw outputs) -> BSDF sample, p~ = p_bsdf, V := 0
    rng = np.random.default_rng(6)
    m = 64
    raw = random_raw(rng, 8, m)
    raw[:, :32] = np.nan
    act = vmf.activate(raw, 8)
    n = random_normals(rng, m)
    u = rng.random((4, m))
    u[3] = 0.9                      # guide branch everywhere (alpha = 0.5)
    w, p, v, tech = guide.combined_sample(act, 8, n, 0.5, u)
    assert (tech[:32] == guide.FALLBACK).all() and (tech[32:] == guide.GUIDE).all()
    wb = guide.bsdf_sample(n, u[0], u[1])
    assert np.allclose(w[:, :32], wb[:, :32])
    assert np.allclose(p[:32], guide.bsdf_pdf(n[:, :32], wb[:, :32]))
    assert (v[:32] == 0).all()


def test_philox_fourth_uniform_is_out3():
    # C-A25: u_sel = (out3 >> 8) 2^-24 of the same counter as u1..u3
    u4 = philox.sample_uniforms(5, 0x1234, 7, count=4)
    u3 = philox.sample_uniforms(5, 0x1234, 7)
    assert np.array_equal(u4[:3], u3)
    o = philox.philox4x32_10((np.arange(7, 12, dtype=np.uint64), np.zeros(5, np.uint64), np.zeros(5, np.uint64),
                              np.zeros(5, np.uint64)), (0x1234, 0))
    assert np.array_equal(u4[3], (o[3] >> np.uint64(8)).astype(np.float64) * 2.0 ** -24)


def suffix_sum_unwind(le, fs, cosv, pdf, depth):
    # independent form: <L_i(x_v)> = sum_{k >= v} L_e[k] prod_{j = v+1..k} f_s cos / p~ at j
    C, D, m = le.shape
    out = np.zeros((C, D, m))
    for p in range(m):
        for v in range(int(depth[p])):
            tot = np.zeros(C)
            thr = np.ones(C)
            for k in range(v, int(depth[p])):
                if k > v:
                    thr = thr * fs[:, k, p] * cosv[k, p] / pdf[k, p]
                tot = tot + thr * le[:, k, p]
            out[:, v, p] = tot
    return out


def test_unwind_matches_suffix_sum():
    rng = np.random.default_rng(7)
    C, D, m = 3, 6, 50
    le = rng.random((C, D, m)) * (rng.random((1, D, m)) < 0.3)
    fs = rng.random((C, D, m)) / np.pi
    cosv = rng.random((D, m))
    pdf = 0.05 + rng.random((D, m))
    depth = rng.integers(0, D + 1, size=m)
    got = guide.unwind_records(le, fs, cosv, pdf, depth)
    assert np.allclose(got, suffix_sum_unwind(le, fs, cosv, pdf, depth), rtol=1e-12, atol=0)
    assert (got[:, np.arange(D)[:, None] >= depth[None, :]] == 0).all()
    prod = guide.unwind_records(le, fs, cosv, pdf, depth, product=True)
    assert np.allclose(prod, fs * got * cosv[None], rtol=1e-12, atol=0)


def test_unwind_golden_3vertex():
    # hand-computed path (tests/golden/unwind_3vertex.txt)
    rows = {}
    with open(os.path.join(GOLDEN, "unwind_3vertex.txt")) as f:
        for line in f:
            line = line.split("#")[0].strip()
            if line:
                k, *vals = line.split()
                rows[k] = np.array([float(x) for x in vals])
    le = rows["le"].reshape(1, 3, 1)
    fs = rows["fs"].reshape(1, 3, 1)
    cosv = rows["cos"].reshape(3, 1)
    pdf = rows["pdf"].reshape(3, 1)
    got = guide.unwind_records(le, fs, cosv, pdf, np.array([3]))
    assert np.allclose(got[0, :, 0], rows["Li"], rtol=1e-15)
    got_p = guide.unwind_records(le, fs, cosv, pdf, np.array([3]), product=True)
    assert np.allclose(got_p[0, :, 0], rows["Dprod"], rtol=1e-15)


def test_unwind_special_cases():
    # black escape -> all zero; one-bounce emitter -> D^ = L_e; p~ = 0 successor ends the path
    z = np.zeros((3, 4, 2))
    assert (guide.unwind_records(z, np.ones((3, 4, 2)), np.ones((4, 2)), np.ones((4, 2)), np.array([4, 2])) == 0).all()
    le = np.zeros((3, 1, 1)); le[:, 0, 0] = [1.0, 2.0, 3.0]
    got = guide.unwind_records(le, np.ones((3, 1, 1)), np.ones((1, 1)), np.ones((1, 1)), np.array([1]))
    assert np.array_equal(got[:, 0, 0], [1.0, 2.0, 3.0])
    le = np.zeros((1, 2, 1)); le[0, 1, 0] = 4.0
    got = guide.unwind_records(le, np.ones((1, 2, 1)), np.ones((2, 1)), np.array([[1.0], [0.0]]), np.array([2]))
    assert got[0, 0, 0] == 0.0 and got[0, 1, 0] == 4.0
