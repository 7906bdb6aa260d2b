"""Guided one-sample MIS and training-record construction:
the steps on either side of the hot path in a wavefront path tracer.  Test
infrastructure only -- see oracle/__init__.py.

* combined_sample: with probability alpha sample the BSDF, else the decoded
  mixture; the returned pdf is the one-sample balance-heuristic mixture
  p~ = alpha p_bsdf(w) + (1 - alpha) V(w), the divisor of the estimator and of
  Eq. 9 ("a combination of the BSDF importance sampling and guiding
  distribution"; "fixing the BSDF selection probability to 50%";
  S:339-347 for the interface and the underflow fallback).
* unwind_records: the MC radiance estimate <L_i> at every path vertex by the
  backward unwind <L_i(x_v)> = L_e(x_{v+1} -> x_v) + f_s cos / p~ <L_i(x_{v+1})>
  ("we collect MC radiance estimates along each traced path");
  D^ = <L_i> (radiance mode) or f_s <L_i> cos (product mode, Eq. 12).

Readings:
  C-A24  BSDF stand-in: Lambertian about the shading normal n,
         p_bsdf(w) = max(n.w, 0) / pi, sampled cosine-weighted with (u1, u2)
         in the Duff ONB of n (the paper's BSDFs belong to its renderer).
  C-A25  Uniforms: u = (u1, u2, u3, u_sel); u1..u3 are C-O11's, u_sel =
         (out3 >> 8) 2^-24 of the same Philox call.  BSDF iff u_sel < alpha.
  C-A26  "Guide pdf underflows": the guide branch was taken and V(w) at the
         guide sample is < 1e-30 or non-finite.  The vertex then uses the BSDF
         sample from (u1, u2) with p~ = p_bsdf (technique 2, counted);
         its reported guide pdf is 0.
  C-A27  Unwind: a vertex whose successor has p~ <= 0 or non-finite p~ ends
         the path there (no throughput term); vertices v >= depth get D^ = 0.
"""
import numpy as np

from . import vmf

V_UNDERFLOW = 1e-30
BSDF, GUIDE, FALLBACK = 0, 1, 2


def bsdf_pdf(n, w):
    """C-A24: max(n.w, 0) / pi.  n, w: [3, m] -> [m]."""
    return np.maximum((np.asarray(n) * np.asarray(w)).sum(axis=0), 0.0) / np.pi


def bsdf_sample(n, u1, u2):
    """C-A24: cosine-weighted hemisphere about n: r = sqrt(u1), phi = 2 pi u2,
    local (r cos phi, r sin phi, sqrt(1 - u1)) in the Duff ONB (t1, t2, n)."""
    n = np.asarray(n, np.float64)
    r = np.sqrt(u1)
    phi = 2 * np.pi * u2
    lz = np.sqrt(np.maximum(1.0 - u1, 0.0))
    t1, t2 = vmf.duff_onb(n)
    return (r * np.cos(phi))[None, :] * t1 + (r * np.sin(phi))[None, :] * t2 + lz[None, :] * n


def combined_sample(act, k, n, alpha, u):
    """One-sample MIS (balance heuristic) of BSDF and guide.

    act: activated mixture (vmf.activate); n: shading normals [3, m];
    u: [4, m] uniforms (C-A25).  Returns (w [3, m], p~ [m], V [m], technique [m])
    with V = V(w) (0 for fallback records, C-A26)."""
    u = np.asarray(u, np.float64)
    w_g, v_g, _ = vmf.sample(act, u[:3], k)
    w_b = bsdf_sample(n, u[0], u[1])
    use_bsdf = u[3] < alpha
    w = np.where(use_bsdf[None, :], w_b, w_g)
    v = vmf.mixture_pdf(w, act)
    p = alpha * bsdf_pdf(n, w) + (1.0 - alpha) * v
    tech = np.where(use_bsdf, BSDF, GUIDE)
    fallback = (~use_bsdf) & ~(np.isfinite(v_g) & (v_g >= V_UNDERFLOW))
    w = np.where(fallback[None, :], w_b, w)
    p = np.where(fallback, bsdf_pdf(n, w_b), p)
    v = np.where(fallback, 0.0, v)
    tech = np.where(fallback, FALLBACK, tech)
    return w, p, v, tech


def unwind_records(le, fs, cosv, pdf, depth, product=False):
    """Backward unwind along each path, literal recurrence.

    le: [C, D, m] radiance arriving at vertex v from the vertex its sampled ray
    hit; fs: [C, D, m] BSDF value at vertex v for its sampled direction;
    cosv: [D, m] |cos theta_i| at v; pdf: [D, m] p~ at v; depth: [m] valid
    vertices per path.  Returns D^ [C, D, m] (radiance: <L_i>; product:
    f_s <L_i> cos, C-A27 for invalid vertices)."""
    le = np.asarray(le, np.float64)
    fs = np.asarray(fs, np.float64)
    cosv = np.asarray(cosv, np.float64)
    pdf = np.asarray(pdf, np.float64)
    C, D, m = le.shape
    li = np.zeros((C, D, m))
    for p in range(m):
        for v in range(int(depth[p]) - 1, -1, -1):
            acc = le[:, v, p].copy()
            if v + 1 < depth[p]:
                q = pdf[v + 1, p]
                if np.isfinite(q) and q > 0:
                    acc = acc + fs[:, v + 1, p] * cosv[v + 1, p] / q * li[:, v + 1, p]
            li[:, v, p] = acc
    if product:
        return fs * li * cosv[None, :, :]
    return li
