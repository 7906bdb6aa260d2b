"""Seeded synthetic workload generator shared by the tests and bench.py.

Holds NONE of the method's arithmetic (no grid encoding, no MLP, no vMF
mixture): it only draws inputs shaped like the paper's workloads.  Both the
CUDA path and the oracle receive exactly these arrays.

Recipe:
  * scene proxy: 256 planar quads in the AABB [-1, 1]^3, centres U[-0.9, 0.9]^3,
    random unit normals, side U[0.1, 0.6]; positions uniform on the quads and
    shuffled (path vertices lie on surfaces; deep-bounce order);
  * training directions drawn from p~ = 0.5 cosine-hemisphere(n) + 0.5 uniform
    sphere, a BSDF stand-in at the paper's 50 % selection probability;
    p~ stored in closed form;
  * targets D^ = D(x, w) * xi with D a two-lobe spatially varying radiance field
    (normalised Phong lobes, exponents 50 and 5, lobe direction rotating with
    x) and xi = Bernoulli(0.5) * LogNormal(-s^2/2, s = 1.5): ~50 % zeros
    (escaped/black paths) and heavy tails ("noisy MC radiance estimates");
  * product mode: w_o uniform on the hemisphere of n, roughness U(0.05, 1),
    D^ multiplied by max(n.w, 0) * a roughness-dependent lobe stand-in (Eq. 12);
  * query directions uniform on the sphere;
  * optional NaN/Inf injection into targets / pdfs (fault-injection rate).
"""
import numpy as np

SEED = 0x4E504D


def _unit(rng, n):
    w = rng.normal(size=(3, n))
    return w / np.linalg.norm(w, axis=0)


def _frame(nrm):
    """Any orthonormal tangent pair for unit normals [3, n] (not the method's ONB)."""
    a = np.where(np.abs(nrm[0:1]) > 0.9, np.array([[0.0], [1.0], [0.0]]), np.array([[1.0], [0.0], [0.0]]))
    t = np.cross(a.T, nrm.T).T
    t /= np.linalg.norm(t, axis=0)
    b = np.cross(nrm.T, t.T).T
    return t, b


def scene_points(rng, n, n_quads=256):
    c = rng.uniform(-0.9, 0.9, (3, n_quads))
    nq = _unit(rng, n_quads)
    side = rng.uniform(0.1, 0.6, n_quads)
    t, b = _frame(nq)
    q = rng.integers(0, n_quads, n)
    s1, s2 = rng.uniform(-0.5, 0.5, n), rng.uniform(-0.5, 0.5, n)
    x = c[:, q] + side[q] * (s1 * t[:, q] + s2 * b[:, q])
    x = np.clip(x, -1.0, 1.0)
    perm = rng.permutation(n)
    return x[:, perm].astype(np.float32), nq[:, q][:, perm]


def bsdf_standin_directions(rng, nrm):
    """w ~ 0.5 cosine-hemisphere(n) + 0.5 uniform; returns (w [3,n], p~ [n])."""
    n = nrm.shape[1]
    uni = _unit(rng, n)
    r1, r2 = rng.uniform(size=n), rng.uniform(size=n)
    rad, ph = np.sqrt(r1), 2 * np.pi * r2
    t, b = _frame(nrm)
    cosw = rad * np.cos(ph)[None, :] * t + rad * np.sin(ph)[None, :] * b + np.sqrt(np.maximum(1 - r1, 0))[None, :] * nrm
    pick = rng.uniform(size=n) < 0.5
    w = np.where(pick[None, :], cosw, uni)
    w /= np.linalg.norm(w, axis=0)
    pdf = 0.5 * np.maximum((nrm * w).sum(0), 0) / np.pi + 0.5 / (4 * np.pi)
    return w, pdf


def radiance_field(x, w):
    """Two normalised Phong lobes; the first rotates with position."""
    m1 = np.stack([np.cos(np.pi * x[0]), np.sin(np.pi * x[1]), 0.5 + 0.5 * x[2]])
    m1 /= np.linalg.norm(m1, axis=0)
    m2 = np.array([[0.3], [-0.5], [0.81]]); m2 /= np.linalg.norm(m2)
    c1 = np.maximum((m1 * w).sum(0), 0.0)
    c2 = np.maximum((m2 * w).sum(0), 0.0)
    return 0.7 * 51 / (2 * np.pi) * c1 ** 50 + 0.3 * 6 / (2 * np.pi) * c2 ** 5


def training_batch(n, seed=SEED, product=False, rgb=False, nan_rate=0.0):
    """SoA training records: dict(x [3,n] f32, wi [3,n], target [C,n], pdf [n],
    wo, nrm [3,n], rough [n]) -- float32 except x kept float32 too."""
    rng = np.random.default_rng(seed)
    x, nrm = scene_points(rng, n)
    wi, pdf = bsdf_standin_directions(rng, nrm)
    d = radiance_field(x.astype(np.float64), wi)
    xi = (rng.uniform(size=n) < 0.5) * rng.lognormal(-1.5 ** 2 / 2, 1.5, n)
    tgt = d * xi
    wo = _unit(rng, n)
    wo = np.where((wo * nrm).sum(0)[None, :] < 0, -wo, wo)
    rough = rng.uniform(0.05, 1.0, n)
    if product:
        cos_i = np.maximum((nrm * wi).sum(0), 0.0)
        refl = 2 * (wo * nrm).sum(0)[None, :] * nrm - wo
        lobe = np.maximum((refl * wi).sum(0), 0.0) ** (2.0 / rough ** 2) * (1.0 / rough ** 2) + 0.2
        tgt = tgt * cos_i * lobe
    if rgb:
        tint = rng.uniform(0.5, 1.5, (3, n))
        target = (tgt[None, :] * tint)
    else:
        target = tgt[None, :]
    if nan_rate > 0:
        k = max(1, int(round(nan_rate * n)))
        bad = rng.choice(n, k, replace=False)
        target[0, bad[: k // 2 + 1]] = np.nan
        pdf = pdf.copy()
        pdf[bad[k // 2 + 1:]] = np.inf if k > 1 else pdf[bad[k // 2 + 1:]]
    return dict(x=x, wi=wi.astype(np.float32), target=target.astype(np.float32),
                pdf=pdf.astype(np.float32), wo=wo.astype(np.float32), nrm=nrm.astype(np.float32),
                rough=rough.astype(np.float32))


def query_batch(n, seed=SEED + 1, product=False):
    """SoA guided queries: positions, (product) w_o, n, roughness, and a
    caller direction per query for the fused pdf (uniform sphere)."""
    rng = np.random.default_rng(seed)
    x, nrm = scene_points(rng, n)
    wq = _unit(rng, n)
    wo = _unit(rng, n)
    wo = np.where((wo * nrm).sum(0)[None, :] < 0, -wo, wo)
    return dict(x=x, wq=wq.astype(np.float32), wo=wo.astype(np.float32), nrm=nrm.astype(np.float32),
                rough=rng.uniform(0.05, 1.0, n).astype(np.float32))


def random_params(layer_dims, n_grid, n_lobes, seed=SEED + 2, feat_sd=0.5, kappa_sd=1.5):
    """Parity parameters in the flat C-ABI layout: per layer W [out][in]
    Xavier-uniform and b [out] (the kappa' rows of the output bias ~ N(0, 1.5^2),
    others 0.1 N(0,1)), then grid features ~ N(0, 0.5^2).  float32."""
    rng = np.random.default_rng(seed)
    parts = []
    for li, (i, o) in enumerate(layer_dims):
        lim = np.sqrt(6.0 / (i + o))
        parts.append(rng.uniform(-lim, lim, o * i))
        b = rng.normal(scale=0.1, size=o)
        if li == len(layer_dims) - 1:
            b[n_lobes:2 * n_lobes] = rng.normal(scale=kappa_sd, size=n_lobes)
        parts.append(b)
    parts.append(rng.normal(scale=feat_sd, size=n_grid))
    return np.concatenate(parts).astype(np.float32)
