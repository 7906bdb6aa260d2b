"""Multi-resolution spatial embedding, Eq. 13 (§5.1).

TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py.

  G(x | Phi_E) = (+)_{l=1..L} bilinear(x, V_l[x])            (Eq. 13)

"L 3D uniform grids G_l, each covering the entire scene with a spatial
resolution of D_l^3 ... D_l grows exponentially ... assign a learnable
embedding v in R^F to each lattice point ... interpolate the features nearby
x for each resolution, and concatenate"; "V_l[x] is the set of
features at the eight corners of the cell enclosing x".

Readings (DESIGN.md / SURVEY §8(c)):
  C-A2  "bilinearly" over "eight corners" -> trilinear.
  C-A3  D_l = lattice points per axis spanning the AABB (corners on its faces);
        D_l = ceil(D_1 b^(l-1) - 1e-9), b = (D_L/D_1)^(1/(L-1)), D_L exact.
  C-A1  the cell index is an fp32 op sequence (no FMA), emulated exactly here
        with numpy float32 ops (IEEE round-to-nearest per op).
  C-A4  levels with D^3 > T use the instant-ngp spatial hash (not in the
        paper: PARITY UNPINNED against the paper, pinned to our convention).
"""
import math
import numpy as np

HASH_PRIMES = (1, 2654435761, 805459861)   # C-A4 convention (not in PAPER.md)
U_MAX = np.float32(1.0 - 1e-6)             # S:163 clamp to [0, 1 - 1e-6]


def level_resolutions(d1, dl, n_levels):
    """C-O2: D_l = ceil(D_1 * b^(l-1) - 1e-9), b = (D_L/D_1)^(1/(L-1)),
    D_L forced exactly ("grows exponentially", P:302 endpoints)."""
    if n_levels == 1:
        return [int(dl)]
    b = (dl / d1) ** (1.0 / (n_levels - 1))
    res = [int(math.ceil(d1 * b ** l - 1e-9)) for l in range(n_levels)]
    res[-1] = int(dl)
    return res


def level_table_sizes(res, log2_hashmap):
    """Entries per level: D^3 when dense (T = 0 or D^3 <= T), else T = 2^log2."""
    out = []
    for d in res:
        if log2_hashmap == 0 or d ** 3 <= (1 << log2_hashmap):
            out.append(d ** 3)
        else:
            out.append(1 << log2_hashmap)
    return out


def inv_extent(lo, hi):
    """C-O1: inv_ext_a = fl32(1 / (hi_a - lo_a)) evaluated in float64."""
    lo = np.asarray(lo, np.float32).astype(np.float64)
    hi = np.asarray(hi, np.float32).astype(np.float64)
    return (1.0 / (hi - lo)).astype(np.float32)


def normalize_position(x, lo, hi):
    """C-O1: u_a = min(max(fl32(fl32(x_a - lo_a) * inv_ext_a), 0), fl32(1-1e-6)).
    C-A32 (the paper is silent on non-finite positions): min / max are IEEE-754
    minNum / maxNum, so a NaN coordinate becomes the lower face (max(NaN, 0) =
    0) and +-inf clamp to the faces.  x: [3, n] float32.  Returns u [3, n] float32."""
    x = np.asarray(x, np.float32)
    lo32 = np.asarray(lo, np.float32).reshape(3, 1)
    inv = inv_extent(lo, hi).reshape(3, 1)
    d = (x - lo32).astype(np.float32)          # fp32 subtract
    u = (d * inv).astype(np.float32)           # fp32 multiply
    u = np.fmin(np.fmax(u, np.float32(0.0)), U_MAX)
    return u.astype(np.float32)


def cell_coords(u, d):
    """C-O3: s = fl32(u * fl32(D - 1)); i = floor(s) clamped to [0, D-2];
    f = s - i (exact in fp32).  Returns (i int64 [3,n], f float64 [3,n])."""
    s = (u * np.float32(d - 1)).astype(np.float32)
    i = np.floor(s).astype(np.int64)
    i = np.clip(i, 0, max(d - 2, 0))
    f = (s - i.astype(np.float32)).astype(np.float32)
    return i, f.astype(np.float64)


def corner_index(p, d, table_size, hashed):
    """C-O4: dense P_x + D (P_y + D P_z); hashed
    (P_x*1 ^ P_y*2654435761 ^ P_z*805459861) mod 2^32 & (T-1)."""
    px, py, pz = (np.asarray(c, np.int64) for c in p)
    if not hashed:
        return px + d * (py + d * pz)
    m = (1 << 32) - 1
    h = ((px * HASH_PRIMES[0]) & m) ^ ((py * HASH_PRIMES[1]) & m) ^ ((pz * HASH_PRIMES[2]) & m)
    return h & (table_size - 1)


def level_corners(u, d, table_size, hashed):
    """For one level: 8 corner indices [8, n] (int64) and trilinear weights
    [8, n] (float64), corner c = c_x + 2 c_y + 4 c_z, w_c = prod_a
    (c_a ? f_a : 1 - f_a)  (C-O4, Eq. 13 "eight corners")."""
    i, f = cell_coords(u, d)
    idx, w = [], []
    for c in range(8):
        cb = ((c >> 0) & 1, (c >> 1) & 1, (c >> 2) & 1)
        p = [i[a] + cb[a] for a in range(3)]
        idx.append(corner_index(p, d, table_size, hashed))
        wc = np.ones(u.shape[1])
        for a in range(3):
            wc = wc * (f[a] if cb[a] else 1.0 - f[a])
        w.append(wc)
    return np.stack(idx), np.stack(w)


def encode(x, lo, hi, res, sizes, log2_hashmap, tables):
    """Eq. 13: G(x) = concat_l sum_c w_c E_l[idx_c], coarsest level first
    (C-O5).  tables: list of [size_l, F] float64.  Returns [L*F, n]."""
    u = normalize_position(x, lo, hi)
    out = []
    for l, d in enumerate(res):
        hashed = sizes[l] != d ** 3
        idx, w = level_corners(u, d, sizes[l], hashed)
        g = np.zeros((tables[l].shape[1], u.shape[1]))
        for c in range(8):
            g += w[c][None, :] * tables[l][idx[c]].T
        out.append(g)
    return np.concatenate(out, axis=0)


def scatter_grad(x, lo, hi, res, sizes, dz, n_features):
    """Backward of Eq. 13 (C-O15): dE_l[idx_c] += w_c * dz_l; colliding hashed
    corners simply accumulate ("optimized with all (and only) its nearby
    samples").  dz: [L*F, n].  Returns list of [size_l, F]."""
    u = normalize_position(x, lo, hi)
    grads = []
    for l, d in enumerate(res):
        hashed = sizes[l] != d ** 3
        idx, w = level_corners(u, d, sizes[l], hashed)
        g = np.zeros((sizes[l], n_features))
        dzl = dz[l * n_features:(l + 1) * n_features]          # [F, n]
        for c in range(8):
            np.add.at(g, idx[c], (w[c][None, :] * dzl).T)
        grads.append(g)
    return grads
