"""Pins for oracle/philox.py and oracle/grid.py (Eq. 13)."""
import os
import numpy as np
import pytest

from oracle import philox, grid

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def load_kat():
    rows = []
    with open(os.path.join(GOLDEN, "philox4x32_10_kat.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            v = [int(t, 16) for t in line.split()]
            rows.append((v[0:4], v[4:6], v[6:10]))
    return rows


def test_philox_known_answer_vectors():
    # Random123 published KAT (tests/golden/philox4x32_10_kat.txt)
    for ctr, key, out in load_kat():
        got = philox.philox4x32_10(ctr, key)
        assert [int(g) for g in got] == out


def test_uniforms_range_and_resolution():
    u = philox.sample_uniforms(10000, seed=0x1234_5678_9ABC, offset=77)
    assert u.shape == (3, 10000)
    assert (u >= 0).all() and (u < 1).all()
    # 24-bit grid
    assert np.all(u * 2 ** 24 == np.floor(u * 2 ** 24))
    # means ~ 1/2 (10000 samples, sd ~ 0.0029)
    assert np.allclose(u.mean(axis=1), 0.5, atol=0.015)
    # counter offset shifts the stream
    u2 = philox.sample_uniforms(10, seed=0x1234_5678_9ABC, offset=78)
    assert np.array_equal(u2[:, :9], u[:, 1:10])


def test_level_schedule_paper_endpoints():
    # D_1 = 8, D_8 = 86; C-A3 ceil reading
    r = grid.level_resolutions(8, 86, 8)
    assert r[0] == 8 and r[-1] == 86
    assert all(a < b for a, b in zip(r, r[1:]))
    assert r == [8, 12, 16, 23, 32, 44, 62, 86]
    # exact geometric case (b = 2): closed form
    assert grid.level_resolutions(2, 16, 4) == [2, 4, 8, 16]
    # c5 endpoints
    r5 = grid.level_resolutions(16, 2048, 16)
    assert r5[0] == 16 and r5[-1] == 2048 and all(a < b for a, b in zip(r5, r5[1:]))


def test_table_sizes_and_param_count():
    res = [8, 12, 16, 23, 32, 44, 62, 86]
    sizes = grid.level_table_sizes(res, 18)
    assert sizes[:7] == [d ** 3 for d in res[:7]] and sizes[7] == 2 ** 18
    assert sum(sizes) * 4 == 2547708            # 2,547,708 grid params
    assert grid.level_table_sizes(res, 0) == [d ** 3 for d in res]


def test_normalize_position_invariants():
    lo, hi = (-1.0, -2.0, 0.5), (1.0, 2.0, 4.5)
    x = np.array([[-1.0, 0.0, 5.0, -7.0], [-2.0, 0.0, 9.0, -3.0], [0.5, 2.5, 4.5, 0.0]], np.float32)
    u = grid.normalize_position(x, lo, hi)
    assert np.all(u[:, 0] == 0)                       # x = aabb.min -> 0
    assert np.allclose(u[:, 1], 0.5, atol=1e-7)      # centre -> 1/2
    assert np.all(u[:, 2] == np.float32(1 - 1e-6))   # beyond max -> clamp
    assert np.all(u[:, 3] == 0)                       # below min -> clamp


def test_lattice_points_exact_index():
    # AABB [0,1], D - 1 = 8: u = k/8 is exact in fp32, so s = k, i = k, f = 0.
    d = 9
    k = np.arange(8)
    x = np.stack([k / 8.0, (7 - k) / 8.0, np.full(8, 3 / 8.0)]).astype(np.float32)
    u = grid.normalize_position(x, (0, 0, 0), (1, 1, 1))
    i, f = grid.cell_coords(u, d)
    assert np.array_equal(i[0], k) and np.array_equal(i[1], 7 - k) and np.all(i[2] == 3)
    assert np.all(f == 0)
    idx, w = grid.level_corners(u, d, d ** 3, False)
    assert np.array_equal(idx[0], k + d * ((7 - k) + d * 3))   # dense index P_x + D(P_y + D P_z)
    assert np.all(w[0] == 1) and np.all(w[1:] == 0)


def _encode_level(tables_fn, d, x, lo=(0, 0, 0), hi=(1, 1, 1)):
    p = np.stack(np.meshgrid(np.arange(d), np.arange(d), np.arange(d), indexing='ij'), -1)
    # dense entry order: index = P_x + D (P_y + D P_z)
    tab = np.zeros((d ** 3, 2))
    px, py, pz = p[..., 0].ravel(), p[..., 1].ravel(), p[..., 2].ravel()
    tab[px + d * (py + d * pz)] = tables_fn(px, py, pz)
    return grid.encode(x, lo, hi, [d], [d ** 3], 0, [tab])


def test_trilinear_reproduces_affine_and_multilinear_fields():
    # Trilinear interpolation is exact for functions that are affine in each
    # lattice coordinate separately (closed form; catches swapped axes, wrong
    # corner weights and wrong dense index).
    rng = np.random.default_rng(1)
    d = 7
    x = rng.uniform(0, 1, (3, 500)).astype(np.float32)
    u = grid.normalize_position(x, (0, 0, 0), (1, 1, 1))
    s = (u * np.float32(d - 1)).astype(np.float32).astype(np.float64)
    f_aff = lambda a, b, c: np.stack([0.3 * a - 1.7 * b + 2.9 * c + 0.25, 1.1 * a * b * c - 0.5 * a * c], -1)
    g = _encode_level(f_aff, d, x)
    exp0 = 0.3 * s[0] - 1.7 * s[1] + 2.9 * s[2] + 0.25
    exp1 = 1.1 * s[0] * s[1] * s[2] - 0.5 * s[0] * s[2]
    assert np.allclose(g[0], exp0, atol=1e-12)
    assert np.allclose(g[1], exp1, atol=1e-12)


def test_cell_centre_is_mean_of_corners():
    d = 5
    rng = np.random.default_rng(2)
    tab = rng.normal(size=(d ** 3, 4))
    # cell (1,2,3) centre: u = (i + 1/2)/(D - 1) = (1.5, 2.5, 3.5)/4 (exact in fp32)
    x = np.array([[1.5 / 4], [2.5 / 4], [3.5 / 4]], np.float32)
    g = grid.encode(x, (0, 0, 0), (1, 1, 1), [d], [d ** 3], 0, [tab])
    corners = [(1 + cx) + d * ((2 + cy) + d * (3 + cz)) for cz in (0, 1) for cy in (0, 1) for cx in (0, 1)]
    assert np.allclose(g[:, 0], tab[corners].mean(axis=0), atol=1e-14)


def test_continuity_across_cell_boundaries():
    d = 6
    rng = np.random.default_rng(3)
    tab = rng.normal(size=(d ** 3, 4))
    t = np.linspace(0.05, 0.95, 4001)
    x = np.stack([t, 0.31 + 0.2 * t, 0.77 - 0.5 * t]).astype(np.float32)
    g = grid.encode(x, (0, 0, 0), (1, 1, 1), [d], [d ** 3], 0, [tab])
    step = np.abs(np.diff(g, axis=1)).max()
    assert step < 0.05            # Lipschitz: |dG| <= C |dx|, no jumps


def test_scatter_is_adjoint_of_encode():
    # encode is linear in the tables: <scatter(dz), T> = sum_n dz_n . G_T(x_n).
    rng = np.random.default_rng(4)
    res, log2 = [3, 5, 9], 6             # last level hashed (729 > 64)
    sizes = grid.level_table_sizes(res, log2)
    x = rng.uniform(-1, 1, (3, 300)).astype(np.float32)
    tabs = [rng.normal(size=(s, 4)) for s in sizes]
    dz = rng.normal(size=(12, 300))
    g = grid.encode(x, (-1, -1, -1), (1, 1, 1), res, sizes, log2, tabs)
    sc = grid.scatter_grad(x, (-1, -1, -1), (1, 1, 1), res, sizes, dz, 4)
    lhs = sum((a * b).sum() for a, b in zip(sc, tabs))
    assert np.isclose(lhs, (dz * g).sum(), rtol=1e-12)
    # weights sum to 1 per level: total scattered mass = total dz per level
    for l in range(3):
        assert np.allclose(sc[l].sum(axis=0), dz[4 * l:4 * l + 4].sum(axis=1), rtol=1e-12)


def test_scatter_touches_only_the_8L_corners():
    rng = np.random.default_rng(5)
    res = [4, 8]
    sizes = grid.level_table_sizes(res, 0)
    x = rng.uniform(-1, 1, (3, 1)).astype(np.float32)
    sc = grid.scatter_grad(x, (-1, -1, -1), (1, 1, 1), res, sizes, np.ones((8, 1)), 4)
    for l, d in enumerate(res):
        assert (np.abs(sc[l]).sum(axis=1) > 0).sum() <= 8


def test_hash_range_and_convention():
    # PARITY UNPINNED vs the paper (C-A4: hash not in PAPER.md); only range +
    # the declared convention's first prime (x * 1) are checked here.
    p = (np.array([0, 1, 0, 0, 123]), np.array([0, 0, 1, 0, 45]), np.array([0, 0, 0, 1, 6789]))
    h = grid.corner_index(p, 86, 1 << 18, True)
    assert np.all((h >= 0) & (h < (1 << 18)))
    assert h[0] == 0 and h[1] == 1


def _hash_golden():
    rows = []
    with open(os.path.join(os.path.dirname(__file__), "golden", "spatial_hash.txt")) as f:
        for line in f:
            if line.strip() and not line.startswith("#"):
                px, py, pz, lt, hy, hz, h, idx = line.split()
                rows.append((int(px), int(py), int(pz), int(lt), int(hy, 16), int(hz, 16), int(h, 16), int(idx)))
    return rows


def test_hash_hand_computed_golden():
    # tests/golden/spatial_hash.txt: the C-A4 hash worked out by hand (products
    # mod 2^32 in hex); pins corner_index against a swapped prime, '+' for XOR,
    # or a missing 32-bit wrap
    rows = _hash_golden()
    assert len(rows) >= 10
    for px, py, pz, lt, hy, hz, h, idx in rows:
        got = grid.corner_index((np.array([px]), np.array([py]), np.array([pz])), 0, 1 << lt, True)
        assert int(got[0]) == idx, (px, py, pz, lt)
        assert (px ^ hy ^ hz) == h and h & ((1 << lt) - 1) == idx   # the file is self-consistent


def test_level_corners_hashed_matches_golden_corner():
    # a position whose cell's (1,1,1) corner is lattice point (1,1,1) on a hashed
    # level with D = 86: corner 7 must be the golden index 77349
    d, t = 86, 1 << 18
    u = np.full((3, 1), np.float32(0.5 / 85), np.float32)   # s = 0.5 -> cell (0,0,0)
    idx, _ = grid.level_corners(u, d, t, True)
    assert int(idx[7, 0]) == 77349 and int(idx[0, 0]) == 0 and int(idx[1, 0]) == 1


def test_non_finite_positions_reading():
    # C-A32: the AABB clamp uses IEEE-754 maxNum / minNum (fmax / fmin): a NaN
    # coordinate is replaced by the clamp bound it meets first (the lower face),
    # +inf clamps to the upper face and -inf to the lower one
    x = np.array([[np.nan, np.inf, -np.inf, 0.0],
                  [0.0, np.nan, 0.0, np.inf],
                  [0.0, 0.0, np.nan, -np.inf]], np.float32)
    u = grid.normalize_position(x, (-1, -1, -1), (1, 1, 1))
    assert np.all(np.isfinite(u))
    assert u[0, 0] == 0 and u[1, 1] == 0 and u[2, 2] == 0
    assert u[0, 1] == grid.U_MAX and u[0, 2] == 0 and u[1, 3] == grid.U_MAX and u[2, 3] == 0
    assert u[1, 0] == np.float32(0.5)
