"""Pins of the CPU oracle against the paper, the SPEC's worked examples,
closed forms and invariants (CPU only).

Each test names the passage it pins (P:n = PAPER.md, S:n = SPEC.md).  Expected
values come from tests/golden/spec_examples.json (cited there) or from
mathematics (closed forms, invariants) — never from the oracle itself.
"""
import numpy as np
import pytest

import oracle
from paper_2212_00488_b200 import synth


# ------------------------------------------------------------------ core
def test_paper_parameters_are_defaults(golden):
    g = golden["paper_parameters"]
    p = oracle.params()
    assert (p.lambda_ad, p.lambda_mc, p.t_fill) == (g["lambda_ad"], g["lambda_mc"], g["t_fill"])
    assert (p.w_x, p.w_y, p.k_scale, p.m_pool) == (g["w_x"], g["w_y"], g["k_scale"], g["m_pool"])


def test_scaled_max_disparity(golden):
    for D, K, exp in golden["scaled_max_disparity"]["cases"]:
        assert oracle.scaled_max_disparity(D, K) == exp
    for D in range(1, 400):  # D_s * K >= D, and minimal
        for K in (1, 2):
            Ds = oracle.scaled_max_disparity(D, K)
            assert Ds * K >= D and (Ds - 1) * K < D


def test_fixed_bits_rule():
    # R12c: largest f <= 25 with (2 w_x + 1) 2^(f+1) < 2^32
    assert oracle.fixed_bits(21) == 25
    for w in range(0, 255):
        f = oracle.fixed_bits(w)
        assert (2 * w + 1) * 2 ** (f + 1) < 2 ** 32
        assert f == 25 or (2 * w + 1) * 2 ** (f + 2) >= 2 ** 32
        assert f >= 22  # keeps the 1e-5 relative bound (north_star)


# ------------------------------------------------------------------ SD (Eq. 2)
def test_downscale_worked_example(golden):
    g = golden["downscale_4x4"]
    out = oracle.downscale(np.array(g["input"], np.uint8), g["K"], g["m"])
    assert out.tolist() == g["expected"]


def test_downscale_constant_and_shape():
    img = np.full((992, 1436), 100, np.uint8)
    out = oracle.downscale(img, 2, 1)
    assert out.shape == (496, 718) and (out == 100).all()
    odd = np.full((7, 9), 37, np.uint8)
    assert oracle.downscale(odd, 2, 1).shape == (3, 4)  # S:142 floor


def test_downscale_k1_identity():
    rng = np.random.default_rng(0)
    img = rng.integers(0, 256, (13, 17)).astype(np.uint8)
    assert (oracle.downscale(img, 1, 1) == img).all()


def test_downscale_range_and_mean_bounds():
    rng = np.random.default_rng(1)
    img = rng.integers(0, 256, (40, 50)).astype(np.uint8)
    out = oracle.downscale(img, 2, 1).astype(int)
    # interior: mean of the 3x3 block rounded half-up, so |out*9 - sum| <= 4.5
    for y in range(1, 20):
        for x in range(1, 25):
            s = int(img[2 * y - 1:2 * y + 2, 2 * x - 1:2 * x + 2].astype(int).sum())
            assert abs(out[y, x] * 9 - s) <= 4.5 and out[y, x] * 9 - s > -4.5 - 1e-9
            assert s - out[y, x] * 9 <= 4  # half-up: x.5 never happens for /9


# ------------------------------------------------------------------ census (Fig. 3)
def test_census_examples(golden):
    g = golden["census"]
    assert (oracle.census(np.full((5, 5), 77, np.uint8)) == g["constant_code"]).all()
    img = np.full((5, 5), 100, np.uint8)
    img[2, 2] = 200
    assert oracle.census(img)[2, 2] == g["center200_neighbors100_code"]
    yy, xx = np.mgrid[0:5, 0:5]
    assert oracle.census((10 * xx + yy).astype(np.uint8))[2, 2] == g["ramp_10x_plus_y_at_2_2_code"]


def test_census_codes_are_6bit_and_pattern_order():
    rng = np.random.default_rng(2)
    img = rng.integers(0, 256, (9, 11)).astype(np.uint8)
    c = oracle.census(img)
    assert c.max() < 64
    # bit i follows offset i: a pattern permutation permutes the bits
    pat = oracle.DEFAULT_CENSUS
    perm = [5, 0, 4, 1, 3, 2]
    c2 = oracle.census(img, [pat[i] for i in perm])
    for y in range(9):
        for x in range(11):
            bits = [(int(c[y, x]) >> i) & 1 for i in range(6)]
            assert int(c2[y, x]) == sum(bits[perm[k]] << k for k in range(6))


def test_hamming(golden):
    for a, b, h in golden["hamming6"]["cases"]:
        assert oracle.hamming6(a, b) == h


# ------------------------------------------------------------------ cost (Eqs. 3-6)
def test_cost_closed_forms(golden):
    g = golden["cost_closed_forms"]
    for a, v in g["cost_ad"]:
        assert abs(oracle.cost_ad(a) - v) < g["tol"]
    for h, v in g["cost_mc"]:
        assert abs(oracle.cost_mc(h) - v) < g["tol"]


def test_cost_monotone_bounded():
    ad = [oracle.cost_ad(a) for a in range(256)]
    mc = [oracle.cost_mc(h) for h in range(7)]
    assert ad[0] == 0.0 and mc[0] == 0.0
    assert all(b > a for a, b in zip(ad, ad[1:])) and all(b > a for a, b in zip(mc, mc[1:]))
    assert max(ad) < 1 and max(mc) < 1


def test_fixed_tables_quantise_once():
    f = 25
    qad, qmc = oracle.fixed_tables(0.3, 2.3, f)
    for a in range(256):
        exact = oracle.cost_ad(a) * 2 ** f
        assert abs(int(qad[a]) - exact) <= 0.5
    for h in range(7):
        assert abs(int(qmc[h]) - oracle.cost_mc(h) * 2 ** f) <= 0.5
    assert qad[0] == 0 and qmc[0] == 0
    assert int(qad[255]) + int(qmc[6]) < 2 ** (f + 1)  # BORDER is the supremum


def _tiny(seed, W=12, H=9):
    rng = np.random.default_rng(seed)
    L = rng.integers(0, 256, (H, W)).astype(np.uint8)
    R = rng.integers(0, 256, (H, W)).astype(np.uint8)
    return L, R, oracle.census(L), oracle.census(R)


def test_cost_slice_border_and_identity():
    L, R, cL, cR = _tiny(3)
    c0 = oracle.cost_slice(L, L, cL, cL, 0)           # S:215 identical images, d=0
    assert (c0 == 0).all()
    c3 = oracle.cost_slice(L, R, cL, cR, 3)
    assert (c3[:, :3] == 2.0).all()                   # S:216 x<d band = BORDER
    assert ((c3 >= 0) & (c3 <= 2.0)).all()


@pytest.mark.parametrize("mode", ["double", "fixed"])
def test_eq6_right_base_reuse(mode):
    # Eq. 6, acceptance 2: C^R(x,y,d) = C^L(x+d,y,d)
    f = 25
    tables = oracle.fixed_tables(0.3, 2.3, f)
    for seed in range(20):
        L, R, cL, cR = _tiny(100 + seed, 14, 6)
        for d in range(0, 8):
            kw = dict(mode=mode, tables=tables, border=2 ** (f + 1))
            cl = oracle.cost_slice(L, R, cL, cR, d, "left", **kw)
            cr = oracle.cost_slice(L, R, cL, cR, d, "right", **kw)
            W = L.shape[1]
            assert np.array_equal(cr[:, :W - d], cl[:, d:])
            assert (cr[:, W - d:] == (2.0 if mode == "double" else 2 ** (f + 1))).all()


# ------------------------------------------------------------------ arms
def test_arms_examples(golden):
    g = golden["arms"]
    row = np.full((1, 60), 90, np.uint8)
    m, n = oracle.arms_x(row, g["delta"], 21)
    assert m[0, 30] == n[0, 30] == g["constant_row_cap_x"]
    col = np.full((80, 1), 90, np.uint8)
    M, N = oracle.arms_y(col, g["delta"], 31)
    assert M[40, 0] == N[40, 0] == g["constant_col_cap_y"]
    m, n = oracle.arms_x(np.array([g["step_row"]], np.uint8), g["delta"], 21)
    assert n[0, 2] == g["step_row_plus_at_index2"]
    m, n = oracle.arms_x(np.array([g["fig4_row"]], np.uint8), g["delta"], 21)
    c = g["fig4_center"]
    assert [m[0, c], n[0, c]] == g["fig4_m_n"]
    M, N = oracle.arms_y(np.array(g["fig4_col"], np.uint8)[:, None], g["delta"], 31)
    c = g["fig4_col_center"]
    assert [M[c, 0], N[c, 0]] == g["fig4_M_N"]


def test_arms_invariants_and_transpose():
    rng = np.random.default_rng(5)
    img = (rng.integers(0, 6, (16, 16)) * 9).astype(np.uint8)
    m, n = oracle.arms_x(img, 20, 7)
    H, W = img.shape
    for y in range(H):
        for x in range(W):
            assert 0 <= m[y, x] <= min(7, x) and 0 <= n[y, x] <= min(7, W - 1 - x)
            for k in range(1, n[y, x] + 1):
                assert abs(int(img[y, x + k]) - int(img[y, x])) < 20
            if n[y, x] < min(7, W - 1 - x):                                            # maximal
                assert abs(int(img[y, x + n[y, x] + 1]) - int(img[y, x])) >= 20
    M, N = oracle.arms_y(img, 20, 7)
    mt, nt = oracle.arms_x(np.ascontiguousarray(img.T), 20, 7)
    assert np.array_equal(M, mt.T) and np.array_equal(N, nt.T)


# ------------------------------------------------------------------ aggregation (Eqs. 7-8)
def test_aggregate_closed_forms():
    rng = np.random.default_rng(6)
    H, W = 10, 12
    m = rng.integers(0, 4, (H, W)).astype(np.uint8)
    n = rng.integers(0, 4, (H, W)).astype(np.uint8)
    for y in range(H):
        m[y] = np.minimum(m[y], np.arange(W))
        n[y] = np.minimum(n[y], W - 1 - np.arange(W))
    c = np.full((H, W), 0.25)
    z = np.zeros((H, W), np.uint8)
    Cs = rng.random((H, W))
    assert np.array_equal(oracle.aggregate_x(Cs, z, z), Cs)
    assert np.allclose(oracle.aggregate_x(c, m, n), 0.25 * (m.astype(int) + n + 1))
    Mv = np.minimum(rng.integers(0, 3, (H, W)), np.arange(H)[:, None]).astype(np.uint8)
    Nv = np.minimum(rng.integers(0, 3, (H, W)), H - 1 - np.arange(H)[:, None]).astype(np.uint8)
    assert np.array_equal(oracle.aggregate_y(Cs, z, z), Cs)
    assert np.allclose(oracle.aggregate_y(c, Mv, Nv), 0.25 * (Mv.astype(int) + Nv + 1))
    # linearity
    C2 = rng.random((H, W))
    a, b = 0.7, 1.9
    lhs = oracle.aggregate_x(a * Cs + b * C2, m, n)
    assert np.allclose(lhs, a * oracle.aggregate_x(Cs, m, n) + b * oracle.aggregate_x(C2, m, n),
                       atol=1e-9)
    # the u64 (fixed) path agrees exactly with integer direct sums
    Ci = rng.integers(0, 2 ** 26, (H, W)).astype(np.uint64)
    ax = oracle.aggregate_x(Ci, m, n)
    for y in range(H):
        for x in range(W):
            assert ax[y, x] == int(Ci[y, x - m[y, x]:x + n[y, x] + 1].astype(object).sum())


# ------------------------------------------------------------------ WTA (Eq. 9)
def test_wta_examples(golden):
    g = golden["wta"]
    vol = np.array(g["costs"], np.float64).reshape(4, 1, 1)
    assert oracle.wta(vol)[0, 0] == g["expected"]
    assert oracle.wta(np.array(g["costs"], np.uint64).reshape(4, 1, 1))[0, 0] == g["expected"]
    assert (oracle.wta(np.random.default_rng(0).random((1, 3, 4))) == 0).all()  # D=1 -> 0
    rng = np.random.default_rng(7)
    vol = rng.integers(0, 5, (8, 10, 10)).astype(np.float64)
    ref = np.argmin(vol, axis=0)                       # numpy argmin: first occurrence
    assert np.array_equal(oracle.wta(vol), ref)
    assert np.array_equal(oracle.wta(vol * 3.5), ref)  # S:357 scale invariance


# ------------------------------------------------------------------ cross-check (Eq. 10)
def test_cross_check_examples():
    z = np.zeros((3, 8), np.uint8)
    assert (oracle.cross_check(z, z) == 0).all()
    DL = np.zeros((1, 10), np.uint8)
    DR = np.zeros((1, 10), np.uint8)
    DL[0, 7] = 5
    DR[0, 2] = 4
    DL[0, 2] = 5
    mm = oracle.cross_check(DL, DR)
    assert mm[0, 7] == 255                            # S:341 mismatch
    assert mm[0, 2] == 255                            # S:342 x-k out of bounds
    DR[0, 2] = 5
    assert oracle.cross_check(DL, DR)[0, 7] == 5


def test_cross_check_symmetry():
    rng = np.random.default_rng(8)
    DL = rng.integers(0, 4, (6, 20)).astype(np.uint8)
    DR = rng.integers(0, 4, (6, 20)).astype(np.uint8)
    mm = oracle.cross_check(DL, DR)
    for y, x in zip(*np.nonzero(mm != 255)):
        k = int(DL[y, x])
        assert x - k >= 0 and DR[y, x - k] == k and DL[y, (x - k) + DR[y, x - k]] == k


# ------------------------------------------------------------------ median / fill (Step7)
def test_median_examples(golden):
    g = golden["median"]
    f = np.full((7, 7), g["field_value"], np.uint8)
    assert np.array_equal(oracle.median3x3(f), f)
    f[3, 3] = g["impulse_value"]
    assert oracle.median3x3(f)[3, 3] == g["field_value"]
    inv = np.full((4, 5), 255, np.uint8)
    assert (oracle.median3x3(inv) == 255).all()
    # lower middle of an even count: valid values {2, 9} -> 2
    mm = np.full((3, 3), 255, np.uint8)
    mm[1, 1], mm[0, 0] = 9, 2
    assert oracle.median3x3(mm)[1, 1] == 2


def test_fill_examples(golden):
    g = golden["fill"]
    e = g["interp"]
    row = np.full((1, 5), 255, np.uint8)
    row[0, 0], row[0, 4] = e["Dl"], e["Dr"]
    L = np.zeros((1, 5), np.uint8)
    assert oracle.fill_bilateral(row, L, e["T"])[0, 2] == e["expected"]
    e = g["edge"]
    row = np.array([[e["Dl"], 255, e["Dr"]]], np.uint8)
    Lb = np.array([[50, 52, 90]], np.uint8)          # L(x-1) closer to L(x)
    assert oracle.fill_bilateral(row, Lb, e["T"])[0, 1] == e["expected"]
    Lb2 = np.array([[90, 52, 50]], np.uint8)
    assert oracle.fill_bilateral(row, Lb2, e["T"])[0, 1] == e["Dr"]
    e = g["one_sided"]
    row = np.array([[255, 255, 255, e["Dr"], 255]], np.uint8)
    out = oracle.fill_bilateral(row, np.zeros((1, 5), np.uint8), 3)
    assert out[0, 0] == e["expected"] and out[0, 4] == e["expected"]


def test_fill_invariants():
    # GCPs unchanged, rows dense, interpolations inside the flanks
    rng = np.random.default_rng(9)
    for t in range(50):
        W = int(rng.integers(2, 30))
        row = rng.integers(0, 40, (1, W)).astype(np.uint8)
        row[0, rng.random(W) < 0.5] = 255
        L = rng.integers(0, 256, (1, W)).astype(np.uint8)
        out = oracle.fill_bilateral(row, L, 3)
        v = row[0] != 255
        assert np.array_equal(out[0, v], row[0, v].astype(np.float32))
        assert np.isfinite(out).all()
        cols = np.nonzero(v)[0]
        for x in range(W):
            if v[x] or not len(cols):
                continue
            lft, rgt = cols[cols < x], cols[cols > x]
            if len(lft) and len(rgt):
                a, b = int(row[0, lft[-1]]), int(row[0, rgt[0]])
                assert min(a, b) <= out[0, x] <= max(a, b)


def test_fill_all_invalid_rows():
    med = np.full((4, 5), 255, np.uint8)
    med[1, 3] = 7
    med[1, 1] = 4
    out = oracle.fill_bilateral(med, np.zeros((4, 5), np.uint8), 3)
    assert (out[0] == 4).all()     # nothing above -> first valid of the nearest row below
    assert (out[2] == 7).all() and (out[3] == 7).all()  # last valid preceding in raster order
    assert (oracle.fill_bilateral(np.full((2, 3), 255, np.uint8), np.zeros((2, 3), np.uint8), 3) == 0).all()


# ------------------------------------------------------------------ SU (Step8)
def test_scale_up_examples(golden):
    g = golden["scale_up"]
    v = np.full((6, 8), g["constant"], np.float32)
    Lorg = np.random.default_rng(0).integers(0, 256, (12, 16)).astype(np.uint8)
    assert (oracle.scale_up(v, Lorg) == g["expected"]).all()
    ramp = np.tile(np.arange(8, dtype=np.float32), (6, 1))
    out = oracle.scale_up(ramp, Lorg)
    assert np.array_equal(out[0::2, :15], np.tile(np.arange(15, dtype=np.float32), (6, 1)))
    # odd output sizes: last row / column copy their predecessors
    out = oracle.scale_up(v[:3, :4], np.zeros((7, 9), np.uint8))
    assert out.shape == (7, 9) and (out == 14).all()


def test_scale_up_sharp_edge():
    # a disparity step on a brightness edge stays sharp (|dD| > K*T)
    v = np.array([[10] * 4 + [30] * 4] * 2, np.float32)
    Lorg = np.zeros((4, 16), np.uint8)
    Lorg[:, 8:] = 200
    out = oracle.scale_up(v, Lorg)
    assert set(np.unique(out[0]).tolist()) == {20.0, 60.0}


def test_mde_formula(golden):
    g = golden["mde_per_s"]
    assert round(g["W"] * g["H"] * g["D"] * g["fps"] / 1e6) == g["expected_formula"]


def test_fill_variant_examples(golden):
    """NEXT-3 fill variants (§III.E, Fig. 6 and the printed Eq. 11)."""
    g = golden["fill_variants"]
    for key in ("eq11_literal_spec_example", "eq11_literal_thirds"):
        e = g[key]
        W = e["i"] + e["j"] + 1
        row = np.full((1, W), 255, np.uint8)
        row[0, 0], row[0, W - 1] = e["Dl"], e["Dr"]
        got = oracle.fill_bilateral(row, np.zeros((1, W), np.uint8), e["T"], "eq11_literal")[0, e["i"]]
        want = e["expected"] if "expected" in e else np.float32(e["expected_fraction"][0] / e["expected_fraction"][1])
        assert got == want
    e = g["nearest"]
    W = e["i"] + e["j"] + 1
    row = np.full((1, W), 255, np.uint8)
    row[0, 0], row[0, W - 1] = e["Dl"], e["Dr"]
    out = oracle.fill_bilateral(row, np.zeros((1, W), np.uint8), 3, "nearest")
    assert out[0, e["i"]] == e["expected"]
    assert out[0, W - 2] == e["Dr"]                     # the closer side is the right one
    row2 = np.array([[e["Dl"], 255, 255, 255, e["Dr"]]], np.uint8)
    assert oracle.fill_bilateral(row2, np.zeros((1, 5), np.uint8), 3, "nearest")[0, 2] == e["Dl"]
    e = g["smaller"]
    W = e["i"] + e["j"] + 1
    row = np.full((1, W), 255, np.uint8)
    row[0, 0], row[0, W - 1] = e["Dl"], e["Dr"]
    out = oracle.fill_bilateral(row, np.zeros((1, W), np.uint8), 100, "smaller")
    assert (out[0, 1:W - 1] == e["expected"]).all()
    # the baselines ignore T and brightness; the literal Eq. 11 keeps the edge rule
    row = np.array([[10, 255, 30]], np.uint8)
    Lb = np.array([[90, 52, 50]], np.uint8)
    assert oracle.fill_bilateral(row, Lb, 3, "eq11_literal")[0, 1] == 30.0
    assert oracle.fill_bilateral(row, Lb, 3, "nearest")[0, 1] == 10.0


def test_rgb_to_gray_examples(golden):
    for (r, g, b), want in golden["rgb_to_gray"]["examples"]:
        rgb = np.array([[[r, g, b]]], np.uint8)
        assert oracle.rgb_to_gray(rgb)[0, 0] == want


def test_right_base_arm_cap():
    """w_x_r caps only the right-base x arms; W_y stays common."""
    L = np.full((6, 40), 77, np.uint8)
    r = oracle.pipeline(L, L, 4, oracle.params(k_scale=1, w_x=5, w_x_r=2), "fixed",
                        stages=("armL", "armR"))
    assert r["armL"][0].max() == 5 and r["armL"][1].max() == 5
    assert r["armR"][0].max() == 2 and r["armR"][1].max() == 2
    assert np.array_equal(r["armL"][2:], r["armR"][2:])


def test_depth_eq1():
    """Eq. 1: Z = f B / d; d = 0 is 'at infinity'."""
    d = np.array([[2.0, 0.0, 3.0, 0.5, 144.0]], np.float32)
    Z = oracle.depth(d, 10.0)
    assert Z[0, 0] == 5.0 and np.isinf(Z[0, 1]) and Z[0, 1] > 0
    assert Z[0, 2] == np.float32(10.0) / np.float32(3.0) and Z[0, 3] == 20.0
    # smaller d -> farther
    assert Z[0, 4] < Z[0, 2] < Z[0, 0]
