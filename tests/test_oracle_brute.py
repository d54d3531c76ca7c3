"""The C oracle against an independently written pure-Python brute force
(oracle/brute.py) on tiny random instances (CPU only).

brute.py differs from the C oracle where a plausible mistake would hide:
2-D cross-region enumeration instead of separable Step3/Step5 sums, exact
Fraction arithmetic, sort-based median, tuple-min WTA, set-based fill search.
"""
import math

import numpy as np
import pytest

import oracle
from oracle import brute


def _rand_params(rng):
    pat = oracle.DEFAULT_CENSUS
    if rng.random() < 0.5:  # random distinct census pattern within the 5x5 footprint
        cand = [(dx, dy) for dx in range(-2, 3) for dy in range(-2, 3) if (dx, dy) != (0, 0)]
        idx = rng.choice(len(cand), 6, replace=False)
        pat = tuple(cand[i] for i in idx)
    return dict(delta=int(rng.choice([13, 20, int(rng.integers(1, 60))])),
                w_x=int(rng.integers(0, 6)), w_y=int(rng.integers(0, 6)),
                t_fill=int(rng.integers(0, 5)), census=pat,
                # NEXT-3 variants: right-base x cap, fill mode (§III.E)
                w_x_r=int(rng.choice([-1, int(rng.integers(0, 6))])),
                fill_mode=str(rng.choice(list(oracle.FILL_MODES))))


@pytest.mark.parametrize("seed", range(24))
def test_stages_vs_brute(seed):
    rng = np.random.default_rng(seed)
    K = int(rng.choice([1, 2]))
    W = int(rng.integers(4, 13)) * K + int(rng.integers(0, 2))
    H = int(rng.integers(4, 10)) * K + int(rng.integers(0, 2))
    D = int(rng.integers(1, 7)) * K
    kw = _rand_params(rng)
    levels = int(rng.choice([4, 16, 256]))
    Lorg = (rng.integers(0, levels, (H, W)) * (255 // (levels - 1))).astype(np.uint8)
    Rorg = (rng.integers(0, levels, (H, W)) * (255 // (levels - 1))).astype(np.uint8)
    p = oracle.params(k_scale=K, **kw)
    stages = ("Ls", "Rs", "cenL", "cenR", "armL", "armR", "caL_d", "caR_d", "DL", "DR",
              "masked", "median", "fill", "out")
    r = oracle.pipeline(Lorg, Rorg, D, p, "double", stages=stages)
    rf = oracle.pipeline(Lorg, Rorg, D, p, "fixed", stages=("caL", "DL", "DR"))

    Ls = brute.downscale(Lorg.tolist(), K, 1)
    Rs = brute.downscale(Rorg.tolist(), K, 1)
    assert r["Ls"].tolist() == Ls and r["Rs"].tolist() == Rs
    cL, cR = brute.census(Ls, kw["census"]), brute.census(Rs, kw["census"])
    assert r["cenL"].tolist() == cL and r["cenR"].tolist() == cR
    aL = brute.arms(Ls, kw["delta"], kw["w_x"], kw["w_y"])
    wxr = kw["w_x"] if kw["w_x_r"] < 0 else kw["w_x_r"]
    aR = brute.arms(Rs, kw["delta"], wxr, kw["w_y"])
    assert [a.tolist() for a in r["armL"]] == list(aL)
    assert [a.tolist() for a in r["armR"]] == list(aR)

    Ds = math.ceil(D / K)
    volL, volR = [], []
    for d in range(Ds):
        for base, arms_, vol, key in (("left", aL, volL, "caL_d"), ("right", aR, volR, "caR_d")):
            Cs = brute.costs_double(Ls, Rs, cL, cR, d, 0.3, 2.3, base)
            ca = brute.aggregate_cross(Cs, *arms_)
            vol.append(ca)
            got = r[key][d]
            exact = np.array([[float(v) for v in row] for row in ca])
            assert np.allclose(got, exact, rtol=1e-12, atol=1e-12)
    # WTA on exact rationals vs the double-mode oracle: they agree unless two
    # candidates are within rounding of each other (none expected here)
    DLb, DRb = brute.wta(volL), brute.wta(volR)
    assert r["DL"].tolist() == DLb and r["DR"].tolist() == DRb
    # fixed mode reaches the same maps at this size (no near-ties)
    assert np.array_equal(rf["DL"], r["DL"]) and np.array_equal(rf["DR"], r["DR"])

    mm = brute.cross_check(DLb, DRb)
    assert r["masked"].tolist() == mm
    med = brute.median3x3(mm)
    assert r["median"].tolist() == med
    fl = brute.fill(med, Ls, kw["t_fill"], kw["fill_mode"])
    assert np.array_equal(r["fill"], np.array(fl, np.float32))
    out = brute.scale_up(fl, Lorg.tolist(), K, kw["t_fill"])
    assert np.array_equal(r["out"], np.array(out, np.float32))


@pytest.mark.parametrize("seed", range(6))
def test_fixed_mode_equals_quantised_sums(seed):
    """Fixed mode: CA equals the exact integer sum of the once-quantised terms
    over the cross region (enumerated by brute force)."""
    rng = np.random.default_rng(50 + seed)
    W, H, D = 11, 8, 5
    L = rng.integers(0, 256, (H, W)).astype(np.uint8)
    R = rng.integers(0, 256, (H, W)).astype(np.uint8)
    p = oracle.params(k_scale=1, w_x=3, w_y=2)
    r = oracle.pipeline(L, R, D, p, "fixed", stages=("caL", "caR", "cenL", "cenR", "armL", "armR"))
    f = oracle.fixed_bits(3)
    qad, qmc = oracle.fixed_tables(0.3, 2.3, f)
    aL = [a.tolist() for a in r["armL"]]
    aR = [a.tolist() for a in r["armR"]]
    cL, cR = r["cenL"].tolist(), r["cenR"].tolist()
    for d in range(D):
        QL = [[(int(qad[abs(int(L[y, x]) - int(R[y, x - d]))]) +
                int(qmc[bin(cL[y][x] ^ cR[y][x - d]).count("1")])) if x >= d else 2 ** (f + 1)
               for x in range(W)] for y in range(H)]
        QR = [[(int(qad[abs(int(R[y, x]) - int(L[y, x + d]))]) +
                int(qmc[bin(cR[y][x] ^ cL[y][x + d]).count("1")])) if x + d < W else 2 ** (f + 1)
               for x in range(W)] for y in range(H)]
        assert r["caL"][d].tolist() == [[int(v) for v in row] for row in brute.aggregate_cross(QL, *aL)]
        assert r["caR"][d].tolist() == [[int(v) for v in row] for row in brute.aggregate_cross(QR, *aR)]


@pytest.mark.parametrize("mode", list(oracle.FILL_MODES))
@pytest.mark.parametrize("seed", range(4))
def test_fill_modes_vs_brute(mode, seed):
    """Every §III.E filling mode on random sparse maps (many non-GCP runs,
    rows without any valid pixel)."""
    rng = np.random.default_rng(900 + seed)
    H, W = 7, 17
    med = rng.integers(0, 40, (H, W)).astype(np.uint8)
    med[rng.random((H, W)) < 0.6] = 255
    med[3] = 255
    Limg = rng.integers(0, 256, (H, W)).astype(np.uint8)
    T = int(rng.integers(0, 12))
    got = oracle.fill_bilateral(med, Limg, T, mode)
    ref = np.array(brute.fill(med.tolist(), Limg.tolist(), T, mode), np.float32)
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))


def test_rgb_to_gray_vs_brute():
    rng = np.random.default_rng(7)
    rgb = rng.integers(0, 256, (9, 13, 3)).astype(np.uint8)
    assert oracle.rgb_to_gray(rgb).tolist() == brute.rgb_to_gray(rgb.tolist())
