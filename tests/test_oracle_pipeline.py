"""End-to-end pins of the oracle pipeline (CPU only): synthetic ground truth,
GCP soundness, fixed-vs-double tolerance, determinism across thread counts.
SPEC acceptance criteria S:632-641; BASELINE.json north_star tolerances.
"""
import numpy as np
import pytest

import oracle
from paper_2212_00488_b200 import synth


@pytest.mark.parametrize("s", [2, 4, 5, 6])
def test_shift_pair_recovery_k1(s):
    # S:637 (acceptance 4): >= 95% of interior pixels exactly s without scaling;
    # S:638 (acceptance 5): every GCP equals s, GCP fraction >= 80%
    W, H, D = 64, 48, 16
    L, R = synth.shift_pair(W, H, s, seed=s)
    p = oracle.params(k_scale=1)
    r = oracle.pipeline(L, R, D, p, "fixed", stages=("DL", "masked", "out"))
    lo, hi = s + p.w_x, W - s - p.w_x
    assert (r["DL"][:, s + p.w_x:] == s).mean() >= 0.95
    m = r["masked"][:, lo:hi]
    assert (m[m != 255] == s).all()
    assert (m != 255).mean() >= 0.80
    assert (np.abs(r["out"][:, s + p.w_x:] - s) == 0).mean() >= 0.95


@pytest.mark.parametrize("s", [4, 6])
def test_shift_pair_recovery_k2(s):
    # with K=2 and even s, >= 90% of interior within 1.0 after scale-up
    W, H, D = 160, 96, 32
    L, R = synth.shift_pair(W, H, s, seed=10 + s)
    r = oracle.pipeline(L, R, D, oracle.params(), "fixed", stages=("out",))
    b = s + 2 * 21 + 4
    assert (np.abs(r["out"][4:-4, b:W - b] - s) <= 1.0).mean() >= 0.90


def test_identical_images_all_gcp():
    # identical pair -> disparity 0 everywhere, 100% GCP
    L, _ = synth.shift_pair(48, 32, 0, seed=3)
    r = oracle.pipeline(L, L, 8, oracle.params(k_scale=1), "fixed", stages=("DL", "masked"))
    assert (r["DL"] == 0).all() and (r["masked"] == 0).all()


def test_fixed_vs_double_tolerance():
    # north_star: aggregated costs within 1e-5 relative; <= 0.01% of D^L/D^R
    # pixels differ and only at (near-)ties within the quantisation bound.
    L, R, _ = synth.scene(96, 72, 24, seed=4)
    p = oracle.params(k_scale=1)
    f = oracle.fixed_bits(p.w_x)
    rf = oracle.pipeline(L, R, 24, p, "fixed", stages=("caL", "caR", "DL", "DR"))
    rd = oracle.pipeline(L, R, 24, p, "double", stages=("caL_d", "caR_d", "DL", "DR"))
    for a, b in (("caL", "caL_d"), ("caR", "caR_d")):
        q = rf[a].astype(np.float64) / 2.0 ** f
        d = rd[b]
        rel = np.abs(q - d) / np.maximum(np.abs(d), 1e-300)
        rel[d == 0] = np.abs(q - d)[d == 0]
        assert rel.max() <= 1e-5
        # closed-form bound: 0.5 * 2^-f / c_AD(1) per term
        assert rel.max() <= 0.5 * 2.0 ** -f / oracle.cost_ad(1) + 1e-15
    for m in ("DL", "DR"):
        diff = rf[m] != rd[m]
        assert diff.mean() <= 1e-4
        vol = rd["caL_d" if m == "DL" else "caR_d"]
        for y, x in zip(*np.nonzero(diff)):
            a, b = vol[rf[m][y, x], y, x], vol[rd[m][y, x], y, x]
            assert abs(a - b) <= 1e-5 * abs(b)


def test_threads_determinism():
    # S:636 (acceptance 3): bit-identical for worker counts {1, 2, 8}
    L, R, _ = synth.scene(120, 80, 32, seed=5)
    p = oracle.params()
    outs = [oracle.pipeline(L, R, 32, p, "fixed", nthreads=t, stages=("out", "DL", "DR"))
            for t in (1, 2, 8)]
    for o in outs[1:]:
        for k in o:
            assert np.array_equal(o[k], outs[0][k])


def test_invalid_params_rejected():
    L = np.zeros((8, 8), np.uint8)
    for kw in (dict(lambda_ad=0.0), dict(lambda_mc=-1.0), dict(delta=0), dict(t_fill=-1),
               dict(w_x=-1), dict(k_scale=3)):
        with pytest.raises(ValueError):
            oracle.pipeline(L, L, 4, oracle.params(**kw))
