"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle's
fixed mode, element by element, on seeded synthetic inputs.

Integer stages (scaled images, census, arms, CA_x, CA, D^L, D^R, masked,
median) must be bit-identical; the binary32 stages (fill, scale-up) must be
bit-identical too (one correctly-rounded division / exact halvings, see
DESIGN.md §2 R26, R30).  Tolerance vs the IEEE-double definition is covered
by tests/test_oracle_pipeline.py::test_fixed_vs_double_tolerance plus
test_ca_volume_tolerance_vs_double below.
"""
import numpy as np
import pytest

import oracle
from paper_2212_00488_b200 import abi, synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

DEV = "cuda:0"


def _run_gpu(L, R, D, st=None, **kw):
    H, W = L.shape
    own = st is None
    if own:
        st = abi.Stereo(W, H, D, **kw)
    Lt = torch.from_numpy(np.ascontiguousarray(L)).to(DEV)
    Rt = torch.from_numpy(np.ascontiguousarray(R)).to(DEV)
    out = torch.full((H, W), float("nan"), dtype=torch.float32, device=DEV)
    st.compute(Lt, Rt, out)
    torch.cuda.synchronize()
    res = {"out": out.cpu().numpy()}
    i = st.info
    pixL, pixR = st.download(abi.BUF_PIX_L), st.download(abi.BUF_PIX_R)
    res["Ls"], res["cenL"] = abi.unpack_pix(pixL)
    res["Rs"], res["cenR"] = abi.unpack_pix(pixR)
    res["armL"] = abi.unpack_arms(st.download(abi.BUF_ARM_L))
    res["armR"] = abi.unpack_arms(st.download(abi.BUF_ARM_R))
    for name, b in (("DL", abi.BUF_DL), ("DR", abi.BUF_DR), ("masked", abi.BUF_MASKED),
                    ("median", abi.BUF_MEDIAN)):
        res[name] = st.download(b)
    if kw.get("k_scale", 2) == 2:
        res["fill"] = st.download(abi.BUF_FILL)
    if i.Ds * i.Hs * i.cax_pitch * 4 <= 64 << 20:
        res["caxL"] = st.download(abi.BUF_CAX_L)[:, :, :i.Ws]
        res["caxR"] = st.download(abi.BUF_CAX_R)[:, :, :i.Ws]
    if own:
        st.close()
    return res


def _oracle_params(kw):
    m = dict(kw)
    census = m.pop("census", None)
    if census is not None:
        m["census"] = census
    return oracle.params(**m)


def _compare(L, R, D, kw, volumes=True):
    stages = ["Ls", "Rs", "cenL", "cenR", "armL", "armR", "DL", "DR", "masked", "median", "out"]
    if kw.get("k_scale", 2) == 2:
        stages.append("fill")
    if volumes:
        stages += ["caxL", "caxR"]
    ref = oracle.pipeline(L, R, D, _oracle_params(kw), "fixed", stages=tuple(stages))
    got = _run_gpu(L, R, D, **kw)
    for s in stages:
        if s not in got:
            continue
        a, b = got[s], ref[s]
        assert a.shape == b.shape, (s, a.shape, b.shape)
        if a.dtype == np.float32:
            same = a.view(np.uint32) == b.view(np.uint32)
        else:
            same = a == b
        if not same.all():
            idx = np.argwhere(~same)[:5]
            raise AssertionError(f"stage {s}: {int((~same).sum())} mismatches, first at {idx.tolist()}: "
                                 f"gpu={[a[tuple(i)] for i in idx]} oracle={[b[tuple(i)] for i in idx]}")
    return got, ref


# ---------------------------------------------------------------- tables
def test_tables_identical_to_oracle():
    for w_x in (0, 5, 21, 41, 141, 254):
        st = abi.Stereo(64, 48, 16, w_x=w_x, k_scale=1)
        qad, qmc, border = st.tables()
        f = oracle.fixed_bits(w_x)
        oqad, oqmc = oracle.fixed_tables(0.3, 2.3, f)
        assert st.info.frac_bits == f
        assert np.array_equal(qad, oqad) and np.array_equal(qmc, oqmc) and border == 2 ** (f + 1)
        st.close()


# ---------------------------------------------------------------- BASELINE configs
def test_c1_shift_pair_bit_exact():
    L, R = synth.shift_pair(64, 48, 5, seed=0)
    got, ref = _compare(L, R, 16, dict(k_scale=1))
    assert (got["DL"][:, 26:] == 5).all()


@pytest.mark.parametrize("seed", range(100))
def test_random_small_instances(seed):
    """SPEC acceptance 1: >=100 seeds, sizes up to 64x48, D<=16, random
    delta / W / T / census pattern; every stage bit-exact."""
    rng = np.random.default_rng(1000 + seed)
    K = int(rng.choice([1, 2]))
    W = int(rng.integers(1 * K, 65))
    H = int(rng.integers(1 * K, 49))
    W, H = max(W, K), max(H, K)
    D = int(rng.integers(1, 17))
    cand = [(dx, dy) for dx in range(-2, 3) for dy in range(-2, 3) if (dx, dy) != (0, 0)]
    pat = [cand[i] for i in rng.choice(len(cand), 6, replace=False)] if rng.random() < 0.5 \
        else list(oracle.DEFAULT_CENSUS)
    kw = dict(k_scale=K, delta=int(rng.integers(1, 60)), w_x=int(rng.integers(0, 30)),
              w_y=int(rng.integers(0, 40)), t_fill=int(rng.integers(0, 6)),
              m_pool=int(rng.integers(0, 3)), census=pat)
    if rng.random() < 0.3:  # NEXT-3 variants: right-base x cap, fill modes
        kw["w_x_r"] = int(rng.integers(0, 30))
    if rng.random() < 0.4:
        kw["fill_mode"] = int(rng.integers(0, 4))
    kind = rng.integers(0, 3)
    if kind == 0:
        L, R = synth.random_pair(W, H, seed, levels=int(rng.choice([2, 8, 256])))
    elif kind == 1:
        L, R = synth.shift_pair(W, H, int(rng.integers(0, 6)), seed)
    else:
        L, R, _ = synth.scene(W, H, max(D, 2), seed)
    _compare(L, R, D, kw)


@pytest.mark.parametrize("seed", range(16))
def test_random_medium_instances(seed):
    """Random parameters at sizes with interior tiles (the word-load strip
    paths of PREP, several x-pass lane chunks, several y-pass bands, several
    POST CTAs); every stage bit-exact."""
    rng = np.random.default_rng(5000 + seed)
    K = int(rng.choice([1, 2]))
    W = int(rng.integers(160, 420))
    H = int(rng.integers(90, 220))
    D = int(rng.integers(8, 72))
    cand = [(dx, dy) for dx in range(-2, 3) for dy in range(-2, 3) if (dx, dy) != (0, 0)]
    pat = [cand[i] for i in rng.choice(len(cand), 6, replace=False)] if rng.random() < 0.5 \
        else list(oracle.DEFAULT_CENSUS)
    kw = dict(k_scale=K, delta=int(rng.choice([int(rng.integers(1, 60)), int(rng.integers(128, 300))])),
              w_x=int(rng.integers(0, 45)), w_y=int(rng.integers(0, 45)), t_fill=int(rng.integers(0, 6)),
              m_pool=int(rng.integers(0, 3)), census=pat)
    if rng.random() < 0.3:
        kw["w_x_r"] = int(rng.integers(0, 45))
    if rng.random() < 0.4:
        kw["fill_mode"] = int(rng.integers(0, 4))
    if rng.random() < 0.5:
        L, R, _ = synth.scene(W, H, max(D * K, 2), seed)
    else:
        L, R = synth.random_pair(W, H, seed, levels=int(rng.choice([8, 256])))
    _compare(L, R, D * K, kw, volumes=False)


@pytest.mark.parametrize("W,H,D,K", [
    (33, 17, 40, 1),      # D_s > W_s: every candidate beyond the image for many x
    (737, 9, 64, 1),      # Ws > 736: next lane-chunk template, ragged tail
    (100, 130, 1, 1),     # D = 1 (single candidate)
    (1, 40, 5, 1),        # single column
    (50, 1, 8, 1),        # single row
    (131, 77, 33, 2),     # odd sizes with K = 2 (extra last column/row copies)
    (2, 2, 3, 2),         # 1x1 scaled image
    (290, 200, 100, 2),   # several xpass units, several ypass tiles, ragged strips
])
def test_edge_shapes(W, H, D, K):
    L, R, _ = synth.scene(W, H, D, seed=W + H)
    _compare(L, R, D, dict(k_scale=K))


@pytest.mark.parametrize("delta", [127, 128, 129, 200, 255, 256, 1000])
@pytest.mark.parametrize("K", [1, 2])
def test_prep_delta_extremes(delta, K):
    """PREP's byte-SIMD similarity test across its cases: delta < 128, the
    delta >= 128 template, delta = 255 and delta > 255 (every neighbour
    similar, arms = caps); noise at 256 levels and a scene."""
    L, R = synth.random_pair(97, 61, seed=delta + K, levels=256)
    _compare(L, R, 12, dict(k_scale=K, delta=delta))
    L, R, _ = synth.scene(130, 70, 20, seed=delta)
    _compare(L, R, 20, dict(k_scale=K, delta=delta, w_x=40, w_y=25))


@pytest.mark.parametrize("w_x,w_y", [(254, 112), (253, 3), (252, 0), (0, 112)])
def test_prep_arm_caps_extremes(w_x, w_y):
    """Arm caps at the top of the u8 range (the saturating tail group of the
    byte-SIMD scans beyond 252 steps) on flat rows that let the arms reach
    them; K = 1 so that 300 columns stay 300."""
    rng = np.random.default_rng(w_x + w_y)
    L = np.full((24, 300), 90, np.uint8)
    L[:, 150:] = 160                     # one step edge: arms stop there
    L[5] = rng.integers(0, 256, 300)     # a textured row
    R = np.roll(L, 3, axis=1)
    _compare(L, R, 6, dict(k_scale=1, w_x=w_x, w_y=w_y, delta=20))


@pytest.mark.parametrize("W,H,D,kw", [
    (4032, 40, 60, dict(k_scale=2)),                       # W_s = 2016: widest lane chunk (C = 63)
    (1000, 30, 510, dict(k_scale=2, w_y=20)),              # D_s = 255: the largest u8 disparity range
    (300, 260, 40, dict(k_scale=2, w_y=112, w_x=60)),      # w_y = 112: tallest y window
])
def test_maximum_sizes_bit_exact(W, H, D, kw):
    """The ABI's upper limits (W_s <= 2016, D_s <= 255, w_y <= 112) bit-exact."""
    L, R, _ = synth.scene(W, H, min(D, W // 2), seed=W + D)
    _compare(L, R, D, kw, volumes=False)


def test_c2_quarter_scene_bit_exact():
    L, R, _ = synth.scene(450, 375, 64, seed=1)
    _compare(L, R, 64, dict(k_scale=1))


def test_c3_paper_workload_bit_exact():
    """BASELINE config c3 in the launch configuration bench.py times."""
    L, R, _ = synth.scene(1436, 992, 145, seed=0)
    got, ref = _compare(L, R, 145, dict(), volumes=False)
    assert got["out"].shape == (992, 1436)


@pytest.mark.slow
def test_c5_high_res_bit_exact():
    L, R, _ = synth.scene(2872, 1984, 290, seed=0)
    _compare(L, R, 290, dict(), volumes=False)


def test_large_windows_next2():
    """NEXT-2 window sizes (W_x=41, W_y=61) at K=1."""
    L, R, _ = synth.scene(300, 200, 64, seed=5)
    _compare(L, R, 64, dict(k_scale=1, w_x=41, w_y=61))


# ---------------------------------------------------------------- CA volume
def test_ca_volume_bit_exact_and_tolerance_vs_double():
    L, R, _ = synth.scene(96, 72, 24, seed=4)
    kw = dict(k_scale=1)
    st = abi.Stereo(96, 72, 24, **kw)
    st.set_debug(abi.DEBUG_CA, True)
    _run_gpu(L, R, 24, st=st, **kw)
    caL, caR = st.download(abi.BUF_CA_L), st.download(abi.BUF_CA_R)
    f = st.info.frac_bits
    st.close()
    ref = oracle.pipeline(L, R, 24, oracle.params(k_scale=1), "fixed", stages=("caL", "caR"))
    assert np.array_equal(caL, ref["caL"]) and np.array_equal(caR, ref["caR"])
    dbl = oracle.pipeline(L, R, 24, oracle.params(k_scale=1), "double", stages=("caL_d", "caR_d"))
    for a, b in ((caL, dbl["caL_d"]), (caR, dbl["caR_d"])):
        q = a.astype(np.float64) / 2.0 ** f
        rel = np.abs(q - b) / np.maximum(b, 1e-300)
        rel[b == 0] = np.abs(q - b)[b == 0]
        assert rel.max() <= 1e-5  # north_star tolerance


def _ca_volumes(L, R, D, kw):
    H, W = L.shape
    st = abi.Stereo(W, H, D, **kw)
    st.set_debug(abi.DEBUG_CA, True)
    _run_gpu(L, R, D, st=st, **kw)
    caL, caR, DL, DR = (st.download(b) for b in (abi.BUF_CA_L, abi.BUF_CA_R, abi.BUF_DL, abi.BUF_DR))
    st.close()
    return caL, caR, DL, DR


@pytest.mark.parametrize("case", [
    # several 16-column strips and row bands, odd D_s (the last disparity pair
    # has one member), ragged last strip / band
    dict(W=301, H=263, D=45, kw=dict(k_scale=1), img="scene"),
    # the largest vertical window the y tile allows (2*112+1 = 225 rows) with
    # x sums at their maximum (every term BORDER for x < d, or AD = 255):
    # exercises the exact lo/hi split of the column prefix at its limits
    dict(W=60, H=300, D=40, kw=dict(k_scale=1, w_y=112), img="flat"),
    dict(W=60, H=300, D=12, kw=dict(k_scale=1, w_y=112, w_x=60), img="extreme"),
])
def test_ca_volume_split_prefix_extremes(case):
    W, H, D, kw = case["W"], case["H"], case["D"], case["kw"]
    if case["img"] == "scene":
        L, R, _ = synth.scene(W, H, D, seed=9)
    elif case["img"] == "flat":
        L = np.full((H, W), 90, np.uint8)
        R = L.copy()
    else:  # maximal AD everywhere, flat (arms at their caps)
        L = np.zeros((H, W), np.uint8)
        R = np.full((H, W), 255, np.uint8)
    caL, caR, DL, DR = _ca_volumes(L, R, D, kw)
    ref = oracle.pipeline(L, R, D, _oracle_params(kw), "fixed", stages=("caL", "caR", "DL", "DR"))
    for a, b in ((caL, ref["caL"]), (caR, ref["caR"]), (DL, ref["DL"]), (DR, ref["DR"])):
        assert np.array_equal(a, b)
    if case["img"] != "scene":  # the windows really reach the split's limits
        f = oracle.fixed_bits(kw.get("w_x", 21))
        assert int(caL.max()) >= 200 * (2 ** 24) and int(caL.max()) < 2 ** 41 and f >= 22


@pytest.mark.parametrize("W,H,D", [
    (1444, 960, 380),   # NEXT-2 (i): Vintage-shaped, D_s = 190
    (1482, 994, 128),   # NEXT-2 (ii): Pipes-shaped
])
def test_next2_workloads_bit_exact(W, H, D):
    L, R, _ = synth.scene(W, H, D, seed=3)
    _compare(L, R, D, dict(), volumes=False)


@pytest.mark.parametrize("mode", ["bilateral", "nearest", "smaller", "eq11_literal"])
def test_next3_fill_modes_bit_exact(mode):
    """NEXT-3: the Fig. 6 baselines and the printed Eq. 11 (§III.E), c2 scene
    (many occlusion non-GCPs) with K = 2 so the scale-up sees every mode."""
    L, R, _ = synth.scene(450, 376, 64, seed=12)
    _compare(L, R, 64, dict(fill_mode=oracle.FILL_MODES[mode]), volumes=False)


@pytest.mark.parametrize("w_x,w_x_r", [(21, 5), (7, 41), (0, 21)])
def test_next3_asymmetric_x_windows_bit_exact(w_x, w_x_r):
    """NEXT-3: different x aggregation caps for D^L and D^R."""
    L, R, _ = synth.scene(300, 160, 48, seed=w_x + w_x_r)
    got, ref = _compare(L, R, 48, dict(k_scale=1, w_x=w_x, w_x_r=w_x_r))
    assert got["armR"][0].max() <= w_x_r and got["armL"][0].max() <= w_x


def test_rgb_front_end_bit_exact():
    """§III item 1: gray front end + pipeline == oracle(rgb_to_gray)."""
    W, H, D = 320, 200, 48
    L, R, _ = synth.scene(W, H, D, seed=21)
    rng = np.random.default_rng(5)
    # colour images whose luma is not the gray scene: the conversion matters
    Lrgb = np.clip(L[..., None].astype(np.int32) + rng.integers(-40, 41, (H, W, 3)), 0, 255).astype(np.uint8)
    Rrgb = np.clip(R[..., None].astype(np.int32) + rng.integers(-40, 41, (H, W, 3)), 0, 255).astype(np.uint8)
    gL, gR = oracle.rgb_to_gray(Lrgb), oracle.rgb_to_gray(Rrgb)
    ref = oracle.pipeline(gL, gR, D, oracle.params(), "fixed", stages=("out",))["out"]
    st = abi.Stereo(W, H, D)
    out = torch.zeros((H, W), dtype=torch.float32, device=DEV)
    st.compute_rgb(torch.from_numpy(Lrgb).to(DEV), torch.from_numpy(Rrgb).to(DEV), out)
    g = torch.zeros((H, W), dtype=torch.uint8, device=DEV)
    abi.rgb_to_gray(torch.from_numpy(Lrgb).to(DEV), g)
    torch.cuda.synchronize()
    assert np.array_equal(g.cpu().numpy(), gL)
    assert np.array_equal(out.cpu().numpy().view(np.uint32), ref.view(np.uint32))
    st.close()


def test_depth_eq1_bit_exact():
    """NEXT-4: Eq. 1 on a computed disparity map (d = 0 -> +inf)."""
    L, R, _ = synth.scene(200, 120, 32, seed=4)
    st = abi.Stereo(200, 120, 32)
    out = torch.zeros((120, 200), dtype=torch.float32, device=DEV)
    st.compute(torch.from_numpy(L).to(DEV), torch.from_numpy(R).to(DEV), out)
    out[0, :5] = torch.tensor([0.0, 1.0, 3.0, 0.5, 144.0])
    Z = torch.empty_like(out)
    abi.disparity_to_depth(out, Z, 1234.5)
    torch.cuda.synchronize()
    ref = oracle.depth(out.cpu().numpy(), 1234.5)
    assert np.array_equal(Z.cpu().numpy().view(np.uint32), ref.view(np.uint32))
    st.close()


@pytest.mark.parametrize("case", [(450, 375, 64, 1, 2), (300, 200, 48, 2, 5), (160, 120, 32, 1, 9)])
def test_disparity_maps_vs_double_definition(case):
    """<= 0.01% of D^L/D^R pixels may differ from the double-mode oracle, and
    every one of them only where the two candidates' double costs tie within
    1e-5 relative (north_star; the quantisation bound 0.5*2^-f/c_AD(1) per
    term)."""
    W, H, D, K, seed = case
    L, R, _ = synth.scene(W, H, D, seed=seed)
    got = _run_gpu(L, R, D, k_scale=K)
    dbl = oracle.pipeline(L, R, D, oracle.params(k_scale=K), "double",
                          stages=("DL", "DR", "caL_d", "caR_d"))
    for m, vol in (("DL", "caL_d"), ("DR", "caR_d")):
        diff = got[m] != dbl[m]
        assert diff.mean() <= 1e-4
        v = dbl[vol]
        for y, x in zip(*np.nonzero(diff)):
            a, b = v[got[m][y, x], y, x], v[dbl[m][y, x], y, x]
            assert abs(a - b) <= 1e-5 * abs(b), (m, y, x, a, b)


# ---------------------------------------------------------------- stage isolation
def test_stage_isolation_ypass_from_oracle_cax():
    """Feed the oracle's CA_x and arms into the y pass alone."""
    L, R, _ = synth.scene(200, 90, 40, seed=7)
    p = oracle.params(k_scale=1)
    ref = oracle.pipeline(L, R, 40, p, "fixed", stages=("caxL", "caxR", "armL", "armR", "DL", "DR"))
    st = abi.Stereo(200, 90, 40, k_scale=1)
    i = st.info
    pad = lambda v: np.pad(v, ((0, 0), (0, 0), (0, i.cax_pitch - i.Ws)))
    st.upload(abi.BUF_CAX_L, pad(ref["caxL"]))
    st.upload(abi.BUF_CAX_R, pad(ref["caxR"]))
    pack = lambda a: (a[0].astype(np.uint32) | a[1].astype(np.uint32) << 8 |
                      a[2].astype(np.uint32) << 16 | a[3].astype(np.uint32) << 24)
    st.upload(abi.BUF_ARM_L, pack(ref["armL"]))
    st.upload(abi.BUF_ARM_R, pack(ref["armR"]))
    st.run_stage(abi.STAGE_YPASS)
    torch.cuda.synchronize()
    assert np.array_equal(st.download(abi.BUF_DL), ref["DL"])
    assert np.array_equal(st.download(abi.BUF_DR), ref["DR"])
    st.close()


def test_stage_isolation_post_from_oracle_maps():
    """Feed the oracle's D^L / D^R into the fused post stage alone."""
    L, R, _ = synth.scene(160, 100, 32, seed=8)
    p = oracle.params()
    ref = oracle.pipeline(L, R, 32, p, "fixed",
                          stages=("DL", "DR", "masked", "median", "fill", "out", "Ls", "cenL"))
    st = abi.Stereo(160, 100, 32)
    st.upload(abi.BUF_DL, ref["DL"])
    st.upload(abi.BUF_DR, ref["DR"])
    st.upload(abi.BUF_PIX_L, ref["Ls"].astype(np.uint16) | (ref["cenL"].astype(np.uint16) << 8))
    Lt = torch.from_numpy(L).to(DEV)
    out = torch.zeros((100, 160), dtype=torch.float32, device=DEV)
    st.run_stage(abi.STAGE_POST, L=Lt, out=out)
    torch.cuda.synchronize()
    assert np.array_equal(st.download(abi.BUF_MASKED), ref["masked"])
    assert np.array_equal(st.download(abi.BUF_MEDIAN), ref["median"])
    assert np.array_equal(st.download(abi.BUF_FILL).view(np.uint32), ref["fill"].view(np.uint32))
    assert np.array_equal(out.cpu().numpy().view(np.uint32), ref["out"].view(np.uint32))
    st.close()


@pytest.mark.parametrize("K", [1, 2])
def test_all_invalid_rows_rule_d(K):
    """Rule (d): rows without any valid pixel (constructed via uploaded maps),
    including the first rows and an odd output height."""
    Ws, Hs = 40, 12
    W, H = Ws * K + (K - 1), Hs * K + (K - 1)
    st = abi.Stereo(W, H, 8, k_scale=K)
    rng = np.random.default_rng(3)
    DL = rng.integers(0, 8, (Hs, Ws)).astype(np.uint8)
    DR = np.full((Hs, Ws), 200, np.uint8)  # nothing cross-checks ...
    for y in (4, 5, 9):                    # ... except rows 4, 5 and 9
        DR[y] = DL[y] = rng.integers(0, 3)
        DL[y, :3] = 0
        DR[y, :3] = 0
    Ls = rng.integers(0, 256, (Hs, Ws)).astype(np.uint8)
    Lorg = rng.integers(0, 256, (H, W)).astype(np.uint8)
    st.upload(abi.BUF_DL, DL)
    st.upload(abi.BUF_DR, DR)
    st.upload(abi.BUF_PIX_L, Ls.astype(np.uint16))
    out = torch.zeros((H, W), dtype=torch.float32, device=DEV)
    Lt = torch.from_numpy(Lorg).to(DEV)
    for _ in range(2):  # twice: the grid-wide counter must reset itself
        st.run_stage(abi.STAGE_POST, L=Lt, out=out)
    torch.cuda.synchronize()
    med = oracle.median3x3(oracle.cross_check(DL, DR))
    fill = oracle.fill_bilateral(med, Ls, 3)
    ref = fill if K == 1 else oracle.scale_up(fill, Lorg, 2, 3)
    assert np.array_equal(out.cpu().numpy(), ref)
    st.close()


# ---------------------------------------------------------------- API behaviour
def test_batch_host_and_repeat_determinism():
    W, H, D = 200, 120, 48
    frames = synth.stream(W, H, D, 7, seed=3)
    st = abi.Stereo(W, H, D)
    Lb = torch.from_numpy(np.stack([f[0] for f in frames])).to(DEV)
    Rb = torch.from_numpy(np.stack([f[1] for f in frames])).to(DEV)
    out = torch.zeros((7, H, W), dtype=torch.float32, device=DEV)
    st.compute_batch(Lb, Rb, out, 7)
    torch.cuda.synchronize()
    outs = out.cpu().numpy()
    for k, (L, R) in enumerate(frames):
        ref = oracle.pipeline(L, R, D, oracle.params(), "fixed", stages=("out",))["out"]
        assert np.array_equal(outs[k], ref)
    # host-buffer (end-to-end) path
    Lh = torch.from_numpy(frames[2][0]).pin_memory()
    Rh = torch.from_numpy(frames[2][1]).pin_memory()
    oh = torch.zeros((H, W), dtype=torch.float32).pin_memory()
    st.compute_host(Lh, Rh, oh)
    torch.cuda.synchronize()
    assert np.array_equal(oh.numpy(), outs[2])
    # a second stream gives the same bits
    s2 = torch.cuda.Stream()
    o2 = torch.zeros((H, W), dtype=torch.float32, device=DEV)
    with torch.cuda.stream(s2):
        st.compute(Lb[4], Rb[4], o2, stream=s2)
    s2.synchronize()
    assert np.array_equal(o2.cpu().numpy(), outs[4])
    st.close()


@pytest.mark.parametrize("nb,n,K", [(1, 3, 2), (3, 7, 2), (8, 8, 1), (5, 11, 1), (4, 6, 2)])
def test_batch_capacity_bit_exact(nb, n, K):
    """stereo_create_batch: one launch sequence per chunk of nb frames (the x
    and y passes see a chunk as one tall image); every frame bit-exact,
    including chunk tails and frames that need fill rule (d)."""
    W, H, D = 61, 47, 16
    frames = []
    for i in range(n):
        if i % 3 == 2:  # unrelated noise: all-invalid rows (rule (d))
            frames.append(synth.random_pair(W, H, seed=40 + i, levels=256))
        else:
            frames.append(synth.scene(W, H, D, seed=40 + i)[:2])
    st = abi.Stereo(W, H, D, max_frames=nb, k_scale=K)
    assert st.info.max_frames == nb
    Lb = torch.from_numpy(np.stack([f[0] for f in frames])).to(DEV)
    Rb = torch.from_numpy(np.stack([f[1] for f in frames])).to(DEV)
    out = torch.full((n, H, W), float("nan"), dtype=torch.float32, device=DEV)
    for _ in range(2):  # twice: the per-frame rule-(d) counters reset themselves
        st.compute_batch(Lb, Rb, out, n)
    torch.cuda.synchronize()
    outs = out.cpu().numpy()
    for k, (L, R) in enumerate(frames):
        ref = oracle.pipeline(L, R, D, oracle.params(k_scale=K), "fixed", stages=("out",))["out"]
        assert np.array_equal(outs[k].view(np.uint32), ref.view(np.uint32)), k
    st.close()


def test_batch_capacity_c3_two_frames():
    W, H, D = 1436, 992, 145
    frames = [synth.scene(W, H, D, seed=s)[:2] for s in (21, 22, 23)]
    st1 = abi.Stereo(W, H, D)
    st2 = abi.Stereo(W, H, D, max_frames=2)
    Lb = torch.from_numpy(np.stack([f[0] for f in frames])).to(DEV)
    Rb = torch.from_numpy(np.stack([f[1] for f in frames])).to(DEV)
    o1 = torch.zeros((3, H, W), dtype=torch.float32, device=DEV)
    o2 = torch.ones((3, H, W), dtype=torch.float32, device=DEV)
    st1.compute_batch(Lb, Rb, o1, 3)
    st2.compute_batch(Lb, Rb, o2, 3)
    torch.cuda.synchronize()
    assert torch.equal(o1.view(torch.int32), o2.view(torch.int32))
    ref = oracle.pipeline(frames[1][0], frames[1][1], D, oracle.params(), "fixed", stages=("out",))["out"]
    assert np.array_equal(o2[1].cpu().numpy().view(np.uint32), ref.view(np.uint32))
    st1.close()
    st2.close()


def test_large_and_small_handles_alive_together():
    """the per-kernel dynamic shared-memory limit is process-wide;
    a later, smaller handle must not break an earlier, larger one."""
    big = abi.Stereo(2872, 1984, 290)
    small = abi.Stereo(200, 120, 32)
    for st, (W, H, D) in ((big, (2872, 1984, 290)), (small, (200, 120, 32)), (big, (2872, 1984, 290))):
        L, R, _ = synth.scene(W, H, D, seed=1) if W < 1000 else (None, None, None)
        if L is None:
            L = np.random.default_rng(0).integers(0, 256, (H, W), dtype=np.uint8)
            R = np.roll(L, -20, axis=1)
        out = torch.zeros((H, W), dtype=torch.float32, device=DEV)
        st.compute(torch.from_numpy(L).to(DEV), torch.from_numpy(R).to(DEV), out)
        torch.cuda.synchronize()  # a launch failure would raise at the next call
        assert torch.isfinite(out).all()
    big.close()
    small.close()


def test_binding_rejects_bad_arguments():
    st = abi.Stereo(64, 48, 16, k_scale=1)
    L = torch.zeros((48, 64), dtype=torch.uint8, device=DEV)
    out = torch.zeros((48, 64), dtype=torch.float32, device=DEV)
    with pytest.raises(ValueError):
        st.compute(L.cpu(), L, out)            # host tensor
    with pytest.raises(ValueError):
        st.compute(L.float(), L, out)          # dtype
    with pytest.raises(ValueError):
        st.compute(L[:40], L, out)             # shape
    with pytest.raises(ValueError):
        st.compute(L, L, out.double())
    with pytest.raises(ValueError):
        st.compute_host(np.zeros((48, 64), np.uint8), np.zeros((48, 64), np.uint8),
                        np.zeros((48, 63), np.float32))
    st.close()


@pytest.mark.parametrize("nb,case", [(8, (1436, 992, 145, 2)), (3, (200, 120, 32, 2)),
                                     (5, (160, 100, 24, 1)), (64, (96, 70, 16, 1))])
def test_l2_band_staging_bit_exact(nb, case, monkeypatch):
    """NEXT-1 prototype (STEREO_L2_BANDS): the x and y passes alternate over
    row bands, CA_x rows discarded from L2 once dead; every output bit-exact
    (the CA_x volumes themselves are then undefined after a frame)."""
    W, H, D, K = case
    monkeypatch.setenv("STEREO_L2_BANDS", str(nb))
    frames = [synth.scene(W, H, D, seed=s)[:2] for s in (31, 32)]
    st = abi.Stereo(W, H, D, k_scale=K)
    monkeypatch.delenv("STEREO_L2_BANDS")
    out = torch.zeros((H, W), dtype=torch.float32, device=DEV)
    for _ in range(2):  # twice: the previous frame's tail discard
        for L, R in frames:
            st.compute(torch.from_numpy(L).to(DEV), torch.from_numpy(R).to(DEV), out)
            torch.cuda.synchronize()
            ref = oracle.pipeline(L, R, D, oracle.params(k_scale=K), "fixed", stages=("out",))["out"]
            assert np.array_equal(out.cpu().numpy().view(np.uint32), ref.view(np.uint32))
    st.close()


def test_stage_timers():
    W, H, D = 1436, 992, 145
    L, R, _ = synth.scene(W, H, D, seed=0)
    st = abi.Stereo(W, H, D)
    Lt, Rt = torch.from_numpy(L).to(DEV), torch.from_numpy(R).to(DEV)
    out = torch.zeros((H, W), dtype=torch.float32, device=DEV)
    st.set_timing(True)
    for _ in range(3):
        st.compute(Lt, Rt, out)
    ms, n = st.stage_times_ms()
    assert n == 3 and all(v > 0 for v in ms.values())
    st.close()


def test_racecheck_variant_bit_exact():
    """The sanitizer build (lib/racecheck, -DSTEREO_RACECHECK: x-pass ring
    refills ordered by CTA barriers, the edge compute-sanitizer's racecheck
    models) gives the same bits as the oracle (run in a subprocess that loads
    that library instead of the product one)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    lib_rc = os.path.join(root, "paper_2212_00488_b200", "lib", "racecheck", "libstereo_b200.so")
    if not os.path.exists(lib_rc):
        pytest.skip("racecheck variant not built (STEREO_SKIP_RACECHECK_BUILD)")
    code = r'''
import sys, numpy as np, torch
sys.path.insert(0, ROOT)
import oracle
from paper_2212_00488_b200 import abi, synth
assert abi.LIB_PATH.endswith("racecheck/libstereo_b200.so")
for (W, H, D, K) in ((64, 48, 16, 1), (131, 77, 33, 2), (450, 375, 64, 1), (2880, 64, 40, 2)):
    L, R, _ = synth.scene(W, H, D, seed=3)
    st = abi.Stereo(W, H, D, k_scale=K)
    out = torch.empty((H, W), dtype=torch.float32, device="cuda")
    st.compute(torch.from_numpy(L).cuda(), torch.from_numpy(R).cuda(), out)
    torch.cuda.synchronize()
    ref = oracle.pipeline(L, R, D, oracle.params(k_scale=K), "fixed", stages=("out",))["out"]
    assert np.array_equal(out.cpu().numpy().view(np.uint32), ref.view(np.uint32)), (W, H, D, K)
    st.close()
print("ok")
'''.replace("ROOT", repr(root))
    env = dict(os.environ, STEREO_B200_LIB=lib_rc)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]


@pytest.mark.parametrize("case", [(1436, 992, 145, 2), (300, 200, 48, 1)])
def test_ypass_v2_wide_strips_bit_exact(case, monkeypatch):
    """The 32-column y pass (STEREO_YPASS_V=2, a measured-slower experiment
    kept selectable) gives the same bits as the oracle."""
    W, H, D, K = case
    monkeypatch.setenv("STEREO_YPASS_V", "2")
    L, R, _ = synth.scene(W, H, D, seed=12)
    got = _run_gpu(L, R, D, k_scale=K)
    monkeypatch.delenv("STEREO_YPASS_V")
    ref = oracle.pipeline(L, R, D, oracle.params(k_scale=K), "fixed", stages=("DL", "DR", "out"))
    for s in ("DL", "DR"):
        assert np.array_equal(got[s], ref[s])
    assert np.array_equal(got["out"].view(np.uint32), ref["out"].view(np.uint32))


@pytest.mark.parametrize("case", [(1436, 992, 145, 2, 0), (300, 200, 48, 1, 3), (131, 77, 33, 2, 5),
                                  (64, 48, 16, 1, 7)])
def test_fused_next1_bit_exact(case, monkeypatch):
    """NEXT-1 prototype (STEREO_FUSED=1): cost + CA_x + CA + WTA in one
    kernel, CA_x never written to global memory; every stage bit-exact."""
    W, H, D, K, seed = case
    monkeypatch.setenv("STEREO_FUSED", "1")
    L, R, _ = synth.scene(W, H, D, seed=seed)
    got = _run_gpu(L, R, D, k_scale=K)
    monkeypatch.delenv("STEREO_FUSED")
    ref = oracle.pipeline(L, R, D, oracle.params(k_scale=K), "fixed", stages=("DL", "DR", "out"))
    for s in ("DL", "DR"):
        assert np.array_equal(got[s], ref[s]), s
    assert np.array_equal(got["out"].view(np.uint32), ref["out"].view(np.uint32))


def test_batch_handle_single_frame_calls():
    """A handle of batch capacity 4 serves single frames too (stereo_compute,
    stereo_compute_host use frame slot 0) and an empty batch is a no-op."""
    W, H, D = 120, 90, 24
    L, R, _ = synth.scene(W, H, D, seed=17)
    ref = oracle.pipeline(L, R, D, oracle.params(), "fixed", stages=("out",))["out"]
    st = abi.Stereo(W, H, D, max_frames=4)
    out = torch.zeros((H, W), dtype=torch.float32, device=DEV)
    st.compute(torch.from_numpy(L).to(DEV), torch.from_numpy(R).to(DEV), out)
    oh = torch.zeros((H, W), dtype=torch.float32).pin_memory()
    st.compute_host(torch.from_numpy(L).pin_memory(), torch.from_numpy(R).pin_memory(), oh)
    e = torch.zeros((0, H, W), dtype=torch.uint8, device=DEV)
    st.compute_batch(e, e, torch.zeros((0, H, W), dtype=torch.float32, device=DEV), 0)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy().view(np.uint32), ref.view(np.uint32))
    assert np.array_equal(oh.numpy().view(np.uint32), ref.view(np.uint32))
    st.close()


@pytest.mark.parametrize("nb,n", [(1, 3), (3, 7), (4, 4)])
def test_compute_host_batch_bit_exact(nb, n):
    """stereo_compute_host_batch: pinned host frames in, host maps out, per
    chunk of max_frames frames one copy in / launch sequence / copy out."""
    W, H, D = 100, 70, 20
    frames = [synth.scene(W, H, D, seed=60 + i)[:2] for i in range(n)]
    st = abi.Stereo(W, H, D, max_frames=nb)
    Lh = torch.from_numpy(np.stack([f[0] for f in frames])).pin_memory()
    Rh = torch.from_numpy(np.stack([f[1] for f in frames])).pin_memory()
    Oh = torch.zeros((n, H, W), dtype=torch.float32).pin_memory()
    st.compute_host_batch(Lh, Rh, Oh, n)
    torch.cuda.synchronize()
    for k, (L, R) in enumerate(frames):
        ref = oracle.pipeline(L, R, D, oracle.params(), "fixed", stages=("out",))["out"]
        assert np.array_equal(Oh[k].numpy().view(np.uint32), ref.view(np.uint32)), k
    st.close()
