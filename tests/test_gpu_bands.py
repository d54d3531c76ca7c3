"""Row-band mode on the GPU through the band
calls of the C ABI: P band handles of one frame (emulated on one GPU: the
halo exchange is slicing, the MAX all-reduce of the summaries is torch.max)
must reassemble to the single-GPU full-frame output bit for bit, including
frames whose fill rule (d) needs rows of another band (resolved on the device
by stereo_band_finish).  tests/test_dist_gloo.py covers the real exchange."""
import numpy as np
import pytest

import oracle
from paper_2212_00488_b200 import abi
from paper_2212_00488_b200 import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def _full(L, R, D, **kw):
    H, W = L.shape
    st = abi.Stereo(W, H, D, **kw)
    out = torch.empty((H, W), dtype=torch.float32, device=DEV)
    st.compute(torch.from_numpy(L).to(DEV), torch.from_numpy(R).to(DEV), out)
    torch.cuda.synchronize()
    st.close()
    return out.cpu().numpy()


def _bands(L, R, D, P, check_cone=True, **kw):
    H, W = L.shape
    p = abi.default_params(**kw)
    K = p.k_scale
    bss, outs, Lbs = [], [], []
    for r in range(P):
        y0, rows = abi.band_rows(H, P, r, p)
        bs = abi.StereoBand(W, H, D, y0, rows, params=p)
        if check_cone:  # y aggregation + WTA only for the own rows + the 3-row cone
            assert bs.info.ypass_rows <= rows // K + 4
        Lb = torch.from_numpy(np.ascontiguousarray(L[bs.sub_y0:bs.sub_y0 + bs.sub_rows])).to(DEV)
        Rb = torch.from_numpy(np.ascontiguousarray(R[bs.sub_y0:bs.sub_y0 + bs.sub_rows])).to(DEV)
        o = torch.full((rows, W), float("nan"), dtype=torch.float32, device=DEV)
        bs.compute(Lb, Rb, o)
        bss.append(bs)
        outs.append(o)
        Lbs.append(Lb)
    # the summaries' MAX all-reduce, emulated
    summs = [torch.empty((H // K, 2), dtype=torch.int32, device=DEV) for _ in range(P)]
    for bs, sm in zip(bss, summs):
        bs.summary(sm)
    summ = torch.stack(summs).amax(dim=0).contiguous()
    for bs, Lb, o in zip(bss, Lbs, outs):
        bs.finish(summ, Lb, o)
    torch.cuda.synchronize()
    got = np.zeros((H, W), np.float32)
    for bs, o in zip(bss, outs):
        got[bs.y0:bs.y0 + bs.rows] = o.cpu().numpy()
        bs.close()
    return got, summ.cpu().numpy()


@pytest.mark.parametrize("P", [2, 3, 8])
def test_c3_bands_bit_exact(P):
    L, R, _ = synth.scene(1436, 992, 145, seed=2)
    full = _full(L, R, 145)
    got, _ = _bands(L, R, 145, P)
    assert np.array_equal(got.view(np.uint32), full.view(np.uint32))


@pytest.mark.parametrize("case", [
    (10, 90, 16, 2, 1, 3, 5, 1),   # rows 26..30 without any GCP straddle a band edge
    (24, 60, 16, 1, 3, 2, 5, 1),
    (31, 77, 12, 2, 2, 4, 9, 1),   # odd sizes
    (40, 96, 16, 2, 4, 3, 5, 0),   # m_pool = 0 with rule (d)
    (40, 97, 16, 2, 4, 3, 5, 3),
])
def test_degenerate_rows_need_global_patch(case):
    W, H, D, K, w_y, P, seed, m = case
    L, R = synth.random_pair(W, H, seed=seed)
    kw = dict(k_scale=K, w_y=w_y, m_pool=m)
    full = _full(L, R, D, **kw)
    ref = oracle.pipeline(L, R, D, oracle.params(**kw), "fixed", stages=("out",))["out"]
    assert np.array_equal(full, ref)
    got, summ = _bands(L, R, D, P, check_cone=False, **kw)
    if case[0] == 10:  # the first case is built to need the frame-wide rule (d)
        assert (summ[:, 0] < 0).any()
    assert np.array_equal(got.view(np.uint32), full.view(np.uint32))


@pytest.mark.parametrize("m", [0, 1, 2, 3])
def test_bands_every_pool_radius(m):
    L, R, _ = synth.scene(300, 258, 48, seed=m)
    full = _full(L, R, 48, m_pool=m, w_y=9)
    got, _ = _bands(L, R, 48, 3, m_pool=m, w_y=9)
    assert np.array_equal(got.view(np.uint32), full.view(np.uint32))


def test_band_handle_rejects_other_calls():
    bs = abi.StereoBand(200, 120, 32, 0, 60)
    L = torch.zeros((bs.sub_rows, 200), dtype=torch.uint8, device=DEV)
    o = torch.zeros((60, 200), dtype=torch.float32, device=DEV)
    # the plain call on a band handle
    rc = abi.lib().stereo_compute(bs._h, L.data_ptr(), L.data_ptr(), o.data_ptr(), None)
    assert rc == abi.STEREO_EINVAL
    rc = abi.lib().stereo_compute_band(bs._h, L.data_ptr(), L.data_ptr(), 2, 60, bs.top, bs.bot,
                                       o.data_ptr(), None)
    assert rc == abi.STEREO_EINVAL  # wrong y0
    bs.close()


@pytest.mark.slow
def test_c5_eight_bands_bit_exact():
    L, R, _ = synth.scene(2872, 1984, 290, seed=0)
    full = _full(L, R, 290)
    got, _ = _bands(L, R, 290, 8)
    assert np.array_equal(got.view(np.uint32), full.view(np.uint32))


@pytest.mark.parametrize("seed", range(24))
def test_random_band_splits(seed):
    """Random frames, parameters (delta, w_x, w_y, T, pool radius, census
    pattern, fill mode) and band counts: the bands reassemble to the whole
    frame bit for bit (the library's halo covers the cone; rule (d) from the
    frame-wide summaries)."""
    import oracle
    rng = np.random.default_rng(500 + seed)
    K = int(rng.choice([1, 2]))
    W = int(rng.integers(8, 160))
    H = int(rng.integers(12 * K, 140))
    D = int(rng.integers(1, 40))
    cand = [(dx, dy) for dx in range(-2, 3) for dy in range(-2, 3) if (dx, dy) != (0, 0)]
    pat = [cand[i] for i in rng.choice(len(cand), 6, replace=False)]
    kw = dict(k_scale=K, delta=int(rng.integers(1, 60)), w_x=int(rng.integers(0, 30)),
              w_y=int(rng.integers(0, 40)), t_fill=int(rng.integers(0, 6)),
              m_pool=int(rng.integers(0, 4)), census=pat, fill_mode=int(rng.integers(0, 4)))
    if rng.random() < 0.5:
        L, R, _ = synth.scene(W, H, max(D, 2), seed=seed)
    else:
        L, R = synth.random_pair(W, H, seed=seed, levels=int(rng.integers(2, 257)))
    P = int(rng.integers(1, min(6, H // K) + 1))
    full = _full(L, R, D, **kw)
    ref = oracle.pipeline(L, R, D, oracle.params(**kw), "fixed", stages=("out",))["out"]
    assert np.array_equal(full.view(np.uint32), ref.view(np.uint32))
    got, _ = _bands(L, R, D, P, check_cone=False, **kw)
    assert np.array_equal(got.view(np.uint32), full.view(np.uint32)), (W, H, D, P, kw)
