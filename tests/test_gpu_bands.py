"""Row-band mode on the GPU: P bands of one frame
computed independently through the C ABI (emulated on one GPU, the exchange
replaced by slicing; tests/test_dist_gloo.py covers the real P2P exchange) must
reassemble to the single-GPU full-frame output bit for bit, including frames
whose fill rule (d) needs rows of another band."""
import numpy as np
import pytest

import oracle
from paper_2212_00488_b200 import abi
from paper_2212_00488_b200 import dist as sdist
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


def _bands(L, R, D, P, **kw):
    H, W = L.shape
    bss = [sdist.BandStereo(W, H, D, P, r, **kw) for r in range(P)]
    outs, Lbs = [], []
    for bs in bss:
        b = bs.b
        Lb = torch.from_numpy(np.ascontiguousarray(L[b.r0:b.r1])).to(DEV)
        Rb = torch.from_numpy(np.ascontiguousarray(R[b.r0:b.r1])).to(DEV)
        o = torch.empty((b.rows, W), dtype=torch.float32, device=DEV)
        bs.compute(Lb, Rb, o)
        outs.append(o)
        Lbs.append(Lb)
    torch.cuda.synchronize()
    patched = 0
    if any(bs.needs_patch_local() for bs in bss):  # the all_reduce(MAX) of dist.py
        Hs = H // bss[0].K
        summ = np.zeros((3, Hs), np.int64)         # the all_gather of dist.py
        for bs in bss:
            summ[:, bs.b.ys0:bs.b.ys1] = bs.local_summaries()
        for bs, Lb, o in zip(bss, Lbs, outs):
            patched += bs.patch(summ, Lb, o)
    got = np.zeros((H, W), np.float32)
    for bs, o in zip(bss, outs):
        got[bs.b.o0:bs.b.o1] = o[bs.own_slice()].cpu().numpy()
        bs.close()
    return got, patched


@pytest.mark.parametrize("P", [2, 3, 8])
def test_c3_bands_bit_exact(P):
    L, R, _ = synth.scene(1436, 992, 145, seed=2)
    full = _full(L, R, 145)
    got, _ = _bands(L, R, 145, P)
    assert np.array_equal(got.view(np.uint32), full.view(np.uint32))


@pytest.mark.parametrize("case", [
    (10, 90, 16, 2, 1, 3, 5),   # rows 26..30 without any GCP straddle a band edge
    (24, 60, 16, 1, 3, 2, 5),
    (31, 77, 12, 2, 2, 4, 9),   # odd sizes
])
def test_degenerate_rows_need_global_patch(case):
    W, H, D, K, w_y, P, seed = case
    L, R = synth.random_pair(W, H, seed=seed)
    full = _full(L, R, D, k_scale=K, w_y=w_y)
    ref = oracle.pipeline(L, R, D, oracle.params(k_scale=K, w_y=w_y), "fixed", stages=("out",))["out"]
    assert np.array_equal(full, ref)
    got, patched = _bands(L, R, D, P, k_scale=K, w_y=w_y)
    assert np.array_equal(got.view(np.uint32), full.view(np.uint32))


@pytest.mark.slow
def test_c5_eight_bands_bit_exact():
    L, R, _ = synth.scene(2872, 1984, 290, seed=0)
    full = _full(L, R, 290)
    got, _ = _bands(L, R, 290, 8)
    assert np.array_equal(got.view(np.uint32), full.view(np.uint32))
