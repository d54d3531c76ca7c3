"""Middlebury evaluation harness (NEXT-4, paper_2212_00488_b200/middlebury.py):
PFM / calib I/O and the bad-N metric pinned by the format definition and the
SPEC examples; a GPU run on a synthetic Middlebury-format scene."""
import math
import os
import struct

import numpy as np
import pytest

from paper_2212_00488_b200 import middlebury as mb


def test_pfm_header_example_bottom_row_first():
    # header "Pf\n2 2\n-1.0\n" + 16 bytes -> 2x2 map, bottom row first
    raw = b"Pf\n2 2\n-1.0\n" + struct.pack("<4f", 1.0, 2.0, 3.0, 4.0)
    d = mb.read_pfm(raw)
    assert d.dtype == np.float32 and d.shape == (2, 2)
    assert d.tolist() == [[3.0, 4.0], [1.0, 2.0]]


def test_pfm_big_endian_positive_scale():
    raw = b"Pf\n3 1\n1.0\n" + struct.pack(">3f", 0.5, -2.0, 7.25)
    assert mb.read_pfm(raw).tolist() == [[0.5, -2.0, 7.25]]


def test_pfm_round_trip_with_invalid(tmp_path):
    rng = np.random.default_rng(3)
    d = rng.normal(50, 20, (37, 53)).astype(np.float32)
    d[rng.random(d.shape) < 0.1] = np.inf  # Middlebury: +inf = unknown
    p = tmp_path / "d.pfm"
    mb.write_pfm(str(p), d)
    back = mb.read_pfm(str(p))
    assert np.array_equal(back.view(np.uint32), d.view(np.uint32))


def test_pfm_rejects_nan_and_bad_headers():
    with pytest.raises(ValueError):
        mb.write_pfm(None, np.array([[np.nan]], dtype=np.float32))
    for raw in (b"P6\n2 2\n255\n", b"PF\n1 1\n-1.0\n" + b"\0" * 12, b"Pf\n2 2\n0\n" + b"\0" * 16,
                b"Pf\n2 2\n-1.0\n" + b"\0" * 15):
        with pytest.raises(ValueError):
            mb.read_pfm(raw)


def test_calib():
    c = mb.read_calib("cam0=[...]\nndisp=145\nwidth=1436\nheight=992\n")
    assert (c["ndisp"], c["width"], c["height"]) == (145, 1436, 992)  # Table II Adirondack(H)
    with pytest.raises(ValueError):
        mb.read_calib("width=10\n")


def test_eval_bad_examples():
    rng = np.random.default_rng(0)
    gt = rng.uniform(0, 100, (40, 60))
    assert mb.eval_bad(gt, gt).bad_rate_all == 0.0
    assert mb.eval_bad(gt + 3.0, gt, 2.0).bad_rate_all == 100.0
    half = gt.copy()
    half[:, :30] += 5.0
    r = mb.eval_bad(half, gt, 2.0)
    assert r.bad_rate_all == 50.0
    assert math.isclose(r.avg_abs_err, 2.5)


def test_eval_bad_invalid_handling():
    gt = np.full((4, 4), 10.0)
    gt[0, 0] = np.inf                       # GT-unknown: not counted
    pred = np.full((4, 4), 10.5)
    pred[1, 1] = np.inf                     # predicted INVALID counts as bad
    r = mb.eval_bad(pred, gt, 2.0, occ_mask=np.eye(4) == 0)
    assert math.isclose(r.bad_rate_all, 100.0 / 15)
    assert r.bad_rate_nonocc == 0.0         # (1,1) is on the diagonal: masked out
    assert math.isclose(r.avg_abs_err, 0.5)
    assert math.isclose(r.coverage, 15 / 16)
    with pytest.raises(ValueError):
        mb.eval_bad(pred[:3], gt)


@pytest.mark.gpu
def test_run_scene_on_synthetic_middlebury_layout(tmp_path):
    """A synthetic scene written in the Middlebury layout (im0/im1 PNG, GT PFM,
    calib) goes through the GPU path (colour front end) and is scored; the score
    equals the one of the device map computed directly from the gray pair
    (BT.601 of a gray pixel is itself)."""
    import torch
    from PIL import Image

    from paper_2212_00488_b200 import abi, synth
    W, H, D = 360, 248, 64
    L, R, dgt = synth.scene(W, H, D, seed=5)
    sd = tmp_path / "Synth"
    sd.mkdir()
    Image.fromarray(np.repeat(L[:, :, None], 3, axis=2)).save(sd / "im0.png")
    Image.fromarray(np.repeat(R[:, :, None], 3, axis=2)).save(sd / "im1.png")
    mb.write_pfm(str(sd / "disp0GT.pfm"), dgt.astype(np.float32))
    (sd / "calib.txt").write_text(f"ndisp={D}\nwidth={W}\nheight={H}\n")
    res = mb.run_dataset(str(tmp_path))
    rep = res["Synth"]
    st = abi.Stereo(W, H, D, k_scale=2)
    out = torch.empty((H, W), dtype=torch.float32, device="cuda")
    st.compute(torch.from_numpy(L).cuda(), torch.from_numpy(R).cuda(), out)
    torch.cuda.synchronize()
    st.close()
    ref = mb.eval_bad(out.cpu().numpy(), dgt.astype(np.float32))
    assert rep.bad_rate_all == ref.bad_rate_all
    assert rep.coverage == 1.0              # dense output (§8(b))
    assert rep.bad_rate_all < 35.0          # SPEC acceptance 7's bound, on synthetic data
    assert res["average"] == rep.bad_rate_all
