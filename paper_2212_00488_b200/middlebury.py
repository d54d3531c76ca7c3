"""Middlebury evaluation harness (the step after the path).

The paper reports accuracy as the bad-2.0 error rate on the Middlebury
benchmark set ("error rate (Bad 2.0) of our system (24.09%)", Table I
P:536-549).  This module is host-side plumbing around the GPU path — no part
of the method's arithmetic lives here:

* ``read_pfm`` / ``write_pfm``: the Middlebury v3 ground-truth format:
  "Pf" header, width height, scale (negative = little-endian), rows stored
  bottom-up, +inf = invalid / unknown;
* ``read_calib``: ``calib.txt`` key=value lines (ndisp, width, height);
* ``eval_bad``: bad-N over GT-valid pixels: a pixel is bad when
  |pred - gt| > N or pred is invalid (non-finite); optional non-occluded mask;
* ``run_dataset``: for each scene directory holding im0.png, im1.png,
  disp0GT.pfm (+ calib.txt, mask0nocc.png) runs the GPU path
  (``stereo_compute_rgb`` — BT.601 gray front end, reading R31) and evaluates.
  It only runs when the dataset is present (no data ships with the repo, there
  is no network): the accuracy figure stays out of the parity claims.
"""
from __future__ import annotations

import dataclasses
import math
import os
import re
import sys

import numpy as np


# ---------------------------------------------------------------- PFM
def read_pfm(path_or_bytes) -> np.ndarray:
    """Single-channel PFM -> float32 [H][W], top row first (the file stores rows
    bottom-up).  Raises ValueError on a malformed header or a colour PFM."""
    data = path_or_bytes if isinstance(path_or_bytes, (bytes, bytearray)) else open(path_or_bytes, "rb").read()
    # header: three whitespace-separated tokens after the magic, then exactly one
    # whitespace byte before the raster
    m = re.match(rb"(P[fF])\s+(\d+)\s+(\d+)\s+([-+0-9.eE]+)\s", data)
    if not m:
        raise ValueError("malformed PFM header")
    if m.group(1) != b"Pf":
        raise ValueError("colour PFM (PF) is not a disparity map")
    w, h, scale = int(m.group(2)), int(m.group(3)), float(m.group(4))
    if w < 1 or h < 1 or scale == 0.0 or not math.isfinite(scale):
        raise ValueError("malformed PFM header (dimensions / scale)")
    off = m.end()
    need = 4 * w * h
    if len(data) - off < need:
        raise ValueError("truncated PFM raster")
    dt = np.dtype("<f4") if scale < 0 else np.dtype(">f4")
    img = np.frombuffer(data, dtype=dt, count=w * h, offset=off).reshape(h, w)
    return np.ascontiguousarray(img[::-1].astype(np.float32))


def write_pfm(path, d: np.ndarray) -> bytes:
    """float32 [H][W] (top row first; +inf = invalid) -> little-endian PFM with
    scale -1.0.  NaN is rejected.  Returns the bytes; writes them to
    ``path`` unless it is None."""
    d = np.asarray(d, dtype=np.float32)
    if d.ndim != 2:
        raise ValueError("disparity map must be 2-D")
    if np.isnan(d).any():
        raise ValueError("NaN in disparity map")
    h, w = d.shape
    out = f"Pf\n{w} {h}\n-1.0\n".encode() + d[::-1].astype("<f4").tobytes()
    if path is not None:
        with open(path, "wb") as f:
            f.write(out)
    return out


def read_calib(path_or_text) -> dict:
    """calib.txt -> {"ndisp": int, "width": int, "height": int, ...}; ndisp is
    required."""
    text = open(path_or_text).read() if os.path.exists(path_or_text) else path_or_text
    kv = {}
    for line in text.splitlines():
        if "=" in line:
            k, v = line.split("=", 1)
            kv[k.strip()] = v.strip()
    if "ndisp" not in kv:
        raise ValueError("calib: missing ndisp")
    out = dict(kv)
    for k in ("ndisp", "width", "height"):
        if k in kv:
            out[k] = int(float(kv[k]))
    return out


# ---------------------------------------------------------------- metric
@dataclasses.dataclass
class EvalReport:
    bad_threshold: float
    bad_rate_all: float          # % of GT-valid pixels
    bad_rate_nonocc: float | None  # % of GT-valid non-occluded pixels (mask given)
    avg_abs_err: float           # over GT-valid pixels with a valid prediction
    coverage: float              # fraction of pixels with a valid prediction


def eval_bad(pred: np.ndarray, gt: np.ndarray, threshold: float = 2.0,
             occ_mask: np.ndarray | None = None) -> EvalReport:
    """bad-N: 100 * |{p: gt valid, pred invalid or |pred-gt| > N}| /
    |{p: gt valid}|; gt valid = finite; pred invalid = non-finite.
    occ_mask: True (or nonzero) where the pixel is NOT occluded."""
    pred = np.asarray(pred, dtype=np.float64)
    gt = np.asarray(gt, dtype=np.float64)
    if pred.shape != gt.shape:
        raise ValueError(f"dimension mismatch: pred {pred.shape} vs gt {gt.shape}")
    gv = np.isfinite(gt)
    pv = np.isfinite(pred)
    err = np.abs(np.where(pv & gv, pred, 0.0) - np.where(gv, gt, 0.0))
    bad = gv & (~pv | (err > threshold))
    n = int(gv.sum())
    rate = 100.0 * int(bad.sum()) / n if n else 0.0
    nonocc = None
    if occ_mask is not None:
        m = gv & (np.asarray(occ_mask) != 0)
        nm = int(m.sum())
        nonocc = 100.0 * int((bad & m).sum()) / nm if nm else 0.0
    both = gv & pv
    aae = float(err[both].mean()) if both.any() else 0.0
    return EvalReport(threshold, rate, nonocc, aae, float(pv.mean()) if pv.size else 0.0)


# ---------------------------------------------------------------- dataset run
def _load_rgb(path) -> np.ndarray:
    from PIL import Image  # host-side image decoding only
    im = Image.open(path)
    if im.mode not in ("RGB", "L", "RGBA"):
        raise ValueError(f"{path}: unsupported image mode {im.mode}")
    return np.array(im.convert("RGB"), dtype=np.uint8)  # writable copy


def run_scene(scene_dir: str, threshold: float = 2.0, k_scale: int = 2, **params) -> EvalReport:
    """One Middlebury scene directory through the GPU path (cuda:0)."""
    import torch

    from . import abi
    L = _load_rgb(os.path.join(scene_dir, "im0.png"))
    R = _load_rgb(os.path.join(scene_dir, "im1.png"))
    gt = read_pfm(os.path.join(scene_dir, "disp0GT.pfm"))
    cal = os.path.join(scene_dir, "calib.txt")
    D = read_calib(cal)["ndisp"] if os.path.exists(cal) else int(np.nanmax(gt[np.isfinite(gt)])) + 1
    H, W = L.shape[:2]
    dev = torch.device("cuda:0")
    st = abi.Stereo(W, H, D, k_scale=k_scale, **params)
    out = torch.empty((H, W), dtype=torch.float32, device=dev)
    st.compute_rgb(torch.from_numpy(L).to(dev), torch.from_numpy(R).to(dev), out)
    torch.cuda.synchronize()
    st.close()
    mask = None
    mp = os.path.join(scene_dir, "mask0nocc.png")
    if os.path.exists(mp):
        from PIL import Image
        mask = np.asarray(Image.open(mp)) == 255  # Middlebury: 255 = non-occluded
    return eval_bad(out.cpu().numpy(), gt, threshold, mask)


def run_dataset(root: str, threshold: float = 2.0, **params) -> dict:
    """Every scene directory under ``root`` with im0.png / im1.png / disp0GT.pfm;
    returns {scene: EvalReport, "average": bad_rate_all mean} (Table I's
    "average error rate")."""
    res = {}
    for name in sorted(os.listdir(root)):
        d = os.path.join(root, name)
        if all(os.path.exists(os.path.join(d, f)) for f in ("im0.png", "im1.png", "disp0GT.pfm")):
            res[name] = run_scene(d, threshold, **params)
    if res:
        res["average"] = float(np.mean([r.bad_rate_all for r in res.values()]))
    return res


def main(argv=None) -> int:
    import argparse
    ap = argparse.ArgumentParser(description="bad-N of the GPU path on a Middlebury-format directory")
    ap.add_argument("root", help="directory of scene folders (im0.png, im1.png, disp0GT.pfm, calib.txt)")
    ap.add_argument("--bad", type=float, default=2.0)
    a = ap.parse_args(argv)
    if not os.path.isdir(a.root):
        print(f"no dataset at {a.root}", file=sys.stderr)
        return 2
    res = run_dataset(a.root, a.bad)
    for k, v in res.items():
        print(k, v)
    return 0


if __name__ == "__main__":
    sys.exit(main())
