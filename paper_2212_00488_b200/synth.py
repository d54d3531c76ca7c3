"""Seeded synthetic stereo inputs (SURVEY.md §8(d) "Synthetic inputs").

This module is the ONE piece shared by the CUDA path's tests/bench and the CPU
oracle's tests.  It contains none of the method's arithmetic (no cost, no
aggregation, no matching): only random textures and a forward warp that renders
a right view from a left view and a ground-truth disparity field.

Recipe (restated in DESIGN.md §3):

* ``patchy(W, H, rng)`` — Middlebury-like texture: background 128, about
  W*H/60 axis-aligned rectangles (sides 2..13 px, intensity U[0,255]), then
  U[-4,4] integer noise, clipped to u8.  Flat runs (long cross arms) plus
  edges (short arms), as in the paper's half-size Middlebury scenes.
* ``shift_pair(W, H, s, seed)`` — texture T of width W+s; L = T[:, 0:W],
  R = T[:, s:s+W], hence R(x - s, y) = T(x, y) = L(x, y): every left pixel at x >= s has
  true disparity s ("L(x,y) is compared with R(x-d,y)").
* ``scene(W, H, D, seed)`` — slanted background plane with d in [0.1D, 0.4D],
  4..8 fronto-parallel elliptic blobs with d in [0.4D, 0.95D]; R is rendered
  by forward-warping L with a z-buffer (larger d wins), disocclusions get fresh
  texture; independent U[-2,2] noise per view.  Gives occlusions (non-GCPs,
  P:111-121).
* ``stream(W, H, D, n, seed)`` — n frames of one scene whose content
  translates by 1..3 px per frame (config c4).
"""
from __future__ import annotations

import numpy as np

__all__ = ["patchy", "shift_pair", "scene", "stream", "random_pair", "CONFIGS"]

# BASELINE.json "configs" (c1..c5): (W, H, D, K)
CONFIGS = {
    "c1": dict(W=64, H=48, D=16, K=1, kind="shift", s=5),
    "c2": dict(W=450, H=375, D=64, K=1, kind="scene"),
    "c3": dict(W=1436, H=992, D=145, K=2, kind="scene"),
    "c4": dict(W=1436, H=992, D=145, K=2, kind="stream", frames=256),
    "c5": dict(W=2872, H=1984, D=290, K=2, kind="scene"),
}


def patchy(W: int, H: int, rng: np.random.Generator, noise: int = 4) -> np.ndarray:
    """Background 128 + ~W*H/60 random rectangles + U[-noise, noise]; u8 [H][W]."""
    img = np.full((H, W), 128, dtype=np.int32)
    n = max(1, (W * H) // 60)
    xs = rng.integers(0, W, n)
    ys = rng.integers(0, H, n)
    ws = rng.integers(2, 14, n)
    hs = rng.integers(2, 14, n)
    vs = rng.integers(0, 256, n)
    for x, y, w, h, v in zip(xs, ys, ws, hs, vs):
        img[y:y + h, x:x + w] = v
    if noise:
        img += rng.integers(-noise, noise + 1, (H, W))
    return np.clip(img, 0, 255).astype(np.uint8)


def shift_pair(W: int, H: int, s: int, seed: int = 0):
    """(L, R) with L(x, y) = R(x - s, y); u8 [H][W] each."""
    rng = np.random.default_rng(seed)
    T = patchy(W + s, H, rng)
    L = np.ascontiguousarray(T[:, 0:W])
    R = np.ascontiguousarray(T[:, s:s + W])
    return L, R


def _disparity_field(W, H, D, rng):
    yy, xx = np.mgrid[0:H, 0:W].astype(np.float64)
    lo, hi = 0.1 * D, 0.4 * D
    a, b = rng.uniform(-1, 1, 2)
    plane = (a * xx / max(W - 1, 1) + b * yy / max(H - 1, 1))
    plane = (plane - plane.min()) / max(plane.max() - plane.min(), 1e-9)
    d = lo + (hi - lo) * plane
    for _ in range(int(rng.integers(4, 9))):
        cx, cy = rng.uniform(0, W), rng.uniform(0, H)
        rx, ry = rng.uniform(0.04, 0.15) * W, rng.uniform(0.04, 0.15) * H
        dv = rng.uniform(0.4 * D, 0.95 * D)
        m = ((xx - cx) / rx) ** 2 + ((yy - cy) / ry) ** 2 <= 1.0
        d[m] = dv
    return d


def _render(T, dgt, fresh, rng, view_noise):
    """Forward-warp base texture T (the left view) to the right view."""
    H, W = T.shape
    di = np.rint(dgt).astype(np.int64)
    xr = np.arange(W)[None, :] - di
    yy = np.broadcast_to(np.arange(H)[:, None], (H, W))
    ok = xr >= 0
    zbuf = np.full((H, W), -1, dtype=np.int64)
    np.maximum.at(zbuf, (yy[ok], xr[ok]), di[ok])
    R = fresh.astype(np.int32).copy()
    win = ok.copy()
    win[ok] = di[ok] == zbuf[yy[ok], xr[ok]]
    R[yy[win], xr[win]] = T[win]
    Ln = T.astype(np.int32)
    if view_noise:
        Ln = Ln + rng.integers(-view_noise, view_noise + 1, (H, W))
        R = R + rng.integers(-view_noise, view_noise + 1, (H, W))
    return (np.clip(Ln, 0, 255).astype(np.uint8), np.clip(R, 0, 255).astype(np.uint8))


def scene(W: int, H: int, D: int, seed: int = 0, view_noise: int = 2):
    """(L, R, dgt): Middlebury-shaped synthetic scene; dgt is float64 [H][W]."""
    rng = np.random.default_rng(seed)
    T = patchy(W, H, rng, noise=0)
    fresh = patchy(W, H, rng, noise=0)
    dgt = _disparity_field(W, H, D, rng)
    L, R = _render(T, dgt, fresh, rng, view_noise)
    return L, R, dgt


def stream(W: int, H: int, D: int, n: int, seed: int = 0, view_noise: int = 2, idx=None):
    """n frames (L, R) of one scene translating 1..3 px/frame; list of tuples.

    idx: the frame indices to render (default: all n).  Every frame draws its
    own noise from a generator keyed by (seed, frame), so a rank renders just
    its slice of the stream (config c4, dist.stream_slice) and gets the same
    frames as a whole-stream render."""
    rng = np.random.default_rng(seed)
    T = patchy(W, H, rng, noise=0)
    fresh = patchy(W, H, rng, noise=0)
    dgt = _disparity_field(W, H, D, rng)
    offs = np.concatenate([[0], np.cumsum(rng.integers(1, 4, max(n - 1, 0)))]).astype(int)
    frames = []
    for i in (range(n) if idx is None else idx):
        off = int(offs[i])
        Ts = np.roll(T, off, axis=1)
        ds = np.roll(dgt, off, axis=1)
        frames.append(_render(Ts, ds, fresh, np.random.default_rng([seed, 7, i]), view_noise))
    return frames


def random_pair(W: int, H: int, seed: int = 0, levels: int = 256):
    """Unstructured (L, R) u8 noise pair; for parity tests of arbitrary inputs."""
    rng = np.random.default_rng(seed)
    L = rng.integers(0, levels, (H, W)).astype(np.uint8)
    R = rng.integers(0, levels, (H, W)).astype(np.uint8)
    if levels < 256:
        L = (L * (255 // max(levels - 1, 1))).astype(np.uint8)
        R = (R * (255 // max(levels - 1, 1))).astype(np.uint8)
    return L, R
