"""Pure-Python brute-force second implementation, for TINY inputs only.

TEST INFRASTRUCTURE ONLY.  Used by tests/test_oracle_brute.py to pin the C
oracle against a formulation that is different where it matters:

* aggregation enumerates the 2-D cross support region instead of the
  separable x-then-y loops of Steps 3/5;
* the median uses ``sorted`` (BASELINE.json north_star: "a sort-based median");
* WTA is an exhaustive ``min`` over (cost, d) tuples;
* rounding uses exact ``fractions.Fraction`` arithmetic;
* the fill searches the set of valid columns instead of scanning.

Inputs are nested lists / numpy arrays of ints; outputs are Python lists.
"""
from __future__ import annotations

import math
from fractions import Fraction

import numpy as np

INVALID = 255


def clamp(v, lo, hi):
    return max(lo, min(hi, v))


def downscale(img, K, m):
    """Eq. 2: round-half-up of the exact block mean, border clamped."""
    H, W = len(img), len(img[0])
    if K == 1:
        return [list(r) for r in img]
    out = []
    for y in range(H // K):
        row = []
        for x in range(W // K):
            vals = [img[clamp(K * y + j, 0, H - 1)][clamp(K * x + i, 0, W - 1)]
                    for j in range(-m, m + 1) for i in range(-m, m + 1)]
            row.append(math.floor(Fraction(sum(vals), len(vals)) + Fraction(1, 2)))
        out.append(row)
    return out


def census(img, pattern):
    H, W = len(img), len(img[0])
    return [[sum(1 << i for i, (dx, dy) in enumerate(pattern)
                 if img[clamp(y + dy, 0, H - 1)][clamp(x + dx, 0, W - 1)] < img[y][x])
             for x in range(W)] for y in range(H)]


def _run(seq, c, delta, cap):
    n = 0
    for v in seq[:cap]:
        if abs(v - c) >= delta:
            break
        n += 1
    return n


def arms(img, delta, wx, wy):
    """Returns (m, n, M, N) grids: runs of |I - I(c)| < delta, capped."""
    H, W = len(img), len(img[0])
    m = [[_run(img[y][:x][::-1], img[y][x], delta, wx) for x in range(W)] for y in range(H)]
    n = [[_run(img[y][x + 1:], img[y][x], delta, wx) for x in range(W)] for y in range(H)]
    col = lambda x: [img[y][x] for y in range(H)]
    M = [[_run(col(x)[:y][::-1], img[y][x], delta, wy) for x in range(W)] for y in range(H)]
    N = [[_run(col(x)[y + 1:], img[y][x], delta, wy) for x in range(W)] for y in range(H)]
    return m, n, M, N


def costs_double(L, R, cL, cR, d, lad, lmc, base):
    """Eqs. 3-6 with math.exp; BORDER 2.0."""
    H, W = len(L), len(L[0])
    out = [[2.0] * W for _ in range(H)]
    for y in range(H):
        for x in range(W):
            if base == "left" and x - d >= 0:
                a, b, ca, cb = L[y][x], R[y][x - d], cL[y][x], cR[y][x - d]
            elif base == "right" and x + d < W:
                a, b, ca, cb = R[y][x], L[y][x + d], cR[y][x], cL[y][x + d]
            else:
                continue
            h = bin(ca ^ cb).count("1")
            out[y][x] = (1 - math.exp(-(abs(a - b) / 255) / lad)) + (1 - math.exp(-h / lmc))
    return out


def aggregate_cross(Cs, m, n, M, N):
    """Sum over the 2-D cross region {(x+dx, y+dy): -M<=dy<=N, -m(x,y+dy)<=dx<=n(x,y+dy)}
    -- Eq. 7 then Eq. 8, with the x arms of each row of the vertical segment.
    Exact rational sum (Fractions) so the order of summation cannot matter."""
    H, W = len(Cs), len(Cs[0])
    out = [[None] * W for _ in range(H)]
    for y in range(H):
        for x in range(W):
            s = Fraction(0)
            for yy in range(y - M[y][x], y + N[y][x] + 1):
                for xx in range(x - m[yy][x], x + n[yy][x] + 1):
                    s += Fraction(Cs[yy][xx])
            out[y][x] = s
    return out


def wta(vols):
    """vols[d][y][x] -> argmin with the smallest d on ties."""
    D, H, W = len(vols), len(vols[0]), len(vols[0][0])
    return [[min((vols[d][y][x], d) for d in range(D))[1] for x in range(W)] for y in range(H)]


def cross_check(DL, DR):
    H, W = len(DL), len(DL[0])
    return [[DL[y][x] if (x - DL[y][x] >= 0 and DR[y][x - DL[y][x]] == DL[y][x]) else INVALID
             for x in range(W)] for y in range(H)]


def median3x3(mm):
    H, W = len(mm), len(mm[0])
    out = [[INVALID] * W for _ in range(H)]
    for y in range(H):
        for x in range(W):
            if mm[y][x] == INVALID:
                continue
            vals = sorted(v for v in (mm[clamp(y + j, 0, H - 1)][clamp(x + i, 0, W - 1)]
                                      for j in (-1, 0, 1) for i in (-1, 0, 1)) if v != INVALID)
            out[y][x] = vals[(len(vals) - 1) // 2]
    return out


def fill(med, Limg, T, mode="bilateral"):
    """§III.E: mode 'bilateral' (Eq. 11 read as interpolation),
    'nearest' / 'smaller' (Fig. 6 (a)/(b)), 'eq11_literal' (P:292
    as printed)."""
    H, W = len(med), len(med[0])
    out = [[0.0] * W for _ in range(H)]
    valid_rows = [[x for x in range(W) if med[y][x] != INVALID] for y in range(H)]
    for y in range(H):
        cols = valid_rows[y]
        if not cols:
            above = [yy for yy in range(y) if valid_rows[yy]]
            below = [yy for yy in range(y + 1, H) if valid_rows[yy]]
            if above:
                v = med[above[-1]][valid_rows[above[-1]][-1]]
            elif below:
                v = med[below[0]][valid_rows[below[0]][0]]
            else:
                v = 0
            out[y] = [float(v)] * W
            continue
        for x in range(W):
            if med[y][x] != INVALID:
                out[y][x] = float(med[y][x])
                continue
            left = [c for c in cols if c < x]
            right = [c for c in cols if c > x]
            if left and right:
                i, j = x - left[-1], right[0] - x
                Dl, Dr = med[y][left[-1]], med[y][right[0]]
                if mode == "nearest":
                    out[y][x] = float(Dl if i <= j else Dr)   # equal distance -> left
                elif mode == "smaller":
                    out[y][x] = float(min(Dl, Dr))
                elif abs(Dl - Dr) <= T:
                    if mode == "eq11_literal":  # D_l + i*(D_l - D_r)/(i+j), rounded once
                        v = Fraction(Dl) + i * Fraction(Dl - Dr, i + j)
                    else:                       # D_l + i*(D_r - D_l)/(i+j), rounded once
                        v = Fraction(Dl) + i * Fraction(Dr - Dl, i + j)
                    out[y][x] = _f32_of_fraction(v)
                else:
                    c = Limg[y][x]
                    out[y][x] = float(Dl if abs(Limg[y][x - i] - c) <= abs(Limg[y][x + j] - c) else Dr)
            else:
                out[y][x] = float(med[y][left[-1]] if left else med[y][right[0]])
    return out


def _f32_of_fraction(v: Fraction) -> float:
    """Round an exact rational once to binary32 (via the correctly-rounded
    double: |numerator| < 2^24, denominator < 2^12, so no double rounding)."""
    return float(np.float32(v.numerator / v.denominator))


def rgb_to_gray(rgb):
    """BT.601 luma rounded half up (reading R31), via exact rationals."""
    out = []
    for row in rgb:
        o = []
        for r, g, b in row:
            v = Fraction(299, 1000) * r + Fraction(587, 1000) * g + Fraction(114, 1000) * b
            o.append(math.floor(v + Fraction(1, 2)))
        out.append(o)
    return out


def scale_up(v, Lorg, K, T):
    """Step8 per output pixel, binary32 via numpy.float32."""
    f32 = np.float32
    Hs, Ws = len(v), len(v[0])
    H, W = len(Lorg), len(Lorg[0])
    if K == 1:
        return [[float(a) for a in r] for r in v]

    def xrow(y):
        Y = 2 * y
        r = [None] * W
        for X in range(W):
            if X % 2 == 0 and X // 2 < Ws:
                r[X] = f32(2) * f32(v[y][X // 2])
        for X in range(1, W, 2):
            a = r[X - 1]
            if X + 1 < W and (X + 1) // 2 < Ws:
                b = f32(2) * f32(v[y][(X + 1) // 2])
                if abs(f32(a - b)) <= f32(K * T):
                    r[X] = f32(f32(a + b) * f32(0.5))
                else:
                    c = Lorg[Y][X]
                    r[X] = a if abs(Lorg[Y][X - 1] - c) <= abs(Lorg[Y][X + 1] - c) else b
            else:
                r[X] = a
        for X in range(W):
            if r[X] is None:
                r[X] = r[X - 1]
        return r

    rows = {y: xrow(y) for y in range(Hs)}
    out = [None] * H
    for Y in range(H):
        if Y % 2 == 0 and Y // 2 < Hs:
            out[Y] = rows[Y // 2]
        elif Y % 2 == 1 and Y + 1 < H and (Y + 1) // 2 < Hs:
            up, dn = rows[(Y - 1) // 2], rows[(Y + 1) // 2]
            out[Y] = [f32(f32(a + b) * f32(0.5)) for a, b in zip(up, dn)]
        else:
            out[Y] = out[Y - 1]
    return [[float(a) for a in r] for r in out]
