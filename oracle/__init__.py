"""CPU oracle of the stereo hot path (ctypes front-end of stereo_oracle.c).

TEST INFRASTRUCTURE ONLY.  Only tests/, ``__graft_entry__.smoke()`` and
bench.py's ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  It shares no code with ``paper_2212_00488_b200`` (the CUDA path);
the only common module is the seeded input generator
``paper_2212_00488_b200.synth``, which holds none of the method's arithmetic.

Every function here is a thin numpy wrapper; the arithmetic is the literal C
in ``stereo_oracle.c`` (each function there cites its PAPER.md passage).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "stereo_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

INVALID = 255
MODES = {"fixed": 0, "double": 1}


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (strict IEEE: no fast-math, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "stereo_oracle.h"))
    ):
        tmp = _LIB + f".tmp{os.getpid()}"
        cmd = ["gcc", "-O2", "-std=c11", "-fno-fast-math", "-ffp-contract=off", "-fopenmp",
               "-fPIC", "-shared", "-Wall", "-o", tmp, _SRC, "-lm"]
        subprocess.run(cmd, check=True)
        os.replace(tmp, _LIB)
    return _LIB


class Params(C.Structure):
    _fields_ = [
        ("lambda_ad", C.c_double), ("lambda_mc", C.c_double), ("t_fill", C.c_int32),
        ("w_x", C.c_int32), ("w_y", C.c_int32), ("delta", C.c_int32),
        ("k_scale", C.c_int32), ("m_pool", C.c_int32),
        ("census_dx", C.c_int32 * 6), ("census_dy", C.c_int32 * 6),
        ("w_x_r", C.c_int32), ("fill_mode", C.c_int32),
    ]


# §III.E non-GCP filling modes (oracle/stereo_oracle.h OR_FILL_*)
FILL_MODES = {"bilateral": 0, "nearest": 1, "smaller": 2, "eq11_literal": 3}


# S:92 default pattern (reading R8): (0,-2)(-1,-1)(+1,-1)(-1,+1)(+1,+1)(0,+2)
DEFAULT_CENSUS = ((0, -2), (-1, -1), (1, -1), (-1, 1), (1, 1), (0, 2))


def params(lambda_ad=0.3, lambda_mc=2.3, t_fill=3, w_x=21, w_y=31, delta=20, k_scale=2,
           m_pool=1, census=DEFAULT_CENSUS, w_x_r=-1, fill_mode=0) -> Params:
    """P:609 (lambda_AD, lambda_MC, T), P:621-622 (W_x, W_y), S:90 (delta), P:155 (K);
    w_x_r: right-base x cap (-1 = w_x); fill_mode: FILL_MODES value or name."""
    p = Params()
    p.lambda_ad, p.lambda_mc, p.t_fill = lambda_ad, lambda_mc, t_fill
    p.w_x, p.w_y, p.delta, p.k_scale, p.m_pool = w_x, w_y, delta, k_scale, m_pool
    p.w_x_r = w_x_r
    p.fill_mode = FILL_MODES[fill_mode] if isinstance(fill_mode, str) else fill_mode
    for i, (dx, dy) in enumerate(census):
        p.census_dx[i], p.census_dy[i] = dx, dy
    return p


class _Outputs(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in (
        "Ls", "Rs", "cenL", "cenR", "armL", "armR", "caxL", "caxR", "caL", "caR",
        "caxL_d", "caxR_d", "caL_d", "caR_d", "DL", "DR", "masked", "median", "fill", "out")]


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = C.CDLL(_LIB)
            u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
            u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
            u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
            f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
            f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
            i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
            sig = {
                "or_scaled_max_disparity": (C.c_int, [C.c_int, C.c_int]),
                "or_fixed_bits": (C.c_int, [C.c_int]),
                "or_cost_ad": (C.c_double, [C.c_int, C.c_double]),
                "or_cost_mc": (C.c_double, [C.c_int, C.c_double]),
                "or_fixed_tables": (None, [C.c_double, C.c_double, C.c_int, u32p, u32p]),
                "or_hamming6": (C.c_int, [C.c_int, C.c_int]),
                "or_downscale": (None, [u8p, C.c_int, C.c_int, C.c_int, C.c_int, u8p]),
                "or_census": (None, [u8p, C.c_int, C.c_int, i32p, i32p, u8p]),
                "or_arms_x": (None, [u8p, C.c_int, C.c_int, C.c_int, C.c_int, u8p, u8p]),
                "or_arms_y": (None, [u8p, C.c_int, C.c_int, C.c_int, C.c_int, u8p, u8p]),
                "or_cost_left_double": (None, [u8p, u8p, u8p, u8p, C.c_int, C.c_int, C.c_int,
                                               C.c_double, C.c_double, f64p]),
                "or_cost_right_double": (None, [u8p, u8p, u8p, u8p, C.c_int, C.c_int, C.c_int,
                                                C.c_double, C.c_double, f64p]),
                "or_cost_left_fixed": (None, [u8p, u8p, u8p, u8p, C.c_int, C.c_int, C.c_int,
                                              u32p, u32p, C.c_uint32, u32p]),
                "or_cost_right_fixed": (None, [u8p, u8p, u8p, u8p, C.c_int, C.c_int, C.c_int,
                                               u32p, u32p, C.c_uint32, u32p]),
                "or_aggregate_x_double": (None, [f64p, u8p, u8p, C.c_int, C.c_int, f64p]),
                "or_aggregate_y_double": (None, [f64p, u8p, u8p, C.c_int, C.c_int, f64p]),
                "or_aggregate_x_u64": (None, [u64p, u8p, u8p, C.c_int, C.c_int, u64p]),
                "or_aggregate_y_u64": (None, [u64p, u8p, u8p, C.c_int, C.c_int, u64p]),
                "or_wta_double": (None, [f64p, C.c_int, C.c_int, C.c_int, u8p]),
                "or_wta_u64": (None, [u64p, C.c_int, C.c_int, C.c_int, u8p]),
                "or_cross_check": (None, [u8p, u8p, C.c_int, C.c_int, u8p]),
                "or_median3x3": (None, [u8p, C.c_int, C.c_int, u8p]),
                "or_fill_bilateral": (None, [u8p, u8p, C.c_int, C.c_int, C.c_int, C.c_int, f32p]),
                "or_rgb_to_gray": (None, [u8p, C.c_int, C.c_int, u8p]),
                "or_depth": (None, [f32p, C.c_int, C.c_float, f32p]),
                "or_scale_up": (None, [f32p, C.c_int, C.c_int, u8p, C.c_int, C.c_int, C.c_int,
                                       C.c_int, f32p]),
                "or_pipeline": (C.c_int, [u8p, u8p, C.c_int, C.c_int, C.c_int, C.POINTER(Params),
                                          C.c_int, C.c_int, C.POINTER(_Outputs)]),
            }
            for name, (res, args) in sig.items():
                fn = getattr(L, name)
                fn.restype, fn.argtypes = res, args
            _lib = L
    return _lib


def _u8(a):
    return np.ascontiguousarray(a, dtype=np.uint8)


# ---------------------------------------------------------------- stage wrappers
def scaled_max_disparity(D, K):
    return lib().or_scaled_max_disparity(D, K)


def fixed_bits(w_x):
    return lib().or_fixed_bits(w_x)


def cost_ad(a, lambda_ad=0.3):
    return lib().or_cost_ad(int(a), lambda_ad)


def cost_mc(h, lambda_mc=2.3):
    return lib().or_cost_mc(int(h), lambda_mc)


def hamming6(a, b):
    return lib().or_hamming6(int(a), int(b))


def fixed_tables(lambda_ad=0.3, lambda_mc=2.3, f=25):
    qad = np.zeros(256, np.uint32)
    qmc = np.zeros(7, np.uint32)
    lib().or_fixed_tables(lambda_ad, lambda_mc, f, qad, qmc)
    return qad, qmc


def downscale(img, K=2, m=1):
    img = _u8(img)
    H, W = img.shape
    out = np.zeros((H // K, W // K), np.uint8)
    lib().or_downscale(img, W, H, K, m, out)
    return out


def census(img, pattern=DEFAULT_CENSUS):
    img = _u8(img)
    H, W = img.shape
    dx = np.array([p[0] for p in pattern], np.int32)
    dy = np.array([p[1] for p in pattern], np.int32)
    out = np.zeros_like(img)
    lib().or_census(img, W, H, dx, dy, out)
    return out


def arms_x(img, delta=20, w=21):
    img = _u8(img)
    H, W = img.shape
    m, n = np.zeros_like(img), np.zeros_like(img)
    lib().or_arms_x(img, W, H, delta, w, m, n)
    return m, n


def arms_y(img, delta=20, w=31):
    img = _u8(img)
    H, W = img.shape
    m, n = np.zeros_like(img), np.zeros_like(img)
    lib().or_arms_y(img, W, H, delta, w, m, n)
    return m, n


def cost_slice(L, R, cL, cR, d, base="left", mode="double", lambda_ad=0.3, lambda_mc=2.3,
               tables=None, border=None):
    L, R, cL, cR = map(_u8, (L, R, cL, cR))
    H, W = L.shape
    if mode == "double":
        out = np.zeros((H, W), np.float64)
        fn = lib().or_cost_left_double if base == "left" else lib().or_cost_right_double
        fn(L, R, cL, cR, W, H, d, lambda_ad, lambda_mc, out)
    else:
        qad, qmc = tables
        out = np.zeros((H, W), np.uint32)
        fn = lib().or_cost_left_fixed if base == "left" else lib().or_cost_right_fixed
        fn(L, R, cL, cR, W, H, d, qad, qmc, border, out)
    return out


def aggregate_x(Cs, minus, plus):
    H, W = Cs.shape
    if Cs.dtype == np.float64:
        out = np.zeros_like(Cs)
        lib().or_aggregate_x_double(np.ascontiguousarray(Cs), _u8(minus), _u8(plus), W, H, out)
    else:
        Cs = np.ascontiguousarray(Cs, dtype=np.uint64)
        out = np.zeros_like(Cs)
        lib().or_aggregate_x_u64(Cs, _u8(minus), _u8(plus), W, H, out)
    return out


def aggregate_y(Cs, minus, plus):
    H, W = Cs.shape
    if Cs.dtype == np.float64:
        out = np.zeros_like(Cs)
        lib().or_aggregate_y_double(np.ascontiguousarray(Cs), _u8(minus), _u8(plus), W, H, out)
    else:
        Cs = np.ascontiguousarray(Cs, dtype=np.uint64)
        out = np.zeros_like(Cs)
        lib().or_aggregate_y_u64(Cs, _u8(minus), _u8(plus), W, H, out)
    return out


def wta(vol):
    D, H, W = vol.shape
    out = np.zeros((H, W), np.uint8)
    if vol.dtype == np.float64:
        lib().or_wta_double(np.ascontiguousarray(vol), W, H, D, out)
    else:
        lib().or_wta_u64(np.ascontiguousarray(vol, dtype=np.uint64), W, H, D, out)
    return out


def cross_check(DL, DR):
    DL, DR = _u8(DL), _u8(DR)
    H, W = DL.shape
    out = np.zeros_like(DL)
    lib().or_cross_check(DL, DR, W, H, out)
    return out


def median3x3(m):
    m = _u8(m)
    H, W = m.shape
    out = np.zeros_like(m)
    lib().or_median3x3(m, W, H, out)
    return out


def fill_bilateral(med, Limg, T=3, mode=0):
    med, Limg = _u8(med), _u8(Limg)
    H, W = med.shape
    out = np.zeros((H, W), np.float32)
    mode = FILL_MODES[mode] if isinstance(mode, str) else mode
    lib().or_fill_bilateral(med, Limg, W, H, T, mode, out)
    return out


def depth(disp, fB):
    """Eq. 1: Z = fl32(fB / d), d = 0 -> +inf."""
    disp = np.ascontiguousarray(disp, dtype=np.float32)
    out = np.zeros_like(disp)
    lib().or_depth(disp.reshape(-1), disp.size, fB, out.reshape(-1))
    return out


def rgb_to_gray(rgb):
    """§III item 1, BT.601 reading: rgb u8 [H][W][3] -> u8 [H][W]."""
    rgb = _u8(rgb)
    H, W, _ = rgb.shape
    out = np.zeros((H, W), np.uint8)
    lib().or_rgb_to_gray(rgb, W, H, out)
    return out


def scale_up(v, Lorg, K=2, T=3):
    v = np.ascontiguousarray(v, dtype=np.float32)
    Lorg = _u8(Lorg)
    Hs, Ws = v.shape
    H, W = Lorg.shape
    out = np.zeros((H, W), np.float32)
    lib().or_scale_up(v, Ws, Hs, Lorg, W, H, K, T, out)
    return out


STAGES = ("Ls", "Rs", "cenL", "cenR", "armL", "armR", "caxL", "caxR", "caL", "caR",
          "caxL_d", "caxR_d", "caL_d", "caR_d", "DL", "DR", "masked", "median", "fill", "out")


def pipeline(L, R, D, p: Params | None = None, mode="fixed", nthreads=0, stages=("out",)):
    """Run the whole oracle; returns {stage: ndarray} for the requested stages.

    Volumes (caxL/caxR/caL/caR and the _d variants) are [Ds][Hs][Ws] and are
    only produced in the matching mode; request them only for small inputs.
    """
    L, R = _u8(L), _u8(R)
    H, W = L.shape
    p = p or params()
    K = p.k_scale
    Ws, Hs, Ds = W // K, H // K, scaled_max_disparity(D, K)
    shapes = {
        "Ls": ((Hs, Ws), np.uint8), "Rs": ((Hs, Ws), np.uint8),
        "cenL": ((Hs, Ws), np.uint8), "cenR": ((Hs, Ws), np.uint8),
        "armL": ((4, Hs, Ws), np.uint8), "armR": ((4, Hs, Ws), np.uint8),
        "caxL": ((Ds, Hs, Ws), np.uint32), "caxR": ((Ds, Hs, Ws), np.uint32),
        "caL": ((Ds, Hs, Ws), np.uint64), "caR": ((Ds, Hs, Ws), np.uint64),
        "caxL_d": ((Ds, Hs, Ws), np.float64), "caxR_d": ((Ds, Hs, Ws), np.float64),
        "caL_d": ((Ds, Hs, Ws), np.float64), "caR_d": ((Ds, Hs, Ws), np.float64),
        "DL": ((Hs, Ws), np.uint8), "DR": ((Hs, Ws), np.uint8),
        "masked": ((Hs, Ws), np.uint8), "median": ((Hs, Ws), np.uint8),
        "fill": ((Hs, Ws), np.float32), "out": ((H, W), np.float32),
    }
    res, outs = {}, _Outputs()
    for s in stages:
        shp, dt = shapes[s]
        res[s] = np.zeros(shp, dt)
        setattr(outs, s, res[s].ctypes.data)
    rc = lib().or_pipeline(L, R, W, H, D, C.byref(p), MODES[mode], nthreads, C.byref(outs))
    if rc != 0:
        raise ValueError("oracle: invalid parameters")
    return res
