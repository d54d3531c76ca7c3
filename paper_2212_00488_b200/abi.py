"""Thin ctypes binding of include/stereo.h (argument marshalling only).

Every function here forwards to the same-named C entry point of
``paper_2212_00488_b200/lib/libstereo_b200.so``; all computation happens in
that library's sm_100a kernels.  There is no CPU fallback: if the library is
missing or cannot be loaded, :func:`lib` raises ``StereoLibraryError``.

Device buffers are passed as raw pointers; :class:`Stereo` accepts torch CUDA
tensors (PyTorch supplies device memory and streams only) and numpy arrays
for the host (end-to-end) path.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("STEREO_B200_LIB", os.path.join(_HERE, "lib", "libstereo_b200.so"))

STEREO_ABI_VERSION = 3
STEREO_OK, STEREO_EINVAL, STEREO_ENOMEM, STEREO_ECUDA, STEREO_EUNSUPPORTED = 0, -1, -2, -3, -4

(BUF_PIX_L, BUF_PIX_R, BUF_ARM_L, BUF_ARM_R, BUF_CAX_L, BUF_CAX_R, BUF_CA_L, BUF_CA_R,
 BUF_DL, BUF_DR, BUF_MASKED, BUF_MEDIAN, BUF_FILL, BUF_ROWS) = range(14)
(STAGE_SD, STAGE_PREP, STAGE_XPASS, STAGE_YPASS, STAGE_POST) = range(5)
STAGE_NAMES = ("SD", "PREP", "XPASS", "YPASS", "POST")
STAGE_COUNT = 5
DEBUG_CA = 1
# non-GCP filling modes (include/stereo.h STEREO_FILL_*, §III.E)
FILL_BILATERAL, FILL_NEAREST, FILL_SMALLER, FILL_EQ11_LITERAL = range(4)
FILL_MODES = {"bilateral": 0, "nearest": 1, "smaller": 2, "eq11_literal": 3}

# every symbol include/stereo.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "stereo_default_params", "stereo_create", "stereo_compute", "stereo_compute_batch",
    "stereo_compute_host", "stereo_destroy", "stereo_last_error", "stereo_get_info",
    "stereo_get_tables", "stereo_debug_download", "stereo_debug_upload", "stereo_set_debug",
    "stereo_run_stage", "stereo_set_timing", "stereo_stage_times_ms",
    "stereo_rgb_to_gray", "stereo_compute_rgb", "stereo_disparity_to_depth",
    "stereo_create_batch", "stereo_band_rows", "stereo_create_band", "stereo_band_halo",
    "stereo_compute_band", "stereo_band_summary", "stereo_band_finish",
    "stereo_compute_host_batch",
)


class StereoLibraryError(RuntimeError):
    pass


class StereoError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"stereo error {code}: {msg}")
        self.code = code


class Params(C.Structure):
    _fields_ = [
        ("abi_version", C.c_uint32), ("lambda_ad", C.c_double), ("lambda_mc", C.c_double),
        ("t_fill", C.c_int32), ("w_x", C.c_int32), ("w_y", C.c_int32), ("delta", C.c_int32),
        ("k_scale", C.c_int32), ("m_pool", C.c_int32),
        ("census_dx", C.c_int8 * 6), ("census_dy", C.c_int8 * 6),
        ("w_x_r", C.c_int32), ("fill_mode", C.c_int32),
    ]


class Info(C.Structure):
    _fields_ = [
        ("W", C.c_int32), ("H", C.c_int32), ("D", C.c_int32),
        ("Ws", C.c_int32), ("Hs", C.c_int32), ("Ds", C.c_int32),
        ("frac_bits", C.c_int32), ("device", C.c_int32),
        ("device_bytes", C.c_uint64), ("cax_bytes", C.c_uint64),
        ("launches_per_frame", C.c_int32), ("ypass_block_rows", C.c_int32),
        ("cax_pitch", C.c_int32),
        ("max_frames", C.c_int32), ("band", C.c_int32),
        ("band_y0_org", C.c_int32), ("band_rows_org", C.c_int32),
        ("band_halo_top_org", C.c_int32), ("band_halo_bot_org", C.c_int32),
        ("ypass_rows", C.c_int32),
    ]


_lib = None
_lock = threading.Lock()


def lib():
    """Load libstereo_b200.so (raises StereoLibraryError if absent: no fallback)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise StereoLibraryError(
                f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                " (or tools/build_lib.sh); there is no CPU fallback")
        try:
            L = C.CDLL(LIB_PATH)
        except OSError as e:
            raise StereoLibraryError(f"cannot load {LIB_PATH}: {e}") from e
        vp, i32 = C.c_void_p, C.c_int
        sig = {
            "stereo_default_params": (None, [C.POINTER(Params)]),
            "stereo_create": (i32, [i32, i32, i32, C.POINTER(Params), C.POINTER(vp)]),
            "stereo_compute": (i32, [vp, vp, vp, vp, vp]),
            "stereo_compute_batch": (i32, [vp, vp, vp, i32, vp, vp]),
            "stereo_compute_host": (i32, [vp, vp, vp, vp, vp]),
            "stereo_compute_host_batch": (i32, [vp, vp, vp, i32, vp, vp]),
            "stereo_destroy": (None, [vp]),
            "stereo_last_error": (C.c_char_p, []),
            "stereo_get_info": (i32, [vp, C.POINTER(Info)]),
            "stereo_get_tables": (i32, [vp, vp, vp, vp]),
            "stereo_debug_download": (i32, [vp, i32, vp, C.c_size_t]),
            "stereo_debug_upload": (i32, [vp, i32, vp, C.c_size_t]),
            "stereo_set_debug": (i32, [vp, i32, i32]),
            "stereo_run_stage": (i32, [vp, i32, vp, vp, vp, vp]),
            "stereo_set_timing": (i32, [vp, i32]),
            "stereo_stage_times_ms": (i32, [vp, vp, C.POINTER(C.c_int)]),
            "stereo_create_batch": (i32, [i32, i32, i32, C.POINTER(Params), i32, C.POINTER(vp)]),
            "stereo_band_rows": (i32, [i32, C.POINTER(Params), i32, i32, C.POINTER(i32),
                                       C.POINTER(i32)]),
            "stereo_create_band": (i32, [i32, i32, i32, C.POINTER(Params), i32, i32, C.POINTER(vp)]),
            "stereo_band_halo": (i32, [i32, C.POINTER(Params), i32, i32, C.POINTER(i32),
                                       C.POINTER(i32)]),
            "stereo_compute_band": (i32, [vp, vp, vp, i32, i32, i32, i32, vp, vp]),
            "stereo_band_summary": (i32, [vp, vp, vp]),
            "stereo_band_finish": (i32, [vp, vp, vp, vp, vp]),
            "stereo_rgb_to_gray": (i32, [vp, vp, i32, i32, vp]),
            "stereo_compute_rgb": (i32, [vp, vp, vp, vp, vp]),
            "stereo_disparity_to_depth": (i32, [vp, vp, i32, C.c_float, vp]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype, fn.argtypes = res, args
        _lib = L
        return L


def _check(rc):
    if rc != STEREO_OK:
        raise StereoError(rc, lib().stereo_last_error().decode(errors="replace"))


def default_params(**overrides) -> Params:
    p = Params()
    lib().stereo_default_params(C.byref(p))
    census = overrides.pop("census", None)
    if isinstance(overrides.get("fill_mode"), str):
        overrides["fill_mode"] = FILL_MODES[overrides["fill_mode"]]
    for k, v in overrides.items():
        setattr(p, k, v)
    if census is not None:
        for i, (dx, dy) in enumerate(census):
            p.census_dx[i], p.census_dy[i] = dx, dy
    return p


def _ptr(t):
    """Raw pointer of a torch tensor / numpy array / int."""
    if t is None:
        return None
    if isinstance(t, int):
        return t
    if isinstance(t, np.ndarray):
        if not t.flags["C_CONTIGUOUS"]:
            raise ValueError("arrays must be C-contiguous")
        return t.ctypes.data
    if not t.is_contiguous():
        raise ValueError("tensors must be contiguous")
    return t.data_ptr()


_DT = {"u8": (np.uint8, "torch.uint8"), "f32": (np.float32, "torch.float32"),
       "i32": (np.int32, "torch.int32")}


def _dev(t, name, dtype, shape, device):
    """A CUDA tensor on the handle's device with the given dtype and shape."""
    if isinstance(t, int):  # raw device pointer: the caller vouches for it
        return t
    if isinstance(t, np.ndarray) or not getattr(t, "is_cuda", False):
        raise ValueError(f"{name} must be a CUDA tensor on cuda:{device}")
    if t.device.index != device:
        raise ValueError(f"{name} is on cuda:{t.device.index}, the handle on cuda:{device}")
    if str(t.dtype) != _DT[dtype][1]:
        raise ValueError(f"{name} must be {_DT[dtype][1]}, got {t.dtype}")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")
    return _ptr(t)


def _host(a, name, dtype, shape):
    """A host buffer (numpy array or CPU tensor) of the given dtype and shape."""
    if isinstance(a, int):
        return a
    if getattr(a, "is_cuda", False):
        raise ValueError(f"{name} must be a HOST buffer")
    ok = (a.dtype == _DT[dtype][0]) if isinstance(a, np.ndarray) else (str(a.dtype) == _DT[dtype][1])
    if not ok:
        raise ValueError(f"{name} must be {dtype}, got {a.dtype}")
    if tuple(a.shape) != tuple(shape):
        raise ValueError(f"{name} must have shape {tuple(shape)}, got {tuple(a.shape)}")
    return _ptr(a)


def _stream_ptr(stream):
    if stream is None:
        try:
            import torch
            return torch.cuda.current_stream().cuda_stream
        except Exception:  # pragma: no cover
            return None
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


class Stereo:
    """Owns one stereo_t handle (device-bound; not re-entrant across streams)."""

    def __init__(self, W: int, H: int, D: int, params: Params | None = None,
                 max_frames: int = 1, **overrides):
        self.params = params if params is not None else default_params(**overrides)
        h = C.c_void_p()
        if max_frames == 1:
            _check(lib().stereo_create(W, H, D, C.byref(self.params), C.byref(h)))
        else:
            _check(lib().stereo_create_batch(W, H, D, C.byref(self.params), max_frames, C.byref(h)))
        self._h = h
        self.info = Info()
        _check(lib().stereo_get_info(self._h, C.byref(self.info)))
        self.W, self.H, self.D = W, H, D
        self.device = self.info.device

    # ------------------------------------------------------------ lifetime
    def close(self):
        if getattr(self, "_h", None):
            lib().stereo_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # ------------------------------------------------------------ compute
    def compute(self, L, R, out, stream=None):
        """L, R: CUDA u8 [H][W]; out: CUDA f32 [H][W]. Enqueued, not synchronised."""
        hw, d = (self.H, self.W), self.device
        _check(lib().stereo_compute(self._h, _dev(L, "L", "u8", hw, d), _dev(R, "R", "u8", hw, d),
                                    _dev(out, "out", "f32", hw, d), _stream_ptr(stream)))
        return out

    def compute_rgb(self, L_rgb, R_rgb, out, stream=None):
        """L_rgb, R_rgb: CUDA u8 [H][W][3]; gray front end (§III item 1) + pipeline."""
        hw3, d = (self.H, self.W, 3), self.device
        _check(lib().stereo_compute_rgb(self._h, _dev(L_rgb, "L_rgb", "u8", hw3, d),
                                        _dev(R_rgb, "R_rgb", "u8", hw3, d),
                                        _dev(out, "out", "f32", (self.H, self.W), d),
                                        _stream_ptr(stream)))
        return out

    def compute_batch(self, L, R, out, nframes, stream=None):
        """L, R: CUDA u8 [n][H][W]; out: CUDA f32 [n][H][W], n = nframes; one
        launch sequence per chunk of max_frames frames."""
        nhw, d = (nframes, self.H, self.W), self.device
        _check(lib().stereo_compute_batch(self._h, _dev(L, "L", "u8", nhw, d), _dev(R, "R", "u8", nhw, d),
                                          nframes, _dev(out, "out", "f32", nhw, d),
                                          _stream_ptr(stream)))
        return out

    def compute_host(self, L, R, out, stream=None):
        """HOST buffers (pinned for async copies); caller synchronises the stream."""
        hw = (self.H, self.W)
        _check(lib().stereo_compute_host(self._h, _host(L, "L", "u8", hw), _host(R, "R", "u8", hw),
                                         _host(out, "out", "f32", hw), _stream_ptr(stream)))
        return out

    def compute_host_batch(self, L, R, out, nframes, stream=None):
        """HOST u8 [n][H][W] x 2 -> HOST f32 [n][H][W]; per chunk of max_frames
        frames one copy in, one launch sequence, one copy out."""
        nhw = (nframes, self.H, self.W)
        _check(lib().stereo_compute_host_batch(self._h, _host(L, "L", "u8", nhw), _host(R, "R", "u8", nhw),
                                               nframes, _host(out, "out", "f32", nhw),
                                               _stream_ptr(stream)))
        return out

    # ------------------------------------------------------------ debug / stages
    def tables(self):
        qad = np.zeros(256, np.uint32)
        qmc = np.zeros(7, np.uint32)
        border = C.c_uint32()
        _check(lib().stereo_get_tables(self._h, qad.ctypes.data, qmc.ctypes.data, C.byref(border)))
        return qad, qmc, border.value

    def _shape(self, buf):
        i = self.info
        n2 = (i.Hs, i.Ws)
        return {
            BUF_PIX_L: (n2, np.uint16), BUF_PIX_R: (n2, np.uint16),
            BUF_ARM_L: (n2, np.uint32), BUF_ARM_R: (n2, np.uint32),
            BUF_CAX_L: (((i.Ds + 1) // 2, i.Hs, i.cax_pitch, 2), np.uint32),
            BUF_CAX_R: (((i.Ds + 1) // 2, i.Hs, i.cax_pitch, 2), np.uint32),
            BUF_CA_L: ((i.Ds, i.Hs, i.Ws), np.uint64), BUF_CA_R: ((i.Ds, i.Hs, i.Ws), np.uint64),
            BUF_DL: (n2, np.uint8), BUF_DR: (n2, np.uint8), BUF_MASKED: (n2, np.uint8),
            BUF_MEDIAN: (n2, np.uint8), BUF_FILL: (n2, np.float32),
            BUF_ROWS: ((4, i.Hs), np.int32),
        }[buf]

    def download(self, buf):
        """Host copy of a stage buffer; CA_x volumes come back as [Ds][Hs][pitch]
        (the device interleaves disparity pairs, see include/stereo.h)."""
        shp, dt = self._shape(buf)
        a = np.zeros(shp, dt)
        _check(lib().stereo_debug_download(self._h, buf, a.ctypes.data, a.nbytes))
        if buf in (BUF_CAX_L, BUF_CAX_R):
            i = self.info
            a = a.transpose(0, 3, 1, 2).reshape(-1, i.Hs, i.cax_pitch)[:i.Ds].copy()
        return a

    def upload(self, buf, arr):
        shp, dt = self._shape(buf)
        if buf in (BUF_CAX_L, BUF_CAX_R):  # [Ds][Hs][pitch] -> disparity pairs interleaved
            i = self.info
            v = np.zeros((shp[0] * 2, i.Hs, i.cax_pitch), dt)
            v[:i.Ds] = np.asarray(arr, dtype=dt).reshape(i.Ds, i.Hs, i.cax_pitch)
            arr = v.reshape(shp[0], 2, i.Hs, i.cax_pitch).transpose(0, 2, 3, 1)
        a = np.ascontiguousarray(arr, dtype=dt).reshape(shp)
        _check(lib().stereo_debug_upload(self._h, buf, a.ctypes.data, a.nbytes))

    def set_debug(self, what, enable=True):
        _check(lib().stereo_set_debug(self._h, what, int(enable)))

    def run_stage(self, stage, L=None, R=None, out=None, stream=None):
        _check(lib().stereo_run_stage(self._h, stage, _ptr(L), _ptr(R), _ptr(out),
                                      _stream_ptr(stream)))

    def set_timing(self, enable=True):
        _check(lib().stereo_set_timing(self._h, int(enable)))

    def stage_times_ms(self):
        ms = np.zeros(STAGE_COUNT, np.float64)
        n = C.c_int()
        _check(lib().stereo_stage_times_ms(self._h, ms.ctypes.data, C.byref(n)))
        return dict(zip(STAGE_NAMES, ms.tolist())), n.value


def band_rows(H, nbands, band, params: Params | None = None, **overrides):
    """The library's band partition: (y0_org, rows_org) of band `band`."""
    p = params if params is not None else default_params(**overrides)
    y0, rows = C.c_int(), C.c_int()
    _check(lib().stereo_band_rows(H, C.byref(p), nbands, band, C.byref(y0), C.byref(rows)))
    return y0.value, rows.value


def band_halo(H, y0_org, rows_org, params: Params | None = None, **overrides):
    """Halo rows (above, below) the band needs (stereo_band_halo; host only)."""
    p = params if params is not None else default_params(**overrides)
    top, bot = C.c_int(), C.c_int()
    _check(lib().stereo_band_halo(H, C.byref(p), y0_org, rows_org, C.byref(top), C.byref(bot)))
    return top.value, bot.value


class StereoBand:
    """A row-band handle (stereo_create_band): own original rows
    [y0_org, y0_org + rows_org) of a W x H frame, computed from the band plus
    the halo rows stereo_band_halo names; see include/stereo.h."""

    def __init__(self, W, H, D, y0_org, rows_org, params: Params | None = None, **overrides):
        self.params = params if params is not None else default_params(**overrides)
        h = C.c_void_p()
        _check(lib().stereo_create_band(W, H, D, C.byref(self.params), y0_org, rows_org,
                                        C.byref(h)))
        self._h = h
        self.info = Info()
        _check(lib().stereo_get_info(self._h, C.byref(self.info)))
        self.W, self.H, self.D = W, H, D
        self.y0, self.rows = y0_org, rows_org
        self.top, self.bot = self.info.band_halo_top_org, self.info.band_halo_bot_org
        self.sub_rows = self.top + self.rows + self.bot  # rows of L_band / R_band
        self.sub_y0 = y0_org - self.top                   # frame row of L_band[0]
        self.Hs = H // self.params.k_scale
        self.device = self.info.device

    def compute(self, L_band, R_band, out_band, stream=None):
        """L_band, R_band: CUDA u8 [sub_rows][W]; out_band: CUDA f32 [rows][W]."""
        d, sh = self.device, (self.sub_rows, self.W)
        _check(lib().stereo_compute_band(self._h, _dev(L_band, "L_band", "u8", sh, d),
                                         _dev(R_band, "R_band", "u8", sh, d), self.y0, self.rows,
                                         self.top, self.bot,
                                         _dev(out_band, "out_band", "f32", (self.rows, self.W), d),
                                         _stream_ptr(stream)))
        return out_band

    def summary(self, summ, stream=None):
        """summ: CUDA int32 [H/K][2] (frame-wide; own rows written, -1 elsewhere)."""
        _check(lib().stereo_band_summary(self._h, _dev(summ, "summ", "i32", (self.Hs, 2), self.device),
                                         _stream_ptr(stream)))
        return summ

    def finish(self, summ, L_band, out_band, stream=None):
        """Fill rule (d) from the frame-wide summaries (all bands assembled)."""
        d = self.device
        _check(lib().stereo_band_finish(self._h, _dev(summ, "summ", "i32", (self.Hs, 2), d),
                                        _dev(L_band, "L_band", "u8", (self.sub_rows, self.W), d),
                                        _dev(out_band, "out_band", "f32", (self.rows, self.W), d),
                                        _stream_ptr(stream)))
        return out_band

    def close(self):
        if getattr(self, "_h", None):
            lib().stereo_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def unpack_pix(pix):
    """u16 I | census << 8 -> (image u8, census u8)."""
    return (pix & 255).astype(np.uint8), (pix >> 8).astype(np.uint8)


def unpack_arms(arm):
    """u32 m | n<<8 | M<<16 | N<<24 -> u8 [4][H][W] (m, n, M, N)."""
    return np.stack([(arm >> s) & 255 for s in (0, 8, 16, 24)]).astype(np.uint8)


def rgb_to_gray(rgb, gray, stream=None):
    """CUDA u8 [H][W][3] -> CUDA u8 [H][W] (BT.601, §III item 1), enqueued."""
    H, W = int(rgb.shape[0]), int(rgb.shape[1])
    _check(lib().stereo_rgb_to_gray(_ptr(rgb), _ptr(gray), W, H, _stream_ptr(stream)))
    return gray


def disparity_to_depth(disp, Z, fB, stream=None):
    """Eq. 1: CUDA f32 disparities -> CUDA f32 depth Z = fB / d (d <= 0 -> inf)."""
    _check(lib().stereo_disparity_to_depth(_ptr(disp), _ptr(Z), int(disp.numel()), float(fB),
                                           _stream_ptr(stream)))
    return Z
