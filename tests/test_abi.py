"""Host-only checks of the C ABI boundary (no GPU needed): the library loads,
exports every symbol include/stereo.h declares, and validates parameters in
the SPEC's order before touching any device."""
import ctypes as C
import os
import re
import subprocess

import pytest

from paper_2212_00488_b200 import abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "stereo.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(stereo_[a-z_]+)\s*\(", src)))


def test_library_loads_and_exports_every_declared_symbol():
    L = abi.lib()
    declared = _declared()
    assert declared, "no declarations parsed"
    assert set(declared) == set(abi.EXPORTS)
    for name in declared:
        assert hasattr(L, name), name
    nm = subprocess.run(["nm", "-D", "--defined-only", abi.LIB_PATH], capture_output=True,
                        text=True).stdout
    for name in declared:
        assert re.search(rf"\bT {name}\b", nm), f"{name} not exported with C linkage"


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", abi.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_default_params_are_the_papers():
    p = abi.default_params()
    assert p.abi_version == abi.STEREO_ABI_VERSION
    assert (p.lambda_ad, p.lambda_mc, p.t_fill) == (0.3, 2.3, 3)
    assert (p.w_x, p.w_y, p.k_scale, p.m_pool) == (21, 31, 2, 1)
    assert p.delta == 20                                           # S:90 (reading R13)
    assert list(zip(p.census_dx, p.census_dy)) == [(0, -2), (-1, -1), (1, -1), (-1, 1), (1, 1), (0, 2)]
    assert (p.w_x_r, p.fill_mode) == (-1, abi.FILL_BILATERAL)      # NEXT-3 variants off


def _create(W=64, H=48, D=16, **kw):
    p = abi.default_params(**kw)
    h = C.c_void_p()
    rc = abi.lib().stereo_create(W, H, D, C.byref(p), C.byref(h))
    return rc, abi.lib().stereo_last_error().decode()


@pytest.mark.parametrize("kw,code,msg", [
    (dict(lambda_ad=0.0), abi.STEREO_EINVAL, "lambda_ad must be > 0"),
    (dict(lambda_mc=-1.0), abi.STEREO_EINVAL, "lambda_mc must be > 0"),
    (dict(delta=0), abi.STEREO_EINVAL, "delta must be > 0"),
    (dict(t_fill=-1), abi.STEREO_EINVAL, "t_fill"),
    (dict(w_x=-1), abi.STEREO_EINVAL, "w_x"),
    (dict(w_y=-2), abi.STEREO_EINVAL, "w_y"),
    (dict(k_scale=0), abi.STEREO_EINVAL, "k_scale"),
    (dict(k_scale=3), abi.STEREO_EUNSUPPORTED, "k_scale must be 1 or 2"),
    (dict(w_x=255), abi.STEREO_EUNSUPPORTED, "254"),
    (dict(m_pool=4), abi.STEREO_EUNSUPPORTED, "m_pool"),
    (dict(w_x_r=-2), abi.STEREO_EINVAL, "w_x_r"),
    (dict(w_x_r=255), abi.STEREO_EUNSUPPORTED, "254"),
    (dict(fill_mode=4), abi.STEREO_EINVAL, "fill_mode"),
    (dict(fill_mode=-1), abi.STEREO_EINVAL, "fill_mode"),
    (dict(abi_version=7), abi.STEREO_EINVAL, "abi_version"),
    (dict(census=[(0, -2), (0, -2), (1, -1), (-1, 1), (1, 1), (0, 2)]), abi.STEREO_EINVAL, "distinct"),
    (dict(census=[(0, 0), (-1, -1), (1, -1), (-1, 1), (1, 1), (0, 2)]), abi.STEREO_EINVAL, "zero"),
    (dict(census=[(0, -3), (-1, -1), (1, -1), (-1, 1), (1, 1), (0, 2)]), abi.STEREO_EUNSUPPORTED, "2"),
])
def test_validation_errors(kw, code, msg):
    rc, err = _create(**kw)
    assert rc == code and msg in err


def test_validation_order_first_violation_named():
    # "reports the first violated invariant by name"
    rc, err = _create(lambda_ad=0.0, delta=0)
    assert rc == abi.STEREO_EINVAL and "lambda_ad" in err


def test_size_errors():
    assert _create(D=0)[0] == abi.STEREO_EINVAL
    assert _create(W=0)[0] == abi.STEREO_EINVAL
    assert _create(W=1, H=1, k_scale=2)[0] == abi.STEREO_EINVAL       # empty scaled image
    assert _create(D=600, k_scale=2)[0] == abi.STEREO_EUNSUPPORTED    # ceil(D/K) > 255


def test_null_arguments():
    L = abi.lib()
    assert L.stereo_create(8, 8, 4, None, C.byref(C.c_void_p())) == abi.STEREO_EINVAL
    assert L.stereo_compute(None, None, None, None, None) == abi.STEREO_EINVAL
    assert L.stereo_get_info(None, None) == abi.STEREO_EINVAL
    assert L.stereo_compute_rgb(None, None, None, None, None) == abi.STEREO_EINVAL
    assert L.stereo_rgb_to_gray(None, None, 4, 4, None) == abi.STEREO_EINVAL
    assert L.stereo_disparity_to_depth(None, None, 4, 1.0, None) == abi.STEREO_EINVAL
    L.stereo_destroy(None)  # no-op


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    monkeypatch.setattr(abi, "LIB_PATH", str(tmp_path / "nope.so"))
    monkeypatch.setattr(abi, "_lib", None)
    with pytest.raises(abi.StereoLibraryError):
        abi.lib()


def test_header_is_plain_c_and_host_calls_link(tmp_path):
    """include/stereo.h compiles as C11 (no C++ constructs cross the boundary)
    and a C program links against libstereo_b200.so and runs the host-only
    calls (defaults, validation, the band partition and halo) without a GPU."""
    src = tmp_path / "use.c"
    src.write_text(r'''
#include <stdio.h>
#include "stereo.h"
int main(void) {
  stereo_params p;
  stereo_default_params(&p);
  if (p.abi_version != STEREO_ABI_VERSION || p.w_x != 21 || p.w_y != 31 || p.k_scale != 2) return 1;
  int y0, rows, top, bot, total = 0;
  for (int b = 0; b < 8; ++b) {
    if (stereo_band_rows(992, &p, 8, b, &y0, &rows) != STEREO_OK) return 2;
    if (y0 != total) return 3;
    total += rows;
    if (stereo_band_halo(992, &p, y0, rows, &top, &bot) != STEREO_OK) return 4;
    if (y0 > 0 && top < 68) return 5;
  }
  if (total != 992) return 6;
  stereo_t* h = 0;
  p.lambda_ad = -1.0;  /* validation happens before any device call */
  if (stereo_create(64, 48, 16, &p, &h) != STEREO_EINVAL || h) return 7;
  printf("ok %s\n", stereo_last_error());
  return 0;
}
''')
    exe = tmp_path / "use"
    libdir = os.path.dirname(abi.LIB_PATH)
    r = subprocess.run(["gcc", "-std=c11", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                        str(src), "-L", libdir, "-lstereo_b200", f"-Wl,-rpath,{libdir}", "-o", str(exe)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 0 and r.stdout.startswith("ok lambda_ad"), (r.returncode, r.stdout, r.stderr)
