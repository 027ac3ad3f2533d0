"""CPU: the C-ABI library loads, exports every symbol include/ocean_b200.h
declares, and its host-evaluated scalar entry points agree with the oracle.
No device compute here (there is no GPU in the build container)."""
import ctypes as C
import math

import numpy as np
import pytest

from helpers import config2_params
from paper_2503_03326_b200 import _abi
from paper_2503_03326_b200._types import SliceConfig, SpectrumParams


@pytest.fixture(scope="module")
def L():
    return _abi.lib()


def test_exports_every_declared_symbol(L):
    syms = _abi.header_symbols()
    assert len(syms) >= 70
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    assert set(_abi.SIGNATURES) == set(syms), set(_abi.SIGNATURES) ^ set(syms)
    assert L.ocn_abi_version() == 2


def test_no_silent_cpu_fallback(L):
    """Without a usable B200 the product path must fail loudly."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    h = C.c_void_p()
    st = L.ocn_ctx_create(0, C.byref(h))
    assert st == _abi.OCN_ERR_CUDA
    assert b"CUDA" in L.ocn_last_error(None) or b"device" in L.ocn_last_error(None)
    from paper_2503_03326_b200 import ocean
    with pytest.raises(ocean.OceanCudaError):
        ocean.Context(0)


def test_host_scalars_match_oracle(L, port):
    p = config2_params()
    p0 = SpectrumParams.make()
    for pp in (p, p0):
        assert L.ocn_alpha(C.byref(pp)) == port.scalar("alpha", pp)
        assert L.ocn_peak_omega(C.byref(pp)) == port.scalar("peak_omega", pp)
        for w in (0.3, 0.9, 1.7, 5.0):
            for th in (-2.0, 0.0, 0.4, 3.1):
                assert L.ocn_directional(w, th, C.byref(pp)) == port.scalar("directional", w, th, pp)
        out = C.c_double()
        assert L.ocn_jonswap(0.8, C.byref(pp), C.byref(out)) == 0
        assert out.value == port.jonswap(0.8, pp)
        assert L.ocn_jonswap(0.0, C.byref(pp), C.byref(out)) == _abi.OCN_ERR_DOMAIN
    for r in (0.3, 0.94, 0.95, 1.0, 1.59, 1.6, 4.0, 150.0):
        assert L.ocn_beta_s(r) == port.scalar("beta_s", r)
        assert L.ocn_q_dbxi_approx(r) == port.scalar("q_dbxi_approx", r)
    assert L.ocn_q_dbxi_quadrature(0.8, 1.0, 4096) == port.scalar("q_dbxi_quadrature", 0.8, 1.0, 4096)
    assert L.ocn_damping_factor(2.5, 0.98, 0.999, 5.0) == pytest.approx(0.9895)
    for cfg in (SliceConfig.make(count=32), SliceConfig.make(count=7, distribution=1)):
        d = np.zeros(cfg.count)
        assert L.ocn_slice_depths(C.byref(cfg), d.ctypes.data_as(_abi.d)) == 0
        np.testing.assert_array_equal(d, port.slice_depths(cfg))
    bad = SliceConfig.make(count=1)
    assert L.ocn_slice_depths(C.byref(bad), np.zeros(1).ctypes.data_as(_abi.d)) == _abi.OCN_ERR_CONFIG
    bad_p = SpectrumParams.make(swell=2.0)
    assert L.ocn_spectrum_validate(C.byref(bad_p)) == _abi.OCN_ERR_CONFIG


def test_hypot_matches_host_libm():
    """|k| is computed with the reference libm's hypot algorithm (glibc e_hypot
    non-FMA kernel), which is what makes the band mask bit-exact."""
    import subprocess, os, tempfile
    src = r'''
#include <cstdio>
#include <cmath>
#include <initializer_list>
#include "paper_2503_03326_b200/csrc/spectrum_math.cuh"
int main(){ const double kPi=3.14159265358979323846; long bad=0;
 for (double L : {1024.0, 256.0, 16.0, 4.0, 4096.0}) { double dk = 2.0*kPi/L;
  for (int i=0;i<512;i+=3) for (int j=0;j<1024;++j) { double kx=dk*(i-512), kz=dk*(j-512);
   if (hypot(kx,kz) != ocn::sm::hypot_ref(kx,kz)) ++bad; } }
 printf("%ld\n", bad); return 0; }'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with tempfile.TemporaryDirectory() as d:
        f = os.path.join(d, "h.cpp")
        open(f, "w").write(src)
        exe = os.path.join(d, "h")
        subprocess.run(["g++", "-O2", "-std=c++17", "-I", root, "-I", os.path.join(root, "include"),
                        f, "-o", exe], check=True)
        out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout.strip()
    assert out == "0"


def test_struct_layouts_match_header():
    """Every POD struct of include/ocean_b200.h has the same size and field
    offsets in the C compiler's layout and in the ctypes mirror."""
    import os
    import subprocess
    import tempfile
    from paper_2503_03326_b200 import _types as T
    pairs = {"ocn_spectrum_params": T.SpectrumParams, "ocn_slice_config": T.SliceConfig,
             "ocn_pose": T.Pose, "ocn_fluid": T.Fluid, "ocn_hydro_report": T.HydroReport,
             "ocn_triangle_state": T.TriangleState, "ocn_fdm_config": T.FdmConfig,
             "ocn_mask_params": T.MaskParams, "ocn_mask_frame": T.MaskFrame,
             "ocn_zone_state": T.ZoneState, "ocn_body_frame": T.BodyFrame,
             "ocn_xform_info": T.XformInfo, "ocn_sim_config": T.SimConfig,
             "ocn_sim_body": T.SimBody}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "ocean_b200.h"', 'int main(void){']
    for cname, py in pairs.items():
        lines.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for fname, _ in py._fields_:
            lines.append(f'printf("{cname} {fname} %zu\\n", offsetof({cname}, {fname}));')
    lines.append("return 0;}")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "layout.c")
        open(src, "w").write("\n".join(lines))
        exe = os.path.join(d, "layout")
        subprocess.run(["gcc", "-std=c99", "-I", os.path.join(root, "include"), src, "-o", exe],
                       check=True)
        out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split("\n")
    got = {}
    for ln in out:
        if ln:
            parts = ln.split()
            got[tuple(parts[:-1])] = int(parts[-1])
    for cname, py in pairs.items():
        assert got[(cname, "size")] == C.sizeof(py), cname
        for fname, _ in py._fields_:
            assert got[(cname, fname)] == getattr(py, fname).offset, (cname, fname)
