"""GPU: the C++ drop-in API (include/ocean/*.hpp -> libocean_api.so -> C-ABI)
driven like reference callers (tests/cpp/test_api.cpp), outputs vs the oracle."""
import math
import os
import subprocess

import numpy as np
import pytest

from helpers import CONFIG2_CUTOFFS, CONFIG2_LENGTHS, config2_params, normwise_rel
from paper_2503_03326_b200._types import SliceConfig

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "paper_2503_03326_b200", "build", "test_api")


def test_cpp_api(tmp_path, port):
    if not os.path.exists(EXE):
        from paper_2503_03326_b200 import build
        build.build()
    r = subprocess.run([EXE, str(tmp_path)], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stderr
    p = config2_params()
    want = port.generate_maps(64, CONFIG2_LENGTHS, CONFIG2_CUTOFFS, p, 1.5)
    for c in range(4):
        for f in range(8):
            got = np.fromfile(tmp_path / f"maps_{c}_{f}.bin").reshape(64, 64)
            assert normwise_rel(got, want[c, f]) < 1e-4, (c, f)
    xs = np.array([[3.0, 7.0], [-100.5, 33.25], [512.0, -4.0]])
    h = np.fromfile(tmp_path / "heights.bin")
    h_ref = port.height_at(64, CONFIG2_LENGTHS, want, xs)
    assert np.abs(h - h_ref).max() <= 1e-4 * np.abs(want[:, 0]).max()
    cfg = SliceConfig.make(count=8)
    d_ref, s_ref = port.build_slices(64, CONFIG2_LENGTHS, CONFIG2_CUTOFFS, p, 1.5, cfg)
    v = np.fromfile(tmp_path / "velocity.bin")
    v_ref = port.velocity_at_port(64, CONFIG2_LENGTHS, d_ref, cfg, s_ref, np.array([[3.0, 7.0, -2.0]]))[0]
    assert np.linalg.norm(v - v_ref) <= 1e-4 * np.linalg.norm(v_ref)
    dv = np.fromfile(tmp_path / "direct.bin")
    dv_ref = port.direct_velocity(64, CONFIG2_LENGTHS, CONFIG2_CUTOFFS, p, 1.5, np.array([[3.0, 7.0, -2.0]]))[0]
    assert np.linalg.norm(dv - dv_ref) <= 1e-4 * np.linalg.norm(dv_ref)
