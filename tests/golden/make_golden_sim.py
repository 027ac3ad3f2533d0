"""Generate tests/golden/sim_ref.npz: a 2-body Simulation (sim.cpp:16-131)
stepped by the REFERENCE library (oracle/_ref, ref_sim_run in ref_shim.cpp).

Run here (where /root/reference exists):  python tests/golden/make_golden_sim.py
The scene is sim_scene() below, shared with tests/test_gpu_sim.py.
"""
import ctypes as C
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from paper_2503_03326_b200._types import FdmConfig, SliceConfig, SpectrumParams  # noqa: E402
from paper_2503_03326_b200.meshgen import uv_ellipsoid  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def sim_scene():
    """Two 10 m x 6 m x 20 m hulls side by side ~1 m apart (overlapping wake zones), config-2 sea at N = 64."""
    p = SpectrumParams.make(wind_speed=20.0, fetch=1e5, wind_direction=0.4, swell=0.5,
                            direction_mix=0.5, rng_seed=42)
    p.has_peak_omega_override = 1
    p.peak_omega_override = p.standard_peak_omega()
    v, t = uv_ellipsoid(24, 17, (5.0, 3.0, 10.0))
    return dict(
        n=64, lengths=[1024.0, 256.0, 16.0, 4.0],
        cutoffs=[12 * math.pi / 256, 12 * math.pi / 16, 12 * math.pi / 4], params=p,
        slices=SliceConfig.make(count=8), vertices=v, triangles=t,
        bodies=[dict(position=(0.0, -0.5, 0.0), yaw=0.2, velocity=(1.0, 0.0, 3.0), density=480.0),
                dict(position=(11.0, -1.0, 3.0), yaw=-0.4, velocity=(-0.5, 0.0, 2.0), density=520.0)],
        fdm=FdmConfig.make(grid_size=128, margin=16), angular_damping=0.1, wind=(5.0, 0.0, 2.0),
        dt=1.0 / 60.0, steps=24)


def main():
    from oracle.oracle import build
    build(reference=True)
    s = sim_scene()
    L = C.CDLL(os.path.join(ROOT, "oracle", "_ref", "libocean_ref.so"))
    dp = C.POINTER(C.c_double)
    P = lambda a: np.ascontiguousarray(a, np.float64).ctypes.data_as(dp)
    nb, steps = len(s["bodies"]), s["steps"]
    cfg = np.array([[*b["position"], b["yaw"], *b["velocity"], b["density"]] for b in s["bodies"]],
                   np.float64)
    out_pose = np.zeros((steps, nb, 13))
    out_vw = np.zeros((steps, nb))
    tris = np.ascontiguousarray(s["triangles"], np.int32)
    verts = np.ascontiguousarray(s["vertices"], np.float64)
    lengths = np.array(s["lengths"], np.float64)
    cutoffs = np.array(s["cutoffs"] + [0.0], np.float64)
    wind = np.array(s["wind"], np.float64)
    L.ref_sim_run.restype = C.c_int
    st = L.ref_sim_run(C.c_int(s["n"]), C.c_int(len(lengths)), P(lengths), P(cutoffs),
                       C.byref(s["params"]), C.byref(s["slices"]), C.c_int(len(verts)), P(verts),
                       C.c_int(len(tris)), tris.ctypes.data_as(C.POINTER(C.c_int32)), C.c_int(nb),
                       P(cfg), C.byref(s["fdm"]), C.c_double(s["angular_damping"]), P(wind),
                       C.c_double(s["dt"]), C.c_int(steps), out_pose.ctypes.data_as(dp),
                       out_vw.ctypes.data_as(dp))
    assert st == 0, st
    np.savez_compressed(os.path.join(OUT, "sim_ref.npz"), pose=out_pose, submerged_volume=out_vw)
    print("sim_ref.npz: final poses\n", out_pose[-1], "\nsubmerged volumes", out_vw[-1])


if __name__ == "__main__":
    main()
