"""A few device-simulation steps (10 bodies, config-2 sea) for ncu launch lists;
not a benchmark.   python tools/prof_sim.py [steps] [bodies]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import math  # noqa: E402

from paper_2503_03326_b200 import ocean as oc  # noqa: E402
from paper_2503_03326_b200._types import FdmConfig, SliceConfig, SpectrumParams  # noqa: E402
from paper_2503_03326_b200.meshgen import uv_ellipsoid  # noqa: E402
from paper_2503_03326_b200.sim import BodyConfig, DeviceSimulation  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 10
p = SpectrumParams.make(wind_speed=20.0, fetch=1e5, wind_direction=0.4, swell=0.5,
                        direction_mix=0.5, rng_seed=42)
p.has_peak_omega_override = 1
p.peak_omega_override = p.standard_peak_omega()
v, t = uv_ellipsoid(64, 33, (2.0, 1.5, 6.0))
bodies = [BodyConfig(vertices=v, triangles=t, position=(15.0 * (b % 5), -0.3, 20.0 * (b // 5)),
                     yaw=0.1 * b, initial_velocity=(0.0, 0.0, 2.0), density=500.0,
                     fdm=FdmConfig.make(grid_size=256, margin=16)) for b in range(nb)]
cc = oc.CascadeConfig(1024, [1024.0, 256.0, 16.0, 4.0],
                      [12 * math.pi / 256, 12 * math.pi / 16, 12 * math.pi / 4])
sim = DeviceSimulation(cc, p, SliceConfig.make(count=32), bodies, pipelined=False)
for _ in range(steps):
    sim.step()
print("ok")
