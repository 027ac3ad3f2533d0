"""Wall-clock ms per Simulation::step (sim.py over the device path) for the
paper's ten-solids setting (XP2: 10 bodies) on the config-2
sea (4 cascades x 1024^2, 32 velocity slices). Host wall time per step,
including the per-body report reads and the host rigid integration."""
import math
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2503_03326_b200 import ocean as oc  # noqa: E402
from paper_2503_03326_b200._types import FdmConfig, SliceConfig, SpectrumParams  # noqa: E402
from paper_2503_03326_b200.meshgen import uv_ellipsoid  # noqa: E402
from paper_2503_03326_b200.sim import BodyConfig, DeviceSimulation, Simulation  # noqa: E402


def main(n_bodies=10, steps=60, n=1024, pipelined=False, native=False, concurrent=False,
         device=False):
    p = SpectrumParams.make(wind_speed=20.0, fetch=1e5, wind_direction=0.4, swell=0.5,
                            direction_mix=0.5, rng_seed=42)
    p.has_peak_omega_override = 1
    p.peak_omega_override = p.standard_peak_omega()
    v, t = uv_ellipsoid(64, 33, (2.0, 1.5, 6.0))  # 4,096 triangles (the XP2 hulls carry 4,135 in total)
    bodies = [BodyConfig(vertices=v, triangles=t, position=(15.0 * (b % 5), -0.3, 20.0 * (b // 5)),
                         yaw=0.1 * b, initial_velocity=(0.0, 0.0, 2.0), density=500.0,
                         fdm=FdmConfig.make(grid_size=256, margin=16)) for b in range(n_bodies)]
    cc = oc.CascadeConfig(n, [1024.0, 256.0, 16.0, 4.0],
                          [12 * math.pi / 256, 12 * math.pi / 16, 12 * math.pi / 4])
    if device:
        sim = DeviceSimulation(cc, p, SliceConfig.make(count=32), bodies, pipelined=pipelined)
    else:
        sim = Simulation(cc, p, SliceConfig.make(count=32), bodies, pipelined=pipelined,
                         native=native, concurrent=concurrent)
    for _ in range(5):
        sim.step()
    t0 = time.perf_counter()
    for _ in range(steps):
        sim.step()
    ms = (time.perf_counter() - t0) * 1e3 / steps
    print(f"simulation: {n_bodies} bodies x {len(t)} triangles, {n}^2 x 4 cascades + 32 slices: "
          f"{ms:.3f} ms/step (host wall, {steps} steps, {'concurrent bodies' if concurrent else 'pipelined' if pipelined else 'serial'}, "
          f"{'ocn_sim (C++ step)' if device else 'ocn_bodies_step' if native and not concurrent else 'per-body calls'})")


if __name__ == "__main__":
    main()
    main(native=True)
    main(pipelined=True)
    main(pipelined=True, native=True)
    main(concurrent=True)
    main(device=True)
    main(device=True, pipelined=True)
    for nb in (1, 2, 5):
        main(n_bodies=nb, device=True, pipelined=True)
