"""Time the device DirectVelocityEvaluator at config 2:
4 cascades x 1024^2, mode-list build and evaluation at P points (CUDA events
are not needed: each call synchronises; wall time over repeated calls)."""
import math
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2503_03326_b200 import ocean as oc  # noqa: E402
from paper_2503_03326_b200._types import SpectrumParams  # noqa: E402


def main(points=(1000, 100000)):
    p = SpectrumParams.make(wind_speed=20.0, fetch=1e5, wind_direction=0.4, swell=0.5,
                            direction_mix=0.5, rng_seed=42)
    p.has_peak_omega_override = 1
    p.peak_omega_override = p.standard_peak_omega()
    cs = oc.CascadeSet(oc.CascadeConfig(1024, [1024.0, 256.0, 16.0, 4.0],
                                        [12 * math.pi / 256, 12 * math.pi / 16, 12 * math.pi / 4]), p)
    oc.DirectVelocityEvaluator(cs, 1.0)
    t0 = time.perf_counter()
    ev = oc.DirectVelocityEvaluator(cs, 1.0)
    build_ms = (time.perf_counter() - t0) * 1e3
    M = ev.mode_count
    rng = np.random.default_rng(0)
    for P in points:
        xz = rng.uniform(-500, 500, size=(P, 2))
        y = rng.uniform(-20, 0, size=P)
        ev(xz, y)
        t0 = time.perf_counter()
        reps = 3
        for _ in range(reps):
            ev(xz, y)
        ms = (time.perf_counter() - t0) * 1e3 / reps
        print(f"direct velocity: modes {M}, points {P}: {ms:.3f} ms "
              f"({M * P / (ms * 1e-3) / 1e9:.0f} G mode-points/s); mode build {build_ms:.2f} ms")


if __name__ == "__main__":
    main()
