"""Where a Simulation::step goes: host enqueue time vs device completion, by body count."""
import sys
import time

sys.path.insert(0, ".")
import tools.bench_sim as bs  # noqa: E402
from paper_2503_03326_b200 import ocean as oc  # noqa: E402


def run(nb):
    import math
    from paper_2503_03326_b200._types import FdmConfig, SliceConfig, SpectrumParams
    from paper_2503_03326_b200.meshgen import uv_ellipsoid
    from paper_2503_03326_b200.sim import BodyConfig, Simulation
    p = SpectrumParams.make(wind_speed=20.0, fetch=1e5, wind_direction=0.4, swell=0.5,
                            direction_mix=0.5, rng_seed=42)
    p.has_peak_omega_override = 1
    p.peak_omega_override = p.standard_peak_omega()
    v, t = uv_ellipsoid(64, 33, (2.0, 1.5, 6.0))
    bodies = [BodyConfig(vertices=v, triangles=t, position=(15.0 * (b % 5), -0.3, 20.0 * (b // 5)),
                         yaw=0.1 * b, initial_velocity=(0.0, 0.0, 2.0), density=500.0,
                         fdm=FdmConfig.make(grid_size=256, margin=16)) for b in range(nb)]
    sim = Simulation(oc.CascadeConfig(1024, [1024.0, 256.0, 16.0, 4.0],
                                      [12 * math.pi / 256, 12 * math.pi / 16, 12 * math.pi / 4]), p,
                     SliceConfig.make(count=32), bodies)
    for _ in range(5):
        sim.step()
    K = 40
    t0 = time.perf_counter()
    for _ in range(K):
        sim.step()
    ms = (time.perf_counter() - t0) * 1e3 / K
    # spectral step alone (device-bound)
    t0 = time.perf_counter()
    for _ in range(K):
        oc.spectral_step(sim.maps, sim.slices, 1.0)
    sim.ctx.synchronize() if hasattr(sim.ctx, "synchronize") else oc.lib().ocn_ctx_synchronize(sim.ctx.h)
    spec = (time.perf_counter() - t0) * 1e3 / K
    # one body's hull stages, synchronous, repeated
    b = sim.bodies[0]
    fluid = oc.FluidQuery(maps=sim.maps, slices=sim.slices, zones=[x.zone for x in sim.bodies[1:]])
    pose = b.rigid.pose()
    t0 = time.perf_counter()
    for _ in range(K):
        oc.aggregate(b.mesh, pose, fluid, sync=False)
    enq = (time.perf_counter() - t0) * 1e3 / K
    oc.lib().ocn_ctx_synchronize(sim.ctx.h)
    t0 = time.perf_counter()
    for _ in range(K):
        oc.aggregate(b.mesh, pose, fluid, sync=True)
    agg = (time.perf_counter() - t0) * 1e3 / K
    print(f"bodies {nb}: step {ms:.3f} ms | spectral {spec:.3f} | one aggregate enqueue {enq:.3f}, "
          f"synchronous {agg:.3f} ms")


if __name__ == "__main__":
    for nb in (1, 2, 5, 10):
        run(nb)
