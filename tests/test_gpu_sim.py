"""GPU parity: Simulation::step (sim.cpp:59-131) over the device path — two
bodies whose wake zones overlap, so each hull's depths include the other's zone
(compose_height, sim.cpp:44-51), with deferred masks and rigid integration —
against the reference library stepping the same scene
(tests/golden/make_golden_sim.py -> sim_ref.npz)."""
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))

from make_golden_sim import sim_scene  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", params=[(False, False, False), (False, True, False),
                                        (True, False, False), (True, True, False),
                                        (True, False, True)],
                ids=["serial-calls", "serial-native", "pipelined", "pipelined-native",
                     "concurrent"])
def run(request):
    from paper_2503_03326_b200 import ocean as oc
    from paper_2503_03326_b200.sim import BodyConfig, Simulation
    s = sim_scene()
    bodies = [BodyConfig(vertices=s["vertices"], triangles=s["triangles"], position=b["position"],
                         yaw=b["yaw"], initial_velocity=b["velocity"], density=b["density"],
                         angular_damping=s["angular_damping"], fdm=s["fdm"]) for b in s["bodies"]]
    sim = Simulation(oc.CascadeConfig(s["n"], s["lengths"], s["cutoffs"]), s["params"], s["slices"],
                     bodies, dt=s["dt"], wind=s["wind"], pipelined=request.param[0], native=request.param[1],
                     concurrent=request.param[2])
    v0 = sim.poses()[:, 7:10].copy()
    poses, vw = [], []
    for _ in range(s["steps"]):
        sim.step()
        poses.append(sim.poses())
        vw.append([b.report.submerged_volume for b in sim.bodies])
    ref = np.load(os.path.join(HERE, "golden", "sim_ref.npz"))
    return sim, np.array(poses), np.array(vw), v0, ref


def test_submerged_volume(run):
    _, _, vw, _, ref = run
    assert np.abs(vw - ref["submerged_volume"]).max() <= 1e-4 * np.abs(ref["submerged_volume"]).max()


def test_body_states(run):
    _, poses, _, v0, ref = run
    rp = ref["pose"]
    for s in range(rp.shape[0]):
        for b in range(rp.shape[1]):
            g, r = poses[s, b], rp[s, b]
            dv_g, dv_r = g[7:10] - v0[b], r[7:10] - v0[b]
            assert np.linalg.norm(dv_g - dv_r) <= 1e-4 * np.linalg.norm(dv_r), (s, b, dv_g, dv_r)
            assert np.linalg.norm(g[10:13] - r[10:13]) <= 1e-3 * np.linalg.norm(r[10:13]) + 1e-9, (s, b)
            assert np.abs(g[0:3] - r[0:3]).max() <= 1e-5, (s, b)
            assert np.abs(g[3:7] - r[3:7]).max() <= 1e-6, (s, b)


def test_zone_coupling_is_live(run):
    """Each zone is non-zero after the masks, and compose_height(exclude_body=i) adds the other
    body's zone: at body 1's hull it differs from height_at; at body 0's hull the same call
    excluding body 1 is plain height_at (sim.cpp:44-51)."""
    from paper_2503_03326_b200 import ocean as oc
    sim = run[0]
    assert all(np.abs(b.zone.field()).max() > 0.0 for b in sim.bodies)
    w1, _ = sim.bodies[1].report.vertices()
    xz1 = np.ascontiguousarray(w1[:, [0, 2]])
    d1 = sim.compose_height(xz1, exclude_body=0) - oc.height_at(sim.maps, xz1)
    assert np.abs(d1).max() > 0.0
    w0, _ = sim.bodies[0].report.vertices()
    xz0 = np.ascontiguousarray(w0[:, [0, 2]])
    d0 = sim.compose_height(xz0, exclude_body=0) - oc.height_at(sim.maps, xz0)
    # after 24 steps body 1's wake has crossed the gap: body 0's hull depths (and the
    # reference-parity forces above) include it
    assert np.abs(d0).max() > 1e-6


@pytest.mark.parametrize("pipelined", [False, True])
def test_device_simulation_matches_reference(pipelined):
    """The C++ Simulation over device-resident state (ocn_sim: one C-ABI call per
    step, all bodies' hulls in one batched launch set, rigid integration in C++)
    against the reference library stepping the same two-body scene."""
    from paper_2503_03326_b200 import ocean as oc
    from paper_2503_03326_b200.sim import BodyConfig, DeviceSimulation
    s = sim_scene()
    bodies = [BodyConfig(vertices=s["vertices"], triangles=s["triangles"], position=b["position"],
                         yaw=b["yaw"], initial_velocity=b["velocity"], density=b["density"],
                         angular_damping=s["angular_damping"], fdm=s["fdm"]) for b in s["bodies"]]
    sim = DeviceSimulation(oc.CascadeConfig(s["n"], s["lengths"], s["cutoffs"]), s["params"],
                           s["slices"], bodies, dt=s["dt"], wind=s["wind"], pipelined=pipelined)
    sim.set_timing(True)
    v0 = sim.poses()[:, 7:10].copy()
    ref = np.load(os.path.join(HERE, "golden", "sim_ref.npz"))
    rp = ref["pose"]
    for st in range(s["steps"]):
        sim.step()
        poses = sim.poses()
        vw = [r.submerged_volume for r in sim.reports()]
        assert np.abs(np.array(vw) - ref["submerged_volume"][st]).max() <= \
            1e-4 * np.abs(ref["submerged_volume"]).max(), st
        for b in range(rp.shape[1]):
            g, r = poses[b], rp[st, b]
            dv_g, dv_r = g[7:10] - v0[b], r[7:10] - v0[b]
            assert np.linalg.norm(dv_g - dv_r) <= 1e-4 * np.linalg.norm(dv_r), (st, b)
            assert np.abs(g[0:3] - r[0:3]).max() <= 1e-5, (st, b)
            assert np.abs(g[3:7] - r[3:7]).max() <= 1e-6, (st, b)
    # Simulation::timing() stages (sim.hpp:50-54): device time of the fused
    # spectral step, hulls, zones; host time of the integration
    tm = sim.timing()
    assert list(tm) == ["surface", "velocity", "hydro", "zones", "integrate"]
    assert tm["surface"] > 0 and tm["hydro"] > 0 and tm["zones"] > 0 and tm["integrate"] > 0, tm
    assert tm["velocity"] == 0.0
