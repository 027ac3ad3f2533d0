"""GPU parity: hull clipping / forces (K5-K8), waterline, mask (K9), FDM (K10)."""
import math

import numpy as np
import pytest

from helpers import (CONFIG2_CUTOFFS, CONFIG2_LENGTHS, config2_params, config3_pose, normwise_rel,
                     vec_rel)
from paper_2503_03326_b200._types import FdmConfig, MaskFrame, MaskParams, Pose, SliceConfig
from paper_2503_03326_b200.meshgen import icosphere, unit_cube, uv_ellipsoid

pytestmark = pytest.mark.gpu
TOL = 1e-4


@pytest.fixture(scope="module")
def oc():
    from paper_2503_03326_b200 import ocean
    return ocean


def _report_close(g, r, tol=TOL):
    assert g.state_count == r["state_count"]
    assert g.waterline_loops == r["waterline_loops"]
    assert abs(g.submerged_volume - r["submerged_volume"]) <= tol * max(abs(r["submerged_volume"]), 1.0)
    for k in ("buoyancy_force", "water_drag", "air_drag", "force", "torque"):
        assert vec_rel(getattr(g, k), r[k]) <= tol, (k, getattr(g, k), r[k])
    for k in ("water_center", "air_center"):
        assert vec_rel(getattr(g, k), r[k]) <= tol, k
    if r["has_center_of_immersion"]:
        assert vec_rel(g.center_of_immersion, r["center_of_immersion"]) <= tol


def test_clip_structure_bit_exact(oc, port):
    """Same vertex depths -> identical states (count / order / parent / status) and
    identical waterline loops (bit-exact mesh traversal)."""
    v, t = uv_ellipsoid(128, 97)
    mesh_o = port.mesh_build(v, t)
    mesh_g = oc.TriMesh(v, t)
    np.testing.assert_array_equal(mesh_g.triangles, mesh_o["tris"])
    np.testing.assert_array_equal(mesh_g.normals, mesh_o["normals"])
    np.testing.assert_array_equal(mesh_g.areas, mesh_o["areas"])
    pose = config3_pose(mesh_o["centroid"])
    rng = np.random.default_rng(4)
    # a wavy synthetic sea evaluated on the oracle side only -> explicit depths
    world = np.array([[0.0]])
    wpos = np.zeros((v.shape[0], 3))
    dd = np.zeros(v.shape[0])
    import ctypes as C
    from oracle.oracle import P
    from oracle.oracle_structs import OrcFluid
    fl = OrcFluid()
    fl.water_density, fl.air_density, fl.cd_water, fl.cd_air = 1025.0, 1.204, 1.0, 1.0
    f = port.lib.orc_vertex_depths
    f.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    f(v.shape[0], P(v), C.byref(pose), C.byref(fl), P(wpos), P(dd))
    depth = wpos[:, 1] - 0.7 * np.sin(0.3 * wpos[:, 0]) * np.cos(0.2 * wpos[:, 2]) - 0.1
    rep_o, st_o, loops_o = port.aggregate(v, mesh_o, pose, vertex_depth=depth, wind=(5, 0, 2))
    res = oc.aggregate(mesh_g, pose, oc.FluidQuery(wind=(5, 0, 2)), vertex_depth=depth)
    st_g = res.states()
    assert st_g.shape == st_o.shape
    assert np.array_equal(st_g["parent"], st_o["parent"])
    assert np.array_equal(st_g["status"], st_o["status"])
    for k in ("area", "centroid", "depth", "normal"):
        assert np.allclose(st_g[k], st_o[k], rtol=1e-12, atol=1e-12), k
    loops_g = res.waterline()
    assert len(loops_g) == len(loops_o) and len(loops_g) >= 1
    for a, b in zip(loops_g, loops_o):
        assert a.shape == b.shape
        assert np.allclose(a, b, rtol=1e-12, atol=1e-12)
    _report_close(res, rep_o, 1e-9)


def test_spec_cube_and_sphere(oc):
    """SPEC.md:420-450 known answers on the device (flat water)."""
    v, t = unit_cube()
    mesh = oc.TriMesh(v, t)
    still = oc.FluidQuery()
    r = oc.aggregate(mesh, Pose.make(position=(0, -10, 0)), still)
    assert r.submerged_volume == pytest.approx(1.0, abs=1e-9)
    assert r.submerged_area == pytest.approx(6.0, abs=1e-9)
    r = oc.aggregate(mesh, Pose.make(position=(0, 10, 0)), still)
    assert r.submerged_volume == 0.0 and r.center_of_immersion is None
    r = oc.aggregate(mesh, Pose.make(position=(0, 1e-7, 0)), still)
    assert r.submerged_volume == pytest.approx(0.5, abs=1e-6)
    assert r.buoyancy_force[1] == pytest.approx(1025 * 9.80665 * 0.5, rel=1e-5)
    loops = r.waterline()
    assert len(loops) == 1 and np.allclose(loops[0][0], loops[0][-1])
    assert np.sum(np.linalg.norm(np.diff(loops[0], axis=0), axis=1)) == pytest.approx(4.0, rel=1e-9)
    iv, it = icosphere(2.0, 3)
    ico = oc.TriMesh(iv, it)
    r = oc.aggregate(ico, Pose.make(position=(0, -10, 0)), still)
    assert r.submerged_volume == pytest.approx(ico.volume, rel=1e-6)


@pytest.mark.parametrize("n", [128])
def test_aggregate_end_to_end(oc, port, n):
    """Config-3 pipeline at a reduced grid: device maps + slices + hull -> report
    within 1e-4 of the oracle run on its own fp64 maps / slices."""
    p = config2_params()
    t = 1.0 / 60.0
    cfg = SliceConfig.make(count=32)
    cs = oc.CascadeSet(oc.CascadeConfig(n, CONFIG2_LENGTHS, CONFIG2_CUTOFFS), p)
    maps = oc.generate_maps(cs, t)
    vs = oc.build_slices(cs, t, cfg)
    v, tr = uv_ellipsoid()
    mesh_g = oc.TriMesh(v, tr)
    mesh_o = port.mesh_build(v, tr)
    pose = config3_pose(mesh_o["centroid"])
    res = oc.aggregate(mesh_g, pose, oc.FluidQuery(maps=maps, slices=vs, wind=(5, 0, 2)))
    m_ref = port.generate_maps(n, CONFIG2_LENGTHS, CONFIG2_CUTOFFS, p, t)
    d_ref, s_ref = port.build_slices(n, CONFIG2_LENGTHS, CONFIG2_CUTOFFS, p, t, cfg)
    rep, st, loops = port.aggregate(v, mesh_o, pose, n=n, lengths=CONFIG2_LENGTHS, maps=m_ref,
                                    slices=s_ref, depths=d_ref, slice_cfg=cfg, wind=(5, 0, 2))
    _report_close(res, rep)
    # vertex depths within tolerance of the oracle's
    w, dg = res.vertices()
    wpos = np.zeros_like(w)


def test_mask_bit_exact_from_loops(oc, port, golden):
    """compute_mask on identical loops -> identical cell set and heights."""
    fc = FdmConfig.make(grid_size=128, margin=8)
    zo = port.zone(fc, 12.0, 3.0, 7.0, 1.0 / 60.0)
    zg = oc.FdmZone(fc, 12.0, (3.0, 7.0), 1.0 / 60.0)
    for z in (zo, zg):
        z.update_stability(math.hypot(1, 4), 1.0 / 60.0)
    frame = MaskFrame.make(center_x=0.0, half_beam=12.0, z_min=-6.0, z_max=6.0, mesh_height=12.0,
                           volume_ratio=0.4)
    mp = MaskParams.make(back_height=0.1)
    loops = [golden["agg_loop0"]]
    ij_o, h_o = zo.compute_mask(loops, 0.3, 3.0, 7.0, math.hypot(1, 4), frame, mp)
    ij_g, h_g = oc.compute_mask(zg, loops, 0.3, (3.0, 7.0), math.hypot(1, 4), frame, mp)
    assert len(h_o) > 0
    assert np.array_equal(ij_g, ij_o)
    assert np.array_equal(h_g, h_o)


def test_fdm_steps(oc, port):
    fc = FdmConfig.make(grid_size=256, margin=16)
    zo = port.zone(fc, 20.0, 0.0, 0.0, 1.0 / 60.0)
    zg = oc.FdmZone(fc, 20.0, (0.0, 0.0), 1.0 / 60.0)
    rng = np.random.default_rng(9)
    f0 = np.zeros((256, 256))
    f0[16:-16, 16:-16] = rng.normal(size=(224, 224))
    zo.set_field(f0)
    zg.set_fields(f0, np.zeros_like(f0))
    pos = np.array([0.0, 0.0])
    for k in range(6):
        speed = 2.0 + k
        for z in (zo, zg):
            z.update_stability(speed, 1.0 / 60.0)
        pos = pos + np.array([speed / 60.0, 0.5 * speed / 60.0])
        zo.step(1.0 / 60.0, *pos)
        zg.step(1.0 / 60.0, pos)
        assert normwise_rel(zg.field(), zo.field()) < 1e-5
        st = zg.state()
        so = zo.state()
        assert st.spacing == so["spacing"] and st.origin[0] == so["origin"][0]
    # teleport: wake dropped (interactive.cpp:74-82)
    zo.step(1.0 / 60.0, 500.0, 0.0)
    zg.step(1.0 / 60.0, (500.0, 0.0))
    assert zg.state().dropped_wake == 1 == zo.state()["dropped_wake"]
    assert normwise_rel(zg.field(), zo.field()) < 1e-5 or np.abs(zo.field()).max() == 0.0
    xz = rng.uniform(-10, 10, size=(100, 2))
    assert np.allclose(zg.sample(xz), [zo.sample(x, z) for x, z in xz], atol=1e-5)
    assert zg.cfl_ratio(1.0 / 60.0) == pytest.approx(0.49)


def test_frame_pipeline_mask_from_hydro(oc, port):
    """sim.cpp:74-109 on the device: aggregate -> mask from the device waterline /
    volume -> apply -> step; the mask equals compute_mask on the downloaded loops."""
    n, p, t = 64, config2_params(), 0.5
    cs = oc.CascadeSet(oc.CascadeConfig(n, CONFIG2_LENGTHS, CONFIG2_CUTOFFS), p)
    maps = oc.generate_maps(cs, t)
    v, tr = uv_ellipsoid(96, 73)
    mesh = oc.TriMesh(v, tr)
    pose = config3_pose(mesh.centroid)
    res = oc.aggregate(mesh, pose, oc.FluidQuery(maps=maps, wind=(5, 0, 2)))
    fc = FdmConfig.make(grid_size=1024, margin=16)
    zone = oc.FdmZone(fc, 40.0, (3.0, 7.0), 1.0 / 60.0)
    zone.update_stability(math.hypot(1, 4), 1.0 / 60.0)
    ext = mesh.bbox_max - mesh.bbox_min
    frame = MaskFrame.make(center_x=0.0, half_beam=ext[0], z_min=mesh.bbox_min[2],
                           z_max=mesh.bbox_max[2], mesh_height=mesh.height(),
                           volume_ratio=res.submerged_volume / mesh.volume)
    mp = MaskParams.make()
    yaw = 0.3
    oc.mask_from_hydro(zone, mesh, yaw, (3.0, 7.0), math.hypot(1, 4), frame, mp)
    ij, h = zone.mask_cells()
    zo = port.zone(fc, 40.0, 3.0, 7.0, 1.0 / 60.0)
    zo.update_stability(math.hypot(1, 4), 1.0 / 60.0)
    ij_o, h_o = zo.compute_mask(res.waterline(), yaw, 3.0, 7.0, math.hypot(1, 4), frame, mp)
    assert len(h) > 1000
    assert np.array_equal(ij, ij_o)
    assert np.allclose(h, h_o, rtol=1e-12, atol=1e-12)
    f = zone.field()
    assert np.allclose(f[ij[:, 0], ij[:, 1]], h, rtol=1e-6, atol=1e-6)
