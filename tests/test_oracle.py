"""CPU: pin the oracle restatement against the reference (golden fixtures made
by the reference build, and the live reference build where it exists)."""
import math

import numpy as np
import pytest

from helpers import (CONFIG2_CUTOFFS, CONFIG2_LENGTHS, DEFAULT_CUTOFFS, DEFAULT_LENGTHS,
                     config2_params, config3_pose, pose_from_array)
from paper_2503_03326_b200._types import (FdmConfig, MaskFrame, MaskParams, SliceConfig,
                                          SpectrumParams)
from paper_2503_03326_b200.meshgen import icosphere, unit_cube, uv_ellipsoid


def test_philox_and_gaussian_bit_exact(port, golden):
    for k, want in zip(golden["philox_in"], golden["philox_out"]):
        got = port.philox(*[int(x) for x in k])
        assert np.array_equal(got, want)
    for a, want in zip(golden["gauss_in"], golden["gauss_out"]):
        z = port.gaussian_complex(*[int(x) for x in a])
        assert z.real == want[0] and z.imag == want[1]


def test_scalar_known_answers(port, golden):
    p = config2_params()
    p0 = SpectrumParams.make()
    got = [
        port.scalar("dispersion", 1.0, 9.80665), port.scalar("beta_s", 1.0),
        port.scalar("beta_s", 0.5), port.scalar("beta_s", 1.6), port.scalar("q_dbxi_approx", 0.5),
        port.scalar("q_dbxi_approx", 150.0), port.scalar("damping_factor", 2.5, 0.98, 0.999, 5.0),
        port.jonswap(2.0 * port.scalar("peak_omega", p), p), port.scalar("directional", 0.9, 0.3, p),
        port.scalar("directional", 0.9, 0.3, p0),
        port.scalar("h0_variance", 0.03, -0.02, math.hypot(0.03, -0.02),
                    math.sqrt(9.80665 * math.hypot(0.03, -0.02)), 1024.0, p),
        port.scalar("q_dbxi_quadrature", 0.8, 1.0, 4096),
        port.scalar("swell_spread", 1.0, math.pi / 2, 1.0, 1.0), port.scalar("alpha", p),
        port.scalar("peak_omega", p0), port.scalar("standard_peak_omega", p0),
    ]
    np.testing.assert_array_equal(np.array(got), golden["scalars"])
    # SPEC.md known answers
    assert abs(got[0] - 3.131557) < 1e-6           # dispersion(1)
    assert got[1] == pytest.approx(2.28)            # beta_s(1)
    # q_dbxi_approx(0.5) (SPEC.md:102 quotes "2.81013..."; the printed coefficients give 2.8100996)
    assert got[4] == pytest.approx(7.1467551 * 0.25 - 13.4662001 * 0.5 + 7.75651088, abs=1e-12)
    assert got[6] == pytest.approx(0.9895)          # damping_factor(2.5)
    with pytest.raises(Exception):
        port.jonswap(0.0, p)


def test_generate_h0_bit_exact(port, golden):
    p = config2_params()
    for c in range(4):
        bmin = 0.0 if c == 0 else CONFIG2_CUTOFFS[c - 1]
        bmax = CONFIG2_CUTOFFS[c] if c < 3 else 1e300
        h0, h0cn, band, _ = port.generate_h0(16, CONFIG2_LENGTHS[c], bmin, bmax, p, c)
        assert np.array_equal(band, golden["c2_band"][c])
        assert np.array_equal(h0, golden["c2_h0"][c])
        assert np.array_equal(h0cn, golden["c2_h0cn"][c])
    h0, h0cn, band, waves = port.generate_h0(32, 256.0, 0.0, 1e300, SpectrumParams.make(), 0)
    assert np.array_equal(h0, golden["c1_h0"]) and np.array_equal(band, golden["c1_band"])
    assert np.array_equal(waves, golden["c1_waves"])


def test_fft_bit_exact(port, golden):
    for n in (8, 16):
        assert np.array_equal(port.ifft2_centered(golden[f"fft{n}_x"]), golden[f"fft{n}_centered"])
        re, im = port.ifft2_pair(golden[f"fft{n}_x"], golden[f"fft{n}_y"])
        assert np.array_equal(re, golden[f"fft{n}_re"]) and np.array_equal(im, golden[f"fft{n}_im"])


def test_maps_and_slices_bit_exact(port, golden):
    p = config2_params()
    assert np.array_equal(port.generate_maps(16, CONFIG2_LENGTHS, CONFIG2_CUTOFFS, p, 1 / 60.0),
                          golden["c2_maps_t1"])
    assert np.array_equal(port.generate_maps(16, CONFIG2_LENGTHS, CONFIG2_CUTOFFS, p, 10.0, 1.3),
                          golden["c2_maps_t10"])
    d, s = port.build_slices(16, CONFIG2_LENGTHS, CONFIG2_CUTOFFS, p, 1 / 60.0, SliceConfig.make(count=5))
    assert np.array_equal(d, golden["c2_depths5"]) and np.array_equal(s, golden["c2_slices5"])
    assert np.array_equal(port.generate_maps(32, [256.0], [], SpectrumParams.make(), 0.5),
                          golden["c1_maps"])


def test_samplers_bit_exact(port, golden):
    p = config2_params()
    maps = golden["c2_maps_t1"]
    xz = golden["samp_xz"]
    assert np.array_equal(port.height_at(16, CONFIG2_LENGTHS, maps, xz), golden["samp_height"])
    assert np.array_equal(port.sample_displacement(16, CONFIG2_LENGTHS, maps, xz), golden["samp_disp"])
    hv, it = port.height_at_tolerance(16, CONFIG2_LENGTHS, maps, xz, 0.01, 16)
    assert np.array_equal(hv, golden["samp_htol"]) and np.array_equal(it, golden["samp_htol_it"])
    cfg = SliceConfig.make(count=5)
    d, s = golden["c2_depths5"], golden["c2_slices5"]
    xzy = golden["samp_xzy"]
    assert np.array_equal(port.velocity_at_port(16, CONFIG2_LENGTHS, d, cfg, s, xzy, 0),
                          golden["samp_vel_exp"])
    assert np.array_equal(port.velocity_at_port(16, CONFIG2_LENGTHS, d, cfg, s, xzy, 1),
                          golden["samp_vel_lin"])
    assert np.array_equal(port.direct_velocity(16, CONFIG2_LENGTHS, CONFIG2_CUTOFFS, p, 1 / 60.0,
                                               xzy[:16]), golden["samp_direct"])


def test_mesh_and_aggregate_bit_exact(port, golden):
    mesh = port.mesh_build(golden["mesh_v"], golden["mesh_t"])
    for k in ("tris", "normals", "areas", "inertia", "centroid", "bbox_min", "bbox_max"):
        assert np.array_equal(np.asarray(mesh[k]), golden["mesh_" + k]), k
    cfg = SliceConfig.make(count=5)
    pose = pose_from_array(golden["pose"])
    rep, st, loops = port.aggregate(golden["mesh_v"], mesh, pose, n=16, lengths=CONFIG2_LENGTHS,
                                    maps=golden["c2_maps_t1"], slices=golden["c2_slices5"],
                                    depths=golden["c2_depths5"], slice_cfg=cfg, wind=(5, 0, 2))
    got = np.array([rep["submerged_volume"]] + rep["center_of_immersion"] + rep["buoyancy_force"]
                   + rep["water_drag"] + rep["air_drag"] + rep["water_center"] + rep["air_center"]
                   + [rep["submerged_area"], rep["dry_area"]] + rep["force"] + rep["torque"])
    np.testing.assert_array_equal(got, golden["agg_report"])
    assert [rep["state_count"], rep["waterline_loops"], rep["waterline_points"], rep["volume_clamped"],
            rep["has_center_of_immersion"], rep["degenerate_skipped"]] == list(golden["agg_counts"])
    assert np.array_equal(st["parent"], golden["agg_states_parent"])
    assert np.array_equal(st["status"], golden["agg_states_status"])
    assert np.array_equal(loops[0], golden["agg_loop0"])


def test_mask_and_fdm_bit_exact(port, golden):
    fc = FdmConfig.make(grid_size=128, margin=8)
    z = port.zone(fc, 12.0, 3.0, 7.0, 1.0 / 60.0)
    z.update_stability(math.hypot(1, 4), 1.0 / 60.0)
    mesh_vol = port.mesh_build(golden["mesh_v"], golden["mesh_t"])["volume"]
    frame = MaskFrame.make(center_x=0.0, half_beam=12.0, z_min=-6.0, z_max=6.0, mesh_height=12.0,
                           volume_ratio=golden["agg_report"][0] / mesh_vol)
    mp = MaskParams.make(back_height=0.1, intensity=1.0, amplitude=1.0)
    ij, h = z.compute_mask([golden["agg_loop0"]], 0.3, 3.0, 7.0, math.hypot(1, 4), frame, mp)
    assert np.array_equal(ij, golden["mask_ij"]) and np.array_equal(h, golden["mask_h"])
    z.apply_cells(ij, h)
    z.step(1.0 / 60.0, 3.0 + 1.0 / 60.0, 7.0 + 4.0 / 60.0)
    z.step(1.0 / 60.0, 3.0 + 2.0 / 60.0, 7.0 + 8.0 / 60.0)
    assert np.array_equal(z.field(), golden["fdm_field2"])
    st = z.state()
    np.testing.assert_array_equal([st["spacing"], st["wave_speed"], st["damping"]] + list(st["origin"]),
                                  golden["fdm_state"])


def test_spec_clipping_known_answers(port):
    """SPEC.md:420-450 unit-cube clipping / volume known answers (flat water)."""
    from paper_2503_03326_b200._types import Pose
    v, t = unit_cube()
    mesh = port.mesh_build(v, t)
    assert mesh["volume"] == pytest.approx(1.0)
    for y, vol, sub_area in [(-10.0, 1.0, 6.0), (10.0, 0.0, 0.0)]:
        rep, _, loops = port.aggregate(v, mesh, Pose.make(position=(0, y, 0)))
        assert rep["submerged_volume"] == pytest.approx(vol, abs=1e-9)
        assert rep["submerged_area"] == pytest.approx(sub_area, abs=1e-9)
        assert not loops
    # half submerged, tilted by a tiny yaw so no vertex sits exactly on y = 0
    rep, _, loops = port.aggregate(v, mesh, Pose.make(position=(0, 1e-7, 0)))
    assert rep["submerged_volume"] == pytest.approx(0.5, abs=1e-6)
    assert rep["center_of_immersion"][1] == pytest.approx(-0.25, abs=1e-3)
    assert rep["buoyancy_force"][1] == pytest.approx(1025 * 9.80665 * 0.5, rel=1e-5)
    assert len(loops) == 1 and np.allclose(loops[0][0], loops[0][-1])
    ico_v, ico_t = icosphere(2.0, 3)
    mesh = port.mesh_build(ico_v, ico_t)
    rep, _, _ = port.aggregate(ico_v, mesh, Pose.make(position=(0, -10, 0)))
    assert rep["submerged_volume"] == pytest.approx(mesh["volume"], rel=1e-6)


def test_theorem1_pair_equivalence(port):
    """SPEC.md:767 (Appendix C): packed pair == two separate transforms for Hermitian input."""
    rng = np.random.default_rng(3)
    for n in (8, 64):
        for _ in range(3):
            def herm():
                a = rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))
                ni = [(-i) % n if i else 0 for i in range(n)]
                b = np.conj(a[np.ix_(ni, ni)])
                h = 0.5 * (a + b)
                return h
            x, y = herm(), herm()
            re, im = port.ifft2_pair(x, y)
            np.testing.assert_allclose(re, port.ifft2_centered(x).real, atol=1e-9)
            np.testing.assert_allclose(im, port.ifft2_centered(y).real, atol=1e-9)


@pytest.mark.parametrize("n", [32, 64])
def test_port_matches_reference_live(port, ref, n):
    """Larger cases against the live reference build (skipped on the GPU box)."""
    p = config2_params(seed=9)
    mp = port.generate_maps(n, CONFIG2_LENGTHS, CONFIG2_CUTOFFS, p, 3.7)
    mr = ref.generate_maps(n, CONFIG2_LENGTHS, CONFIG2_CUTOFFS, p, 3.7)
    assert np.array_equal(mp, mr)
    cfg = SliceConfig.make(count=6, distribution=1)
    dp, sp = port.build_slices(n, DEFAULT_LENGTHS, DEFAULT_CUTOFFS, p, 2.0, cfg)
    dr, sr = ref.build_slices(n, DEFAULT_LENGTHS, DEFAULT_CUTOFFS, p, 2.0, cfg)
    assert np.array_equal(dp, dr) and np.array_equal(sp, sr)
    v, t = uv_ellipsoid(64, 49)
    mesh = port.mesh_build(v, t)
    pose = config3_pose(mesh["centroid"])
    cfg8 = SliceConfig.make(count=8)
    d8, s8 = port.build_slices(n, CONFIG2_LENGTHS, CONFIG2_CUTOFFS, p, 3.7, cfg8)
    a = port.aggregate(v, mesh, pose, n=n, lengths=CONFIG2_LENGTHS, maps=mp, slices=s8, depths=d8,
                       slice_cfg=cfg8, wind=(5, 0, 2))
    b = ref.aggregate(v, mesh, pose, n=n, lengths=CONFIG2_LENGTHS, maps=mr, slice_cfg=cfg8,
                      cutoffs=CONFIG2_CUTOFFS, params=p, t=3.7, wind=(5, 0, 2))
    assert a[0] == b[0]
    assert np.array_equal(a[1], b[1])
    assert all(np.array_equal(x, y) for x, y in zip(a[2], b[2]))


@pytest.mark.parametrize("n", [256, 1024])
def test_band_rows_outside_row_half_are_zero(port, n):
    """The premise of the device's band skipping: for every
    cascade, spectrum rows and columns with |i - N/2| >= row_half carry no mode
    of the band, so h0 there is exactly zero in the reference algorithm."""
    import math
    from helpers import CONFIG2_CUTOFFS, CONFIG2_LENGTHS, config2_params
    p = config2_params()
    for c, L in enumerate(CONFIG2_LENGTHS):
        bmin = 0.0 if c == 0 else CONFIG2_CUTOFFS[c - 1]
        bmax = CONFIG2_CUTOFFS[c] if c < len(CONFIG2_CUTOFFS) else 1e300
        h0, h0cn, band, _ = port.generate_h0(n, L, bmin, bmax, p, c)
        dk = 2 * math.pi / L
        rh = math.ceil(bmax * (1 + 1e-9) / dk)
        if rh > n // 2:
            continue  # every row may carry the band
        far = np.abs(np.arange(n) - n // 2) >= rh
        assert not band[far, :].any() and not band[:, far].any(), c
        assert np.all(h0[far, :] == 0) and np.all(h0[:, far] == 0), c
        assert np.all(h0cn[far, :] == 0), c


def test_surface_pair_large_equals_generate_maps(port):
    """The large-grid pair (per-mode h0 on the fly, threaded row / column
    transforms) used for the 16384^2 parity test is bit-identical to the
    restatement's generate_maps on the same grid, and its direct sums at grid
    nodes equal the transform to fp64 rounding."""
    from helpers import config2_params
    p = config2_params(seed=7)
    n, L, t = 128, 32.0, 10.0
    want = port.generate_maps(n, [L], [], p, t, 0.8)[0]
    ab = np.array([[0, 0], [5, 77], [127, 64], [64, 1]])
    for pair in range(4):
        re, im, direct = port.surface_pair_large(n, L, 0.0, 1e300, p, t, pair, choppiness=0.8,
                                                 threads=3, ab=ab)
        assert np.array_equal(re, want[2 * pair]) and np.array_equal(im, want[2 * pair + 1])
        at = re[ab[:, 0], ab[:, 1]] + 1j * im[ab[:, 0], ab[:, 1]]
        assert np.abs(direct - at).max() <= 1e-12 * max(np.abs(re).max(), np.abs(im).max())
