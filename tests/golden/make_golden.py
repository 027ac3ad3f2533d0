"""Generate tests/golden/*.npz from the REFERENCE build (oracle/_ref/libocean_ref.so).

Run here (where /root/reference exists):  python tests/golden/make_golden.py
The fixtures pin the oracle restatement (tests/test_oracle.py) and travel to
the GPU box, where /root/reference does not exist. Every array is produced by
the unmodified reference library compiled from /root/reference/proj/src.
"""
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import Oracle, build  # noqa: E402
from paper_2503_03326_b200._types import (FdmConfig, MaskFrame, MaskParams, Pose,  # noqa: E402
                                          SliceConfig, SpectrumParams)
from paper_2503_03326_b200.meshgen import icosphere, uv_ellipsoid  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

CONFIG2_LENGTHS = [1024.0, 256.0, 16.0, 4.0]
CONFIG2_CUTOFFS = [12 * math.pi / 256, 12 * math.pi / 16, 12 * math.pi / 4]


def config2_params(seed=42):
    """U=20, F=1e5, theta0=0.4, xi=0.5, delta=0.5, standard peak."""
    p = SpectrumParams.make(wind_speed=20.0, fetch=1e5, wind_direction=0.4, swell=0.5,
                            direction_mix=0.5, rng_seed=seed)
    p.has_peak_omega_override = 1
    p.peak_omega_override = p.standard_peak_omega()
    return p


def main():
    build(reference=True)
    r = Oracle("reference")
    g = {}
    # ---- rng.hpp: Philox words and Gaussian draws
    keys = [(0, 0x6F63656E00000000, 0, 0), (42, 0x6F63656E00000003, (5 << 32) | 7, 0),
            (2**64 - 1, 2**63 + 5, 123456789, 987654321)]
    g["philox_in"] = np.array(keys, dtype=np.uint64)
    g["philox_out"] = np.array([r.philox(*k) for k in keys], dtype=np.uint32)
    gin = [(0, 0, 0, 0), (42, 3, 511, 17), (7, 1, 1023, 1023), (2**40 + 3, 2, 9, 250)]
    g["gauss_in"] = np.array(gin, dtype=np.uint64)
    gz = [r.gaussian_complex(*a) for a in gin]
    g["gauss_out"] = np.array([[z.real, z.imag] for z in gz])
    # ---- spectrum scalars (SPEC known answers + config-2 params)
    p = config2_params()
    p0 = SpectrumParams.make()
    g["scalars"] = np.array([
        r.scalar("dispersion", 1.0, 9.80665), r.scalar("beta_s", 1.0), r.scalar("beta_s", 0.5),
        r.scalar("beta_s", 1.6), r.scalar("q_dbxi_approx", 0.5), r.scalar("q_dbxi_approx", 150.0),
        r.scalar("damping_factor", 2.5, 0.98, 0.999, 5.0), r.jonswap(2.0 * r.scalar("peak_omega", p), p),
        r.scalar("directional", 0.9, 0.3, p), r.scalar("directional", 0.9, 0.3, p0),
        r.scalar("h0_variance", 0.03, -0.02, math.hypot(0.03, -0.02),
                 math.sqrt(9.80665 * math.hypot(0.03, -0.02)), 1024.0, p),
        r.scalar("q_dbxi_quadrature", 0.8, 1.0, 4096), r.scalar("swell_spread", 1.0, math.pi / 2, 1.0, 1.0),
        r.scalar("alpha", p), r.scalar("peak_omega", p0), r.scalar("standard_peak_omega", p0),
    ])
    # ---- generate_h0 / CascadeSet at N=16 (config-2 params) and N=32 (defaults, 1 cascade)
    n = 16
    h0, h0cn, band = [], [], []
    for c in range(4):
        bmin = 0.0 if c == 0 else CONFIG2_CUTOFFS[c - 1]
        bmax = CONFIG2_CUTOFFS[c] if c < 3 else 1e300
        a, b, m, _ = r.generate_h0(n, CONFIG2_LENGTHS[c], bmin, bmax, p, c)
        h0.append(a)
        h0cn.append(b)
        band.append(m)
    g["c2_h0"], g["c2_h0cn"], g["c2_band"] = np.array(h0), np.array(h0cn), np.array(band)
    g["c2_maps_t1"] = r.generate_maps(n, CONFIG2_LENGTHS, CONFIG2_CUTOFFS, p, 1.0 / 60.0)
    g["c2_maps_t10"] = r.generate_maps(n, CONFIG2_LENGTHS, CONFIG2_CUTOFFS, p, 10.0, choppiness=1.3)
    cfg = SliceConfig.make(count=5)
    d, s = r.build_slices(n, CONFIG2_LENGTHS, CONFIG2_CUTOFFS, p, 1.0 / 60.0, cfg)
    g["c2_depths5"], g["c2_slices5"] = d, s
    p1 = SpectrumParams.make()
    a, b, m, w = r.generate_h0(32, 256.0, 0.0, 1e300, p1, 0)
    g["c1_h0"], g["c1_h0cn"], g["c1_band"], g["c1_waves"] = a, b, m, w
    g["c1_maps"] = r.generate_maps(32, [256.0], [], p1, 0.5)
    # ---- FFT
    rng = np.random.default_rng(7)
    for nn in (8, 16):
        x = rng.normal(size=(nn, nn)) + 1j * rng.normal(size=(nn, nn))
        y = rng.normal(size=(nn, nn)) + 1j * rng.normal(size=(nn, nn))
        g[f"fft{nn}_x"], g[f"fft{nn}_y"] = x, y
        g[f"fft{nn}_centered"] = r.ifft2_centered(x)
        re, im = r.ifft2_pair(x, y)
        g[f"fft{nn}_re"], g[f"fft{nn}_im"] = re, im
    # ---- samplers on the N=16 config-2 maps
    xz = rng.uniform(-600, 600, size=(64, 2))
    g["samp_xz"] = xz
    g["samp_height"] = r.height_at(n, CONFIG2_LENGTHS, g["c2_maps_t1"], xz)
    g["samp_disp"] = r.sample_displacement(n, CONFIG2_LENGTHS, g["c2_maps_t1"], xz)
    hv, it = r.height_at_tolerance(n, CONFIG2_LENGTHS, g["c2_maps_t1"], xz, 0.01, 16)
    g["samp_htol"], g["samp_htol_it"] = hv, it
    xzy = np.concatenate([xz, rng.uniform(-125.0, 4.5, size=(64, 1))], axis=1)
    xzy[0, 2], xzy[1, 2], xzy[2, 2] = -125.0, 4.5, d[2]  # endpoints and an exact slice depth
    g["samp_xzy"] = xzy
    g["samp_vel_exp"] = r.velocity_at_ref(n, CONFIG2_LENGTHS, CONFIG2_CUTOFFS, p, 1.0 / 60.0, cfg, xzy, 0)
    g["samp_vel_lin"] = r.velocity_at_ref(n, CONFIG2_LENGTHS, CONFIG2_CUTOFFS, p, 1.0 / 60.0, cfg, xzy, 1)
    g["samp_direct"] = r.direct_velocity(n, CONFIG2_LENGTHS, CONFIG2_CUTOFFS, p, 1.0 / 60.0, xzy[:16])
    # ---- mesh + aggregate (icosphere r=6 on the N=16 maps)
    v, t = icosphere(6.0, 2)
    mesh = r.mesh_build(v, t)
    g["mesh_v"], g["mesh_t"] = v, t
    for k in ("tris", "normals", "areas", "inertia", "centroid", "bbox_min", "bbox_max"):
        g["mesh_" + k] = np.asarray(mesh[k])
    g["mesh_scalars"] = np.array([mesh["volume"], mesh["total_area"], mesh["degenerate"]])
    yaw = 0.3
    pose = Pose.make(position=(3.0, 0.5, 7.0), orientation=(math.cos(yaw / 2), 0, math.sin(yaw / 2), 0),
                     linear_velocity=(1, 0, 4), angular_velocity=(0.01, 0.05, 0.02),
                     com_body=mesh["centroid"])
    g["pose"] = np.array(list(pose.position) + list(pose.orientation) + list(pose.linear_velocity)
                         + list(pose.angular_velocity) + list(pose.com_body))
    rep, states, loops = r.aggregate(v, mesh, pose, n=n, lengths=CONFIG2_LENGTHS, maps=g["c2_maps_t1"],
                                     slice_cfg=cfg, cutoffs=CONFIG2_CUTOFFS, params=p, t=1.0 / 60.0,
                                     wind=(5, 0, 2))
    g["agg_report"] = np.array([rep["submerged_volume"]] + rep["center_of_immersion"]
                               + rep["buoyancy_force"] + rep["water_drag"] + rep["air_drag"]
                               + rep["water_center"] + rep["air_center"]
                               + [rep["submerged_area"], rep["dry_area"]] + rep["force"] + rep["torque"])
    g["agg_counts"] = np.array([rep["state_count"], rep["waterline_loops"], rep["waterline_points"],
                                rep["volume_clamped"], rep["has_center_of_immersion"],
                                rep["degenerate_skipped"]])
    g["agg_states_parent"] = states["parent"]
    g["agg_states_status"] = states["status"]
    g["agg_states_f"] = np.concatenate([states["area"][:, None], states["centroid"],
                                        states["depth"][:, None], states["normal"]], axis=1)
    g["agg_loop0"] = loops[0] if loops else np.zeros((0, 3))
    # ---- FDM zone + mask (N=128 zone)
    fc = FdmConfig.make(grid_size=128, margin=8)
    z = r.zone(fc, 12.0, 3.0, 7.0, 1.0 / 60.0)
    z.update_stability(math.hypot(1, 4), 1.0 / 60.0)
    frame = MaskFrame.make(center_x=0.0, half_beam=12.0, z_min=-6.0, z_max=6.0, mesh_height=12.0,
                           volume_ratio=rep["submerged_volume"] / mesh["volume"])
    mp = MaskParams.make(back_height=0.1, intensity=1.0, amplitude=1.0)
    ij, hh = z.compute_mask(loops, yaw, 3.0, 7.0, math.hypot(1, 4), frame, mp)
    g["mask_ij"], g["mask_h"] = ij, hh
    z.apply_cells(ij, hh)
    z.step(1.0 / 60.0, 3.0 + 1.0 / 60.0, 7.0 + 4.0 / 60.0)
    z.step(1.0 / 60.0, 3.0 + 2.0 / 60.0, 7.0 + 8.0 / 60.0)
    g["fdm_field2"] = z.field()
    st = z.state()
    g["fdm_state"] = np.array([st["spacing"], st["wave_speed"], st["damping"]] + list(st["origin"]))
    np.savez_compressed(os.path.join(OUT, "golden_ref.npz"), **g)
    print("wrote", os.path.join(OUT, "golden_ref.npz"), len(g), "arrays")


if __name__ == "__main__":
    main()
