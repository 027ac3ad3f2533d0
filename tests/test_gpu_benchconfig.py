"""GPU parity at the benchmarked configurations themselves, not at
reduced sizes: the CUDA path through the C-ABI against the fp64 CPU oracle.

* config 2/3 spectral step: 4 x 1024^2 maps + 32 logarithmic velocity slices
  through the fused plan the bench runs (ocn_spectral_step(maps, slices)), at
  t = 1/60 and t = 10 s, including which transforms the plan drops as exactly
  zero and the spectrum row band each executed transform keeps;
* config 3 forces: the 100,352-triangle hull over those maps and slices;
* config 4: four of the 64 instances of the batched 3 x 512^2 set;
* config 5: packed 16384^2 transforms of the slab path against
  ifft2_hermitian_pair (fft.cpp:79-101) and against direct spectral sums.
"""
import math

import numpy as np
import pytest

from helpers import (CONFIG2_CUTOFFS, CONFIG2_LENGTHS, config2_params, config3_pose, normwise_rel,
                     vec_rel)
from paper_2503_03326_b200._types import SliceConfig

pytestmark = pytest.mark.gpu
TOL = 1e-4  # BASELINE.json north_star: max relative error <= 1e-4
N = 1024
DEPTHS = 32
LOG2E = 1.4426950408889634


@pytest.fixture(scope="module")
def oc():
    from paper_2503_03326_b200 import ocean
    return ocean


@pytest.fixture(scope="module")
def bench_set(oc):
    """The bench's spectral set (bench.py Frame): config-2 spectrum, seed 42."""
    p = config2_params()
    cfg = SliceConfig.make(count=DEPTHS)
    cs = oc.CascadeSet(oc.CascadeConfig(N, CONFIG2_LENGTHS, CONFIG2_CUTOFFS), p)
    maps = oc.SurfaceMaps(cs)
    vs = oc.VelocitySlices(cs, cfg)
    return p, cfg, cs, maps, vs


@pytest.fixture(scope="module")
def oracle_frame(port, bench_set):
    """Oracle maps + slices at t = 1/60 (shared by the spectral and force tests)."""
    p, cfg, _, _, _ = bench_set
    t = 1.0 / 60.0
    tables = port.cascade_tables(N, CONFIG2_LENGTHS, CONFIG2_CUTOFFS, p)
    m = port.generate_maps(N, CONFIG2_LENGTHS, CONFIG2_CUTOFFS, p, t, tables=tables)
    d, s = port.build_slices(N, CONFIG2_LENGTHS, CONFIG2_CUTOFFS, p, t, cfg, tables=tables)
    return t, tables, m, d, s


def _check_frame(oc, maps, vs, m_ref, d_ref, s_ref):
    np.testing.assert_array_equal(vs.depths(), d_ref)
    got = maps.all_fields()
    for c in range(len(CONFIG2_LENGTHS)):
        for f in range(8):
            err = normwise_rel(got[c, f], m_ref[c, f])
            assert err < TOL, f"maps cascade {c} field {f}: {err:.3e}"
    sl = vs.all_fields()
    worst = 0.0
    for d in range(DEPTHS):
        for k in range(3):
            err = normwise_rel(sl[d, :, k], s_ref[d, :, k])
            worst = max(worst, err)
            assert err < TOL, f"slice depth {d} comp {k}: {err:.3e}"
    return worst


def _expected_plan(depths):
    """The drop / row-band rules restated from first principles: grid c holds
    modes with band_min <= |k| < band_max only; a velocity coefficient at depth
    y < 0 carries exp(|k| y), which the fp32 row pass evaluates as
    ex2.approx(|k| y log2 e) and flushes to 0 below 2^-132."""
    bmin = [0.0] + CONFIG2_CUTOFFS
    bmax = CONFIG2_CUTOFFS + [1e300]
    out = []
    for c, L in enumerate(CONFIG2_LENGTHS):
        dk = 2 * math.pi / L
        rg = math.ceil(bmax[c] * (1 + 1e-9) / dk)
        grid_rows = N // 2 + 1 if rg > N // 2 else rg

        def rows(y):
            if not y < 0:
                return N // 2 + 1
            kmax = 132.0 / (-y * LOG2E) * (1 + 1e-5)
            r = math.ceil(kmax / dk)
            return N // 2 + 1 if r > N // 2 else r

        def dead(y):
            return y < 0 and bmin[c] * (1 - 1e-5) * (-y) * LOG2E >= 132.0

        ys = [float(np.float32(y)) for y in depths]
        for d in range(DEPTHS):
            out.append((c, 4, d, min(grid_rows, rows(ys[d])), not dead(ys[d])))
        for d0 in range(0, DEPTHS, 2):
            out.append((c, 5, d0, min(grid_rows, max(rows(ys[d0]), rows(ys[d0 + 1]))),
                        not (dead(ys[d0]) and dead(ys[d0 + 1]))))
    return out


def test_bench_spectral_step_t_first_frame(oc, bench_set, oracle_frame):
    """ocn_spectral_step at the bench's own configuration, first frame (t = 1/60)."""
    _, _, _, maps, vs = bench_set
    t, _, m_ref, d_ref, s_ref = oracle_frame
    oc.spectral_step(maps, vs, t)
    worst = _check_frame(oc, maps, vs, m_ref, d_ref, s_ref)
    print(f"1024^2 x 32 slices, t = 1/60: worst slice error {worst:.2e}")


def test_bench_spectral_step_t10(oc, port, bench_set, oracle_frame):
    """Same plan at t = 10 s (phases ~1e3 rad, SURVEY 7 hard part 3)."""
    p, cfg, _, maps, vs = bench_set
    _, tables, _, _, _ = oracle_frame
    t = 10.0
    oc.spectral_step(maps, vs, t)
    m_ref = port.generate_maps(N, CONFIG2_LENGTHS, CONFIG2_CUTOFFS, p, t, tables=tables)
    d_ref, s_ref = port.build_slices(N, CONFIG2_LENGTHS, CONFIG2_CUTOFFS, p, t, cfg, tables=tables)
    _check_frame(oc, maps, vs, m_ref, d_ref, s_ref)


def test_bench_plan_drops_and_row_bands(oc, bench_set, oracle_frame):
    """The transforms the bench plan drops (44 of 208 at config 3) and the row
    band each executed transform keeps, against (1) the rule restated here and
    (2) the oracle's own fields: a dropped transform's planes are below 1e-30 of
    the slice scale in fp64, and the spectrum rows a transform skips carry no
    more than 1e-12 of its largest coefficient (forward FFT of the oracle planes)."""
    _, _, _, maps, vs = bench_set
    _, _, m_ref, d_ref, s_ref = oracle_frame
    plan = oc.spectral_plan(maps, vs)
    assert len(plan) == 4 * 4 + 4 * (DEPTHS + DEPTHS // 2)
    surf, vel = plan[:16], plan[16:]
    assert all(x["executed"] == 1 for x in surf)
    # ceil(band_max (1 + 1e-9) / dk) per grid: rows |i - N/2| < 25, 97, 25 (all for the last)
    grid_rows = [25, 97, 25, N // 2 + 1]
    for x in surf:
        assert x["row_half"] == grid_rows[x["cascade"]], x
    want = _expected_plan(d_ref)
    got = [(x["cascade"], x["kind"], x["index0"], x["row_half"], bool(x["executed"])) for x in vel]
    assert got == want
    dropped = [x for x in vel if not x["executed"]]
    assert len(dropped) == 44
    assert sum(1 for x in dropped if x["cascade"] == 3) == 31
    assert sum(1 for x in dropped if x["cascade"] == 2) == 13
    scale = [np.abs(s_ref[d]).max() for d in range(DEPTHS)]
    for x in dropped:
        c, d0 = x["cascade"], x["index0"]
        ds = [d0] if x["kind"] == 4 else [d0, x["index1"]]
        comps = [0, 2] if x["kind"] == 4 else [1]
        for d in ds:
            for k in comps:
                assert np.abs(s_ref[d, c, k]).max() <= 1e-30 * scale[d], (x, d, k)
    # skipped rows of the executed velocity transforms: the forward FFT of the
    # oracle's packed output recovers its coefficient spectrum (fft.cpp:69-77);
    # the coefficients in the skipped rows can move the slice by at most their
    # L1 norm, which must vanish against the slice scale (fp64 noise ~1e-13)
    ii = np.arange(N)
    sign = np.where(((ii[:, None] + ii[None, :]) & 1) == 1, -1.0, 1.0)
    checked = 0
    for x in vel:
        if not x["executed"] or x["row_half"] > N // 2:
            continue
        c, d0 = x["cascade"], x["index0"]
        if x["kind"] == 4:
            packed = s_ref[d0, c, 0] + 1j * s_ref[d0, c, 2]
            ds = [d0]
        else:
            packed = s_ref[d0, c, 1] + 1j * s_ref[x["index1"], c, 1]
            ds = [d0, x["index1"]]
        coef = np.abs(np.fft.fft2(packed * sign)) / N**2
        outside = np.abs(ii - N // 2) >= x["row_half"]
        assert coef[outside].sum() <= 1e-10 * min(scale[d] for d in ds), x
        checked += 1
    assert checked == 143


def test_bench_forces_full_size(oc, port, bench_set, oracle_frame):
    """Config 3 forces: 100,352-triangle hull at the bench pose over the 4 x 1024^2
    maps and 32 slices (device) vs the oracle on its own fp64 maps / slices.
    Forces, torque, submerged volume and centre within 1e-4; vertex depth sign
    flips (fp32 vs fp64 maps) and the resulting state / loop deltas reported."""
    from paper_2503_03326_b200.meshgen import uv_ellipsoid
    _, cfg, _, maps, vs = bench_set
    t, _, m_ref, d_ref, s_ref = oracle_frame
    oc.spectral_step(maps, vs, t)
    v, tr = uv_ellipsoid()
    assert tr.shape[0] == 100352 and v.shape[0] == 50178
    mesh_g = oc.TriMesh(v, tr)
    mesh_o = port.mesh_build(v, tr)
    pose = config3_pose(mesh_o["centroid"])
    res = oc.aggregate(mesh_g, pose, oc.FluidQuery(maps=maps, slices=vs, wind=(5, 0, 2)))
    rep, st, loops = port.aggregate(v, mesh_o, pose, n=N, lengths=CONFIG2_LENGTHS, maps=m_ref,
                                    slices=s_ref, depths=d_ref, slice_cfg=cfg, wind=(5, 0, 2))
    for k in ("buoyancy_force", "water_drag", "air_drag", "force", "torque", "water_center",
              "air_center", "center_of_immersion"):
        err = vec_rel(getattr(res, k), rep[k])
        assert err <= TOL, (k, err, getattr(res, k), rep[k])
    assert abs(res.submerged_volume - rep["submerged_volume"]) <= TOL * rep["submerged_volume"]
    _, dg = res.vertices()
    # oracle vertex depths on its own fp64 maps (same pose transform)
    import ctypes as C
    from oracle.oracle import P
    from oracle.oracle_structs import OrcFluid
    wpos = np.zeros((v.shape[0], 3))
    do = np.zeros(v.shape[0])
    surf = port._surface(N, CONFIG2_LENGTHS, m_ref)
    fl = OrcFluid()
    fl.surface = C.cast(C.pointer(surf), C.c_void_p)
    f = port.lib.orc_vertex_depths
    f.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    f(v.shape[0], P(v), C.byref(pose), C.byref(fl), P(wpos), P(do))
    flips = int(np.sum((dg >= 0) != (do >= 0)))
    assert normwise_rel(dg, do) < TOL
    print(f"config 3 forces: states {res.state_count} vs {rep['state_count']}, loops "
          f"{res.waterline_loops} vs {rep['waterline_loops']}, vertex sign flips {flips}")
    if flips == 0:
        assert res.state_count == rep["state_count"]
        assert res.waterline_loops == rep["waterline_loops"]
    else:
        assert abs(res.state_count - rep["state_count"]) <= 2 * flips


def test_config4_instances_full_size(oc, port):
    """Config 4: the 64-instance batched 3 x 512^2 set the bench runs; instances
    0, 21, 42 and 63 (own seeds) against their own oracle generate_maps."""
    lengths = [256.0, 16.0, 4.0]
    cutoffs = [12 * math.pi / 16, 12 * math.pi / 4]
    params = [config2_params(seed=s) for s in range(64)]
    inst = oc.CascadeInstances(oc.CascadeConfig(512, lengths, cutoffs), params)
    maps = oc.SurfaceMaps(inst)
    t = 10.0
    maps.generate(t)
    for k in (0, 21, 42, 63):
        want = port.generate_maps(512, lengths, cutoffs, params[k], t)
        for c in range(3):
            for f in range(8):
                err = normwise_rel(maps.field(3 * k + c, f), want[c, f])
                assert err < TOL, (k, c, f, err)


@pytest.mark.parametrize("pair", [0, 2])
def test_config5_packed_transform_16384(port, pair):
    """Config 5 at full size: the slab path (1 rank) builds the 16384^2 surface;
    packed pair `pair` (surface.cpp:77-80) against the oracle's
    ifft2_hermitian_pair of the same coefficients (fft.cpp:79-101), and 16 grid
    nodes against the direct spectral sum of the packed spectrum."""
    import torch
    from paper_2503_03326_b200.slab import SlabSurface, tile_layout
    n, L, t = 16384, 4096.0, 10.0
    p = config2_params(seed=7)
    slab = SlabSurface(n, 1, 0, L, p)
    _, total = tile_layout(slab.rows, 1)
    buf = torch.empty(2 * total, dtype=torch.float32, device="cuda:0")
    slab.rows_pass(t, buf.data_ptr())
    slab.cols_pass(buf.data_ptr())
    slab.ctx.synchronize()
    del buf
    torch.cuda.empty_cache()
    rng = np.random.default_rng(pair)
    ab = np.concatenate([[[0, 0], [n - 1, n - 1], [n // 2, 7]], rng.integers(0, n, size=(13, 2))])
    re_ref, im_ref, direct = port.surface_pair_large(n, L, 0.0, 1e300, p, t, pair, ab=ab)
    got_re = slab.field(2 * pair)
    assert normwise_rel(got_re, re_ref) < TOL
    got_at = got_re[ab[:, 0], ab[:, 1]]
    del got_re
    got_im = slab.field(2 * pair + 1)
    assert normwise_rel(got_im, im_ref) < TOL
    got_at = got_at + 1j * got_im[ab[:, 0], ab[:, 1]]
    del got_im
    ref_at = re_ref[ab[:, 0], ab[:, 1]] + 1j * im_ref[ab[:, 0], ab[:, 1]]
    scale = max(np.abs(re_ref).max(), np.abs(im_ref).max())
    # the oracle FFT equals the definition (fp64 rounding) and the device equals both
    assert np.abs(direct - ref_at).max() <= 1e-9 * scale
    assert np.abs(got_at - direct).max() <= TOL * scale


def _assembly_ref(maps_c):
    """SURVEY 8a row 10 applied to one grid's oracle maps [8][N][N]."""
    hx, hz = maps_c[6], maps_c[7]
    dxdx, dzdx, dzdz = maps_c[3], maps_c[4], maps_c[5]
    inv = 1.0 / np.sqrt(hx * hx + 1.0 + hz * hz)
    return np.stack([-hx * inv, inv, -hz * inv, (1.0 - dxdx) * (1.0 - dzdz) - dzdx * dzdx])


def test_bench_assembly_grid_full_size(oc, bench_set, oracle_frame):
    """North-star item 3 as a grid product at config 2: per-texel normal and
    Jacobian written by the spectral step, against the formula on the oracle's
    fp64 maps (every grid, every component, 1e-4 normwise)."""
    _, _, _, maps, vs = bench_set
    t, _, m_ref, _, _ = oracle_frame
    maps.set_assembly(True)
    try:
        oc.spectral_step(maps, vs, t)
        for c in range(len(CONFIG2_LENGTHS)):
            got = maps.assembly(c)
            want = _assembly_ref(m_ref[c])
            for k in range(4):
                err = normwise_rel(got[k], want[k])
                assert err < TOL, (c, k, err)
    finally:
        maps.set_assembly(False)


def test_config1_frames_full_size(oc, port):
    """Config 1: reference defaults, one 256^2 cascade, 600 frames at
    t_f = (f + 1) / 60 synthesised by one batched spectral step; frames 0, 299
    and 599 against the oracle's generate_maps at their times, and every checked
    frame bit-identical to a single-frame step at the same t."""
    from paper_2503_03326_b200._types import SpectrumParams
    p = SpectrumParams.make()
    cfg = oc.CascadeConfig(256, [256.0], [])
    dt = 1.0 / 60.0
    frames = oc.CascadeFrames(cfg, p, 600, dt)
    maps = oc.SurfaceMaps(frames)
    maps.generate_batch(dt, dt)
    single = oc.SurfaceMaps(oc.CascadeSet(cfg, p))
    for f in (0, 299, 599):
        t = dt + f * dt
        want = port.generate_maps(256, [256.0], [], p, t)[0]
        single.generate(t)
        for k in range(8):
            got = maps.field(f, k)
            assert normwise_rel(got, want[k]) < TOL, (f, k)
            assert np.array_equal(got, single.field(0, k)), (f, k)
