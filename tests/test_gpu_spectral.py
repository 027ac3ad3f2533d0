"""GPU parity: K1 spectrum init, fused coefficient + packed 2D IFFT, samplers
(CUDA path through the C-ABI) against the fp64 CPU oracle."""
import math

import numpy as np
import pytest

from helpers import (CONFIG2_CUTOFFS, CONFIG2_LENGTHS, DEFAULT_CUTOFFS, DEFAULT_LENGTHS,
                     config2_params, normwise_rel)
from paper_2503_03326_b200._types import SliceConfig, SpectrumParams

pytestmark = pytest.mark.gpu

TOL = 1e-4  # BASELINE.json north_star: max relative error <= 1e-4 (normwise per field)


@pytest.fixture(scope="module")
def oc():
    from paper_2503_03326_b200 import ocean
    return ocean


@pytest.mark.parametrize("n,params,lengths,cutoffs", [
    (64, "c2", CONFIG2_LENGTHS, CONFIG2_CUTOFFS),
    (256, "default", DEFAULT_LENGTHS, DEFAULT_CUTOFFS),
    (1024, "c2", CONFIG2_LENGTHS, CONFIG2_CUTOFFS),
])
def test_spectrum_init_band_bit_exact(oc, port, n, params, lengths, cutoffs):
    p = config2_params() if params == "c2" else SpectrumParams.make()
    cs = oc.CascadeSet(oc.CascadeConfig(n, lengths, cutoffs), p)
    for c, g in enumerate(cs.grids()):
        bmin = 0.0 if c == 0 else cutoffs[c - 1]
        bmax = cutoffs[c] if c + 1 < len(lengths) else 1e300
        h0, h0cn, band, waves = port.generate_h0(n, lengths[c], bmin, bmax, p, c)
        assert np.array_equal(g.in_band(), band), f"band mask differs in cascade {c}"
        np.testing.assert_array_equal(g.waves()[..., :2], waves[..., :2])
        assert np.array_equal(g.waves()[..., 2], waves[..., 2])  # |k| bit-exact (hypot)
        assert normwise_rel(g.h0(), h0) < 1e-12
        assert normwise_rel(g.h0_conj_neg(), h0cn) < 1e-12


@pytest.mark.parametrize("n", [2, 4, 8, 16, 32, 64, 128, 256, 512, 1024, 2048])
def test_ifft2_pair_and_centered(oc, port, n):
    rng = np.random.default_rng(n)
    x = rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))
    y = rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))
    re, im = oc.ifft2_hermitian_pair(x, y)
    r0, i0 = port.ifft2_pair(x, y)
    assert normwise_rel(re, r0) < 1e-5 and normwise_rel(im, i0) < 1e-5
    c = oc.ifft2_centered(x)
    assert normwise_rel(c, port.ifft2_centered(x)) < 1e-5


def test_ifft_errors(oc):
    with pytest.raises(oc.ConfigError):
        oc.ifft2_centered(np.zeros((6, 6), complex))


def _maps_case(oc, port, n, lengths, cutoffs, p, t, chop=1.0):
    cs = oc.CascadeSet(oc.CascadeConfig(n, lengths, cutoffs), p)
    maps = oc.generate_maps(cs, t, oc.SurfaceGenOptions(choppiness=chop))
    got = maps.all_fields()
    want = port.generate_maps(n, lengths, cutoffs, p, t, chop)
    for c in range(len(lengths)):
        for f in range(8):
            err = normwise_rel(got[c, f], want[c, f])
            assert err < TOL, f"cascade {c} field {f}: {err:.3e}"
    return cs, maps, want


def test_generate_maps_config1(oc, port):
    """reference defaults, single cascade 256^2 (Nyquist leak case)."""
    p = SpectrumParams.make()
    for t in (1.0 / 60.0, 10.0):
        _maps_case(oc, port, 256, [256.0], [], p, t)


def test_generate_maps_config2_small(oc, port):
    _maps_case(oc, port, 64, CONFIG2_LENGTHS, CONFIG2_CUTOFFS, config2_params(), 3.0, 1.3)


def test_generate_maps_config2_full(oc, port):
    """Config 2 surface at full size (4 x 1024^2), t = 10 s (phases ~1e3 rad)."""
    _maps_case(oc, port, 1024, CONFIG2_LENGTHS, CONFIG2_CUTOFFS, config2_params(), 10.0)


@pytest.mark.parametrize("n", [2048, 4096])
def test_generate_maps_large(oc, port, n):
    """Large single grids: the TMA column pass at 8 / 4 / 2 columns per tile
    and its store epilogues (TMA store up to 2048, direct stores at 4096)."""
    _maps_case(oc, port, n, [float(n)], [], config2_params(seed=3), 4.0, 0.8)


@pytest.mark.parametrize("n,count,dist", [(64, 7, 0), (128, 8, 1), (256, 32, 0), (1024, 3, 0)])
def test_build_slices(oc, port, n, count, dist):
    p = config2_params(seed=5)
    cfg = SliceConfig.make(count=count, distribution=dist)
    cs = oc.CascadeSet(oc.CascadeConfig(n, CONFIG2_LENGTHS, CONFIG2_CUTOFFS), p)
    vs = oc.build_slices(cs, 2.5, cfg)
    d_ref, s_ref = port.build_slices(n, CONFIG2_LENGTHS, CONFIG2_CUTOFFS, p, 2.5, cfg)
    np.testing.assert_array_equal(vs.depths(), d_ref)
    got = vs.all_fields()
    # Tolerance per slice and component, normalised by the slice's scale over all
    # cascades (velocity_at sums the cascades): deep slices of the short cascades
    # are ~1e-130 in fp64 and underflow to 0 in fp32, which is physically exact.
    for d in range(count):
        for k in range(3):
            err = normwise_rel(got[d, :, k], s_ref[d, :, k])
            assert err < TOL, f"depth {d} comp {k}: {err:.3e}"


def test_samplers(oc, port):
    n, p = 128, config2_params(seed=11)
    cfg = SliceConfig.make(count=8)
    cs = oc.CascadeSet(oc.CascadeConfig(n, CONFIG2_LENGTHS, CONFIG2_CUTOFFS), p)
    maps = oc.generate_maps(cs, 1.5)
    vs = oc.build_slices(cs, 1.5, cfg)
    want_maps = port.generate_maps(n, CONFIG2_LENGTHS, CONFIG2_CUTOFFS, p, 1.5)
    d_ref, s_ref = port.build_slices(n, CONFIG2_LENGTHS, CONFIG2_CUTOFFS, p, 1.5, cfg)
    rng = np.random.default_rng(1)
    xz = rng.uniform(-800, 800, size=(4096, 2))
    h = oc.height_at(maps, xz)
    assert normwise_rel(h, port.height_at(n, CONFIG2_LENGTHS, want_maps, xz)) < TOL
    d = maps.sample_displacement(xz)
    assert normwise_rel(d, port.sample_displacement(n, CONFIG2_LENGTHS, want_maps, xz)) < TOL
    ht, it = oc.height_at_tolerance(maps, xz, 0.01, 16)
    ht_ref, it_ref = port.height_at_tolerance(n, CONFIG2_LENGTHS, want_maps, xz, 0.01, 16)
    assert normwise_rel(ht, ht_ref) < 1e-3 and np.mean(it == it_ref) > 0.98
    y = rng.uniform(-125.0, 4.5, size=4096)
    xzy = np.concatenate([xz, y[:, None]], axis=1)
    for interp in (0, 1):
        v = oc.velocity_at(vs, xz, y, interp)
        v_ref = port.velocity_at_port(n, CONFIG2_LENGTHS, d_ref, cfg, s_ref, xzy, interp)
        assert normwise_rel(v, v_ref) < TOL
    for i in (0, 5, 7):
        assert normwise_rel(vs.sample_slice(i, xz),
                            port.sample_slice_port(n, CONFIG2_LENGTHS, d_ref, cfg, s_ref, i, xz)) < TOL
    with pytest.raises(oc.DomainError):
        oc.velocity_at(vs, xz[:2], [-200.0, 0.0])
    vc = oc.velocity_at(vs, xz[:2], [-200.0, 10.0], clamp=True)
    assert np.all(np.isfinite(vc))


def test_slices_vs_direct_sum(oc, port):
    """At a slice depth and grid nodes the slice pipeline equals the direct
    spectral sum (velocity.cpp:24-59) up to the packed-transform Nyquist leak
    the reference itself has (SURVEY 7 hard part 2): the device result must
    deviate from the direct sum exactly as much as the reference does."""
    n, p = 32, config2_params(seed=3)
    cfg = SliceConfig.make(count=6)
    cs = oc.CascadeSet(oc.CascadeConfig(n, CONFIG2_LENGTHS, CONFIG2_CUTOFFS), p)
    vs = oc.build_slices(cs, 0.7, cfg)
    dep = vs.depths()
    d_ref, s_ref = port.build_slices(n, CONFIG2_LENGTHS, CONFIG2_CUTOFFS, p, 0.7, cfg)
    L0 = CONFIG2_LENGTHS[-1]
    xz = np.stack(np.meshgrid(np.arange(4) * L0 / n, np.arange(4) * L0 / n), -1).reshape(-1, 2)
    for di in (1, 3, 5):
        y = np.full(xz.shape[0], dep[di])
        xzy = np.concatenate([xz, y[:, None]], axis=1)
        direct = port.direct_velocity(n, CONFIG2_LENGTHS, CONFIG2_CUTOFFS, p, 0.7, xzy)
        ref = port.velocity_at_port(n, CONFIG2_LENGTHS, d_ref, cfg, s_ref, xzy)
        got = oc.velocity_at(vs, xz, y)
        assert normwise_rel(got, ref) < TOL
        assert abs(normwise_rel(got, direct) - normwise_rel(ref, direct)) < TOL


def test_assembly_properties(oc, port):
    """North-star item 3: J and normal from the sampled derivative maps agree with
    finite differences of the displaced surface X(p) = p + D(p)."""
    n, p = 256, SpectrumParams.make(wind_speed=8.0)
    cs = oc.CascadeSet(oc.CascadeConfig(n, [256.0], []), p)
    maps = oc.generate_maps(cs, 2.0)
    rng = np.random.default_rng(2)
    xz = rng.uniform(0, 256, size=(512, 2))
    a = oc.surface_assemble(maps, xz)
    assert np.allclose(a[:, 1], oc.height_at(maps, xz))
    nrm = a[:, 3:6]
    assert np.allclose(np.linalg.norm(nrm, axis=1), 1.0)
    # finite-difference Jacobian of X(p) = p + D(p) at the Algorithm-1 point p
    pts = xz - a[:, [0, 2]]
    eps = 1e-3
    def disp(q):
        d = maps.sample_displacement(q)
        return q + d[:, [0, 2]]
    jx = (disp(pts + [eps, 0]) - disp(pts - [eps, 0])) / (2 * eps)
    jz = (disp(pts + [0, eps]) - disp(pts - [0, eps])) / (2 * eps)
    J_fd = jx[:, 0] * jz[:, 1] - jx[:, 1] * jz[:, 0]
    corr = np.corrcoef(J_fd, a[:, 6])[0, 1]
    assert corr > 0.9, corr


def test_instances_batched(oc, port):
    """Config 4 shape: independent instances (own seeds) synthesised by one
    spectral step over a multi-grid set; each instance equals its own oracle run."""
    from paper_2503_03326_b200._types import SpectrumParams
    cfg = oc.CascadeConfig(64, [256.0, 16.0, 4.0], [12 * math.pi / 16, 12 * math.pi / 4])
    params = [config2_params(seed=s) for s in (0, 7, 63)]
    inst = oc.CascadeInstances(cfg, params)
    maps = oc.SurfaceMaps(inst)
    maps.generate(2.0)
    for k, p in enumerate(params):
        want = port.generate_maps(64, list(cfg.lengths), list(cfg.cutoffs), p, 2.0)
        for c in range(3):
            for f in range(8):
                got = maps.field(3 * k + c, f)
                assert normwise_rel(got, want[c, f]) < TOL, (k, c, f)


def test_frames_batch_small(oc, port):
    """Time-batched set (config 1 shape, 3 cascades): frame f at t0 + f dt."""
    p = config2_params(seed=2)
    cfg = oc.CascadeConfig(64, CONFIG2_LENGTHS[1:], CONFIG2_CUTOFFS[1:])
    frames = oc.CascadeFrames(cfg, p, 5, 0.25)
    maps = oc.SurfaceMaps(frames)
    maps.generate_batch(1.0, 0.5)  # the call's dt overrides the set's
    for f in range(5):
        want = port.generate_maps(64, cfg.lengths, cfg.cutoffs, p, 1.0 + 0.5 * f)
        for c in range(3):
            for k in range(8):
                assert normwise_rel(maps.field(3 * f + c, k), want[c, k]) < TOL, (f, c, k)
    maps.generate(2.0)  # the set's own spacing
    want = port.generate_maps(64, cfg.lengths, cfg.cutoffs, p, 2.0 + 0.25 * 4)
    assert normwise_rel(maps.field(3 * 4 + 1, 0), want[1, 0]) < TOL
    with pytest.raises(oc.ConfigError):
        oc.height_at(maps, [[0.0, 0.0]])


def test_assembly_grid_small(oc, port):
    p = config2_params(seed=4)
    cs = oc.CascadeSet(oc.CascadeConfig(128, CONFIG2_LENGTHS, CONFIG2_CUTOFFS), p)
    maps = oc.SurfaceMaps(cs).set_assembly(True)
    maps.generate(3.0, 0.9)
    want = port.generate_maps(128, CONFIG2_LENGTHS, CONFIG2_CUTOFFS, p, 3.0, 0.9)
    for c in range(4):
        got = maps.assembly(c)
        hx, hz = want[c, 6], want[c, 7]
        inv = 1.0 / np.sqrt(hx * hx + 1.0 + hz * hz)
        ref = [-hx * inv, inv, -hz * inv,
               (1 - want[c, 3]) * (1 - want[c, 5]) - want[c, 4] ** 2]
        for k in range(4):
            assert normwise_rel(got[k], ref[k]) < TOL, (c, k)
