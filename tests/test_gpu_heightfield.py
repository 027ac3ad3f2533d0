"""GPU parity: the composed surface (Simulation::compose_height, sim.cpp:44-51)
and the ABHF writers fed from device fields (heightfield_io.cpp:30-45,
dump_fields main.cpp:59-90), against the CPU oracle."""
import math
import os

import numpy as np
import pytest

from helpers import CONFIG2_CUTOFFS, CONFIG2_LENGTHS, config2_params, normwise_rel
from paper_2503_03326_b200._types import FdmConfig

pytestmark = pytest.mark.gpu
TOL = 1e-4
N = 64
T = 0.75


@pytest.fixture(scope="module")
def oc():
    from paper_2503_03326_b200 import ocean
    return ocean


@pytest.fixture(scope="module")
def scene(oc, port):
    p = config2_params()
    cs = oc.CascadeSet(oc.CascadeConfig(N, CONFIG2_LENGTHS, CONFIG2_CUTOFFS), p)
    maps = oc.SurfaceMaps(cs).generate(T)
    want = port.generate_maps(N, CONFIG2_LENGTHS, CONFIG2_CUTOFFS, p, T)
    rng = np.random.default_rng(5)
    fc = FdmConfig.make(grid_size=128, margin=16)
    zones, ozones = [], []
    for body, size in (((3.0, 7.0), 40.0), ((-20.0, 5.0), 30.0)):
        f = np.zeros((128, 128))
        f[16:-16, 16:-16] = rng.normal(scale=0.3, size=(96, 96))
        f = f.astype(np.float32).astype(np.float64)  # the device zone field is fp32
        zg = oc.FdmZone(fc, size, body, 1.0 / 60.0)
        zg.set_fields(f, np.zeros_like(f))
        zo = port.zone(fc, size, body[0], body[1], 1.0 / 60.0)
        zo.set_field(f)
        zones.append(zg)
        ozones.append(zo)
    return maps, want, zones, ozones


def _oracle_compose(port, want, ozones, xz):
    h = port.height_at(N, CONFIG2_LENGTHS, want, xz)
    for zo in ozones:
        h = h + np.array([zo.sample(x, z) for x, z in xz])
    return h


def test_compose_height(oc, port, scene):
    maps, want, zones, ozones = scene
    rng = np.random.default_rng(11)
    xz = np.concatenate([rng.uniform(-40, 40, size=(400, 2)), rng.uniform(-3000, 3000, size=(100, 2))])
    got = oc.compose_height(maps, xz, zones)
    ref = _oracle_compose(port, want, ozones, xz)
    assert normwise_rel(got, ref) <= TOL
    # no zones: exactly height_at (the same device Algorithm 1)
    assert np.array_equal(oc.compose_height(maps, xz), oc.height_at(maps, xz))
    # excluding a body = leaving its zone out of the list (sim.cpp:47)
    ref1 = _oracle_compose(port, want, ozones[1:], xz)
    assert normwise_rel(oc.compose_height(maps, xz, zones[1:]), ref1) <= TOL


def test_compose_grid(oc, port, scene):
    maps, want, zones, ozones = scene
    res, extent = 48, CONFIG2_LENGTHS[0]
    got = oc.compose_grid(maps, res, extent, zones)
    i, j = np.meshgrid(np.arange(res), np.arange(res), indexing="ij")
    xz = np.stack([extent * i / res, extent * j / res], -1).reshape(-1, 2)
    ref = _oracle_compose(port, want, ozones, xz).reshape(res, res)
    assert normwise_rel(got, ref) <= TOL
    assert np.array_equal(got.ravel(), oc.compose_height(maps, xz, zones))


def test_field_file(oc, scene, tmp_path):
    maps = scene[0]
    for c, f in ((0, 0), (3, 7), (1, 4)):
        p = tmp_path / f"c{c}f{f}.abhf"
        oc.write_field_heightfield(str(p), maps, c, f, T)
        data, hdr = oc.read_heightfield(str(p))
        assert hdr == {"resolution": N, "cascade": c, "time": float(np.float32(T))}
        # the device field bytes, unchanged (fp32 on the device already)
        assert np.array_equal(data, maps.field(c, f))
        assert os.path.getsize(p) == 16 + 4 * N * N


def test_composed_file_and_dump(oc, scene, tmp_path):
    maps, _, zones, _ = scene
    res, extent = 40, CONFIG2_LENGTHS[0]
    p = tmp_path / "composed.abhf"
    oc.write_composed_heightfield(str(p), maps, res, extent, T, zones)
    data, hdr = oc.read_heightfield(str(p))
    assert hdr == {"resolution": res, "cascade": -1, "time": float(np.float32(T))}
    grid = oc.compose_grid(maps, res, extent, zones)
    np.testing.assert_allclose(data, grid.astype(np.float32), rtol=2e-7, atol=1e-7 * np.abs(grid).max())
    d = tmp_path / "dump"
    oc.dump_fields(maps, str(d), T, res, zones)
    names = sorted(os.listdir(d))
    assert len(names) == 1 + 4 * 8 and "surface_composed_t0.750.abhf" in names
    assert "cascade3_dh_dz_t0.750.abhf" in names
    h, hdr = oc.read_heightfield(str(d / "cascade2_h_t0.750.abhf"))
    assert hdr["cascade"] == 2 and np.array_equal(h, maps.field(2, 0))


def test_errors(oc, scene, tmp_path):
    maps = scene[0]
    with pytest.raises(oc.IoError, match="cannot open for writing"):
        oc.write_field_heightfield(str(tmp_path / "no" / "x.abhf"), maps, 0, 0, T)
    with pytest.raises(oc.ConfigError):
        oc.compose_grid(maps, 0, 1.0)
    with pytest.raises(oc.ArgumentError):
        oc.write_field_heightfield(str(tmp_path / "x.abhf"), maps, 4, 0, T)
