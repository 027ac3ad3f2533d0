"""The reference's own caller on the drop-in: the reference's
sim.cpp, rigid_body.cpp and scenario.cpp, unmodified, compiled against this
repo's include/ and linked with libocean_api.so (oracle/Makefile target
`caller` -> oracle/_ref/ref_caller_b200), step a two-body JSON scenario; the
same driver over the reference library itself (ref_caller_cpu) is the oracle.

Simulation::step builds FluidQuery from host lambdas (sim.cpp:77-80): the
surface sampler runs per vertex through the drop-in's height_at / zone
sampling, the velocity sampler is called back by ocn_hydro_aggregate with the
submerged states batched (ocn_fluid::host_velocity)."""
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
B200 = os.path.join(ROOT, "oracle", "_ref", "ref_caller_b200")
CPU = os.path.join(ROOT, "oracle", "_ref", "ref_caller_cpu")


def _run(exe, *args):
    if not os.path.exists(exe):
        pytest.skip(f"{os.path.basename(exe)} not built (needs /root/reference at build time)")
    r = subprocess.run([exe, *args], capture_output=True, text=True, timeout=600)
    return r.returncode, r.stdout


def _parse(out):
    rows, heights = [], []
    for ln in out.splitlines():
        if ln.startswith("H "):
            heights.append([float(x) for x in ln.split()[1:]])
        elif ln and ln[0].isdigit():
            rows.append([float(x) for x in ln.split()])
    return np.array(rows), np.array(heights)


def test_reference_simulation_runs_on_dropin():
    rc_g, out_g = _run(B200, "twobody", "24")
    rc_c, out_c = _run(CPU, "twobody", "24")
    assert rc_c == 0, out_c
    assert rc_g == 0, out_g
    g, hg = _parse(out_g)
    c, hc = _parse(out_c)
    assert g.shape == c.shape == (48, 23)
    assert np.array_equal(g[:, :3], c[:, :3])  # step, body, time
    pos, vel, quat = slice(3, 6), slice(6, 9), slice(9, 13)
    assert np.abs(g[:, pos] - c[:, pos]).max() <= 1e-5  # metres
    assert np.abs(g[:, vel] - c[:, vel]).max() <= 1e-4 * np.abs(c[:, vel]).max()
    assert np.abs(g[:, quat] - c[:, quat]).max() <= 1e-6
    vol = c[:, 13]
    assert np.all(np.abs(g[:, 13] - vol) <= 1e-4 * vol)
    for cols in (slice(14, 15), slice(15, 18), slice(18, 21)):  # buoyancy, water / air drag
        ref = c[:, cols]
        den = np.linalg.norm(ref, axis=1)
        err = np.linalg.norm(g[:, cols] - ref, axis=1)
        assert np.all(err <= 1e-4 * np.maximum(den, 1e-9)), (cols, (err / den).max())
    # mask cell counts: the same waterline gives the same cells, up to cells
    # whose centre lies within rounding of the fp32-surface waterline
    assert np.all(np.abs(g[:, 22] - c[:, 22]) <= 0.01 * c[:, 22] + 2)
    scale = np.abs(hc[:, 2]).max()
    assert np.abs(hg[:, 2] - hc[:, 2]).max() <= 1e-4 * scale


@pytest.mark.parametrize("primitive", ["box", "hull"])
def test_reference_primitives_throw_like_reference(primitive):
    """make_box / make_hull (mesh.hpp:58-63) fail closed-mesh validation in the
    reference (SURVEY 2 note 1); the drop-in throws the same MeshError."""
    rc_g, out_g = _run(B200, primitive, "1")
    rc_c, out_c = _run(CPU, primitive, "1")
    assert rc_c == 3 and rc_g == 3
    assert out_g == out_c
