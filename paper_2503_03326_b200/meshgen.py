"""Synthetic hull fixtures (host-side, load-time).

The reference's make_box / make_hull always throw MeshError (SURVEY 2 note 1), so
the benchmark hull is a closed UV ellipsoid: `longitudes` x `bands` gives
2 + (bands - 1) * longitudes vertices and 2 * longitudes * (bands - 1) triangles
(256 x 197 -> 50,178 vertices, 100,352 triangles), outward-wound.
"""
import numpy as np


def uv_ellipsoid(longitudes=256, bands=197, half_axes=(5.0, 3.0, 20.0)):
    a, b, c = half_axes
    L, B = longitudes, bands
    theta = np.pi * np.arange(1, B) / B                 # polar angle of inner rings
    phi = 2.0 * np.pi * np.arange(L) / L
    st, ct = np.sin(theta)[:, None], np.cos(theta)[:, None]
    ring = np.stack([a * st * np.cos(phi)[None, :], b * ct * np.ones_like(phi)[None, :],
                     c * st * np.sin(phi)[None, :]], axis=-1).reshape(-1, 3)
    verts = np.concatenate([[[0.0, b, 0.0]], ring, [[0.0, -b, 0.0]]])
    top, bot = 0, verts.shape[0] - 1

    def rv(r, k):  # ring r in [0, B-2], longitude k
        return 1 + r * L + (k % L)

    tris = []
    for k in range(L):
        tris.append((top, rv(0, k + 1), rv(0, k)))
    for r in range(B - 2):
        for k in range(L):
            a0, a1 = rv(r, k), rv(r, k + 1)
            b0, b1 = rv(r + 1, k), rv(r + 1, k + 1)
            tris.append((a0, a1, b1))
            tris.append((a0, b1, b0))
    for k in range(L):
        tris.append((bot, rv(B - 2, k), rv(B - 2, k + 1)))
    return verts.astype(np.float64), np.asarray(tris, dtype=np.int32)


def unit_cube():
    """Closed, outward-wound unit cube centered at the origin (12 triangles)."""
    v = np.array([[x, y, z] for x in (-0.5, 0.5) for y in (-0.5, 0.5) for z in (-0.5, 0.5)])
    idx = lambda x, y, z: 4 * x + 2 * y + z
    quads = [
        (idx(0, 0, 0), idx(0, 0, 1), idx(0, 1, 1), idx(0, 1, 0)),  # -x
        (idx(1, 0, 0), idx(1, 1, 0), idx(1, 1, 1), idx(1, 0, 1)),  # +x
        (idx(0, 0, 0), idx(1, 0, 0), idx(1, 0, 1), idx(0, 0, 1)),  # -y
        (idx(0, 1, 0), idx(0, 1, 1), idx(1, 1, 1), idx(1, 1, 0)),  # +y
        (idx(0, 0, 0), idx(0, 1, 0), idx(1, 1, 0), idx(1, 0, 0)),  # -z
        (idx(0, 0, 1), idx(1, 0, 1), idx(1, 1, 1), idx(0, 1, 1)),  # +z
    ]
    tris = []
    for a, b, c_, d in quads:
        tris += [(a, b, c_), (a, c_, d)]
    return v.astype(np.float64), np.asarray(tris, dtype=np.int32)


def icosphere(radius=1.0, subdivisions=2):
    """Icosphere by midpoint subdivision (same construction family as mesh.cpp:223-258)."""
    t = (1.0 + 5 ** 0.5) / 2.0
    verts = [(-1, t, 0), (1, t, 0), (-1, -t, 0), (1, -t, 0), (0, -1, t), (0, 1, t), (0, -1, -t),
             (0, 1, -t), (t, 0, -1), (t, 0, 1), (-t, 0, -1), (-t, 0, 1)]
    verts = [np.array(v, float) for v in verts]
    faces = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11), (1, 5, 9), (5, 11, 4),
             (11, 10, 2), (10, 7, 6), (7, 1, 8), (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8),
             (3, 8, 9), (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1)]
    for _ in range(subdivisions):
        cache = {}

        def mid(a, b):
            key = (min(a, b), max(a, b))
            if key not in cache:
                cache[key] = len(verts)
                verts.append((verts[a] + verts[b]) / 2.0)
            return cache[key]

        nf = []
        for a, b, c in faces:
            ab, bc, ca = mid(a, b), mid(b, c), mid(c, a)
            nf += [(a, ab, ca), (b, bc, ab), (c, ca, bc), (ab, bc, ca)]
        faces = nf
    v = np.array([x * (radius / np.linalg.norm(x)) for x in verts])
    return v, np.asarray(faces, dtype=np.int32)
