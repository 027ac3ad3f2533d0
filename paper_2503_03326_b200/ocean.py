"""Python mirror of the reference's hot-path API (proj/include/ocean/*.hpp) over
the C-ABI of libocean_b200.so. Same names, argument meaning and error
behaviour (ConfigError / MeshError / NumericError / DomainError); results are
device-resident and materialised on access.

    cs   = CascadeSet(CascadeConfig(resolution=1024, lengths=..., cutoffs=...), params)
    maps = generate_maps(cs, t)                      # surface.hpp:83
    vs   = build_slices(cs, t, SliceConfig(count=32)) # velocity.hpp:89
    h    = height_at(maps, xz)                        # surface.hpp:88 (batched)
    v    = velocity_at(vs, xz, y)                     # velocity.hpp:102
    rep  = aggregate(mesh, pose, FluidQuery(maps, vs, wind=...))   # hydro.hpp:112
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _abi
from ._abi import (ArgumentError, ConfigError, DomainError, IoError, MeshError, NumericError,  # noqa: F401
                   OceanCudaError, OceanError, check, lib)
from ._types import (FdmConfig, Fluid, HydroReport, MaskFrame, MaskParams, Pose, SliceConfig,
                     SpectrumParams, TriangleState, ZoneState)

kGravity = 9.80665
kPi = math.pi
kFieldH, kFieldDx, kFieldDz, kFieldDxDx, kFieldDzDx, kFieldDzDz, kFieldHx, kFieldHz = range(8)
kHeightRetrievalIters = 4


def _dp(a):
    return a.ctypes.data_as(_abi.d)


class Context:
    """One device + one CUDA stream (ocn_ctx)."""

    _default: dict[int, "Context"] = {}

    def __init__(self, device: int = 0, priority: int = 0):
        """priority: 1 highest, -1 lowest, 0 default stream priority."""
        h = C.c_void_p()
        check(lib().ocn_ctx_create_priority(device, priority, C.byref(h)), None, "ocn_ctx_create")
        self.h = h
        self.device = device

    @classmethod
    def default(cls, device: int = 0) -> "Context":
        if device not in cls._default:
            cls._default[device] = Context(device)
        return cls._default[device]

    def synchronize(self):
        check(lib().ocn_ctx_synchronize(self.h), self.h, "synchronize")

    @property
    def stream(self) -> int:
        return lib().ocn_ctx_stream(self.h) or 0

    def kernel_launches(self) -> int:
        return int(lib().ocn_ctx_kernel_launches(self.h))

    def __del__(self):
        try:
            if self.h:
                lib().ocn_ctx_destroy(self.h)
                self.h = None
        except Exception:
            pass


# --------------------------------------------------------------------- spectra
@dataclass
class GridConfig:
    """spectra.hpp:81-87"""
    resolution: int = 256
    length: float = 256.0
    band_min: float = 0.0
    band_max: float = 1e300


@dataclass
class CascadeConfig:
    """surface.hpp:18-25"""
    resolution: int = 256
    lengths: Sequence[float] = (256.0, 16.0, 4.0)
    cutoffs: Sequence[float] = (12.0 * math.pi / 16.0, 12.0 * math.pi / 4.0)

    def validate(self):
        if not self.lengths:
            raise ConfigError("at least one cascade is required")
        if len(self.cutoffs) + 1 != len(self.lengths):
            raise ConfigError("cascade cutoffs must number one less than cascade lengths")
        for i in range(1, len(self.lengths)):
            if not self.lengths[i] < self.lengths[i - 1]:
                raise ConfigError("cascade lengths must be strictly decreasing")
        for i in range(1, len(self.cutoffs)):
            if not self.cutoffs[i] > self.cutoffs[i - 1]:
                raise ConfigError("cascade cutoffs must be increasing")
        n = self.resolution
        if n < 2 or n & (n - 1):
            raise ConfigError("cascade resolution must be a power of two >= 2")


class _Grids:
    """Device spectrum tables for one or more grids of one resolution (ocn_cascades)."""

    def __init__(self, ctx, n, lengths, bmin, bmax, cindex, params: SpectrumParams):
        self.ctx = ctx or Context.default()
        self.params = params
        self.n = n
        self.lengths = list(lengths)
        cnt = len(self.lengths)
        la = np.ascontiguousarray(self.lengths, np.float64)
        bl = np.ascontiguousarray(bmin, np.float64)
        bh = np.ascontiguousarray(bmax, np.float64)
        ci = np.ascontiguousarray(cindex, np.uint32)
        h = C.c_void_p()
        check(lib().ocn_cascades_create(self.ctx.h, n, cnt, _dp(la), _dp(bl), _dp(bh),
                                        ci.ctypes.data_as(_abi.u32), C.byref(params), C.byref(h)),
              self.ctx.h, "generate_h0")
        self.h = h

    def download(self, g):
        n = self.n
        h0 = np.zeros((n, n), np.complex128)
        h0cn = np.zeros((n, n), np.complex128)
        band = np.zeros((n, n), np.uint8)
        waves = np.zeros((n, n, 4))
        check(lib().ocn_cascades_download(self.h, g, _dp(h0.view(np.float64)),
                                          _dp(h0cn.view(np.float64)),
                                          band.ctypes.data_as(_abi.u8), _dp(waves)),
              self.ctx.h, "download")
        return h0, h0cn, band.astype(bool), waves

    def __del__(self):
        try:
            if self.h:
                lib().ocn_cascades_destroy(self.h)
                self.h = None
        except Exception:
            pass


class WaveGrid:
    """spectra.hpp:91-118 — one grid's tables (materialised from the device)."""

    def __init__(self, grids: _Grids, index: int, band_min: float, band_max: float):
        self._g, self._i = grids, index
        self._cache = None
        self.band_min, self.band_max = band_min, band_max

    def _load(self):
        if self._cache is None:
            self._cache = self._g.download(self._i)
        return self._cache

    def resolution(self):
        return self._g.n

    def length(self):
        return self._g.lengths[self._i]

    def gravity(self):
        return self._g.params.gravity

    def h0(self):
        return self._load()[0]

    def h0_conj_neg(self):
        return self._load()[1]

    def in_band(self):
        return self._load()[2]

    def waves(self):
        return self._load()[3]


def generate_h0(config: GridConfig, params: SpectrumParams, cascade_index: int = 0,
                ctx: Context = None) -> WaveGrid:
    """spectra.hpp:122-123, on the device (K1)."""
    g = _Grids(ctx, config.resolution, [config.length], [config.band_min], [config.band_max],
               [cascade_index], params)
    return WaveGrid(g, 0, config.band_min, config.band_max)


class CascadeSet:
    """surface.hpp:27-40"""

    def __init__(self, config: CascadeConfig, params: SpectrumParams, ctx: Context = None):
        config.validate()
        self.config = config
        self.params = params
        C_ = len(config.lengths)
        bmin = [0.0 if c == 0 else config.cutoffs[c - 1] for c in range(C_)]
        bmax = [config.cutoffs[c] if c + 1 < C_ else 1e300 for c in range(C_)]
        self._g = _Grids(ctx, config.resolution, config.lengths, bmin, bmax, list(range(C_)), params)
        self.ctx = self._g.ctx
        self.h = self._g.h
        self._grids = [WaveGrid(self._g, c, bmin[c], bmax[c]) for c in range(C_)]

    def grids(self):
        return self._grids


class CascadeInstances:
    """Batched independent scenes: every instance is a
    CascadeSet of `config` with its own SpectrumParams (e.g. its own seed); one
    spectral step synthesises all of them (ocn_cascades_create_multi)."""

    def __init__(self, config: CascadeConfig, params_list: Sequence[SpectrumParams],
                 ctx: Context = None):
        config.validate()
        self.config = config
        self.instances = len(params_list)
        C_ = len(config.lengths)
        lengths, bmin, bmax, cidx, ps = [], [], [], [], []
        for p in params_list:
            for c in range(C_):
                lengths.append(config.lengths[c])
                bmin.append(0.0 if c == 0 else config.cutoffs[c - 1])
                bmax.append(config.cutoffs[c] if c + 1 < C_ else 1e300)
                cidx.append(c)
                ps.append(p)
        self.ctx = ctx or Context.default()
        arr = (SpectrumParams * len(ps))(*ps)
        la = np.ascontiguousarray(lengths, np.float64)
        bl = np.ascontiguousarray(bmin, np.float64)
        bh = np.ascontiguousarray(bmax, np.float64)
        ci = np.ascontiguousarray(cidx, np.uint32)
        h = C.c_void_p()
        check(lib().ocn_cascades_create_multi(self.ctx.h, config.resolution, len(ps), _dp(la), _dp(bl),
                                              _dp(bh), ci.ctypes.data_as(_abi.u32), arr, C.byref(h)),
              self.ctx.h, "cascade instances")
        self.h = h
        self.grids = len(ps)

    def __del__(self):
        try:
            if self.h:
                lib().ocn_cascades_destroy(self.h)
                self.h = None
        except Exception:
            pass


class CascadeFrames:
    """Time-batched frames of one CascadeSet: frame f is the
    cascade set at t0 + f dt, and one spectral step synthesises every frame
    (ocn_cascades_create_frames; generate_maps is a pure function of t,
    surface.cpp:70-103). Maps of it are [frames][C][8][N][N]."""

    def __init__(self, config: CascadeConfig, params: SpectrumParams, frames: int,
                 dt: float = 1.0 / 60.0, ctx: Context = None):
        config.validate()
        self.config = config
        self.params = params
        self.frames = frames
        self.dt = dt
        C_ = len(config.lengths)
        bmin = [0.0 if c == 0 else config.cutoffs[c - 1] for c in range(C_)]
        bmax = [config.cutoffs[c] if c + 1 < C_ else 1e300 for c in range(C_)]
        self.ctx = ctx or Context.default()
        la = np.ascontiguousarray(config.lengths, np.float64)
        bl = np.ascontiguousarray(bmin, np.float64)
        bh = np.ascontiguousarray(bmax, np.float64)
        ci = np.ascontiguousarray(list(range(C_)), np.uint32)
        h = C.c_void_p()
        check(lib().ocn_cascades_create_frames(self.ctx.h, config.resolution, C_, _dp(la), _dp(bl),
                                               _dp(bh), ci.ctypes.data_as(_abi.u32), C.byref(params),
                                               frames, dt, C.byref(h)),
              self.ctx.h, "cascade frames")
        self.h = h
        self.grids = frames * C_

    def __del__(self):
        try:
            if self.h:
                lib().ocn_cascades_destroy(self.h)
                self.h = None
        except Exception:
            pass


# --------------------------------------------------------------------- surface
@dataclass
class SurfaceGenOptions:
    choppiness: float = 1.0
    single_precision: bool = False  # outputs are fp32 on the device either way


class SurfaceMaps:
    """surface.hpp:65-80 — device-resident fp32 maps; `cascades[c].fields[f]`
    materialise lazily (fp64 numpy arrays)."""

    class _Cascade:
        def __init__(self, maps, c):
            self._m, self._c = maps, c
            self.length = maps.cascade_set.config.lengths[c]

        @property
        def fields(self):
            return [self._m.field(self._c, f) for f in range(8)]

    def __init__(self, cascade_set: CascadeSet):
        self.cascade_set = cascade_set
        self.ctx = cascade_set.ctx
        h = C.c_void_p()
        check(lib().ocn_maps_create(cascade_set.h, C.byref(h)), self.ctx.h, "maps_create")
        self.h = h
        self.time = 0.0

    @property
    def cascades(self):
        return [SurfaceMaps._Cascade(self, c) for c in range(len(self.cascade_set.config.lengths))]

    def generate(self, t, choppiness=1.0):
        check(lib().ocn_surface_generate(self.h, t, choppiness), self.ctx.h, "generate_maps")
        self.time = t
        return self

    def generate_batch(self, t0, dt, choppiness=1.0):
        """Every frame of a CascadeFrames set: frame f at t0 + f dt (async)."""
        check(lib().ocn_surface_generate_batch(self.h, t0, dt, choppiness), self.ctx.h,
              "generate_batch")
        self.time = t0
        return self

    def set_assembly(self, enable: bool = True):
        """Per-texel normal + Jacobian planes written by every spectral step."""
        check(lib().ocn_maps_set_assembly(self.h, int(enable)), self.ctx.h, "set_assembly")
        return self

    def assembly(self, grid) -> np.ndarray:
        """[4][N][N] fp32: nx, ny, nz, J of grid `grid`."""
        n = self.cascade_set.config.resolution
        out = np.zeros((4, n, n), np.float32)
        for k in range(4):
            check(lib().ocn_maps_download_assembly(self.h, grid, k,
                                                   out[k].ctypes.data_as(_abi.f32)),
                  self.ctx.h, "assembly")
        return out

    def field(self, cascade, f) -> np.ndarray:
        n = self.cascade_set.config.resolution
        out = np.zeros((n, n))
        check(lib().ocn_maps_download(self.h, cascade, f, _dp(out)), self.ctx.h, "download")
        return out

    def all_fields(self) -> np.ndarray:
        C_ = len(self.cascade_set.config.lengths)
        return np.stack([np.stack([self.field(c, f) for f in range(8)]) for c in range(C_)])

    def sample(self, f, xz):
        xz = np.ascontiguousarray(np.atleast_2d(xz), np.float64)
        out = np.zeros(xz.shape[0])
        check(lib().ocn_maps_sample(self.h, f, xz.shape[0], _dp(xz), _dp(out)), self.ctx.h, "sample")
        return out

    def sample_displacement(self, xz):
        xz = np.ascontiguousarray(np.atleast_2d(xz), np.float64)
        out = np.zeros((xz.shape[0], 3))
        check(lib().ocn_sample_displacement(self.h, xz.shape[0], _dp(xz), _dp(out)), self.ctx.h,
              "sample_displacement")
        return out

    def __del__(self):
        try:
            if self.h:
                lib().ocn_maps_destroy(self.h)
                self.h = None
        except Exception:
            pass


def generate_maps(cascades: CascadeSet, t: float, options: SurfaceGenOptions = SurfaceGenOptions(),
                  out: SurfaceMaps = None) -> SurfaceMaps:
    """surface.hpp:83-84 (K2 + K4 on the device)."""
    m = out or SurfaceMaps(cascades)
    return m.generate(t, options.choppiness)


def height_at(maps: SurfaceMaps, xz) -> np.ndarray:
    """surface.hpp:88, batched over points (N, 2) -> (N,)."""
    xz = np.ascontiguousarray(np.atleast_2d(xz), np.float64)
    out = np.zeros(xz.shape[0])
    check(lib().ocn_height_at(maps.h, xz.shape[0], _dp(xz), _dp(out)), maps.ctx.h, "height_at")
    return out


def height_at_tolerance(maps: SurfaceMaps, xz, tol: float, max_iters: int):
    """surface.hpp:93-94 -> (heights, iterations)."""
    xz = np.ascontiguousarray(np.atleast_2d(xz), np.float64)
    out = np.zeros(xz.shape[0])
    it = np.zeros(xz.shape[0], np.int32)
    check(lib().ocn_height_at_tolerance(maps.h, xz.shape[0], _dp(xz), tol, max_iters, _dp(out),
                                        it.ctypes.data_as(_abi.i32)), maps.ctx.h, "height_at_tol")
    return out, it


def surface_assemble(maps: SurfaceMaps, xz) -> np.ndarray:
    """North-star item 3: (dx, h, dz, nx, ny, nz, J, DxDx, DzDx, DzDz) per point."""
    xz = np.ascontiguousarray(np.atleast_2d(xz), np.float64)
    out = np.zeros((xz.shape[0], 10))
    check(lib().ocn_surface_assemble(maps.h, xz.shape[0], _dp(xz), _dp(out)), maps.ctx.h, "assemble")
    return out


# -------------------------------------------------------------------- velocity
class VelocitySlices:
    """velocity.hpp:64-86 — device-resident fp32 slices."""

    def __init__(self, cascade_set: CascadeSet, config: SliceConfig):
        self.cascade_set = cascade_set
        self.ctx = cascade_set.ctx
        self.config = config
        h = C.c_void_p()
        check(lib().ocn_slices_create(cascade_set.h, C.byref(config), C.byref(h)), self.ctx.h,
              "build_slices")
        self.h = h
        self._depths = np.zeros(config.count)
        cnt = C.c_int()
        check(lib().ocn_slices_depths(self.h, C.byref(cnt), _dp(self._depths)), self.ctx.h, "depths")

    def depths(self):
        return self._depths.copy()

    def y_min(self):
        return self.config.y_min

    def y_max(self):
        return self.config.y_max

    def build(self, t):
        check(lib().ocn_velocity_build(self.h, t), self.ctx.h, "build_slices")
        return self

    def field(self, depth, cascade, comp) -> np.ndarray:
        n = self.cascade_set.config.resolution
        out = np.zeros((n, n))
        check(lib().ocn_slices_download(self.h, depth, cascade, comp, _dp(out)), self.ctx.h,
              "download")
        return out

    def all_fields(self) -> np.ndarray:
        D, C_ = self.config.count, len(self.cascade_set.config.lengths)
        return np.stack([np.stack([np.stack([self.field(d, c, k) for k in range(3)])
                                   for c in range(C_)]) for d in range(D)])

    def sample_slice(self, i, xz):
        xz = np.ascontiguousarray(np.atleast_2d(xz), np.float64)
        out = np.zeros((xz.shape[0], 3))
        check(lib().ocn_sample_slice(self.h, i, xz.shape[0], _dp(xz), _dp(out)), self.ctx.h,
              "sample_slice")
        return out

    def __del__(self):
        try:
            if self.h:
                lib().ocn_slices_destroy(self.h)
                self.h = None
        except Exception:
            pass


def build_slices(cascades: CascadeSet, t: float, config: SliceConfig,
                 out: VelocitySlices = None) -> VelocitySlices:
    """velocity.hpp:89 (K3 + K4 on the device)."""
    s = out or VelocitySlices(cascades, config)
    return s.build(t)


def velocity_at(slices: VelocitySlices, xz, y, interp: int = 0, clamp: bool = False) -> np.ndarray:
    """velocity.hpp:102-103, batched: xz (N, 2), y (N,) -> (N, 3)."""
    xz = np.atleast_2d(np.asarray(xz, np.float64))
    y = np.broadcast_to(np.asarray(y, np.float64), (xz.shape[0],))
    xzy = np.ascontiguousarray(np.concatenate([xz, y[:, None]], axis=1))
    out = np.zeros((xz.shape[0], 3))
    check(lib().ocn_velocity_at(slices.h, xz.shape[0], _dp(xzy), interp, int(clamp), _dp(out)),
          slices.ctx.h, "velocity_at")
    return out


def spectral_step(maps: Optional[SurfaceMaps], slices: Optional[VelocitySlices], t: float,
                  choppiness: float = 1.0):
    """generate_maps + build_slices of one frame, enqueued together (async)."""
    check(lib().ocn_spectral_step(maps.h if maps else None, slices.h if slices else None, t,
                                  choppiness),
          (maps or slices).ctx.h, "spectral_step")


def spectral_plan(maps: Optional[SurfaceMaps], slices: Optional[VelocitySlices]) -> list:
    """The packed transforms of spectral_step(maps, slices) in plan order
    (ocn_spectral_plan_info): kind, grid, depth / field indices, the skipped
    row band and whether the transform runs per frame."""
    from ._types import XformInfo
    L = lib()
    ctx = (maps or slices).ctx
    n = C.c_int()
    args = (maps.h if maps else None, slices.h if slices else None)
    check(L.ocn_spectral_plan_info(*args, 0, None, C.byref(n)), ctx.h, "plan_info")
    arr = (XformInfo * max(n.value, 1))()
    check(L.ocn_spectral_plan_info(*args, n.value, arr, C.byref(n)), ctx.h, "plan_info")
    return [{k: getattr(x, k) for k, _ in XformInfo._fields_} for x in arr[:n.value]]


# ------------------------------------------------------------------------- fft
def ifft2_centered(field, ctx: Context = None) -> np.ndarray:
    """fft.hpp:29 (device fp32 math)."""
    ctx = ctx or Context.default()
    f = np.ascontiguousarray(field, np.complex128)
    out = np.zeros_like(f)
    check(lib().ocn_ifft2_centered(ctx.h, f.shape[0], _dp(f.view(np.float64)),
                                   _dp(out.view(np.float64))), ctx.h, "ifft2_centered")
    return out


def ifft2_hermitian_pair(x, y, check_symmetry: bool = False, ctx: Context = None):
    """fft.hpp:36-38. The reference never checks inside generate_maps; with
    check_symmetry the precondition is verified (NumericError)."""
    ctx = ctx or Context.default()
    x = np.ascontiguousarray(x, np.complex128)
    y = np.ascontiguousarray(y, np.complex128)
    if x.shape != y.shape:
        raise ConfigError("paired FFT fields must have equal size")
    if check_symmetry and not (is_conjugate_symmetric(x) and is_conjugate_symmetric(y)):
        raise NumericError("ifft2_hermitian_pair: inputs are not conjugate-symmetric")
    n = x.shape[0]
    re = np.zeros((n, n))
    im = np.zeros((n, n))
    check(lib().ocn_ifft2_pair(ctx.h, n, _dp(x.view(np.float64)), _dp(y.view(np.float64)), _dp(re),
                               _dp(im)), ctx.h, "ifft2_hermitian_pair")
    return re, im


def is_conjugate_symmetric(f, tol=1e-9) -> bool:
    """fft.cpp:57-67 (host check of a host array)."""
    n = f.shape[0]
    ni = np.array([0] + [n - i for i in range(1, n)])
    return bool(np.all(np.abs(f - np.conj(f[np.ix_(ni, ni)])) <= tol))


# ------------------------------------------------------------------------ mesh
class TriMesh:
    """mesh.hpp:15-50 — validated closed mesh, re-oriented outward, with the
    per-triangle normals / areas and mass properties (load-time host code,
    mesh.cpp:18-116), uploaded once to the device (ocn_mesh)."""

    def __init__(self, vertices, triangles, ctx: Context = None):
        v = np.ascontiguousarray(vertices, np.float64).reshape(-1, 3)
        t = np.ascontiguousarray(triangles, np.int32).reshape(-1, 3).copy()
        if v.shape[0] == 0 or t.shape[0] == 0:
            raise MeshError("empty mesh")
        nv = v.shape[0]
        a_idx = t.reshape(-1)
        b_idx = t[:, [1, 2, 0]].reshape(-1)
        if (a_idx < 0).any() or (a_idx >= nv).any():
            raise MeshError("mesh: face references a missing vertex")
        if (a_idx == b_idx).any():
            raise MeshError("mesh: face repeats a vertex")
        key = a_idx.astype(np.int64) * nv + b_idx
        if np.unique(key).size != key.size:
            raise MeshError("mesh: duplicated directed edge (inconsistent winding)")
        rev = b_idx.astype(np.int64) * nv + a_idx
        if not np.isin(rev, key).all():
            raise MeshError("mesh: open mesh, an edge has no partner")
        A, B, Cc = v[t[:, 0]], v[t[:, 1]], v[t[:, 2]]
        if (np.einsum("ij,ij->i", A, np.cross(B, Cc)) / 6.0).sum() < 0.0:
            t[:, [1, 2]] = t[:, [2, 1]]
            A, B, Cc = v[t[:, 0]], v[t[:, 1]], v[t[:, 2]]
        n = np.cross(B - A, Cc - A)
        nlen = np.sqrt(n[:, 0] * n[:, 0] + n[:, 1] * n[:, 1] + n[:, 2] * n[:, 2])
        self.areas = 0.5 * nlen
        deg = nlen < 1e-14
        self.normals = np.where(deg[:, None], 0.0, n / np.where(deg, 1.0, nlen)[:, None])
        self.degenerate_count = int(deg.sum())
        self.total_area = float(self.areas.sum())
        vt = np.einsum("ij,ij->i", A, np.cross(B, Cc)) / 6.0
        vol = float(vt.sum())
        if not vol > 0.0:
            raise MeshError("mesh volume must be positive")
        S = A + B + Cc
        self.volume = vol
        self.centroid = (S * (vt / 4.0)[:, None]).sum(0) / vol
        second = np.zeros((3, 3))
        for P in (A, B, Cc, S):
            second += np.einsum("t,ti,tj->ij", vt / 20.0, P, P)
        second -= vol * np.outer(self.centroid, self.centroid)
        self.unit_inertia = np.trace(second) * np.eye(3) - second
        self.bbox_min, self.bbox_max = v.min(0), v.max(0)
        self.vertices, self.triangles = v, t
        self.ctx = ctx or Context.default()
        h = C.c_void_p()
        check(lib().ocn_mesh_create(self.ctx.h, nv, _dp(v), t.shape[0], t.ctypes.data_as(_abi.i32),
                                    _dp(np.ascontiguousarray(self.normals)), _dp(self.areas), vol,
                                    C.byref(h)), self.ctx.h, "TriMesh")
        self.h = h

    def height(self):
        return float(self.bbox_max[1] - self.bbox_min[1])

    def __del__(self):
        try:
            if self.h:
                lib().ocn_mesh_destroy(self.h)
                self.h = None
        except Exception:
            pass


# ----------------------------------------------------------------------- hydro
@dataclass
class FluidQuery:
    """hydro.hpp:38-49 with device samplers: height = height_at(maps) + the
    given zones' samples (Simulation::compose_height), velocity = velocity_at
    (slices), clamped into [y_min, y_max] when velocity_clamp (sim.cpp:39-42)."""
    maps: Optional[SurfaceMaps] = None
    slices: Optional[VelocitySlices] = None
    zones: Sequence["FdmZone"] = ()
    wind: Sequence[float] = (0.0, 0.0, 0.0)
    water_density: float = 1025.0
    air_density: float = 1.204
    density_profile: Sequence[Sequence[float]] = ()
    velocity_clamp: bool = True


@dataclass
class DragCoefficients:
    water: float = 1.0
    air: float = 1.0


def _fluid_struct(fluid: FluidQuery, cd: DragCoefficients):
    f = Fluid()
    keep = []
    f.maps = fluid.maps.h.value if fluid.maps is not None else None
    f.slices = fluid.slices.h.value if fluid.slices is not None else None
    f.velocity_clamp = int(fluid.velocity_clamp)
    if fluid.zones:
        arr = (C.c_void_p * len(fluid.zones))(*[z.h.value for z in fluid.zones])
        keep.append(arr)
        f.n_zones = len(fluid.zones)
        f.zones = C.cast(arr, C.POINTER(C.c_void_p))
    f.wind[:] = list(fluid.wind)
    f.water_density, f.air_density = fluid.water_density, fluid.air_density
    f.cd_water, f.cd_air = cd.water, cd.air
    if fluid.density_profile:
        pr = np.ascontiguousarray(fluid.density_profile, np.float64).reshape(-1, 2)
        keep.append(pr)
        f.n_profile = pr.shape[0]
        f.host_profile = _dp(pr)
    return f, keep


class HydroResult:
    """HydroReport (hydro.hpp:97-109) + access to the states and waterline."""

    def __init__(self, mesh: TriMesh, rep: HydroReport):
        self.mesh = mesh
        self.report = rep
        for name, _ in HydroReport._fields_:
            val = getattr(rep, name)
            setattr(self, name, np.array(list(val)) if hasattr(val, "__len__") else val)
        self.center_of_immersion = self.center_of_immersion if rep.has_center_of_immersion else None

    def states(self):
        n = C.c_int()
        check(lib().ocn_hydro_states(self.mesh.h, 0, None, C.byref(n)), self.mesh.ctx.h, "states")
        buf = (TriangleState * max(n.value, 1))()
        check(lib().ocn_hydro_states(self.mesh.h, n.value, buf, C.byref(n)), self.mesh.ctx.h, "states")
        dt = np.dtype([("parent", "i4"), ("status", "i4"), ("area", "f8"), ("centroid", "f8", 3),
                       ("depth", "f8"), ("normal", "f8", 3)])
        return np.frombuffer(buf, dtype=dt, count=n.value).copy()

    def waterline(self):
        nl, npnt = C.c_int(), C.c_int()
        check(lib().ocn_hydro_waterline(self.mesh.h, C.byref(nl), C.byref(npnt), None, None),
              self.mesh.ctx.h, "waterline")
        off = np.zeros(nl.value + 1, np.int32)
        pts = np.zeros((max(npnt.value, 1), 3))
        check(lib().ocn_hydro_waterline(self.mesh.h, C.byref(nl), C.byref(npnt),
                                        off.ctypes.data_as(_abi.i32), _dp(pts)), self.mesh.ctx.h,
              "waterline")
        return [pts[off[i]:off[i + 1]].copy() for i in range(nl.value)]

    def vertices(self):
        nv = self.mesh.vertices.shape[0]
        w = np.zeros((nv, 3))
        dd = np.zeros(nv)
        check(lib().ocn_hydro_vertices(self.mesh.h, _dp(w), _dp(dd)), self.mesh.ctx.h, "vertices")
        return w, dd


def aggregate(mesh: TriMesh, pose: Pose, fluid: FluidQuery, cd: DragCoefficients = DragCoefficients(),
              vertex_depth=None, sync: bool = True) -> Optional[HydroResult]:
    """hydro.hpp:112-113 — classify_clip + reductions on the device.
    vertex_depth (nv,) replaces the surface sampler (user sampler values)."""
    f, keep = _fluid_struct(fluid, cd)
    vd = None if vertex_depth is None else np.ascontiguousarray(vertex_depth, np.float64)
    rep = HydroReport()
    check(lib().ocn_hydro_aggregate(mesh.h, C.byref(pose), C.byref(f), _dp(vd) if vd is not None else None,
                                    C.byref(rep) if sync else None), mesh.ctx.h, "aggregate")
    return HydroResult(mesh, rep) if sync else None


# ------------------------------------------------------------------ FDM zones
class FdmZone:
    """interactive.hpp:61-104 — device fp32 fields, host scalar state."""

    def __init__(self, config: FdmConfig, body_size: float, body_position, dt: float,
                 ctx: Context = None):
        self.ctx = ctx or Context.default()
        h = C.c_void_p()
        check(lib().ocn_zone_create(self.ctx.h, C.byref(config), body_size, float(body_position[0]),
                                    float(body_position[1]), dt, C.byref(h)), self.ctx.h, "FdmZone")
        self.h = h
        self.n = config.grid_size

    def state(self) -> ZoneState:
        s = ZoneState()
        check(lib().ocn_zone_get_state(self.h, C.byref(s)), self.ctx.h, "state")
        return s

    def spacing(self):
        return self.state().spacing

    def wave_speed(self):
        return self.state().wave_speed

    def cfl_ratio(self, dt):
        s = self.state()
        return s.wave_speed ** 2 * dt * dt / (s.spacing * s.spacing)

    def update_stability(self, speed, dt):
        check(lib().ocn_zone_update_stability(self.h, speed, dt), self.ctx.h, "update_stability")

    def step(self, dt, body_position):
        check(lib().ocn_zone_step(self.h, dt, float(body_position[0]), float(body_position[1])),
              self.ctx.h, "step")

    def apply_mask(self, ij, heights):
        ij = np.ascontiguousarray(ij, np.int32).reshape(-1, 2)
        hh = np.ascontiguousarray(heights, np.float64)
        check(lib().ocn_zone_apply_cells(self.h, hh.shape[0], ij.ctypes.data_as(_abi.i32), _dp(hh)),
              self.ctx.h, "apply_mask")

    def sample(self, xz):
        xz = np.ascontiguousarray(np.atleast_2d(xz), np.float64)
        out = np.zeros(xz.shape[0])
        check(lib().ocn_zone_sample(self.h, xz.shape[0], _dp(xz), _dp(out)), self.ctx.h, "sample")
        return out

    def field(self):
        out = np.zeros((self.n, self.n))
        check(lib().ocn_zone_download(self.h, _dp(out), None), self.ctx.h, "field")
        return out

    def fields(self):
        cur = np.zeros((self.n, self.n))
        prv = np.zeros((self.n, self.n))
        check(lib().ocn_zone_download(self.h, _dp(cur), _dp(prv)), self.ctx.h, "fields")
        return cur, prv

    def set_fields(self, curr=None, prev=None):
        c = None if curr is None else np.ascontiguousarray(curr, np.float64)
        p = None if prev is None else np.ascontiguousarray(prev, np.float64)
        check(lib().ocn_zone_upload(self.h, _dp(c) if c is not None else None,
                                    _dp(p) if p is not None else None), self.ctx.h, "upload")

    def mask_cells(self):
        n = C.c_int()
        check(lib().ocn_zone_mask_download(self.h, 0, None, None, C.byref(n)), self.ctx.h, "mask")
        ij = np.zeros((max(n.value, 1), 2), np.int32)
        hh = np.zeros(max(n.value, 1))
        check(lib().ocn_zone_mask_download(self.h, n.value, ij.ctypes.data_as(_abi.i32), _dp(hh),
                                           C.byref(n)), self.ctx.h, "mask")
        return ij[:n.value], hh[:n.value]

    def __del__(self):
        try:
            if self.h:
                lib().ocn_zone_destroy(self.h)
                self.h = None
        except Exception:
            pass


def compute_mask(zone: FdmZone, loops, body_yaw, body_position, body_speed, frame: MaskFrame,
                 params: MaskParams, apply: bool = False):
    """interactive.hpp:108-111 on the device -> (ij (K, 2), heights (K,))."""
    offs = np.zeros(len(loops) + 1, np.int32)
    for i, l in enumerate(loops):
        offs[i + 1] = offs[i] + len(l)
    pts = np.ascontiguousarray(np.concatenate(loops) if loops else np.zeros((1, 3)), np.float64)
    nc = C.c_int()
    check(lib().ocn_zone_compute_mask(zone.h, len(loops), offs.ctypes.data_as(_abi.i32), _dp(pts),
                                      body_yaw, float(body_position[0]), float(body_position[1]),
                                      body_speed, C.byref(frame), C.byref(params), int(apply),
                                      C.byref(nc)), zone.ctx.h, "compute_mask")
    return zone.mask_cells()


def mask_from_hydro(zone: FdmZone, mesh: TriMesh, body_yaw, body_position, body_speed,
                    frame: MaskFrame, params: MaskParams):
    """sim.cpp:86-109: compute_mask on the device waterline + apply_mask (async)."""
    check(lib().ocn_zone_mask_from_hydro(zone.h, mesh.h, body_yaw, float(body_position[0]),
                                         float(body_position[1]), body_speed, C.byref(frame),
                                         C.byref(params)), zone.ctx.h, "mask_from_hydro")


# ============== composed surface and ABHF heightfields ==============

_FIELD_FILE_NAMES = ("h", "dx", "dz", "ddx_dx", "ddz_dx", "ddz_dz", "dh_dx", "dh_dz")  # main.cpp:76-77


def _zone_array(zones):
    zones = list(zones or ())
    arr = (C.c_void_p * max(1, len(zones)))(*[z.h.value for z in zones])
    return len(zones), C.cast(arr, _abi.pvp), arr


def compose_height(maps: SurfaceMaps, xz, zones: Sequence["FdmZone"] = ()) -> np.ndarray:
    """Simulation::compose_height (sim.cpp:44-51), batched over points (N, 2) -> (N,).

    `zones` are the other bodies' FdmZones (the excluded body's zone left out)."""
    xz = np.ascontiguousarray(np.atleast_2d(xz), np.float64)
    out = np.zeros(xz.shape[0])
    nz, zp, _keep = _zone_array(zones)
    check(lib().ocn_compose_height(maps.h, nz, zp, xz.shape[0], _dp(xz), _dp(out)), maps.ctx.h,
          "compose_height")
    return out


def compose_grid(maps: SurfaceMaps, resolution: int, extent: float,
                 zones: Sequence["FdmZone"] = ()) -> np.ndarray:
    """The composed grid of dump_fields (main.cpp:62-67): [i][j] = compose_height(extent*i/res,
    extent*j/res), evaluated on the device -> (res, res) float64."""
    out = np.zeros((resolution, resolution))
    nz, zp, _keep = _zone_array(zones)
    check(lib().ocn_compose_grid(maps.h, nz, zp, int(resolution), float(extent), _dp(out)),
          maps.ctx.h, "compose_grid")
    return out


def write_field_heightfield(path: str, maps: SurfaceMaps, cascade: int, field: int, t: float):
    """write_heightfield_file (heightfield_io.cpp:73-78) of one device field, header
    {N, cascade, float(t)} (main.cpp:80-85)."""
    check(lib().ocn_heightfield_write_field(maps.h, int(cascade), int(field), float(t),
                                            str(path).encode()), maps.ctx.h, "write_heightfield")


def write_composed_heightfield(path: str, maps: SurfaceMaps, resolution: int, extent: float,
                               t: float, zones: Sequence["FdmZone"] = ()):
    """The composed-surface ABHF file of dump_fields (main.cpp:68-75), computed on the device."""
    nz, zp, _keep = _zone_array(zones)
    check(lib().ocn_heightfield_write_composed(maps.h, nz, zp, int(resolution), float(extent),
                                               float(t), str(path).encode()),
          maps.ctx.h, "write_heightfield")


def write_heightfield(path: str, field, resolution: int = None, cascade: int = -1, t: float = 0.0):
    """write_heightfield_file for a host field (heightfield_io.cpp:30-45, 73-78): "ABHF", u32 N,
    i32 cascade, f32 time, N*N f32 little-endian row-major. IoError on a header / field size
    mismatch or an unwritable path, as the reference."""
    a = np.asarray(field, np.float64)
    res = a.shape[0] if resolution is None else int(resolution)
    if a.ndim != 2 or a.shape[0] != a.shape[1] or a.shape[0] != res:
        raise IoError("heightfield: header resolution does not match field")
    hdr = (b"ABHF" + np.uint32(res).astype("<u4").tobytes() + np.int32(cascade).astype("<i4").tobytes()
           + np.float32(t).astype("<f4").tobytes())
    try:
        with open(path, "wb") as f:
            f.write(hdr)
            f.write(a.astype("<f4").tobytes())
    except OSError:
        raise IoError(f"cannot open for writing: {path}") from None


def read_heightfield(path: str):
    """read_heightfield_file (heightfield_io.cpp:47-63, 80-84) -> (field float64 (N, N),
    {"resolution", "cascade", "time"}). IoError on bad magic, bad resolution or truncation."""
    try:
        with open(path, "rb") as f:
            buf = f.read()
    except OSError:
        raise IoError(f"cannot open: {path}") from None
    if len(buf) < 4 or buf[:4] != b"ABHF":
        raise IoError("heightfield: bad magic, not an ABHF file")
    if len(buf) < 16:
        raise IoError("heightfield: truncated stream")
    res = int(np.frombuffer(buf, "<u4", 1, 4)[0])
    cascade = int(np.frombuffer(buf, "<i4", 1, 8)[0])
    t = float(np.frombuffer(buf, "<f4", 1, 12)[0])
    if res == 0 or res > 1 << 16:
        raise IoError("heightfield: bad resolution")
    if len(buf) < 16 + 4 * res * res:
        raise IoError("heightfield: truncated stream")
    data = np.frombuffer(buf, "<f4", res * res, 16).astype(np.float64).reshape(res, res)
    return data, {"resolution": res, "cascade": cascade, "time": t}


def write_heightfield_csv(path: str, field):
    """write_heightfield_csv_file (heightfield_io.cpp:86-103): one row per grid row, 9 significant
    digits (ostream precision 9, default float format)."""
    a = np.asarray(field, np.float64)
    try:
        with open(path, "w") as f:
            for row in a:
                f.write(",".join(format(float(v), ".9g") for v in row) + "\n")
    except OSError:
        raise IoError(f"cannot open for writing: {path}") from None


def dump_fields(maps: SurfaceMaps, directory: str, t: float, resolution: int,
                zones: Sequence["FdmZone"] = (), fmt: str = "abhf"):
    """dump_fields (main.cpp:59-90): the composed surface over the first cascade's tile plus
    every cascade field, named as the reference CLI names them. Fields come straight from the
    device; only the CSV format formats on the host."""
    import os
    os.makedirs(directory, exist_ok=True)
    tb = "%.3f" % t
    lengths = maps.cascade_set.config.lengths
    extent = lengths[0]
    name = os.path.join(directory, f"surface_composed_t{tb}")
    if fmt == "csv":
        write_heightfield_csv(name + ".csv", compose_grid(maps, resolution, extent, zones))
    else:
        write_composed_heightfield(name + ".abhf", maps, resolution, extent, t, zones)
    for c in range(len(lengths)):
        for f in range(8):
            base = os.path.join(directory, f"cascade{c}_{_FIELD_FILE_NAMES[f]}_t{tb}")
            if fmt == "csv":
                write_heightfield_csv(base + ".csv", maps.field(c, f))
            else:
                write_field_heightfield(base + ".abhf", maps, c, f, t)


# ===================== direct spectral velocity =====================

class DirectVelocityEvaluator:
    """velocity.hpp:24-37 — the exact spectral velocity sum at time t, on the device."""

    def __init__(self, cascades: CascadeSet, t: float):
        self.ctx = cascades.ctx
        h = C.c_void_p()
        check(lib().ocn_direct_create(cascades.h, float(t), C.byref(h)), self.ctx.h,
              "DirectVelocityEvaluator")
        self.h = h
        self.time = t

    @property
    def mode_count(self) -> int:
        n = C.c_int64()
        check(lib().ocn_direct_modes(self.h, C.byref(n)), self.ctx.h, "modes")
        return n.value

    def __call__(self, xz, y) -> np.ndarray:
        """operator()(x, y) batched: xz (N, 2), y scalar or (N,) -> (N, 3)."""
        xz = np.atleast_2d(np.asarray(xz, np.float64))
        xzy = np.ascontiguousarray(np.column_stack([xz, np.broadcast_to(np.asarray(y, np.float64),
                                                                        (xz.shape[0],))]))
        out = np.zeros((xzy.shape[0], 3))
        check(lib().ocn_direct_evaluate(self.h, xzy.shape[0], _dp(xzy), _dp(out)), self.ctx.h,
              "direct velocity")
        return out

    def __del__(self):
        try:
            if self.h:
                lib().ocn_direct_destroy(self.h)
                self.h = None
        except Exception:
            pass


def velocity_direct(cascades: CascadeSet, xz, y, t: float) -> np.ndarray:
    """velocity_direct (velocity.cpp:61-63), batched."""
    return DirectVelocityEvaluator(cascades, t)(xz, y)
