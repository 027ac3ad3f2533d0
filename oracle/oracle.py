"""TEST INFRASTRUCTURE ONLY — ctypes front end of the CPU oracle.

Two back ends with the same Python surface:

* ``Oracle("port")``      -> oracle/liboracle.so, the plain-C fp64 restatement
                             (oracle/ocean_oracle.c) of the reference algorithm;
* ``Oracle("reference")`` -> oracle/_ref/libocean_ref.so, the unmodified reference
                             library compiled from /root/reference/proj/src by
                             oracle/Makefile (only present where it was built).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference arm
may import this module. The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2503_03326_b200._types import (FdmConfig, HydroReport, MaskFrame, MaskParams, Pose,
                                          SliceConfig, SpectrumParams, TriangleState)

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libocean_ref.so")

_d = C.POINTER(C.c_double)
_u8 = C.POINTER(C.c_uint8)
_i32 = C.POINTER(C.c_int32)
_u32 = C.POINTER(C.c_uint32)


def build(reference: bool = True) -> None:
    """Compile liboracle.so (and the reference library when its tree exists)."""
    targets = ["all"]
    if reference and os.path.isdir("/root/reference/proj/src"):
        targets.append("ref")
        # the reference's own Simulation over the drop-in (needs libocean_api.so)
        api = os.path.join(os.path.dirname(HERE), "paper_2503_03326_b200", "lib", "libocean_api.so")
        if os.path.exists(api):
            targets.append("caller")
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def P(a, t=_d):
    return a.ctypes.data_as(t) if a is not None else None


class OracleError(RuntimeError):
    def __init__(self, status, where):
        super().__init__(f"{where} -> status {status}")
        self.status = status


def _chk(st, where):
    if st != 0:
        raise OracleError(st, where)


class Oracle:
    """Same Python API over the restatement ('port') or the reference build."""

    def __init__(self, kind: str = "port"):
        self.kind = kind
        path = PORT_SO if kind == "port" else REF_SO
        if not os.path.exists(path):
            build(reference=(kind != "port"))
        self.lib = C.CDLL(path)
        self.p = "orc_" if kind == "port" else "ref_"
        L = self.lib
        for name, restype in [("alpha", C.c_double), ("peak_omega", C.c_double),
                              ("standard_peak_omega", C.c_double)]:
            f = getattr(L, self.p + name)
            f.argtypes = [C.POINTER(SpectrumParams)]
            f.restype = restype
        for name, n in [("dispersion", 2), ("beta_s", 1), ("directional_kernel", 2),
                        ("donelan_banner", 3), ("swell_spread", 4), ("q_dbxi_approx", 1),
                        ("attenuation", 2)]:
            f = getattr(L, self.p + name)
            f.argtypes = [C.c_double] * n
            f.restype = C.c_double
        getattr(L, self.p + "q_dbxi_quadrature").argtypes = [C.c_double, C.c_double, C.c_int]
        getattr(L, self.p + "q_dbxi_quadrature").restype = C.c_double
        getattr(L, self.p + "directional").argtypes = [C.c_double, C.c_double,
                                                      C.POINTER(SpectrumParams)]
        getattr(L, self.p + "directional").restype = C.c_double
        getattr(L, self.p + "h0_variance").argtypes = [C.c_double] * 5 + [C.POINTER(SpectrumParams)]
        getattr(L, self.p + "h0_variance").restype = C.c_double
        getattr(L, self.p + "damping_factor").argtypes = [C.c_double] * 4
        getattr(L, self.p + "damping_factor").restype = C.c_double
        getattr(L, self.p + "jonswap").argtypes = [C.c_double, C.POINTER(SpectrumParams), _d]
        getattr(L, self.p + "philox").argtypes = [C.c_uint64] * 4 + [_u32]
        getattr(L, self.p + "philox").restype = None
        getattr(L, self.p + "gaussian_complex").argtypes = [C.c_uint64, C.c_uint32, C.c_uint32,
                                                           C.c_uint32, _d]
        getattr(L, self.p + "gaussian_complex").restype = None
        getattr(L, self.p + "generate_h0").argtypes = [C.c_int, C.c_double, C.c_double, C.c_double,
                                                      C.POINTER(SpectrumParams), C.c_uint32, _d, _d,
                                                      _u8, _d]
        getattr(L, self.p + "ifft2_centered").argtypes = [C.c_int, _d]
        getattr(L, self.p + "log_distribution").argtypes = [C.c_double, C.c_double, _d]
        getattr(L, self.p + "exp_interp").argtypes = [C.c_double] * 5 + [_d]
        getattr(L, self.p + "slice_depths").argtypes = [C.POINTER(SliceConfig), _d]
        getattr(L, self.p + "mesh_build").argtypes = [C.c_int, _d, C.c_int, _i32, _d, _d, _d]
        getattr(L, self.p + "mask_height").argtypes = [C.c_double, C.c_double, C.POINTER(MaskFrame),
                                                      C.c_double, C.POINTER(MaskParams), _d]
        if kind == "port":
            L.orc_ifft2_pair.argtypes = [C.c_int, _d, _d, _d, _d]
        else:
            L.ref_ifft2_pair.argtypes = [C.c_int, _d, _d, _d, _d, C.c_int]
            L.ref_last_error.restype = C.c_char_p
            L.ref_set_worker_count.argtypes = [C.c_int]

    # ------------------------------------------------------------- scalars
    def scalar(self, name, *args):
        return getattr(self.lib, self.p + name)(*args)

    def jonswap(self, omega, params):
        out = C.c_double()
        _chk(getattr(self.lib, self.p + "jonswap")(omega, C.byref(params), C.byref(out)), "jonswap")
        return out.value

    def philox(self, key_lo, key_hi, ctr_lo, ctr_hi):
        out = np.zeros(4, np.uint32)
        getattr(self.lib, self.p + "philox")(key_lo, key_hi, ctr_lo, ctr_hi, P(out, _u32))
        return out

    def gaussian_complex(self, seed, stream, i, j):
        out = np.zeros(2)
        getattr(self.lib, self.p + "gaussian_complex")(seed, stream, i, j, P(out))
        return complex(out[0], out[1])

    def log_distribution(self, y, y_min):
        out = C.c_double()
        _chk(getattr(self.lib, self.p + "log_distribution")(y, y_min, C.byref(out)), "log_dist")
        return out.value

    def exp_interp(self, a, fa, b, fb, x):
        out = C.c_double()
        _chk(getattr(self.lib, self.p + "exp_interp")(a, fa, b, fb, x, C.byref(out)), "exp_interp")
        return out.value

    def slice_depths(self, cfg: SliceConfig):
        out = np.zeros(cfg.count)
        _chk(getattr(self.lib, self.p + "slice_depths")(C.byref(cfg), P(out)), "slice_depths")
        return out

    def mask_height(self, x, z, frame, speed, params):
        out = C.c_double()
        _chk(getattr(self.lib, self.p + "mask_height")(x, z, C.byref(frame), speed, C.byref(params),
                                                       C.byref(out)), "mask_height")
        return out.value

    # ------------------------------------------------------------ spectrum
    def generate_h0(self, n, length, band_min, band_max, params, cascade=0):
        """-> (h0 complex [n,n], h0cn complex [n,n], in_band bool [n,n], waves [n,n,4])."""
        h0 = np.zeros(2 * n * n)
        h0cn = np.zeros(2 * n * n)
        band = np.zeros(n * n, np.uint8)
        waves = np.zeros(4 * n * n)
        st = getattr(self.lib, self.p + "generate_h0")(n, length, band_min, band_max,
                                                       C.byref(params), cascade, P(h0), P(h0cn),
                                                       P(band, _u8), P(waves))
        _chk(st, "generate_h0")
        return (h0.view(np.complex128).reshape(n, n), h0cn.view(np.complex128).reshape(n, n),
                band.reshape(n, n).astype(bool), waves.reshape(n, n, 4))

    def cascade_tables(self, n, lengths, cutoffs, params):
        """CascadeSet (surface.cpp:22-37) -> stacked h0 / h0cn / in_band per cascade."""
        C_ = len(lengths)
        h0 = np.zeros((C_, n, n), np.complex128)
        h0cn = np.zeros((C_, n, n), np.complex128)
        band = np.zeros((C_, n, n), bool)
        for c in range(C_):
            bmin = 0.0 if c == 0 else cutoffs[c - 1]
            bmax = cutoffs[c] if c + 1 < C_ else 1e300
            h0[c], h0cn[c], band[c], _ = self.generate_h0(n, lengths[c], bmin, bmax, params, c)
        return h0, h0cn, band

    # ----------------------------------------------------------------- fft
    def ifft2_centered(self, field):
        f = np.ascontiguousarray(field, np.complex128).copy()
        n = f.shape[0]
        _chk(getattr(self.lib, self.p + "ifft2_centered")(n, P(f.view(np.float64))), "ifft2")
        return f

    def ifft2_pair(self, x, y):
        x = np.ascontiguousarray(x, np.complex128)
        y = np.ascontiguousarray(y, np.complex128)
        n = x.shape[0]
        re = np.zeros((n, n))
        im = np.zeros((n, n))
        args = [n, P(x.view(np.float64)), P(y.view(np.float64)), P(re), P(im)]
        if self.kind != "port":
            args.append(0)
        _chk(getattr(self.lib, self.p + "ifft2_pair")(*args), "ifft2_pair")
        return re, im

    # ------------------------------------------------------------- surface
    def generate_maps(self, n, lengths, cutoffs, params, t, choppiness=1.0, single_precision=False,
                      tables=None):
        """-> maps [C, 8, n, n] fp64."""
        C_ = len(lengths)
        maps = np.zeros((C_, 8, n, n))
        lengths_a = np.ascontiguousarray(lengths, np.float64)
        if self.kind == "port":
            h0, h0cn, band = tables if tables is not None else self.cascade_tables(n, lengths, cutoffs,
                                                                                  params)
            f = self.lib.orc_generate_maps
            f.argtypes = [C.c_int, C.c_int, _d, C.c_double, _d, _d, _u8, C.c_double, C.c_double,
                          C.c_int, _d]
            band8 = np.ascontiguousarray(band, np.uint8)
            _chk(f(n, C_, P(lengths_a), params.gravity, P(np.ascontiguousarray(h0).view(np.float64)),
                   P(np.ascontiguousarray(h0cn).view(np.float64)), P(band8, _u8), t, choppiness,
                   int(single_precision), P(maps)), "generate_maps")
        else:
            cut = np.ascontiguousarray(list(cutoffs) + [0.0], np.float64)
            f = self.lib.ref_generate_maps
            f.argtypes = [C.c_int, C.c_int, _d, _d, C.POINTER(SpectrumParams), C.c_double,
                          C.c_double, C.c_int, _d]
            _chk(f(n, C_, P(lengths_a), P(cut), C.byref(params), t, choppiness,
                   int(single_precision), P(maps)), "generate_maps")
        return maps

    def surface_pair_large(self, n, length, band_min, band_max, params, t, pair, choppiness=1.0,
                           cascade=0, threads=None, ab=None):
        """Port only: one packed surface pair of a single large grid (fft.cpp:79-101
        on the surface.cpp:45-66 coefficients, h0 per mode on the fly) -> (re, im)
        [n, n] fp64, plus the direct sums of the packed spectrum at the grid
        nodes ab ([k, 2] ints) -> complex [k] (None without ab)."""
        assert self.kind == "port"
        f = self.lib.orc_surface_pair_large
        f.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double, C.POINTER(SpectrumParams),
                      C.c_uint32, C.c_double, C.c_double, C.c_int, C.c_int, C.c_int, _i32, _d, _d,
                      _d]
        threads = threads or os.cpu_count() or 1
        re = np.zeros((n, n))
        im = np.zeros((n, n))
        npts = 0 if ab is None else len(ab)
        ab_a = np.ascontiguousarray(ab if ab is not None else np.zeros((0, 2)), np.int32)
        direct = np.zeros(2 * max(npts, 1))
        _chk(f(n, length, band_min, band_max, C.byref(params), cascade, t, choppiness, pair, threads,
               npts, P(ab_a, _i32), P(direct), P(re), P(im)), "surface_pair_large")
        return re, im, (direct[:2 * npts].view(np.complex128) if npts else None)

    def build_slices(self, n, lengths, cutoffs, params, t, cfg: SliceConfig, tables=None):
        """-> (depths [D], slices [D, C, 3, n, n])."""
        C_ = len(lengths)
        D = cfg.count
        depths = np.zeros(D)
        sl = np.zeros((D, C_, 3, n, n))
        lengths_a = np.ascontiguousarray(lengths, np.float64)
        if self.kind == "port":
            h0, h0cn, band = tables if tables is not None else self.cascade_tables(n, lengths, cutoffs,
                                                                                  params)
            f = self.lib.orc_build_slices
            f.argtypes = [C.c_int, C.c_int, _d, C.c_double, _d, _d, _u8, C.c_double,
                          C.POINTER(SliceConfig), _d, _d]
            _chk(f(n, C_, P(lengths_a), params.gravity, P(np.ascontiguousarray(h0).view(np.float64)),
                   P(np.ascontiguousarray(h0cn).view(np.float64)),
                   P(np.ascontiguousarray(band, np.uint8), _u8), t, C.byref(cfg), P(depths), P(sl)),
                 "build_slices")
        else:
            cut = np.ascontiguousarray(list(cutoffs) + [0.0], np.float64)
            f = self.lib.ref_build_slices
            f.argtypes = [C.c_int, C.c_int, _d, _d, C.POINTER(SpectrumParams), C.c_double,
                          C.POINTER(SliceConfig), _d, _d]
            _chk(f(n, C_, P(lengths_a), P(cut), C.byref(params), t, C.byref(cfg), P(depths), P(sl)),
                 "build_slices")
        return depths, sl

    # ------------------------------------------------------------ samplers
    def _surface(self, n, lengths, maps):
        from oracle.oracle_structs import OrcSurface
        s = OrcSurface()
        s.n, s.C = n, len(lengths)
        self._keep = (np.ascontiguousarray(lengths, np.float64), np.ascontiguousarray(maps, np.float64))
        s.lengths = P(self._keep[0])
        s.maps = P(self._keep[1])
        return s

    def height_at(self, n, lengths, maps, xz):
        xz = np.ascontiguousarray(xz, np.float64)
        npts = xz.shape[0]
        out = np.zeros(npts)
        if self.kind == "port":
            s = self._surface(n, lengths, maps)
            f = self.lib.orc_height_at
            f.argtypes = [C.c_void_p, C.c_int64, _d, _d]
            _chk(f(C.byref(s), npts, P(xz), P(out)), "height_at")
        else:
            f = self.lib.ref_height_at
            f.argtypes = [C.c_int, C.c_int, _d, _d, C.c_int64, _d, _d]
            la = np.ascontiguousarray(lengths, np.float64)
            ma = np.ascontiguousarray(maps, np.float64)
            _chk(f(n, len(lengths), P(la), P(ma), npts, P(xz), P(out)), "height_at")
        return out

    def sample_displacement(self, n, lengths, maps, xz):
        xz = np.ascontiguousarray(xz, np.float64)
        npts = xz.shape[0]
        out = np.zeros((npts, 3))
        if self.kind == "port":
            s = self._surface(n, lengths, maps)
            f = self.lib.orc_sample_displacement
            f.argtypes = [C.c_void_p, C.c_int64, _d, _d]
            _chk(f(C.byref(s), npts, P(xz), P(out)), "sample_displacement")
        else:
            f = self.lib.ref_sample_displacement
            f.argtypes = [C.c_int, C.c_int, _d, _d, C.c_int64, _d, _d]
            la = np.ascontiguousarray(lengths, np.float64)
            ma = np.ascontiguousarray(maps, np.float64)
            _chk(f(n, len(lengths), P(la), P(ma), npts, P(xz), P(out)), "sample_displacement")
        return out

    def height_at_tolerance(self, n, lengths, maps, xz, tol, max_iters):
        xz = np.ascontiguousarray(xz, np.float64)
        npts = xz.shape[0]
        out = np.zeros(npts)
        it = np.zeros(npts, np.int32)
        if self.kind == "port":
            s = self._surface(n, lengths, maps)
            f = self.lib.orc_height_at_tolerance
            f.argtypes = [C.c_void_p, C.c_int64, _d, C.c_double, C.c_int, _d, _i32]
            _chk(f(C.byref(s), npts, P(xz), tol, max_iters, P(out), P(it, _i32)), "h_tol")
        else:
            f = self.lib.ref_height_at_tolerance
            f.argtypes = [C.c_int, C.c_int, _d, _d, C.c_int64, _d, C.c_double, C.c_int, _d, _i32]
            la = np.ascontiguousarray(lengths, np.float64)
            ma = np.ascontiguousarray(maps, np.float64)
            _chk(f(n, len(lengths), P(la), P(ma), npts, P(xz), tol, max_iters, P(out), P(it, _i32)),
                 "h_tol")
        return out, it

    def _slices(self, n, lengths, depths, cfg, data):
        from oracle.oracle_structs import OrcSlices
        s = OrcSlices()
        s.n, s.C, s.D = n, len(lengths), len(depths)
        self._keep_s = (np.ascontiguousarray(lengths, np.float64),
                        np.ascontiguousarray(depths, np.float64),
                        np.ascontiguousarray(data, np.float64))
        s.lengths = P(self._keep_s[0])
        s.depths = P(self._keep_s[1])
        s.y_min, s.y_max = cfg.y_min, cfg.y_max
        s.data = P(self._keep_s[2])
        return s

    def velocity_at_port(self, n, lengths, depths, cfg, slices, xzy, interp=0, clamp=0):
        """Restatement only: velocity_at on explicit slices."""
        xzy = np.ascontiguousarray(xzy, np.float64)
        npts = xzy.shape[0]
        out = np.zeros((npts, 3))
        s = self._slices(n, lengths, depths, cfg, slices)
        f = self.lib.orc_velocity_at
        f.argtypes = [C.c_void_p, C.c_int64, _d, C.c_int, C.c_int, _d]
        _chk(f(C.byref(s), npts, P(xzy), interp, clamp, P(out)), "velocity_at")
        return out

    def sample_slice_port(self, n, lengths, depths, cfg, slices, depth, xz):
        xz = np.ascontiguousarray(xz, np.float64)
        out = np.zeros((xz.shape[0], 3))
        s = self._slices(n, lengths, depths, cfg, slices)
        f = self.lib.orc_sample_slice
        f.argtypes = [C.c_void_p, C.c_int, C.c_int64, _d, _d]
        _chk(f(C.byref(s), depth, xz.shape[0], P(xz), P(out)), "sample_slice")
        return out

    def velocity_at_ref(self, n, lengths, cutoffs, params, t, cfg, xzy, interp=0, clamp=0):
        """Reference build: build_slices + velocity_at (slices rebuilt inside)."""
        xzy = np.ascontiguousarray(xzy, np.float64)
        out = np.zeros((xzy.shape[0], 3))
        f = self.lib.ref_velocity_at
        f.argtypes = [C.c_int, C.c_int, _d, _d, C.POINTER(SpectrumParams), C.c_double,
                      C.POINTER(SliceConfig), C.c_int64, _d, C.c_int, C.c_int, _d]
        la = np.ascontiguousarray(lengths, np.float64)
        cut = np.ascontiguousarray(list(cutoffs) + [0.0], np.float64)
        _chk(f(n, len(lengths), P(la), P(cut), C.byref(params), t, C.byref(cfg), xzy.shape[0],
               P(xzy), interp, clamp, P(out)), "velocity_at")
        return out

    def direct_velocity(self, n, lengths, cutoffs, params, t, xzy, tables=None):
        xzy = np.ascontiguousarray(xzy, np.float64)
        out = np.zeros((xzy.shape[0], 3))
        la = np.ascontiguousarray(lengths, np.float64)
        if self.kind == "port":
            h0, h0cn, band = tables if tables is not None else self.cascade_tables(n, lengths, cutoffs,
                                                                                  params)
            f = self.lib.orc_direct_velocity
            f.argtypes = [C.c_int, C.c_int, _d, C.c_double, _d, _d, _u8, C.c_double, C.c_int64, _d, _d]
            _chk(f(n, len(lengths), P(la), params.gravity, P(np.ascontiguousarray(h0).view(np.float64)),
                   P(np.ascontiguousarray(h0cn).view(np.float64)),
                   P(np.ascontiguousarray(band, np.uint8), _u8), t, xzy.shape[0], P(xzy), P(out)),
                 "direct_velocity")
        else:
            f = self.lib.ref_direct_velocity
            f.argtypes = [C.c_int, C.c_int, _d, _d, C.POINTER(SpectrumParams), C.c_double, C.c_int64,
                          _d, _d]
            cut = np.ascontiguousarray(list(cutoffs) + [0.0], np.float64)
            _chk(f(n, len(lengths), P(la), P(cut), C.byref(params), t, xzy.shape[0], P(xzy), P(out)),
                 "direct_velocity")
        return out

    # ---------------------------------------------------------------- mesh
    def mesh_build(self, verts, tris):
        """TriMesh ctor -> dict(tris, normals, areas, volume, centroid, inertia, bbox_min, bbox_max,
        total_area, degenerate)."""
        verts = np.ascontiguousarray(verts, np.float64)
        tris = np.ascontiguousarray(tris, np.int32).copy()
        nt = tris.shape[0]
        normals = np.zeros((nt, 3))
        areas = np.zeros(nt)
        props = np.zeros(21)
        _chk(getattr(self.lib, self.p + "mesh_build")(verts.shape[0], P(verts), nt, P(tris, _i32),
                                                      P(normals), P(areas), P(props)), "mesh_build")
        return dict(tris=tris, normals=normals, areas=areas, volume=props[0], centroid=props[1:4],
                    inertia=props[4:13].reshape(3, 3), bbox_min=props[13:16], bbox_max=props[16:19],
                    total_area=props[19], degenerate=int(props[20]))

    # --------------------------------------------------------------- hydro
    def aggregate(self, verts, mesh, pose: Pose, *, n=0, lengths=(), maps=None, slices=None,
                  depths=None, slice_cfg=None, cutoffs=(), params=None, t=0.0, velocity_clamp=1,
                  wind=(0, 0, 0), water_density=1025.0, air_density=1.204, cd_water=1.0,
                  cd_air=1.0, vertex_depth=None, zones=(), profile=None):
        """aggregate (hydro.cpp:253-306). Returns (report dict, states, loops list)."""
        verts = np.ascontiguousarray(verts, np.float64)
        tris = mesh["tris"]
        nt = tris.shape[0]
        cap = 3 * nt + 8
        states = (TriangleState * cap)()
        cap_l, cap_p = nt + 8, 3 * nt + 8
        offs = np.zeros(cap_l, np.int32)
        pts = np.zeros((cap_p, 3))
        rep = HydroReport()
        if self.kind == "port":
            from oracle.oracle_structs import OrcClipOut, OrcFluid
            fl = OrcFluid()
            keep = []
            if maps is not None:
                surf = self._surface(n, lengths, maps)
                keep.append(surf)
                fl.surface = C.cast(C.pointer(surf), C.c_void_p)
            if slices is not None:
                sl = self._slices(n, lengths, depths, slice_cfg, slices)
                keep.append(sl)
                fl.slices = C.cast(C.pointer(sl), C.c_void_p)
            fl.velocity_clamp = velocity_clamp
            if zones:
                zarr = (C.c_void_p * len(zones))(*[z.ptr for z in zones])
                keep.append(zarr)
                fl.n_zones = len(zones)
                fl.zones = C.cast(zarr, C.c_void_p)
            fl.wind[:] = wind
            fl.water_density, fl.air_density, fl.cd_water, fl.cd_air = (
                water_density, air_density, cd_water, cd_air)
            if profile is not None:
                pr = np.ascontiguousarray(profile, np.float64)
                keep.append(pr)
                fl.n_profile = pr.shape[0]
                fl.profile = P(pr)
            co = OrcClipOut()
            co.capacity_states = cap
            co.states = C.cast(states, C.c_void_p)
            co.capacity_loops = cap_l
            co.loop_offsets = P(offs, _i32)
            co.capacity_points = cap_p
            co.points = P(pts)
            f = self.lib.orc_aggregate
            f.argtypes = [C.c_int, _d, C.c_int, _i32, _d, _d, C.c_double, C.POINTER(Pose), C.c_void_p,
                          _d, C.POINTER(HydroReport), C.c_void_p]
            vd = None if vertex_depth is None else np.ascontiguousarray(vertex_depth, np.float64)
            _chk(f(verts.shape[0], P(verts), nt, P(tris, _i32), P(mesh["normals"]), P(mesh["areas"]),
                   mesh["volume"], C.byref(pose), C.byref(fl), P(vd), C.byref(rep), C.byref(co)),
                 "aggregate")
            n_loops = co.n_loops
        else:
            assert vertex_depth is None and not zones and profile is None
            f = self.lib.ref_aggregate
            f.argtypes = [C.c_int, _d, C.c_int, _i32, C.POINTER(Pose), C.c_int, C.c_int, _d, _d, _d,
                          C.POINTER(SpectrumParams), C.c_double, C.c_void_p, C.c_int, _d,
                          C.c_double, C.c_double, C.c_double, C.c_double, C.POINTER(HydroReport),
                          C.c_int, C.c_void_p, C.c_int, _i32, C.c_int, _d]
            la = np.ascontiguousarray(lengths, np.float64)
            ma = None if maps is None else np.ascontiguousarray(maps, np.float64)
            cut = np.ascontiguousarray(list(cutoffs) + [0.0], np.float64)
            wd = np.ascontiguousarray(wind, np.float64)
            sc = C.byref(slice_cfg) if slice_cfg is not None else None
            _chk(f(verts.shape[0], P(verts), nt, P(tris, _i32), C.byref(pose), n, len(lengths),
                   P(la), P(ma), P(cut), C.byref(params) if params is not None else None, t, sc,
                   velocity_clamp, P(wd), water_density, air_density, cd_water, cd_air,
                   C.byref(rep), cap, C.cast(states, C.c_void_p), cap_l, P(offs, _i32), cap_p,
                   P(pts)), "aggregate")
            n_loops = rep.waterline_loops
        st = np.zeros(rep.state_count, dtype=[("parent", "i4"), ("status", "i4"), ("area", "f8"),
                                               ("centroid", "f8", 3), ("depth", "f8"),
                                               ("normal", "f8", 3)])
        raw = np.frombuffer(states, dtype=st.dtype, count=rep.state_count)
        st[:] = raw
        loops = [pts[offs[i]:offs[i + 1]].copy() for i in range(n_loops)]
        return rep.as_dict(), st, loops

    # ------------------------------------------------------------ FDM zone
    def zone(self, cfg: FdmConfig, body_size, bx, bz, dt):
        return _Zone(self, cfg, body_size, bx, bz, dt)


class _Zone:
    """FdmZone through either back end."""

    def __init__(self, o: Oracle, cfg, body_size, bx, bz, dt):
        self.o = o
        L = o.lib
        self.n = cfg.grid_size
        if o.kind == "port":
            L.orc_zone_create.argtypes = [C.POINTER(FdmConfig), C.c_double, C.c_double, C.c_double,
                                          C.c_double, C.POINTER(C.c_void_p)]
            h = C.c_void_p()
            _chk(L.orc_zone_create(C.byref(cfg), body_size, bx, bz, dt, C.byref(h)), "zone_create")
            self.ptr = h.value
        else:
            L.ref_zone_create.argtypes = [C.POINTER(FdmConfig), C.c_double, C.c_double, C.c_double,
                                          C.c_double, C.POINTER(C.c_int)]
            L.ref_zone_create.restype = C.c_void_p
            st = C.c_int()
            self.ptr = L.ref_zone_create(C.byref(cfg), body_size, bx, bz, dt, C.byref(st))
            _chk(st.value, "zone_create")

    def __del__(self):
        try:
            f = getattr(self.o.lib, self.o.p + "zone_destroy")
            f.argtypes = [C.c_void_p]
            f(self.ptr)
        except Exception:
            pass

    def update_stability(self, speed, dt):
        f = getattr(self.o.lib, self.o.p + "zone_update_stability")
        f.argtypes = [C.c_void_p, C.c_double, C.c_double]
        _chk(f(self.ptr, speed, dt), "update_stability")

    def step(self, dt, bx, bz):
        f = getattr(self.o.lib, self.o.p + "zone_step")
        f.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_double]
        _chk(f(self.ptr, dt, bx, bz), "step")

    def apply_cells(self, ij, h):
        ij = np.ascontiguousarray(ij, np.int32)
        h = np.ascontiguousarray(h, np.float64)
        f = getattr(self.o.lib, self.o.p + "zone_apply_cells")
        f.argtypes = [C.c_void_p, C.c_int, _i32, _d]
        _chk(f(self.ptr, h.shape[0], P(ij, _i32), P(h)), "apply")

    def state(self):
        from oracle.oracle_structs import OrcZone
        if self.o.kind == "port":
            z = C.cast(self.ptr, C.POINTER(OrcZone)).contents
            return dict(spacing=z.delta, wave_speed=z.c, damping=z.damping, origin=list(z.origin),
                        dropped_wake=z.dropped_wake)
        out = np.zeros(8)
        f = self.o.lib.ref_zone_state
        f.argtypes = [C.c_void_p, _d]
        f.restype = None
        f(self.ptr, P(out))
        return dict(spacing=out[0], wave_speed=out[1], damping=out[2], origin=[out[3], out[4]],
                    dropped_wake=int(out[5]))

    def field(self):
        n = self.n
        if self.o.kind == "port":
            from oracle.oracle_structs import OrcZone
            z = C.cast(self.ptr, C.POINTER(OrcZone)).contents
            return np.ctypeslib.as_array(z.curr, shape=(n * n,)).reshape(n, n).copy()
        out = np.zeros((n, n))
        f = self.o.lib.ref_zone_get_field
        f.argtypes = [C.c_void_p, _d]
        f.restype = None
        f(self.ptr, P(out))
        return out

    def set_field(self, curr):
        n = self.n
        curr = np.ascontiguousarray(curr, np.float64)
        if self.o.kind == "port":
            from oracle.oracle_structs import OrcZone
            z = C.cast(self.ptr, C.POINTER(OrcZone)).contents
            C.memmove(z.curr, P(curr), n * n * 8)
        else:
            f = self.o.lib.ref_zone_set_field
            f.argtypes = [C.c_void_p, _d]
            f.restype = None
            f(self.ptr, P(curr))

    def sample(self, x, z):
        if self.o.kind == "port":
            f = self.o.lib.orc_zone_sample
        else:
            f = self.o.lib.ref_zone_sample
        f.argtypes = [C.c_void_p, C.c_double, C.c_double]
        f.restype = C.c_double
        return f(self.ptr, x, z)

    def compute_mask(self, loops, yaw, bx, bz, speed, frame, params):
        """loops: list of (m, 3) arrays. -> (ij [K,2], h [K])."""
        offs = np.zeros(len(loops) + 1, np.int32)
        for i, l in enumerate(loops):
            offs[i + 1] = offs[i] + len(l)
        pts = np.ascontiguousarray(np.concatenate(loops) if loops else np.zeros((1, 3)), np.float64)
        cap = self.n * self.n
        ij = np.zeros((cap, 2), np.int32)
        h = np.zeros(cap)
        nc = C.c_int()
        f = getattr(self.o.lib, self.o.p + "compute_mask")
        f.argtypes = [C.c_void_p, C.c_int, _i32, _d, C.c_double, C.c_double, C.c_double, C.c_double,
                      C.POINTER(MaskFrame), C.POINTER(MaskParams), C.c_int, _i32, _d,
                      C.POINTER(C.c_int)]
        _chk(f(self.ptr, len(loops), P(offs, _i32), P(pts), yaw, bx, bz, speed, C.byref(frame),
               C.byref(params), cap, P(ij, _i32), P(h), C.byref(nc)), "compute_mask")
        k = nc.value
        return ij[:k].copy(), h[:k].copy()
