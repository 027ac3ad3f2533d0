"""ctypes binding of the C-ABI in include/ocean_b200.h (libocean_b200.so).

The product path: every call lands in hand-written sm_100a kernels. There is no
CPU fallback — importing works on a CPU-only machine (so the symbol table can
be checked), but creating a context without a B200 raises OceanCudaError.
"""
from __future__ import annotations

import ctypes as C
import os

from ._types import (Fluid, FdmConfig, HydroReport, MaskFrame, MaskParams, Pose, SliceConfig,
                     SpectrumParams, TriangleState, ZoneState, BodyFrame, XformInfo, SimConfig,
                     SimBody)

PKG = os.path.dirname(os.path.abspath(__file__))
# OCN_LIB: an alternative build of the same library (kernel-variant experiments)
LIB_PATH = os.environ.get("OCN_LIB") or os.path.join(PKG, "lib", "libocean_b200.so")
HEADER = os.path.join(os.path.dirname(PKG), "include", "ocean_b200.h")

OCN_OK, OCN_ERR_CONFIG, OCN_ERR_MESH, OCN_ERR_NUMERIC = 0, 2, 3, 4
OCN_ERR_IO, OCN_ERR_DOMAIN, OCN_ERR_CUDA, OCN_ERR_ARG = 5, 6, 7, 8


class OceanError(RuntimeError):
    status = -1


class ConfigError(OceanError):
    status = OCN_ERR_CONFIG


class MeshError(OceanError):
    status = OCN_ERR_MESH


class NumericError(OceanError):
    status = OCN_ERR_NUMERIC


class IoError(OceanError):
    status = OCN_ERR_IO


class DomainError(OceanError):
    status = OCN_ERR_DOMAIN


class OceanCudaError(OceanError):
    status = OCN_ERR_CUDA


class ArgumentError(OceanError):
    status = OCN_ERR_ARG


_BY_STATUS = {c.status: c for c in (ConfigError, MeshError, NumericError, IoError, DomainError,
                                    OceanCudaError, ArgumentError)}

vp = C.c_void_p
d = C.POINTER(C.c_double)
f32 = C.POINTER(C.c_float)
i32 = C.POINTER(C.c_int32)
u32 = C.POINTER(C.c_uint32)
u8 = C.POINTER(C.c_uint8)
ci = C.c_int
cd = C.c_double
i64 = C.c_int64
pvp = C.POINTER(C.c_void_p)

# name -> (restype, argtypes); mirrors include/ocean_b200.h one to one
SIGNATURES = {
    "ocn_abi_version": (ci, []),
    "ocn_ctx_create": (ci, [ci, pvp]),
    "ocn_ctx_create_priority": (ci, [ci, ci, pvp]),
    "ocn_ctx_destroy": (ci, [vp]),
    "ocn_last_error": (C.c_char_p, [vp]),
    "ocn_ctx_synchronize": (ci, [vp]),
    "ocn_ctx_stream": (vp, [vp]),
    "ocn_ctx_kernel_launches": (C.c_uint64, [vp]),
    "ocn_ctx_profile": (ci, [vp, ci]),
    "ocn_ctx_profile_read": (ci, [vp, ci, d, C.POINTER(C.c_uint64)]),
    "ocn_ctx_profile_reset": (ci, [vp]),
    "ocn_spectrum_validate": (ci, [C.POINTER(SpectrumParams)]),
    "ocn_alpha": (cd, [C.POINTER(SpectrumParams)]),
    "ocn_peak_omega": (cd, [C.POINTER(SpectrumParams)]),
    "ocn_standard_peak_omega": (cd, [C.POINTER(SpectrumParams)]),
    "ocn_dispersion": (cd, [cd, cd]),
    "ocn_jonswap": (ci, [cd, C.POINTER(SpectrumParams), d]),
    "ocn_beta_s": (cd, [cd]),
    "ocn_directional_kernel": (cd, [cd, cd]),
    "ocn_donelan_banner": (cd, [cd, cd, cd]),
    "ocn_swell_spread": (cd, [cd, cd, cd, cd]),
    "ocn_q_dbxi_approx": (cd, [cd]),
    "ocn_q_dbxi_quadrature": (cd, [cd, cd, ci]),
    "ocn_directional": (cd, [cd, cd, C.POINTER(SpectrumParams)]),
    "ocn_h0_variance": (cd, [cd, cd, cd, cd, cd, C.POINTER(SpectrumParams)]),
    "ocn_damping_factor": (cd, [cd, cd, cd, cd]),
    "ocn_attenuation": (cd, [cd, cd]),
    "ocn_log_distribution": (ci, [cd, cd, d]),
    "ocn_exp_interp": (ci, [cd, cd, cd, cd, cd, d]),
    "ocn_slice_depths": (ci, [C.POINTER(SliceConfig), d]),
    "ocn_cascades_create": (ci, [vp, ci, ci, d, d, d, u32, C.POINTER(SpectrumParams), pvp]),
    "ocn_cascades_create_multi": (ci, [vp, ci, ci, d, d, d, u32, C.POINTER(SpectrumParams), pvp]),
    "ocn_cascades_create_frames": (ci, [vp, ci, ci, d, d, d, u32, C.POINTER(SpectrumParams), ci, cd,
                                        pvp]),
    "ocn_cascades_destroy": (ci, [vp]),
    "ocn_cascades_info": (ci, [vp, C.POINTER(ci), C.POINTER(ci)]),
    "ocn_cascades_download": (ci, [vp, ci, d, d, u8, d]),
    "ocn_assemble_coefficients": (ci, [vp, ci, cd, cd, d]),
    "ocn_maps_create": (ci, [vp, pvp]),
    "ocn_maps_create_bare": (ci, [vp, ci, ci, d, pvp]),
    "ocn_maps_upload": (ci, [vp, ci, ci, d]),
    "ocn_maps_destroy": (ci, [vp]),
    "ocn_surface_generate": (ci, [vp, cd, cd]),
    "ocn_maps_time": (ci, [vp, d]),
    "ocn_surface_generate_batch": (ci, [vp, cd, cd, cd]),
    "ocn_maps_set_assembly": (ci, [vp, ci]),
    "ocn_maps_download_assembly": (ci, [vp, ci, ci, f32]),
    "ocn_maps_download": (ci, [vp, ci, ci, d]),
    "ocn_maps_download_f32": (ci, [vp, ci, ci, f32]),
    "ocn_maps_device_field": (ci, [vp, ci, ci, C.POINTER(f32)]),
    "ocn_slices_create": (ci, [vp, C.POINTER(SliceConfig), pvp]),
    "ocn_slices_destroy": (ci, [vp]),
    "ocn_velocity_build": (ci, [vp, cd]),
    "ocn_slices_depths": (ci, [vp, C.POINTER(ci), d]),
    "ocn_slices_download": (ci, [vp, ci, ci, ci, d]),
    "ocn_spectral_step": (ci, [vp, vp, cd, cd]),
    "ocn_spectral_plan_info": (ci, [vp, vp, ci, C.POINTER(XformInfo), C.POINTER(ci)]),
    "ocn_ifft2_centered": (ci, [vp, ci, d, d]),
    "ocn_ifft2_pair": (ci, [vp, ci, d, d, d, d]),
    "ocn_maps_sample": (ci, [vp, ci, i64, d, d]),
    "ocn_sample_displacement": (ci, [vp, i64, d, d]),
    "ocn_height_at": (ci, [vp, i64, d, d]),
    "ocn_height_at_tolerance": (ci, [vp, i64, d, cd, ci, d, i32]),
    "ocn_surface_assemble": (ci, [vp, i64, d, d]),
    "ocn_sample_slice": (ci, [vp, ci, i64, d, d]),
    "ocn_velocity_at": (ci, [vp, i64, d, ci, ci, d]),
    "ocn_mesh_create": (ci, [vp, ci, d, ci, i32, d, d, cd, pvp]),
    "ocn_mesh_destroy": (ci, [vp]),
    "ocn_hydro_aggregate": (ci, [vp, C.POINTER(Pose), C.POINTER(Fluid), d, C.POINTER(HydroReport)]),
    "ocn_hydro_aggregate_batch": (ci, [ci, pvp, C.POINTER(Pose), C.POINTER(Fluid),
                                       C.POINTER(HydroReport)]),
    "ocn_hydro_report_get": (ci, [vp, C.POINTER(HydroReport)]),
    "ocn_hydro_reports_get": (ci, [ci, pvp, C.POINTER(HydroReport)]),
    "ocn_hydro_vertices": (ci, [vp, d, d]),
    "ocn_hydro_states": (ci, [vp, ci, C.POINTER(TriangleState), C.POINTER(ci)]),
    "ocn_hydro_waterline": (ci, [vp, C.POINTER(ci), C.POINTER(ci), i32, d]),
    "ocn_zone_create": (ci, [vp, C.POINTER(FdmConfig), cd, cd, cd, cd, pvp]),
    "ocn_zone_destroy": (ci, [vp]),
    "ocn_zone_get_state": (ci, [vp, C.POINTER(ZoneState)]),
    "ocn_zone_update_stability": (ci, [vp, cd, cd]),
    "ocn_zone_step": (ci, [vp, cd, cd, cd]),
    "ocn_zone_apply_cells": (ci, [vp, ci, i32, d]),
    "ocn_zone_compute_mask": (ci, [vp, ci, i32, d, cd, cd, cd, cd, C.POINTER(MaskFrame),
                                   C.POINTER(MaskParams), ci, C.POINTER(ci)]),
    "ocn_zone_mask_from_hydro": (ci, [vp, vp, cd, cd, cd, cd, C.POINTER(MaskFrame),
                                      C.POINTER(MaskParams)]),
    "ocn_zone_mask_download": (ci, [vp, ci, i32, d, C.POINTER(ci)]),
    "ocn_zone_sample": (ci, [vp, i64, d, d]),
    "ocn_zone_download": (ci, [vp, d, d]),
    "ocn_zone_upload": (ci, [vp, d, d]),
    "ocn_slab_create": (ci, [vp, ci, ci, ci, cd, cd, cd, C.c_uint32, C.POINTER(SpectrumParams), pvp]),
    "ocn_slab_destroy": (ci, [vp]),
    "ocn_slab_info": (ci, [vp, C.POINTER(ci), C.POINTER(ci), C.POINTER(C.c_size_t)]),
    "ocn_slab_rows": (ci, [vp, cd, cd, vp]),
    "ocn_slab_cols": (ci, [vp, vp]),
    "ocn_slab_download": (ci, [vp, ci, d]),
    "ocn_comm_unique_id": (ci, [C.c_char_p]),
    "ocn_comm_create": (ci, [vp, C.c_char_p, ci, ci, pvp]),
    "ocn_comm_destroy": (ci, [vp]),
    "ocn_comm_info": (ci, [vp, C.POINTER(ci), C.POINTER(ci)]),
    "ocn_slab_exchange": (ci, [vp, vp, ci, vp, vp]),
    "ocn_slab_frame": (ci, [vp, vp, cd, cd, vp, vp]),
    "ocn_compose_height": (ci, [vp, ci, pvp, i64, d, d]),
    "ocn_compose_grid": (ci, [vp, ci, pvp, ci, cd, d]),
    "ocn_heightfield_write_field": (ci, [vp, ci, ci, C.c_float, C.c_char_p]),
    "ocn_heightfield_write_composed": (ci, [vp, ci, pvp, ci, cd, C.c_float, C.c_char_p]),
    "ocn_zone_mask_from_hydro_deferred": (ci, [vp, vp, cd, cd, cd, cd, C.POINTER(MaskFrame), C.POINTER(MaskParams)]),
    "ocn_zone_apply_last_mask": (ci, [vp]),
    "ocn_bodies_step": (ci, [ci, C.POINTER(BodyFrame), C.POINTER(Fluid), cd, C.POINTER(HydroReport)]),
    "ocn_sim_create": (ci, [vp, C.POINTER(SimConfig), ci, C.POINTER(SimBody), pvp]),
    "ocn_sim_destroy": (ci, [vp]),
    "ocn_sim_step": (ci, [vp, ci]),
    "ocn_sim_body_state": (ci, [vp, ci, d, C.POINTER(HydroReport)]),
    "ocn_sim_timing": (ci, [vp, d]),
    "ocn_sim_set_timing": (ci, [vp, ci]),
    "ocn_sim_info": (ci, [vp, d, C.POINTER(ci), pvp, pvp, pvp]),
    "ocn_direct_create": (ci, [vp, cd, pvp]),
    "ocn_direct_destroy": (ci, [vp]),
    "ocn_direct_modes": (ci, [vp, C.POINTER(C.c_int64)]),
    "ocn_direct_evaluate": (ci, [vp, i64, d, d]),
}

_lib = None


def lib():
    """Load libocean_b200.so (building it first if it is missing and nvcc exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        from . import build as _b
        _b.build()
    L = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def check(status: int, ctx=None, where: str = ""):
    if status == OCN_OK:
        return
    msg = lib().ocn_last_error(ctx)
    msg = msg.decode() if msg else ""
    cls = _BY_STATUS.get(status, OceanError)
    raise cls(f"{where}: {msg}" if where else msg)


def header_symbols() -> list[str]:
    """Every function the public header declares (for the export check)."""
    import re
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^OCN_API\s+[\w\s\*]+?\b(ocn_\w+)\s*\(", txt, flags=re.M)))
