"""TEST INFRASTRUCTURE ONLY — ctypes mirrors of the oracle's own C structs."""
import ctypes as C

from paper_2503_03326_b200._types import FdmConfig

_d = C.POINTER(C.c_double)


class OrcSurface(C.Structure):
    _fields_ = [("n", C.c_int), ("C", C.c_int), ("lengths", _d), ("maps", _d)]


class OrcSlices(C.Structure):
    _fields_ = [("n", C.c_int), ("C", C.c_int), ("D", C.c_int), ("lengths", _d), ("depths", _d),
                ("y_min", C.c_double), ("y_max", C.c_double), ("data", _d)]


class OrcZone(C.Structure):
    _fields_ = [("cfg", FdmConfig), ("n", C.c_int), ("margin", C.c_int), ("delta", C.c_double),
                ("c", C.c_double), ("damping", C.c_double), ("origin", C.c_double * 2),
                ("pos_curr", C.c_double * 2), ("carry", C.c_double * 2),
                ("last_shift", C.c_int * 2), ("dropped_wake", C.c_int), ("curr", _d), ("prev", _d)]


class OrcFluid(C.Structure):
    _fields_ = [("surface", C.c_void_p), ("slices", C.c_void_p), ("velocity_clamp", C.c_int),
                ("n_zones", C.c_int), ("zones", C.c_void_p), ("wind", C.c_double * 3),
                ("water_density", C.c_double), ("air_density", C.c_double),
                ("cd_water", C.c_double), ("cd_air", C.c_double), ("n_profile", C.c_int),
                ("profile", _d)]


class OrcClipOut(C.Structure):
    _fields_ = [("capacity_states", C.c_int), ("states", C.c_void_p), ("n_states", C.c_int),
                ("capacity_loops", C.c_int), ("loop_offsets", C.POINTER(C.c_int32)),
                ("capacity_points", C.c_int), ("points", _d), ("n_loops", C.c_int),
                ("n_points", C.c_int), ("submerged_area", C.c_double), ("dry_area", C.c_double),
                ("degenerate_skipped", C.c_int)]
