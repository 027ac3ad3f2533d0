"""ctypes mirrors of the POD structs of include/ocean_b200.h (layout-exact)."""
import ctypes as C

c_double3 = C.c_double * 3


class SpectrumParams(C.Structure):
    """ocn_spectrum_params — SpectrumParams, spectra.hpp:17-34."""

    _fields_ = [
        ("wind_speed", C.c_double),
        ("fetch", C.c_double),
        ("wind_direction", C.c_double),
        ("swell", C.c_double),
        ("direction_mix", C.c_double),
        ("gravity", C.c_double),
        ("rng_seed", C.c_uint64),
        ("has_peak_omega_override", C.c_int32),
        ("reserved0", C.c_int32),
        ("peak_omega_override", C.c_double),
    ]

    @classmethod
    def make(cls, wind_speed=5.0, fetch=1e5, wind_direction=0.0, swell=0.0, direction_mix=0.0,
             gravity=9.80665, rng_seed=0, peak_omega_override=None):
        p = cls()
        p.wind_speed, p.fetch, p.wind_direction = wind_speed, fetch, wind_direction
        p.swell, p.direction_mix, p.gravity, p.rng_seed = swell, direction_mix, gravity, rng_seed
        if peak_omega_override is not None:
            p.has_peak_omega_override = 1
            p.peak_omega_override = peak_omega_override
        return p

    def standard_peak_omega(self):
        """spectra.cpp:19-21: 22 (g^2 / (U F))^(1/3)."""
        import math
        return 22.0 * math.cbrt(self.gravity * self.gravity / (self.wind_speed * self.fetch))


class SliceConfig(C.Structure):
    """ocn_slice_config — SliceConfig, velocity.hpp:51-58."""

    _fields_ = [
        ("y_min", C.c_double),
        ("y_max", C.c_double),
        ("count", C.c_int32),
        ("distribution", C.c_int32),
        ("single_precision", C.c_int32),
        ("reserved0", C.c_int32),
    ]

    @classmethod
    def make(cls, y_min=-125.0, y_max=4.5, count=8, distribution=0, single_precision=0):
        c = cls()
        c.y_min, c.y_max, c.count, c.distribution, c.single_precision = (
            y_min, y_max, count, distribution, single_precision)
        return c


class Pose(C.Structure):
    """ocn_pose — BodyPose, hydro.hpp:17-35; orientation (w, x, y, z)."""

    _fields_ = [
        ("position", C.c_double * 3),
        ("orientation", C.c_double * 4),
        ("linear_velocity", C.c_double * 3),
        ("angular_velocity", C.c_double * 3),
        ("com_body", C.c_double * 3),
    ]

    @classmethod
    def make(cls, position=(0, 0, 0), orientation=(1, 0, 0, 0), linear_velocity=(0, 0, 0),
             angular_velocity=(0, 0, 0), com_body=(0, 0, 0)):
        p = cls()
        p.position[:] = position
        p.orientation[:] = orientation
        p.linear_velocity[:] = linear_velocity
        p.angular_velocity[:] = angular_velocity
        p.com_body[:] = com_body
        return p


# ocn_velocity_fn: host water_velocity sampler (user, n, xzy[3n] in, out[3n])
VelocityFn = C.CFUNCTYPE(None, C.c_void_p, C.c_int64, C.POINTER(C.c_double), C.POINTER(C.c_double))


class Fluid(C.Structure):
    """ocn_fluid — FluidQuery (hydro.hpp:38-49) + DragCoefficients."""

    _fields_ = [
        ("maps", C.c_void_p),
        ("slices", C.c_void_p),
        ("velocity_clamp", C.c_int32),
        ("n_zones", C.c_int32),
        ("zones", C.POINTER(C.c_void_p)),
        ("wind", C.c_double * 3),
        ("water_density", C.c_double),
        ("air_density", C.c_double),
        ("cd_water", C.c_double),
        ("cd_air", C.c_double),
        ("n_profile", C.c_int32),
        ("reserved0", C.c_int32),
        ("host_profile", C.POINTER(C.c_double)),
        ("host_velocity", VelocityFn),
        ("host_velocity_user", C.c_void_p),
    ]


class HydroReport(C.Structure):
    """ocn_hydro_report — HydroReport, hydro.hpp:97-109 (+ composed load)."""

    _fields_ = [
        ("submerged_volume", C.c_double),
        ("center_of_immersion", C.c_double * 3),
        ("buoyancy_force", C.c_double * 3),
        ("water_drag", C.c_double * 3),
        ("air_drag", C.c_double * 3),
        ("water_center", C.c_double * 3),
        ("air_center", C.c_double * 3),
        ("submerged_area", C.c_double),
        ("dry_area", C.c_double),
        ("force", C.c_double * 3),
        ("torque", C.c_double * 3),
        ("volume_clamped", C.c_int32),
        ("has_center_of_immersion", C.c_int32),
        ("state_count", C.c_int32),
        ("degenerate_skipped", C.c_int32),
        ("waterline_loops", C.c_int32),
        ("waterline_points", C.c_int32),
        ("nonfinite", C.c_int32),
        ("reserved0", C.c_int32),
    ]

    def as_dict(self):
        out = {}
        for name, _ in self._fields_:
            v = getattr(self, name)
            out[name] = list(v) if hasattr(v, "__len__") else v
        return out


class TriangleState(C.Structure):
    """ocn_triangle_state — TriangleState, hydro.hpp:53-60."""

    _fields_ = [
        ("parent", C.c_int32),
        ("status", C.c_int32),
        ("area", C.c_double),
        ("centroid", C.c_double * 3),
        ("depth", C.c_double),
        ("normal", C.c_double * 3),
    ]


class FdmConfig(C.Structure):
    """ocn_fdm_config — FdmConfig + DampingParams, interactive.hpp:16-33."""

    _fields_ = [
        ("grid_size", C.c_int32),
        ("margin", C.c_int32),
        ("delta_min", C.c_double),
        ("delta_max", C.c_double),
        ("delta_rate_limit", C.c_double),
        ("d0", C.c_double),
        ("d_max", C.c_double),
        ("v_max", C.c_double),
    ]

    @classmethod
    def make(cls, grid_size=512, margin=16, delta_min=0.0, delta_max=0.0, delta_rate_limit=0.05,
             d0=0.98, d_max=0.999, v_max=5.0):
        c = cls()
        c.grid_size, c.margin, c.delta_min, c.delta_max = grid_size, margin, delta_min, delta_max
        c.delta_rate_limit, c.d0, c.d_max, c.v_max = delta_rate_limit, d0, d_max, v_max
        return c


class MaskParams(C.Structure):
    _fields_ = [("back_height", C.c_double), ("intensity", C.c_double), ("amplitude", C.c_double)]

    @classmethod
    def make(cls, back_height=0.0, intensity=1.0, amplitude=1.0):
        p = cls()
        p.back_height, p.intensity, p.amplitude = back_height, intensity, amplitude
        return p


class MaskFrame(C.Structure):
    _fields_ = [
        ("center_x", C.c_double),
        ("half_beam", C.c_double),
        ("z_min", C.c_double),
        ("z_max", C.c_double),
        ("mesh_height", C.c_double),
        ("volume_ratio", C.c_double),
    ]

    @classmethod
    def make(cls, center_x=0.0, half_beam=1.0, z_min=-1.0, z_max=1.0, mesh_height=1.0,
             volume_ratio=0.0):
        f = cls()
        f.center_x, f.half_beam, f.z_min, f.z_max = center_x, half_beam, z_min, z_max
        f.mesh_height, f.volume_ratio = mesh_height, volume_ratio
        return f


class ZoneState(C.Structure):
    """ocn_zone_state — scalar state of an FdmZone (interactive.hpp:65-104)."""

    _fields_ = [
        ("grid_size", C.c_int32),
        ("margin", C.c_int32),
        ("spacing", C.c_double),
        ("wave_speed", C.c_double),
        ("damping", C.c_double),
        ("origin", C.c_double * 2),
        ("pos_curr", C.c_double * 2),
        ("carry", C.c_double * 2),
        ("last_shift", C.c_int32 * 2),
        ("dropped_wake", C.c_int32),
        ("reserved0", C.c_int32),
        ("delta_min", C.c_double),
        ("delta_max", C.c_double),
    ]


class BodyFrame(C.Structure):
    """ocn_body_frame — one body of a Simulation step (sim.cpp:73-109)."""

    _fields_ = [
        ("mesh", C.c_void_p),
        ("zone", C.c_void_p),
        ("pose", Pose),
        ("cd_water", C.c_double),
        ("cd_air", C.c_double),
        ("speed", C.c_double),
        ("yaw", C.c_double),
        ("frame", MaskFrame),
        ("mask", MaskParams),
    ]


class XformInfo(C.Structure):
    """ocn_xform_info — one packed transform of a spectral step's plan."""

    _fields_ = [
        ("cascade", C.c_int32),
        ("kind", C.c_int32),
        ("index0", C.c_int32),
        ("index1", C.c_int32),
        ("row_half", C.c_int32),
        ("executed", C.c_int32),
        ("y0", C.c_double),
        ("y1", C.c_double),
    ]


class SimConfig(C.Structure):
    """ocn_sim_config — the scenario part of Simulation (sim.hpp:16-60)."""

    _fields_ = [
        ("resolution", C.c_int32),
        ("count", C.c_int32),
        ("lengths", C.c_double * 16),
        ("cutoffs", C.c_double * 16),
        ("spectrum", SpectrumParams),
        ("slices", SliceConfig),
        ("choppiness", C.c_double),
        ("dt", C.c_double),
        ("wind", C.c_double * 3),
        ("rebuild_stride", C.c_int32),
        ("pipelined", C.c_int32),
    ]


class SimBody(C.Structure):
    """ocn_sim_body — BodyConfig (scenario.hpp:30-47) + the hull's TriMesh properties."""

    _fields_ = [
        ("mesh", C.c_void_p),
        ("volume", C.c_double),
        ("centroid", C.c_double * 3),
        ("bbox_min", C.c_double * 3),
        ("bbox_max", C.c_double * 3),
        ("unit_inertia", C.c_double * 9),
        ("density", C.c_double),
        ("mass", C.c_double),
        ("has_mass", C.c_int32),
        ("box_inertia", C.c_int32),
        ("position", C.c_double * 3),
        ("yaw", C.c_double),
        ("initial_velocity", C.c_double * 3),
        ("cd_water", C.c_double),
        ("cd_air", C.c_double),
        ("angular_damping", C.c_double),
        ("n_thrust", C.c_int32),
        ("reserved0", C.c_int32),
        ("thrust", C.POINTER(C.c_double)),
        ("fdm", FdmConfig),
        ("mask", MaskParams),
    ]
