"""Simulation::step over the device hot path (sim.cpp:16-131).

The caller of the per-frame path: surface maps and velocity slices from one
spectral step, then per body the hull forces against the composed surface
(height_at plus every OTHER body's FDM zone, sim.cpp:44-51), the stability
update and the wake mask, then all masks applied and every zone stepped, then
the rigid-body integration. Every field-sized stage runs on the device
(ocn_spectral_step, ocn_hydro_aggregate with the zone list,
ocn_zone_mask_from_hydro_deferred / ocn_zone_apply_last_mask, ocn_zone_step);
the rigid body (13 doubles per body, rigid_body.cpp:6-61) is host scalar code,
as in the reference. Only the hydro report (forces, centres, volume) crosses
to the host per body and step, read after every body's device stages are
enqueued (one stream synchronisation per step).

Ordering matches sim.cpp exactly: body i's aggregate sees the zones of bodies
< i after their update_stability (the spacing changes immediately) but before
any mask is applied, so masks are computed deferred and applied after every
body's aggregate (sim.cpp:73-109).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import ocean as oc
from ._abi import DomainError, NumericError, check, lib
from ._types import BodyFrame, FdmConfig, HydroReport, MaskFrame, MaskParams, Pose, SliceConfig, SpectrumParams

import ctypes as C


# ---------------------------------------------------------------- quaternions (core.hpp:142-186)
def quat_axis_angle(axis, angle):
    n = math.sqrt(axis[0] ** 2 + axis[1] ** 2 + axis[2] ** 2)
    if n < 1e-300:
        return np.array([1.0, 0.0, 0.0, 0.0])
    h = 0.5 * angle
    s = math.sin(h) / n
    return np.array([math.cos(h), axis[0] * s, axis[1] * s, axis[2] * s])


def quat_mul(a, b):
    w, x, y, z = a
    ow, ox, oy, oz = b
    return np.array([w * ow - x * ox - y * oy - z * oz, w * ox + x * ow + y * oz - z * oy,
                     w * oy - x * oz + y * ow + z * ox, w * oz + x * oy - y * ox + z * ow])


def quat_normalized(q):
    return q / math.sqrt(float(q @ q))


def quat_rotate(q, v):
    u = q[1:]
    t = np.cross(u, v) * 2.0
    return v + t * q[0] + np.cross(u, t)


def quat_matrix(q):
    w, x, y, z = q
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


def pose_yaw(q):
    """BodyPose::yaw, hydro.hpp:31-34."""
    bow = quat_rotate(q, np.array([0.0, 0.0, 1.0]))
    return math.atan2(bow[0], bow[2])


# ---------------------------------------------------------------- rigid body (rigid_body.cpp)
class RigidBody:
    """rigid_body.cpp:6-61: mass, body inertia, pose, angular momentum, force / torque accumulators."""

    def __init__(self, mass, inertia_body, position, orientation, linear_velocity, angular_velocity,
                 com_body):
        if not mass > 0.0:
            raise oc.ConfigError("rigid body mass must be > 0")
        self.mass = float(mass)
        self.inertia_body = np.asarray(inertia_body, np.float64)
        self.inertia_body_inv = np.linalg.inv(self.inertia_body)
        self.position = np.asarray(position, np.float64)
        self.orientation = quat_normalized(np.asarray(orientation, np.float64))
        self.linear_velocity = np.asarray(linear_velocity, np.float64)
        self.angular_velocity = np.asarray(angular_velocity, np.float64)
        self.com_body = np.asarray(com_body, np.float64)
        r = quat_matrix(self.orientation)
        self.angular_momentum = (r @ self.inertia_body @ r.T) @ self.angular_velocity
        self.force = np.zeros(3)
        self.torque = np.zeros(3)

    @classmethod
    def from_mesh(cls, mesh: "oc.TriMesh", density, position, orientation, linear_velocity,
                  box_inertia=False):
        """RigidBody::from_mesh, rigid_body.cpp:16-34."""
        mass = density * mesh.volume
        if box_inertia:
            s = mesh.bbox_max - mesh.bbox_min
            inertia = np.diag([mass / 12.0 * (s[1] ** 2 + s[2] ** 2), mass / 12.0 * (s[0] ** 2 + s[2] ** 2),
                               mass / 12.0 * (s[0] ** 2 + s[1] ** 2)])
        else:
            inertia = mesh.unit_inertia * density
        return cls(mass, inertia, position, orientation, linear_velocity, np.zeros(3), mesh.centroid)

    def pose(self) -> Pose:
        return Pose.make(position=tuple(self.position), orientation=tuple(self.orientation),
                         linear_velocity=tuple(self.linear_velocity),
                         angular_velocity=tuple(self.angular_velocity), com_body=tuple(self.com_body))

    def apply_force(self, f):
        self.force = self.force + f

    def apply_force_at(self, f, world_point):
        """rigid_body.cpp:36-39."""
        self.force = self.force + f
        self.torque = self.torque + np.cross(np.asarray(world_point) - self.position, f)

    def integrate(self, gravity, dt, angular_damping):
        """Semi-implicit Euler, rigid_body.cpp:41-61."""
        if not dt > 0.0:
            raise DomainError("integrate: dt must be > 0")
        self.linear_velocity = self.linear_velocity + (self.force / self.mass + gravity) * dt
        self.angular_momentum = self.angular_momentum + self.torque * dt
        if angular_damping > 0.0:
            self.angular_momentum = self.angular_momentum * (1.0 - angular_damping * dt)
        r = quat_matrix(self.orientation)
        self.angular_velocity = (r @ self.inertia_body_inv @ r.T) @ self.angular_momentum
        self.position = self.position + self.linear_velocity * dt
        w = float(np.linalg.norm(self.angular_velocity))
        if w > 1e-300:
            dq = quat_axis_angle(self.angular_velocity / w, w * dt)
            self.orientation = quat_normalized(quat_mul(dq, self.orientation))
        self.force = np.zeros(3)
        self.torque = np.zeros(3)


# ---------------------------------------------------------------- scene
@dataclass
class BodyConfig:
    """The per-body part of the scenario (scenario.hpp BodyConfig) this path uses."""
    vertices: np.ndarray
    triangles: np.ndarray
    position: Sequence[float] = (0.0, 0.0, 0.0)
    yaw: float = 0.0
    initial_velocity: Sequence[float] = (0.0, 0.0, 0.0)
    density: float = 500.0
    cd_water: float = 1.0
    cd_air: float = 1.0
    angular_damping: float = 0.0
    box_inertia: bool = False
    fdm: FdmConfig = field(default_factory=lambda: FdmConfig.make())
    mask: MaskParams = field(default_factory=lambda: MaskParams.make())
    thrust: Sequence = ()  # [(until, (fx, fy, fz))], body-frame force (sim.cpp:53-57)


class _Body:
    def __init__(self, cfg: BodyConfig, dt: float, ctx):
        self.config = cfg
        self.mesh = oc.TriMesh(cfg.vertices, cfg.triangles, ctx=ctx)
        q = quat_axis_angle((0.0, 1.0, 0.0), cfg.yaw)
        pos = np.asarray(cfg.position, np.float64) + quat_rotate(q, self.mesh.centroid)
        self.rigid = RigidBody.from_mesh(self.mesh, cfg.density, pos, q, cfg.initial_velocity,
                                         cfg.box_inertia)
        ext = self.mesh.bbox_max - self.mesh.bbox_min
        self.zone = oc.FdmZone(cfg.fdm, max(ext[0], ext[2]), (pos[0], pos[2]), dt, ctx=ctx)
        self.report: Optional[oc.HydroResult] = None


class Simulation:
    """sim.cpp:16-131 over the device path. Spectrum, cascades and slice config as
    CascadeSet / SliceConfig; gravity from the spectrum parameters."""

    def __init__(self, cascade_config: "oc.CascadeConfig", spectrum: SpectrumParams,
                 slices: SliceConfig, bodies: Sequence[BodyConfig], dt: float = 1.0 / 60.0,
                 wind=(0.0, 0.0, 0.0), choppiness: float = 1.0, rebuild_stride: int = 1,
                 ctx=None, pipelined: bool = False, device: int = 0, native: bool = False,
                 concurrent: bool = False):
        """pipelined: the spectral step of step f+1 (a pure function of time) runs on a
        low-priority context into the other of two map / slice buffers while step f's
        bodies run on a high-priority one; CUDA events order the buffers (the bench.py
        frame pipeline). Results are identical to the serial order.
        native: the per-body stages go through one ocn_bodies_step call.
        concurrent (implies pipelined): every body gets its own high-priority context, so
        the bodies' latency-bound hull chains overlap; CUDA events keep sim.cpp's order
        (every aggregate after every zone's previous step, every zone's mask / step after
        every other body's aggregate)."""
        if not dt > 0.0:
            raise oc.ConfigError("dt must be > 0")
        if pipelined and rebuild_stride != 1:
            raise oc.ConfigError("pipelined Simulation rebuilds the slices every step (rebuild_stride 1)")
        self.dt = dt
        self.wind = tuple(float(w) for w in wind)
        self.choppiness = choppiness
        self.rebuild_stride = max(1, int(rebuild_stride))
        self.gravity = spectrum.gravity
        pipelined = pipelined or concurrent
        self.pipelined = pipelined
        self.concurrent = concurrent
        self.native = native  # per-body stages in one ocn_bodies_step call
        if pipelined:
            import torch
            self.sctx = oc.Context(device, priority=-1)  # spectral steps
            self.ctx = oc.Context(device, priority=1)    # bodies
            self._S = torch.cuda.ExternalStream(self.sctx.stream, device=f"cuda:{device}")
            self._H = torch.cuda.ExternalStream(self.ctx.stream, device=f"cuda:{device}")
            self._ready = [torch.cuda.Event(), torch.cuda.Event()]
            self._consumed = [torch.cuda.Event(), torch.cuda.Event()]
        else:
            self.ctx = self.sctx = ctx or oc.Context.default()
        nbuf = 2 if pipelined else 1
        self.cascades = oc.CascadeSet(cascade_config, spectrum, ctx=self.sctx)
        self._maps = [oc.SurfaceMaps(self.cascades) for _ in range(nbuf)]
        self._slices = [oc.VelocitySlices(self.cascades, slices) for _ in range(nbuf)]
        self._cur = 0
        oc.spectral_step(self._maps[0], self._slices[0], 0.0, choppiness)  # sim.cpp:18-20
        if concurrent:
            import torch
            self._bctx = [oc.Context(device, priority=1) for _ in bodies]
            self._B = [torch.cuda.ExternalStream(c.stream, device=f"cuda:{device}") for c in self._bctx]
            self._agg = [torch.cuda.Event() for _ in bodies]
            # per map / slice buffer: the aggregates of the step that last read it
            self._aggb = [[torch.cuda.Event() for _ in bodies] for _ in range(nbuf)]
            self._zdone = [torch.cuda.Event() for _ in bodies]
            self.bodies: List[_Body] = [_Body(b, dt, c) for b, c in zip(bodies, self._bctx)]
        else:
            self.bodies = [_Body(b, dt, self.ctx) for b in bodies]
        self.time = 0.0
        self.step_index = 0
        self._prefetched = False
        if pipelined:
            self._ready[0].record(self._S)

    @property
    def maps(self) -> "oc.SurfaceMaps":
        return self._maps[self._cur]

    @property
    def slices(self) -> "oc.VelocitySlices":
        return self._slices[self._cur]

    def _spectral(self, k: int, t: float, with_slices: bool):
        oc.spectral_step(self._maps[k], self._slices[k] if with_slices else None, t, self.choppiness)

    def compose_height(self, xz, exclude_body: int = -1):
        """sim.cpp:44-51, batched on the device."""
        zones = [b.zone for i, b in enumerate(self.bodies) if i != exclude_body]
        return oc.compose_height(self.maps, xz, zones)

    def thrust_force(self, body: _Body):
        for until, f in body.config.thrust:
            if self.time < until:
                return quat_rotate(body.rigid.orientation, np.asarray(f, np.float64))
        return np.zeros(3)

    def _mask_frame(self, body: _Body) -> MaskFrame:
        m = body.mesh
        return MaskFrame.make(half_beam=float(m.bbox_max[0] - m.bbox_min[0]), z_min=float(m.bbox_min[2]),
                              z_max=float(m.bbox_max[2]), mesh_height=m.height())

    def _bodies_native(self, speeds, dt):
        """sim.cpp:73-109 for every body in one library call (ocn_bodies_step)."""
        nb = len(self.bodies)
        frames = (BodyFrame * max(nb, 1))()
        for i, body in enumerate(self.bodies):
            f = frames[i]
            f.mesh, f.zone = body.mesh.h.value, body.zone.h.value
            f.pose = body.rigid.pose()
            f.cd_water, f.cd_air = body.config.cd_water, body.config.cd_air
            f.speed, f.yaw = speeds[i], pose_yaw(body.rigid.orientation)
            f.frame = self._mask_frame(body)
            f.mask = body.config.mask
        fluid, _keep = oc._fluid_struct(oc.FluidQuery(maps=self.maps, slices=self.slices, wind=self.wind),
                                        oc.DragCoefficients())
        check(lib().ocn_bodies_step(nb, frames, C.byref(fluid), dt, None), self.ctx.h, "bodies_step")

    def _bodies_calls(self, speeds, dt):
        """The same stages as separate library calls per body."""
        L = lib()
        for i, body in enumerate(self.bodies):
            others = [b.zone for k, b in enumerate(self.bodies) if k != i]
            fluid = oc.FluidQuery(maps=self.maps, slices=self.slices, zones=others, wind=self.wind)
            # enqueued only: the reports are read once after every body's stages
            oc.aggregate(body.mesh, body.rigid.pose(), fluid,
                         oc.DragCoefficients(body.config.cd_water, body.config.cd_air), sync=False)
            body.zone.update_stability(speeds[i], dt)
            frame = self._mask_frame(body)
            check(L.ocn_zone_mask_from_hydro_deferred(body.zone.h, body.mesh.h,
                                                      pose_yaw(body.rigid.orientation),
                                                      float(body.rigid.position[0]),
                                                      float(body.rigid.position[2]), speeds[i],
                                                      C.byref(frame), C.byref(body.config.mask)),
                  self.ctx.h, "mask")
        for body in self.bodies:
            check(L.ocn_zone_apply_last_mask(body.zone.h), self.ctx.h, "apply_mask")
            body.zone.step(dt, (body.rigid.position[0], body.rigid.position[2]))

    def _bodies_concurrent(self, speeds, dt):
        """_bodies_calls with one stream per body and events for sim.cpp's order."""
        L = lib()
        nb = len(self.bodies)
        for i, body in enumerate(self.bodies):
            B = self._B[i]
            for k in range(nb):
                if k != i:
                    B.wait_event(self._zdone[k])  # zone k's previous step (no-op before the first)
            others = [b.zone for k, b in enumerate(self.bodies) if k != i]
            fluid = oc.FluidQuery(maps=self.maps, slices=self.slices, zones=others, wind=self.wind)
            oc.aggregate(body.mesh, body.rigid.pose(), fluid,
                         oc.DragCoefficients(body.config.cd_water, body.config.cd_air), sync=False)
            body.zone.update_stability(speeds[i], dt)
            frame = self._mask_frame(body)
            check(L.ocn_zone_mask_from_hydro_deferred(body.zone.h, body.mesh.h,
                                                      pose_yaw(body.rigid.orientation),
                                                      float(body.rigid.position[0]),
                                                      float(body.rigid.position[2]), speeds[i],
                                                      C.byref(frame), C.byref(body.config.mask)),
                  body.zone.ctx.h, "mask")
            self._agg[i].record(B)
            if self.pipelined:
                self._aggb[self._cur][i].record(B)
        for k, body in enumerate(self.bodies):
            B = self._B[k]
            for i in range(nb):
                if i != k:
                    B.wait_event(self._agg[i])  # every aggregate that read zone k
            check(L.ocn_zone_apply_last_mask(body.zone.h), body.zone.ctx.h, "apply_mask")
            body.zone.step(dt, (body.rigid.position[0], body.rigid.position[2]))
            self._zdone[k].record(B)

    def step(self):
        """sim.cpp:59-124."""
        dt = self.dt
        t_next = self.time + dt
        if not self.pipelined:
            self._spectral(0, t_next, self.step_index % self.rebuild_stride == 0)
        else:
            k = 1 - self._cur
            if not self._prefetched:  # first step: nothing prefetched yet
                self._S.wait_event(self._consumed[k])
                self._spectral(k, t_next, True)
                self._ready[k].record(self._S)
            self._cur = k
            for st in (self._B if self.concurrent else [self._H]):
                st.wait_event(self._ready[k])
        speeds = [float(np.linalg.norm(b.rigid.linear_velocity)) for b in self.bodies]
        if self.concurrent:
            self._bodies_concurrent(speeds, dt)
        elif self.native:
            self._bodies_native(speeds, dt)
        else:
            self._bodies_calls(speeds, dt)
        if self.pipelined:
            # the bodies' stages are enqueued; the next step's spectral step (a function of
            # time only) goes into the other buffer, whose last readers were the PREVIOUS
            # step's bodies -- so it runs while this step's bodies run
            k = 1 - self._cur
            if self.concurrent:
                for ev in self._aggb[k]:
                    self._S.wait_event(ev)
            else:
                self._consumed[self._cur].record(self._H)
                self._S.wait_event(self._consumed[k])
            self._spectral(k, t_next + dt, True)
            self._ready[k].record(self._S)
            self._prefetched = True
        reports = []
        for body in self.bodies:
            rep = HydroReport()
            check(lib().ocn_hydro_report_get(body.mesh.h, C.byref(rep)), body.mesh.ctx.h, "report")
            reports.append(rep)
        for body, rep in zip(self.bodies, reports):
            body.report = r = oc.HydroResult(body.mesh, rep)
            if r.center_of_immersion is not None:
                body.rigid.apply_force_at(r.buoyancy_force, r.water_center)
                body.rigid.apply_force_at(r.water_drag, r.water_center)
            body.rigid.apply_force_at(r.air_drag, r.air_center)
            body.rigid.apply_force(self.thrust_force(body))
            body.rigid.integrate(np.array([0.0, -self.gravity, 0.0]), dt, body.config.angular_damping)
        self.time = t_next
        self.step_index += 1
        self.check_finite()

    def check_finite(self):
        """sim.cpp:126-135."""
        for i, b in enumerate(self.bodies):
            probe = float(b.rigid.position.sum() + b.rigid.linear_velocity.sum())
            if not math.isfinite(probe):
                raise NumericError(f"non-finite body state (body {i}, step {self.step_index})")

    def poses(self) -> np.ndarray:
        """(bodies, 13): position, orientation (w x y z), linear, angular velocity."""
        return np.array([np.concatenate([b.rigid.position, b.rigid.orientation, b.rigid.linear_velocity,
                                         b.rigid.angular_velocity]) for b in self.bodies])


class DeviceSimulation:
    """Simulation::step (sim.cpp:15-131) run entirely by the C++ library over
    device-resident state (ocn_sim): spectral step, every body's hull in one
    batched launch set, deferred masks, zone steps and the rigid-body
    integration in C++ -- one C-ABI call per step. Same scene description as
    Simulation; poses() / submerged volumes / reports read back per step."""

    def __init__(self, cascade_config: "oc.CascadeConfig", spectrum: SpectrumParams,
                 slices: SliceConfig, bodies: Sequence[BodyConfig], dt: float = 1.0 / 60.0,
                 wind=(0.0, 0.0, 0.0), choppiness: float = 1.0, rebuild_stride: int = 1,
                 pipelined: bool = True, device: int = 0):
        from ._types import SimBody, SimConfig
        cascade_config.validate()
        self.ctx = oc.Context(device, priority=1 if pipelined else 0)
        cfg = SimConfig()
        cfg.resolution = cascade_config.resolution
        cfg.count = len(cascade_config.lengths)
        for c, L in enumerate(cascade_config.lengths):
            cfg.lengths[c] = L
        for c, x in enumerate(cascade_config.cutoffs):
            cfg.cutoffs[c] = x
        cfg.spectrum = spectrum
        cfg.slices = slices
        cfg.choppiness, cfg.dt = choppiness, dt
        cfg.wind[:] = tuple(float(w) for w in wind)
        cfg.rebuild_stride, cfg.pipelined = int(rebuild_stride), int(pipelined)
        self.meshes = [oc.TriMesh(b.vertices, b.triangles, ctx=self.ctx) for b in bodies]
        arr = (SimBody * max(len(bodies), 1))()
        self._thrust = []
        for i, (b, m) in enumerate(zip(bodies, self.meshes)):
            sb = arr[i]
            sb.mesh = m.h
            sb.volume = m.volume
            sb.centroid[:] = tuple(m.centroid)
            sb.bbox_min[:] = tuple(m.bbox_min)
            sb.bbox_max[:] = tuple(m.bbox_max)
            sb.unit_inertia[:] = tuple(np.asarray(m.unit_inertia, np.float64).ravel())
            sb.density = b.density
            sb.box_inertia = int(b.box_inertia)
            sb.position[:] = tuple(b.position)
            sb.yaw = b.yaw
            sb.initial_velocity[:] = tuple(b.initial_velocity)
            sb.cd_water, sb.cd_air, sb.angular_damping = b.cd_water, b.cd_air, b.angular_damping
            th = np.ascontiguousarray([[u, *f] for u, f in b.thrust], np.float64).reshape(-1)
            self._thrust.append(th)
            sb.n_thrust = len(b.thrust)
            sb.thrust = th.ctypes.data_as(C.POINTER(C.c_double)) if len(b.thrust) else None
            sb.fdm, sb.mask = b.fdm, b.mask
        h = C.c_void_p()
        check(lib().ocn_sim_create(self.ctx.h, C.byref(cfg), len(bodies), arr, C.byref(h)),
              self.ctx.h, "sim_create")
        self.h = h
        self.n_bodies = len(bodies)

    def step(self, steps: int = 1):
        check(lib().ocn_sim_step(self.h, steps), self.ctx.h, "sim_step")

    def set_timing(self, enabled: bool = True):
        """Collect stage times from now on (ocn_sim_set_timing; off by default)."""
        check(lib().ocn_sim_set_timing(self.h, 1 if enabled else 0), self.ctx.h, "sim_timing")

    def timing(self) -> dict:
        """Cumulative stage seconds with Simulation::timing()'s names (sim.hpp:50-54);
        surface covers the fused maps + slices step (velocity stays 0). Collected
        while set_timing(True) is on."""
        t = np.zeros(5)
        check(lib().ocn_sim_timing(self.h, t.ctypes.data_as(C.POINTER(C.c_double))), self.ctx.h,
              "sim_timing")
        return dict(zip(("surface", "velocity", "hydro", "zones", "integrate"), t.tolist()))

    def poses(self) -> np.ndarray:
        """(bodies, 13): position, orientation (w x y z), linear, angular velocity."""
        out = np.zeros((self.n_bodies, 13))
        for i in range(self.n_bodies):
            check(lib().ocn_sim_body_state(self.h, i, out[i].ctypes.data_as(C.POINTER(C.c_double)),
                                           None), self.ctx.h, "body_state")
        return out

    def reports(self) -> List[HydroReport]:
        reps = []
        for i in range(self.n_bodies):
            r = HydroReport()
            check(lib().ocn_sim_body_state(self.h, i, None, C.byref(r)), self.ctx.h, "body_state")
            reps.append(r)
        return reps

    def __del__(self):
        try:
            if self.h:
                lib().ocn_sim_destroy(self.h)
                self.h = None
        except Exception:
            pass
