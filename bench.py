#!/usr/bin/env python
"""bench.py — per-frame Arc Blanc hot path on B200 (BASELINE.json metric).

Headline workload (one "step" = one frame): the 4-cascade
1024^2 spectrum (U=20, F=1e5, theta0=0.4, xi=0.5, delta=0.5, standard peak,
seed 42; lengths 1024/256/16/4 m) evolved to t, its 8 surface maps + 32
logarithmic velocity-at-depth slices (208 packed 1024^2 inverse FFTs in the
reference; 164 run per frame here, the other 44 are exactly zero in fp32 at
their depth and their planes are zeroed once), fluid-to-solid forces on the
100,352-triangle UV-ellipsoid hull (height_at + velocity_at samplers,
deterministic reductions, waterline), the waterline mask and one 2048^2
Cords-Staadt FDM step. Metric: ocean grid points / s (= 4 * 1024^2 per frame /
frame time) and ms / frame.

The same run also measures the other SURVEY 8d configurations (the "configs"
object of the line; skip with --no-extra-configs):
  1: 600 frames of the reference-default 256^2 cascade in one batched step
     (frames f mod G across ranks), plus the single-frame latency;
  4: 64 independent 3 x 512^2 instances (64/G per rank);
  5: one 16384^2 grid, row slabs per rank, NCCL all-to-all transpose.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config 1|3|4|5]

N > 1 (torchrun, one rank per GPU): config 3 runs independent replicas (configs
2/3 do not shard), weak scaling; configs 1/4/5 split their fixed
work across the ranks (strong scaling); every time is the max over ranks.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

N_GRID = 1024
LENGTHS = [1024.0, 256.0, 16.0, 4.0]
CUTOFFS = [12 * math.pi / 256, 12 * math.pi / 16, 12 * math.pi / 4]
DEPTHS = 32
DT = 1.0 / 60.0
FDM_N, FDM_MARGIN, BODY_SIZE = 2048, 16, 40.0
WIND = (5.0, 0.0, 2.0)
YAW = 0.3
POINTS_PER_FRAME = len(LENGTHS) * N_GRID * N_GRID
# compulsory bytes of the spectral pipeline per frame: fp32-complex
# h0 read once (8 B / cascade-point) + every output field written once in fp32
SPECTRAL_FIELDS = 8 + 3 * DEPTHS
SPECTRAL_BYTES = POINTS_PER_FRAME * (8 + 4 * SPECTRAL_FIELDS)
WORKLOAD = ("config3: 4 cascades x 1024^2 (8 surface maps + 32 velocity slices: 208 packed "
            "2D iFFTs in the reference, 164 executed per frame + 44 exactly zero in fp32 at their "
            "depth, planes zeroed once) + 100,352-tri hull forces + waterline mask + 2048^2 FDM step")


def _params():
    from paper_2503_03326_b200._types import SpectrumParams
    p = SpectrumParams.make(wind_speed=20.0, fetch=1e5, wind_direction=0.4, swell=0.5,
                            direction_mix=0.5, rng_seed=42)
    p.has_peak_omega_override = 1
    p.peak_omega_override = p.standard_peak_omega()
    return p


def _pose(centroid):
    from paper_2503_03326_b200._types import Pose
    return Pose.make(position=(3.0, 0.5, 7.0), orientation=(math.cos(YAW / 2), 0.0, math.sin(YAW / 2), 0.0),
                     linear_velocity=(1.0, 0.0, 4.0), angular_velocity=(0.01, 0.05, 0.02),
                     com_body=centroid)


# ----------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------- our arm
class _SingleStream:
    """Frames whose work is all on one context stream."""

    def contexts(self):
        return [self.ctx]

    def sync(self):
        self.ctx.synchronize()

    def timed_begin(self, ev):
        import torch
        ev.record(torch.cuda.ExternalStream(self.ctx.stream, device=f"cuda:{self.ctx.device}"))

    def timed_end(self, ev):
        self.timed_begin(ev)

    def finish(self, read_report: bool = False):
        pass


class Frame:
    """One config-3 frame of the hot path through the C-ABI (device-resident state).

    Frames are pipelined: the spectral step runs on a low-priority context
    (stream) into double-buffered maps / slices, forces, mask and FDM on a
    high-priority one, so frame f's latency-bound forces / mask / FDM kernels
    fill the SMs beside frame f+1's spectral kernels. Dependencies are CUDA
    events on the two ocn_ctx_stream streams (ready: spectral done; consumed:
    the last reader of a buffer done). pipelined=False runs everything in order
    on one context."""

    def __init__(self, device: int, pipelined: bool = True):
        from paper_2503_03326_b200 import ocean as oc
        from paper_2503_03326_b200._types import FdmConfig, MaskFrame, MaskParams, SliceConfig
        from paper_2503_03326_b200.meshgen import uv_ellipsoid
        import torch
        self.oc = oc
        self.L = oc.lib()
        self.pipelined = pipelined
        self.sctx = oc.Context(device, priority=-1 if pipelined else 0)  # spectral
        self.ctx = oc.Context(device, priority=1) if pipelined else self.sctx  # the rest
        self.cs = oc.CascadeSet(oc.CascadeConfig(N_GRID, LENGTHS, CUTOFFS), _params(), ctx=self.sctx)
        nbuf = 2 if pipelined else 1
        self.maps = [oc.SurfaceMaps(self.cs) for _ in range(nbuf)]
        self.slices = [oc.VelocitySlices(self.cs, SliceConfig.make(count=DEPTHS)) for _ in range(nbuf)]
        v, t = uv_ellipsoid()
        self.mesh = oc.TriMesh(v, t, ctx=self.ctx)
        self.pose = _pose(self.mesh.centroid)
        self.fluids = [oc._fluid_struct(oc.FluidQuery(maps=self.maps[k], slices=self.slices[k],
                                                      wind=WIND), oc.DragCoefficients())
                       for k in range(nbuf)]
        self.zone = oc.FdmZone(FdmConfig.make(grid_size=FDM_N, margin=FDM_MARGIN), BODY_SIZE,
                               (self.pose.position[0], self.pose.position[2]), DT, ctx=self.ctx)
        ext = self.mesh.bbox_max - self.mesh.bbox_min
        self.frame = MaskFrame.make(center_x=0.0, half_beam=ext[0], z_min=self.mesh.bbox_min[2],
                                    z_max=self.mesh.bbox_max[2], mesh_height=self.mesh.height())
        self.mparams = MaskParams.make()
        self.speed = float(np.linalg.norm(list(self.pose.linear_velocity)))
        self.t = 0.0
        self.f = 0
        from paper_2503_03326_b200._types import HydroReport
        self.report = HydroReport()
        self.S = torch.cuda.ExternalStream(self.sctx.stream, device=f"cuda:{device}")
        self.H = torch.cuda.ExternalStream(self.ctx.stream, device=f"cuda:{device}")
        self.ready = [torch.cuda.Event() for _ in range(nbuf)]
        self.consumed = [torch.cuda.Event() for _ in range(nbuf)]
        self.pending_report = False
        self.serialize = False  # profiling passes: no cross-frame overlap

    def contexts(self):
        return [self.sctx, self.ctx] if self.pipelined else [self.ctx]

    def sync(self):
        for c in self.contexts():
            c.synchronize()

    def timed_begin(self, ev):
        ev.record(self.S)
        self.H.wait_event(ev)

    def timed_end(self, ev):
        self.S.wait_event(self.consumed[(self.f - 1) % len(self.consumed)])
        ev.record(self.S)

    def _read_report(self):
        self.oc.check(self.L.ocn_hydro_report_get(self.mesh.h, C.byref(self.report)), self.ctx.h,
                      "report")

    def step(self, read_report: bool = False):
        """sim.cpp:59-109 minus the rigid integrator: spectral step, forces,
        stability, mask from the device waterline, FDM step (all async). With
        read_report, the previous frame's report is read (its forces are what
        an integrator needs before this frame's forces); finish() reads the last."""
        L, oc = self.L, self.oc
        k = self.f % len(self.maps)
        self.t += DT
        # the buffer's previous readers are done (serialize: the previous frame is)
        self.S.wait_event(self.consumed[(self.f - 1) % len(self.maps) if self.serialize else k])
        oc.check(L.ocn_spectral_step(self.maps[k].h, self.slices[k].h, self.t, 1.0), self.sctx.h,
                 "spectral")
        self.ready[k].record(self.S)
        if read_report and self.pending_report:
            self._read_report()
        self.H.wait_event(self.ready[k])
        fluid, _ = self.fluids[k]
        oc.check(L.ocn_hydro_aggregate(self.mesh.h, C.byref(self.pose), C.byref(fluid), None, None),
                 self.ctx.h, "aggregate")
        oc.check(L.ocn_zone_update_stability(self.zone.h, self.speed, DT), self.ctx.h, "stability")
        px, pz = self.pose.position[0], self.pose.position[2]
        oc.check(L.ocn_zone_mask_from_hydro(self.zone.h, self.mesh.h, YAW, px, pz, self.speed,
                                            C.byref(self.frame), C.byref(self.mparams)), self.ctx.h,
                 "mask")
        # the body advances with its velocity (the rigid integrator is out of scope)
        for q in range(3):
            self.pose.position[q] += self.pose.linear_velocity[q] * DT
        oc.check(L.ocn_zone_step(self.zone.h, DT, self.pose.position[0], self.pose.position[2]),
                 self.ctx.h, "fdm")
        self.consumed[k].record(self.H)
        self.pending_report = True
        self.f += 1
        if read_report and not self.pipelined:
            self._read_report()
            self.pending_report = False

    def finish(self, read_report: bool = False):
        if read_report and self.pending_report:
            self._read_report()
        self.pending_report = False


# ---------------------------------------------------------------- config 1
C1_FRAMES, C1_N, C1_L = 600, 256, 256.0
C1_WORKLOAD = ("config1: reference-default spectrum (U=5, F=1e5, seed 0), one 256^2 cascade "
               "(band [0, inf)), 8 surface maps per frame, 600 frames t_f = (f+1)/60 batched in "
               "one spectral step (one 10 s clip per step); frames f mod G per rank")


class Frame1(_SingleStream):
    """This rank's frames of the 600-frame clip as one time-batched set: rank r
    owns frames f = r, r + G, ... (t_f = (f + 1) / 60), i.e. t0 = (r + 1) / 60
    and spacing G / 60 (no collective)."""

    def __init__(self, device: int, rank: int, world: int):
        from paper_2503_03326_b200 import ocean as oc
        from paper_2503_03326_b200._types import SpectrumParams
        self.oc, self.L = oc, oc.lib()
        self.ctx = oc.Context(device)
        self.per = C1_FRAMES // world
        self.p = SpectrumParams.make()
        self.cfg = oc.CascadeConfig(C1_N, [C1_L], [])
        self.frames = oc.CascadeFrames(self.cfg, self.p, self.per, world * DT, ctx=self.ctx)
        self.maps = oc.SurfaceMaps(self.frames)
        self.t0 = (rank + 1) * DT
        self.dt = world * DT
        self.clip = 0
        self.points = self.per * C1_N * C1_N
        self._h = np.zeros(C1_N * C1_N, np.float32)

    def step(self, read_report: bool = False):
        t0 = self.t0 + self.clip * C1_FRAMES * DT  # successive 10 s clips
        self.clip += 1
        self.oc.check(self.L.ocn_surface_generate_batch(self.maps.h, t0, self.dt, 1.0), self.ctx.h,
                      "generate_batch")
        if read_report:  # the step's result probe: the clip's last frame height map -> host
            self.oc.check(self.L.ocn_maps_download_f32(self.maps.h, self.per - 1, 0,
                                                       self._h.ctypes.data_as(C.POINTER(C.c_float))),
                          self.ctx.h, "download")

    def single_frame_latency(self, reps: int = 50) -> float:
        """One frame through the C-ABI, launch to completion (host wall clock,
        median): ocn_surface_generate on a one-frame set + synchronize."""
        oc = self.oc
        cs = oc.CascadeSet(self.cfg, self.p, ctx=self.ctx)
        m = oc.SurfaceMaps(cs)
        for k in range(5):
            m.generate(DT * (k + 1))
        self.ctx.synchronize()
        ts = []
        for k in range(reps):
            t0 = time.perf_counter()
            self.oc.check(self.L.ocn_surface_generate(m.h, DT * (k + 1), 1.0), self.ctx.h, "gen")
            self.ctx.synchronize()
            ts.append(time.perf_counter() - t0)
        return float(np.median(ts) * 1e3)


# ---------------------------------------------------------------- config 4
C4_INSTANCES, C4_N = 64, 512
C4_LENGTHS = [256.0, 16.0, 4.0]
C4_CUTOFFS = [12 * math.pi / 16, 12 * math.pi / 4]
C4_POINTS = C4_INSTANCES * len(C4_LENGTHS) * C4_N * C4_N
C4_WORKLOAD = ("config4: 64 independent instances x 3 cascades x 512^2 (8 surface maps each), "
               "instances sharded across ranks, no collective")


class Frame4(_SingleStream):
    """This rank's share of the 64 instances as one batched spectral set."""

    def __init__(self, device: int, rank: int, world: int):
        from paper_2503_03326_b200 import ocean as oc
        self.oc, self.L = oc, oc.lib()
        self.ctx = oc.Context(device)
        per = C4_INSTANCES // world
        lo = rank * per
        params = []
        for seed in range(lo, lo + per):
            p = _params()
            p.rng_seed = seed
            params.append(p)
        self.inst = oc.CascadeInstances(oc.CascadeConfig(C4_N, C4_LENGTHS, C4_CUTOFFS), params,
                                        ctx=self.ctx)
        self.maps = oc.SurfaceMaps(self.inst)
        self.points = per * len(C4_LENGTHS) * C4_N * C4_N
        self.t = 0.0
        self.probe = C.c_float()

    def step(self, read_report: bool = False):
        self.t += DT
        self.oc.check(self.L.ocn_surface_generate(self.maps.h, self.t, 1.0), self.ctx.h, "maps")
        if read_report:  # the frame's result: instance 0's height map (fp32) -> host
            self.oc.check(self.L.ocn_maps_download_f32(self.maps.h, 0, 0, self._hmap), self.ctx.h,
                          "download")

    _hmap_arr = np.zeros(C4_N * C4_N, np.float32)

    @property
    def _hmap(self):
        return self._hmap_arr.ctypes.data_as(C.POINTER(C.c_float))


# ---------------------------------------------------------------- config 5
C5_N, C5_L = 16384, 4096.0
C5_WORKLOAD = ("config5: single 16384^2 surface (8 fields, 4 packed transforms), row slabs per "
               "rank, tile all-to-all over NVLink (grouped ncclSend/ncclRecv on the library's "
               "communicator) pipelined per packed pair between the row and column passes")


class Frame5(_SingleStream):
    """This rank's slab of the 16384^2 grid. A step is ocn_slab_frame: per packed
    pair the row pass, the tile all-to-all over NVLink (grouped ncclSend / ncclRecv
    on the library's own communicator, ocn_comm) and the column pass, pipelined
    per pair. Profiling passes (serialize) run rows, the whole exchange and the
    columns one after the other, the exchange timed with CUDA events."""

    def __init__(self, device: int, rank: int, world: int, dist):
        from paper_2503_03326_b200 import ocean as oc
        from paper_2503_03326_b200.slab import Comm, SlabSurface, tile_layout
        import torch
        self.oc, self.L, self.dist = oc, oc.lib(), dist
        self.ctx = oc.Context(device)
        p = _params()
        p.rng_seed = 7
        self.slab = SlabSurface(C5_N, world, rank, C5_L, p, ctx=self.ctx)
        _, total = tile_layout(self.slab.rows, world)
        self.send = torch.empty(2 * total, dtype=torch.float32, device=f"cuda:{device}")
        self.recv = self.send if world == 1 else torch.empty_like(self.send)
        self.comm = None
        if world > 1:
            def share(raw):
                obj = [raw]
                dist.broadcast_object_list(obj, src=0)
                return obj[0]
            self.comm = Comm(self.ctx, world, rank, share)
        self.stream = torch.cuda.ExternalStream(self.ctx.stream, device=f"cuda:{device}")
        self.world = world
        self.t = 0.0
        self.points = C5_N * C5_N // world
        self.a2a_ms = []
        self.timing = False
        self.serialize = False

    def step(self, read_report: bool = False):
        import torch
        self.t += DT
        L, h = self.L, self.slab.h
        comm = self.comm.h if self.comm else None
        sp, rp = C.c_void_p(self.send.data_ptr()), C.c_void_p(self.recv.data_ptr())
        if not self.serialize:
            self.oc.check(L.ocn_slab_frame(h, comm, self.t, 1.0, sp, rp), self.ctx.h, "frame")
        else:
            self.slab.rows_pass(self.t, self.send.data_ptr())
            if self.world > 1:
                if self.timing:
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(self.stream)
                self.oc.check(L.ocn_slab_exchange(h, comm, -1, sp, rp), self.ctx.h, "exchange")
                if self.timing:
                    e1.record(self.stream)
                    self.a2a_ms.append((e0, e1))
            self.slab.cols_pass(self.recv.data_ptr())
        if read_report:  # the frame's result probe: synchronize (fields stay on the device)
            self.oc.check(L.ocn_ctx_synchronize(self.ctx.h), self.ctx.h, "sync")


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws <= 1:
        return None, 0, 1, 0
    import torch
    import torch.distributed as dist
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl")
    return dist, dist.get_rank(), ws, local


def _max_over_ranks(dist, x: float) -> float:
    if dist is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _barrier(dist):
    if dist is not None:
        dist.barrier()


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _traffic():
    """dram bytes per frame of the spectral pipeline from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "roofline_traffic.json")) as f:
            return json.load(f).get("spectral_dram_bytes_per_frame")
    except Exception:
        return None


def _measure(fr, dist, local, steps, warmup, stage_names, kernel_names=None, c5=False):
    """Warm-up, then K timed steps (CUDA events on the frame's streams, barrier +
    synchronize on both sides), a profiled pass per stage, and the e2e pass."""
    import torch
    L = fr.L
    ctxs = fr.contexts()
    for _ in range(max(warmup, 3)):
        fr.step()
    fr.sync()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)

    def n_launches():
        return sum(c.kernel_launches() for c in ctxs)
    launches0 = n_launches()
    with ClockSampler(local) as clk:
        _barrier(dist)
        fr.sync()
        fr.timed_begin(ev0)
        for _ in range(steps):
            fr.step()
        fr.timed_end(ev1)
        fr.sync()
        _barrier(dist)
        ms_total = ev0.elapsed_time(ev1)
        launches = n_launches() - launches0

        # ---- roofline pass: same K steps with CUDA-event windows per stage
        # (mode 2: the spectral step still replays its graph), steps not
        # overlapped so that each window times its own stage ...
        fr.serialize = True

        def profiled(mode, names):
            for c in ctxs:
                L.ocn_ctx_profile(c.h, mode)
                L.ocn_ctx_profile_reset(c.h)
            for _ in range(steps):
                fr.step()
            fr.sync()
            out = {}
            for name, cat in names:
                tot = 0.0
                for c in ctxs:  # each category runs on one of the contexts
                    ms, cnt = C.c_double(), C.c_uint64()
                    L.ocn_ctx_profile_read(c.h, cat, C.byref(ms), C.byref(cnt))
                    tot += ms.value
                out[name] = tot / steps
            for c in ctxs:
                L.ocn_ctx_profile(c.h, 0)
            return out
        if c5:
            fr.timing = True
            stages = profiled(1, [("slab_rows", 1), ("slab_cols", 2)])
            fr.timing = False
            torch.cuda.synchronize()
            a2a = [e0.elapsed_time(e1) for e0, e1 in fr.a2a_ms]
            stages["all_to_all"] = float(np.mean(a2a)) if a2a else 0.0
            stages["spectral"] = stages["slab_rows"] + stages["slab_cols"]
        else:
            stages = profiled(2, stage_names)
        # ... and the kernel split of the spectral step (mode 1: eager launches)
        kernels = profiled(1, kernel_names) if kernel_names else None
        fr.serialize = False
        # ---- e2e: through the C-ABI with host inputs (t, pose) and the host
        # read of each step's result, wall clock
        # (at least 60 frames: a 20-frame wall-clock window moves by ~0.1 ms / frame
        # from box to box)
        e2e_steps = max(steps, 60)
        for _ in range(3):
            fr.step(read_report=True)
        fr.finish(read_report=True)
        _barrier(dist)
        fr.sync()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            fr.step(read_report=True)
        fr.finish(read_report=True)
        fr.sync()
        e2e_s = (time.perf_counter() - t0) * steps / e2e_steps
    return {"ms_step": _max_over_ranks(dist, ms_total / steps),
            "e2e_step": _max_over_ranks(dist, e2e_s / steps),
            "spectral_ms": _max_over_ranks(dist, stages["spectral"]),
            "stages": stages, "kernels": kernels, "launches": int(launches),
            "clocks": clk.summary()}


def _produced_bytes(fr):
    """Bytes the config-3 spectral step actually moves by definition per frame:
    h0 read once (8 B / point) + the output planes of the transforms it executes
    (the 44 exactly-zero transforms' planes are written once, at plan build)."""
    plan = fr.oc.spectral_plan(fr.maps[0], fr.slices[0])
    planes = sum((2 if x["index1"] >= 0 else 1) for x in plan if x["executed"])
    return POINTS_PER_FRAME * 8 + planes * N_GRID * N_GRID * 4, plan


def _roofline(kernel, alg_bytes, spec_ms, peak, peak_kind, traffic=None):
    achieved = alg_bytes / (spec_ms / 1e3) / 1e9
    return {"kernel": kernel, "bound": "hbm", "achieved": achieved, "peak": peak,
            "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
            "algorithmic_bytes_per_frame": alg_bytes}


def _config_line(args, cfgno, dist, rank, world, local, steps, warmup, peak, peak_kind,
                 headline: bool):
    """Measure one SURVEY 8d configuration; returns its line (rank 0) or None."""
    c1, c4, c5 = cfgno == 1, cfgno == 4, cfgno == 5
    if c5:
        fr = Frame5(local, rank, world, dist)
    elif c4:
        fr = Frame4(local, rank, world)
    elif c1:
        fr = Frame1(local, rank, world)
    else:
        fr = Frame(local, pipelined=not args.no_pipeline)
    stage_names = ([("spectral", 6)] if (c1 or c4) else
                   [("spectral", 6), ("hydro", 3), ("mask", 4), ("fdm", 5)])
    kernel_names = None if c5 else [("evolve", 0), ("fft_rows", 1), ("fft_cols", 2),
                                    ("spectral_eager", 6)]
    m = _measure(fr, dist, local, steps, warmup, stage_names, kernel_names, c5=c5)
    extra = {}
    if c1:
        extra["single_frame_latency_ms"] = fr.single_frame_latency()
    if rank != 0:
        return None
    spec_ms = m["spectral_ms"]
    if c5:
        points = C5_N * C5_N
        alg_bytes = fr.points * (16 + 4 * 8)  # h0 + h0 mirror slab read, 8 fp32 fields written
        metric = "ocean grid points/sec (single 16384^2 surface, slab FFT + all-to-all)"
        h2d, d2h = 8, 0
        sent = fr.slab.exchange_bytes * (world - 1) / world
        cfg = {"workload": C5_WORKLOAD, "grid": C5_N, "ranks": world,
               "parallelism": f"row slabs x{world}", "exchange_bytes_per_gpu": sent,
               "l2": "per-frame slabs 4-8 GB > 126 MB L2 (no explicit flush)"}
        scaling = "strong"
        roof = _roofline("slab pipeline (k_slab_evolve + k_slab_rows + k_slab_cols)", alg_bytes,
                         spec_ms, peak, peak_kind)
        if world > 1 and m["stages"].get("all_to_all", 0) > 0:
            gbs = sent / (m["stages"]["all_to_all"] / 1e3) / 1e9
            cfg["all_to_all_GBps_per_gpu"] = gbs
            cfg["nvlink_efficiency_vs_900GBps"] = gbs / 900.0
            cfg["nvlink_efficiency_vs_770GBps_measured_peer_copy"] = gbs / 770.0
    elif c4:
        points = C4_POINTS
        alg_bytes = fr.points * (8 + 4 * 8)  # per rank and frame
        metric = "ocean grid points/sec (64 x 3 x 512^2 instances, surface synthesis)"
        h2d, d2h = 8, C4_N * C4_N * 4
        cfg = {"workload": C4_WORKLOAD, "grid": C4_N, "instances": C4_INSTANCES,
               "cascades_per_instance": len(C4_LENGTHS),
               "parallelism": f"instances sharded {C4_INSTANCES // world}/rank x {world}",
               "l2": "per-frame outputs 1.6 GB / world > 126 MB L2 (no explicit flush)"}
        scaling = "strong"
        roof = _roofline("spectral pipeline (k_evolve + k_rows_w + k_cols_tma)", alg_bytes, spec_ms,
                         peak, peak_kind)
    elif c1:
        points = C1_FRAMES * C1_N * C1_N
        alg_bytes = fr.points * (8 + 4 * 8)
        metric = "ocean grid points/sec (600 frames of a 256^2 cascade, batched)"
        h2d, d2h = 16, C1_N * C1_N * 4
        cfg = {"workload": C1_WORKLOAD, "grid": C1_N, "frames": C1_FRAMES,
               "parallelism": f"frames f mod {world} x {world}" if world > 1 else "1 GPU",
               "l2": "per-step outputs 1.26 GB / world > 126 MB L2 (no explicit flush)"}
        scaling = "strong"
        roof = _roofline("spectral pipeline (k_evolve + k_rows_w + k_cols_tma, one CUDA graph)",
                         alg_bytes, spec_ms, peak, peak_kind)
    else:
        points = world * POINTS_PER_FRAME
        alg_bytes = SPECTRAL_BYTES
        metric = "ocean grid points/sec (spectrum+iFFT+forces) at 1024^2 x 4 cascades"
        h2d, d2h = C.sizeof(fr.pose) + 8, C.sizeof(fr.report)
        cfg = {"workload": WORKLOAD, "grid": N_GRID, "cascades": len(LENGTHS),
               "depth_slices": DEPTHS, "hull_triangles": int(fr.mesh.triangles.shape[0]),
               "fdm_grid": FDM_N, "parallelism": f"replicas x{world}" if world > 1 else "1 GPU",
               "frame_pipeline": ("frame f forces/mask/FDM (high-priority stream) overlap frame "
                                  "f+1 spectral step (low-priority stream), double-buffered "
                                  "maps/slices; stages_ms timed without overlap"
                                  if not args.no_pipeline else "off"),
               "l2": "per-frame working set 1.8 GB of outputs > 126 MB L2 (no explicit flush)"}
        scaling = "weak"
        roof = _roofline("spectral pipeline (k_evolve + k_rows_w + k_cols_tma, one CUDA graph)",
                         alg_bytes, spec_ms, peak, peak_kind, _traffic())
        produced, plan = _produced_bytes(fr)
        roof["produced_bytes_per_frame"] = produced
        roof["achieved_produced"] = produced / (spec_ms / 1e3) / 1e9
        roof["frac_produced"] = roof["achieved_produced"] / peak
        roof["transforms"] = {"reference": len(plan),
                              "executed_per_frame": sum(x["executed"] for x in plan),
                              "exactly_zero_planes_written_once": sum(1 - x["executed"] for x in plan)}
        roof["note"] = ("frac: SURVEY 8d algorithmic bytes (h0 + all 104 output fields, 424 B/pt); "
                        "frac_produced: h0 + the planes of the executed transforms only")
    ms = m["ms_step"]
    line = {
        "metric": metric,
        "value": points / (ms / 1e3),
        "unit": "grid-points/s",
        "n_gpus": world,
        "steps": steps,
        "warmup": max(warmup, 3),
        "ms_per_step": ms,
        "ms_per_frame": ms if not c1 else ms / C1_FRAMES * world,
        "higher_is_better": True,
        "scaling": scaling,
        "vs_baseline": None,
        "dtype": "f32 (fields, FFT) / f64 (spectrum init, phases, samplers, forces)",
        "data": "synthetic (SURVEY 8d spectrum presets; UV-ellipsoid hull)",
        "config": cfg,
        "stages_ms": m["stages"],
        "roofline": roof,
        "e2e": {"value": points / m["e2e_step"], "unit": "grid-points/s",
                "ms_per_step": m["e2e_step"] * 1e3, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "frames_timed": max(steps, 60)},
        "gpu_launches": m["launches"],
        "clocks": m["clocks"],
    }
    st = m["stages"]
    if {"spectral", "hydro", "mask", "fdm"} <= set(st):
        # the same stages under Simulation::timing()'s names (sim.hpp:50-54): the
        # reference's surface and velocity stages are one fused spectral step
        # here; the rigid integrator is out of the frame (north_star scope)
        line["stages_ms_reference_names"] = {"surface+velocity": st["spectral"], "hydro": st["hydro"],
                                             "zones": st["mask"] + st["fdm"], "integrate": None}
    if m["kernels"]:
        line["spectral_kernels_ms_eager"] = m["kernels"]
    line.update(extra)
    if world == 1 and not args.no_cpu_baseline:
        if c4:
            line["cpu_baseline"] = cpu_baseline_c4()
        elif c1:
            line["cpu_baseline"] = cpu_baseline_c1()
        elif not c5 and headline:
            line["cpu_baseline"] = cpu_baseline(frames=1, warmup=0, one_worker=True)
    del fr
    return line


EXTRA_CONFIG_BUDGET_S = 300


def run_ours(args):
    dist, rank, world, local = _dist()
    peak, peak_kind = _peaks()
    line = _config_line(args, args.config, dist, rank, world, local, args.steps, args.warmup, peak,
                        peak_kind, headline=True)
    if args.config == 3 and not args.no_extra_configs:
        import gc
        import torch
        extra = {}
        if line is not None:
            line["configs"] = extra
        for cfgno in (1, 4, 5):
            gc.collect()
            torch.cuda.empty_cache()
            # the headline line must survive a failing or hung secondary config
            # (e.g. a multi-rank exchange that never completes): each runs under
            # a watchdog that prints what was measured so far and exits
            done = threading.Event()

            def watchdog(cfgno=cfgno, done=done):
                if done.wait(EXTRA_CONFIG_BUDGET_S):
                    return
                if line is not None:
                    extra[str(cfgno)] = {"unavailable": f"timed out after {EXTRA_CONFIG_BUDGET_S} s"}
                    print(json.dumps(line), flush=True)
                os._exit(0)

            threading.Thread(target=watchdog, daemon=True).start()
            try:
                sub = _config_line(args, cfgno, dist, rank, world, local, min(args.steps, 10),
                                   args.warmup, peak, peak_kind, headline=False)
            except Exception as e:  # noqa: BLE001 -- reported in the line, headline kept
                sub = {"unavailable": f"{type(e).__name__}: {str(e)[:300]}"}
            finally:
                done.set()
            if sub is not None:
                extra[str(cfgno)] = sub
    if line is not None:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_baseline_c4(sample_instances: int = 2):
    """Reference generate_maps per instance (3 x 512^2, no batch API in the
    reference), `sample_instances` of the 64 timed and scaled."""
    from oracle.oracle import P
    lib = _ref_lib()
    ncpu = os.cpu_count() or 1
    lib.ref_set_worker_count.argtypes = [C.c_int]
    lib.ref_set_worker_count(ncpu)
    f = lib.ref_generate_maps_timed
    f.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_int,
                  C.POINTER(C.c_double)]
    la = np.ascontiguousarray(C4_LENGTHS)
    cu = np.ascontiguousarray(C4_CUTOFFS + [0.0])
    per = []
    for k in range(sample_instances):
        p = _params()
        p.rng_seed = k
        sec = C.c_double()
        f(C4_N, 3, P(la), P(cu), C.byref(p), DT, 1, C.byref(sec))  # generate_maps only
        per.append(sec.value)
    dt = float(np.mean(per)) * C4_INSTANCES
    return {"value": C4_POINTS / dt, "unit": "grid-points/s", "ms_per_frame": dt * 1e3, "cores": ncpu,
            "cpu_model": _cpu_model(), "kind": "reference",
            "sample": f"{sample_instances} of 64 instances: reference generate_maps (3 x 512^2, "
                      f"CascadeSet built outside the timing), scaled x{C4_INSTANCES // sample_instances}"}


def cpu_baseline_c1(sample_frames: int = 60):
    """Reference generate_maps of the config-1 cascade, `sample_frames` of the
    600 frames timed (CascadeSet built outside the timing)."""
    from oracle.oracle import P
    from paper_2503_03326_b200._types import SpectrumParams
    lib = _ref_lib()
    ncpu = os.cpu_count() or 1
    lib.ref_set_worker_count.argtypes = [C.c_int]
    lib.ref_set_worker_count(ncpu)
    f = lib.ref_generate_maps_timed
    f.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_int,
                  C.POINTER(C.c_double)]
    la = np.ascontiguousarray([C1_L])
    cu = np.ascontiguousarray([0.0])
    p = SpectrumParams.make()
    sec = C.c_double()
    f(C1_N, 1, P(la), P(cu), C.byref(p), DT, sample_frames, C.byref(sec))
    per_clip = sec.value * C1_FRAMES
    return {"value": C1_FRAMES * C1_N * C1_N / per_clip, "unit": "grid-points/s",
            "ms_per_frame": sec.value * 1e3, "cores": ncpu, "cpu_model": _cpu_model(),
            "kind": "reference",
            "sample": f"{sample_frames} of the 600 frames: reference generate_maps (1 x 256^2), "
                      f"set_worker_count({ncpu}) (its 4 transforms run as one 256-item chunk, "
                      f"i.e. on one thread, parallel.cpp:29)"}


# ---------------------------------------------------------- reference (CPU)
def _ref_lib():
    from oracle.oracle import REF_SO, build, ref_available
    if not ref_available():
        build(reference=True)
    lib = C.CDLL(REF_SO)
    return lib


def cpu_baseline(frames: int = 1, warmup: int = 0, budget_s: float = 1e9, workers: int = 0,
                 one_worker: bool = False):
    """The reference's own CPU implementation (oracle/_ref: the unmodified
    reference library compiled from its sources) on this host: full config-3
    frames (generate_maps 4 x 1024^2, build_slices at all 32 depths, aggregate,
    compute_mask, FdmZone::step), set_worker_count(workers or nproc). Its
    spectral stages stay single-threaded whatever the worker count (4 C and
    D C jobs <= 256 run as one chunk, parallel.cpp:29). Frames run until
    `budget_s` is spent; `frames` reports how many ran. one_worker: also one
    frame with set_worker_count(1)."""
    from paper_2503_03326_b200._types import FdmConfig, SliceConfig
    from paper_2503_03326_b200.meshgen import uv_ellipsoid
    from oracle.oracle import P
    lib = _ref_lib()
    ncpu = workers or os.cpu_count() or 1
    lib.ref_set_worker_count.argtypes = [C.c_int]
    lib.ref_set_worker_count(ncpu)
    v, t = uv_ellipsoid()
    from oracle.oracle import Oracle
    mesh = Oracle("port").mesh_build(v, t)
    pose = _pose(mesh["centroid"])
    p = _params()
    sc = SliceConfig.make(count=DEPTHS)
    fc = FdmConfig.make(grid_size=FDM_N, margin=FDM_MARGIN)
    la = np.ascontiguousarray(LENGTHS)
    cu = np.ascontiguousarray(CUTOFFS + [0.0])
    wind = np.ascontiguousarray(WIND)
    lib.ref_bench_create.restype = C.c_void_p
    lib.ref_bench_create.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                     C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                     C.c_double, C.c_double, C.c_void_p, C.POINTER(C.c_int)]
    lib.ref_bench_frame.argtypes = [C.c_void_p, C.c_double, C.c_int, C.c_void_p]
    lib.ref_bench_destroy.argtypes = [C.c_void_p]
    st = C.c_int()
    vv = np.ascontiguousarray(v)
    tt = np.ascontiguousarray(mesh["tris"])
    t_init = time.perf_counter()
    b = lib.ref_bench_create(N_GRID, len(LENGTHS), P(la), P(cu), C.byref(p), C.byref(sc), v.shape[0],
                             P(vv), t.shape[0], tt.ctypes.data, C.byref(pose), C.byref(fc), BODY_SIZE,
                             DT, P(wind), C.byref(st))
    t_init = time.perf_counter() - t_init
    if st.value != 0:
        raise RuntimeError("reference bench setup failed")
    stage = np.zeros(5)
    for _ in range(warmup):
        lib.ref_bench_frame(b, DT, DEPTHS, P(stage))
    walls, stages = [], []
    t_start = time.perf_counter()
    for _ in range(max(frames, 1)):
        w0 = time.perf_counter()
        lib.ref_bench_frame(b, DT, DEPTHS, P(stage))
        walls.append(time.perf_counter() - w0)
        stages.append(stage.copy())
        if time.perf_counter() - t_start > budget_s:
            break
    one = None
    if one_worker:
        lib.ref_set_worker_count(1)
        w0 = time.perf_counter()
        lib.ref_bench_frame(b, DT, DEPTHS, P(stage))
        one = time.perf_counter() - w0
        lib.ref_set_worker_count(ncpu)
    lib.ref_bench_destroy(b)
    wall = float(np.mean(walls))
    st_mean = np.mean(stages, axis=0)
    out = {
        "value": POINTS_PER_FRAME / wall,
        "unit": "grid-points/s",
        "ms_per_frame": wall * 1e3,
        "cores": ncpu,
        "cpu_model": _cpu_model(),
        "kind": "reference",
        "frames": len(walls),
        "warmup_frames": warmup,
        "stage_s": {"generate_maps": st_mean[0], "build_slices": st_mean[1], "aggregate": st_mean[2],
                    "stability_mask": st_mean[3], "fdm": st_mean[4], "cascade_init_once": t_init},
        "sample": (f"{len(walls)} full config-3 frame(s) through the reference library (oracle/_ref, "
                   f"g++ -O2): generate_maps + build_slices (all {DEPTHS} depths) + aggregate + "
                   f"compute_mask + FdmZone::step; set_worker_count({ncpu})"),
    }
    if one is not None:
        out["one_worker"] = {"value": POINTS_PER_FRAME / one, "ms_per_frame": one * 1e3, "cores": 1}
    return out


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    warmup = max(args.warmup, 3) if not args.reference_fast_warmup else 1
    # bounded: the warm-up frames plus timed frames until ~100 s are spent
    cb = cpu_baseline(frames=args.steps, warmup=warmup, budget_s=100.0)
    line = {
        "impl": "reference",
        "metric": "ocean grid points/sec (spectrum+iFFT+forces) at 1024^2 x 4 cascades",
        "value": cb["value"],
        "unit": "grid-points/s",
        "n_gpus": world,
        "steps": cb["frames"],
        "steps_requested": args.steps,
        "warmup": warmup,
        "ms_per_step": cb["ms_per_frame"],
        "ms_per_frame": cb["ms_per_frame"],
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (SURVEY 8d spectrum presets; UV-ellipsoid hull)",
        "config": {"workload": WORKLOAD, "grid": N_GRID, "cascades": len(LENGTHS),
                   "depth_slices": DEPTHS, "hull_triangles": 100352, "fdm_grid": FDM_N,
                   "parallelism": "host CPU",
                   "frame_pipeline": "off (the reference steps frames in order)",
                   "l2": "n/a (CPU)"},
        "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "cpu_model", "kind", "sample")},
        "e2e": {"value": cb["value"], "unit": "grid-points/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "stage_s": cb["stage_s"],
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-pipeline", action="store_true",
                    help="config 3: run every frame's stages in order on one stream")
    ap.add_argument("--config", type=int, default=3, choices=[1, 3, 4, 5],
                    help="3: the BASELINE metric frame (default); 1: 600 batched 256^2 frames; "
                         "4: 64 batched 512^2 instances; 5: single 16384^2 grid, slab FFT + "
                         "all-to-all across ranks")
    ap.add_argument("--no-extra-configs", action="store_true",
                    help="config 3: do not also measure configs 1, 4 and 5 in the same run")
    ap.add_argument("--reference-fast-warmup", action="store_true",
                    help="reference arm: one warm-up frame instead of our arm's warm-up count")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
