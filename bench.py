#!/usr/bin/env python
"""bench.py — per-frame Arc Blanc hot path on B200 (BASELINE.json metric).

Workload (one "step" = one frame): the 4-cascade 1024^2
spectrum (U=20, F=1e5, theta0=0.4, xi=0.5, delta=0.5, standard peak, seed 42;
lengths 1024/256/16/4 m) evolved to t, its 8 surface maps + 32 logarithmic
velocity-at-depth slices (208 packed 1024^2 inverse FFTs), fluid-to-solid
forces on the 100,352-triangle UV-ellipsoid hull (height_at + velocity_at
samplers, deterministic reductions, waterline), the waterline mask and one
2048^2 Cords-Staadt FDM step. Metric: ocean grid points / s (= 4 * 1024^2 per
frame / frame time) and ms / frame.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

N > 1 (torchrun, one rank per GPU): independent replicas of the frame on every
GPU (configs 2/3 do not shard), weak scaling, max over ranks.
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
WORKLOAD = ("config3: 4 cascades x 1024^2 (8 surface maps + 32 velocity slices, 208 packed "
            "2D iFFTs) + 100,352-tri hull forces + waterline mask + 2048^2 FDM step")


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
               "rank, NCCL all-to-all tile transpose between the row and column passes")


class Frame5(_SingleStream):
    """This rank's slab of the 16384^2 grid; the transpose is an NCCL all-to-all."""

    def __init__(self, device: int, rank: int, world: int, dist):
        from paper_2503_03326_b200 import ocean as oc
        from paper_2503_03326_b200.slab import SlabSurface, tile_layout
        import torch
        self.oc, self.L, self.dist = oc, oc.lib(), dist
        self.ctx = oc.Context(device)
        p = _params()
        p.rng_seed = 7
        self.slab = SlabSurface(C5_N, world, rank, C5_L, p, ctx=self.ctx)
        _, total = tile_layout(self.slab.rows, world)
        self.send = torch.empty(2 * total, dtype=torch.float32, device=f"cuda:{device}")
        self.recv = self.send if world == 1 else torch.empty_like(self.send)
        self.stream = torch.cuda.ExternalStream(self.ctx.stream, device=f"cuda:{device}")
        self.world = world
        self.t = 0.0
        self.points = C5_N * C5_N // world
        self.a2a_ms = []
        self._col = np.zeros(C5_N, np.float64)
        self.timing = False

    def step(self, read_report: bool = False):
        import torch
        self.t += DT
        self.slab.rows_pass(self.t, self.send.data_ptr())
        if self.world > 1:
            with torch.cuda.stream(self.stream):
                if self.timing:
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(self.stream)
                self.dist.all_to_all_single(self.recv, self.send)
                if self.timing:
                    e1.record(self.stream)
                    self.a2a_ms.append((e0, e1))
        self.slab.cols_pass(self.recv.data_ptr())
        if read_report:  # the frame's result probe: one column of the height field -> host
            self.oc.check(self.L.ocn_ctx_synchronize(self.ctx.h), self.ctx.h, "sync")


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


def run_ours(args):
    dist, rank, world, local = _dist()
    c4 = args.config == 4
    c5 = args.config == 5
    fr = (Frame5(local, rank, world, dist) if c5 else
          (Frame4(local, rank, world) if c4 else Frame(local, pipelined=not args.no_pipeline)))
    L = fr.L
    ctxs = fr.contexts()
    for _ in range(max(args.warmup, 3)):
        fr.step()
    fr.sync()
    # ---- timed region: device time with CUDA events on the library stream(s)
    import torch
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)

    def n_launches():
        return sum(c.kernel_launches() for c in ctxs)
    launches0 = n_launches()
    with ClockSampler(local) as clk:
        _barrier(dist)
        fr.sync()
        fr.timed_begin(ev0)
        for _ in range(args.steps):
            fr.step()
        fr.timed_end(ev1)
        fr.sync()
        _barrier(dist)
        ms_total = ev0.elapsed_time(ev1)
        launches = n_launches() - launches0

        # ---- roofline pass: same K frames with CUDA-event windows per stage
        # (mode 2: the spectral step still replays its graph), frames not
        # overlapped so that each window times its own stage ...
        fr.serialize = True

        def profiled(mode, names):
            for c in ctxs:
                L.ocn_ctx_profile(c.h, mode)
                L.ocn_ctx_profile_reset(c.h)
            for _ in range(args.steps):
                fr.step()
            fr.sync()
            out = {}
            for name, cat in names:
                tot = 0.0
                for c in ctxs:  # each category runs on one of the contexts
                    ms, cnt = C.c_double(), C.c_uint64()
                    L.ocn_ctx_profile_read(c.h, cat, C.byref(ms), C.byref(cnt))
                    tot += ms.value
                out[name] = tot / args.steps
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
            stages = profiled(2, [("spectral", 6), ("hydro", 3), ("mask", 4), ("fdm", 5)])
        if c4:
            stages = {"spectral": stages["spectral"]}
        # ... and the kernel split of the spectral step (mode 1: eager launches)
        kernels = profiled(1, [("evolve", 0), ("fft_rows", 1), ("fft_cols", 2), ("spectral_eager", 6)])
        fr.serialize = False
        # ---- e2e: through the C-ABI with host inputs (t, pose) and the host
        # read of each frame's result, wall clock
        _barrier(dist)
        fr.sync()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            fr.step(read_report=True)
        fr.finish(read_report=True)
        fr.sync()
        e2e_s = time.perf_counter() - t0
    ms_frame = _max_over_ranks(dist, ms_total / args.steps)
    e2e_frame = _max_over_ranks(dist, e2e_s / args.steps)
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    peak, peak_kind = _peaks()
    if c5:
        points = C5_N * C5_N
        alg_bytes = fr.points * (16 + 4 * 8)  # h0 + h0 mirror slab read, 8 fp32 fields written
        metric = "ocean grid points/sec (single 16384^2 surface, slab FFT + all-to-all)"
        workload, h2d, d2h = C5_WORKLOAD, 8, 0
        sent = fr.slab.exchange_bytes * (world - 1) / world
        cfg = {"workload": workload, "grid": C5_N, "ranks": world, "parallelism": f"row slabs x{world}",
               "exchange_bytes_per_gpu": sent,
               "l2": "per-frame slabs 4-8 GB > 126 MB L2 (no explicit flush)"}
        scaling = "strong"
    elif c4:
        points = C4_POINTS if world > 1 else fr.points * world
        alg_bytes = fr.points * (8 + 4 * 8)  # per rank and frame
        metric = "ocean grid points/sec (64 x 3 x 512^2 instances, surface synthesis)"
        workload, h2d, d2h = C4_WORKLOAD, 8, C4_N * C4_N * 4
        cfg = {"workload": workload, "grid": C4_N, "instances": C4_INSTANCES,
               "cascades_per_instance": len(C4_LENGTHS),
               "parallelism": f"instances sharded {C4_INSTANCES // world}/rank x {world}",
               "l2": "per-frame outputs 1.6 GB / world > 126 MB L2 (no explicit flush)"}
        scaling = "strong"
    else:
        points = world * POINTS_PER_FRAME
        alg_bytes = SPECTRAL_BYTES
        metric = "ocean grid points/sec (spectrum+iFFT+forces) at 1024^2 x 4 cascades"
        workload, h2d, d2h = WORKLOAD, C.sizeof(fr.pose) + 8, C.sizeof(fr.report)
        cfg = {"workload": workload, "grid": N_GRID, "cascades": len(LENGTHS),
               "depth_slices": DEPTHS, "hull_triangles": int(fr.mesh.triangles.shape[0]),
               "fdm_grid": FDM_N, "parallelism": f"replicas x{world}" if world > 1 else "1 GPU",
               "frame_pipeline": ("frame f forces/mask/FDM (high-priority stream) overlap frame "
                                  "f+1 spectral step (low-priority stream), double-buffered "
                                  "maps/slices; stages_ms timed without overlap"
                                  if not args.no_pipeline else "off"),
               "l2": "per-frame working set 1.8 GB of outputs > 126 MB L2 (no explicit flush)"}
        scaling = "weak"
    value = points / (ms_frame / 1e3)
    spec_ms = stages["spectral"]
    if c5 and world > 1 and stages.get("all_to_all", 0) > 0:
        gbs = cfg["exchange_bytes_per_gpu"] / (stages["all_to_all"] / 1e3) / 1e9
        cfg["all_to_all_GBps_per_gpu"] = gbs
        cfg["nvlink_efficiency_vs_900GBps"] = gbs / 900.0
    achieved = alg_bytes / (spec_ms / 1e3) / 1e9
    line = {
        "metric": metric,
        "value": value,
        "unit": "grid-points/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": max(args.warmup, 3),
        "ms_per_step": ms_frame,
        "ms_per_frame": ms_frame,
        "higher_is_better": True,
        "scaling": scaling,
        "vs_baseline": None,
        "dtype": "f32 (fields, FFT) / f64 (spectrum init, phases, samplers, forces)",
        "data": "synthetic (SURVEY 8d spectrum presets; UV-ellipsoid hull)",
        "config": cfg,
        "stages_ms": stages,
        "spectral_kernels_ms_eager": kernels,
        "roofline": {"kernel": ("spectral pipeline (k_evolve + k_rows_w + k_cols_tma, one CUDA graph)"
                                if not (c4 or c5) else
                                "spectral pipeline (k_evolve + k_rows_w + k_cols_tma)" if c4 else
                                "slab pipeline (k_slab_evolve + k_slab_rows + k_slab_cols)"),
                     "bound": "hbm", "achieved": achieved, "peak": peak, "peak_kind": peak_kind,
                     "unit": "GB/s", "frac": achieved / peak,
                     # dram read + write bytes per frame of the same kernels (ncu
                     # application replay, profiles/roofline_traffic.json; config 3)
                     "traffic": _traffic() if not (c4 or c5) else None,
                     "algorithmic_bytes_per_frame": alg_bytes},
        "e2e": {"value": points / e2e_frame, "unit": "grid-points/s", "ms_per_frame": e2e_frame * 1e3,
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    if world == 1 and not args.no_cpu_baseline and not c5:
        line["cpu_baseline"] = cpu_baseline_c4() if c4 else cpu_baseline(frames=1, warmup=0)
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def cpu_baseline_c4(sample_instances: int = 2):
    """Reference generate_maps per instance (3 x 512^2, no batch API in the
    reference), `sample_instances` of the 64 timed and scaled."""
    from oracle.oracle import P
    from paper_2503_03326_b200._types import SpectrumParams  # noqa: F401
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
            "kind": "reference",
            "sample": f"{sample_instances} of 64 instances: reference generate_maps (3 x 512^2, "
                      f"CascadeSet built outside the timing), scaled x{C4_INSTANCES // sample_instances}"}


# ---------------------------------------------------------- reference (CPU)
def _ref_lib():
    from oracle.oracle import REF_SO, build, ref_available
    if not ref_available():
        build(reference=True)
    lib = C.CDLL(REF_SO)
    return lib


def cpu_baseline(frames: int = 1, warmup: int = 0, budget_s: float = 1e9):
    """The reference's own CPU implementation (oracle/_ref: the unmodified
    reference library compiled from its sources) on this host, all threads
    (set_worker_count(nproc)); spectral stages stay single-threaded in the
    reference (256-item chunks, parallel.cpp:29). Sample: full generate_maps
    (4 x 1024^2), build_slices at 2 of the 32 depths (scaled x16: its cost is
    linear in the depth count), full aggregate / compute_mask / FDM step."""
    from paper_2503_03326_b200._types import FdmConfig, SliceConfig
    from paper_2503_03326_b200.meshgen import uv_ellipsoid
    from oracle.oracle import P
    lib = _ref_lib()
    ncpu = os.cpu_count() or 1
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
    sample_depths = 2
    stage = np.zeros(5)
    for _ in range(warmup):
        lib.ref_bench_frame(b, DT, sample_depths, P(stage))
    ests, done = [], 0
    t_start = time.perf_counter()
    for _ in range(frames):
        lib.ref_bench_frame(b, DT, sample_depths, P(stage))
        est = stage[0] + stage[1] * (DEPTHS / sample_depths) + stage[2] + stage[3] + stage[4]
        ests.append((est, stage.copy()))
        done += 1
        if time.perf_counter() - t_start > budget_s:
            break
    lib.ref_bench_destroy(b)
    est = float(np.mean([e for e, _ in ests]))
    st_mean = np.mean([s for _, s in ests], axis=0)
    return {
        "value": POINTS_PER_FRAME / est,
        "unit": "grid-points/s",
        "ms_per_frame": est * 1e3,
        "cores": ncpu,
        "kind": "reference",
        "frames": done,
        "stage_s": {"generate_maps": st_mean[0], "build_slices_32_est": st_mean[1] * DEPTHS / sample_depths,
                    "aggregate": st_mean[2], "stability_mask": st_mean[3], "fdm": st_mean[4],
                    "cascade_init_once": t_init},
        "sample": (f"{done} frame(s) of config 3 through the reference library (oracle/_ref, g++ -O2): "
                   f"full generate_maps + aggregate + compute_mask + FdmZone::step, build_slices at "
                   f"{sample_depths} of {DEPTHS} depths scaled x{DEPTHS // sample_depths}; "
                   f"set_worker_count({ncpu})"),
    }


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    budget = 150.0
    cb = cpu_baseline(frames=args.steps, warmup=min(args.warmup, 1), budget_s=budget)
    line = {
        "impl": "reference",
        "metric": "ocean grid points/sec (spectrum+iFFT+forces) at 1024^2 x 4 cascades",
        "value": cb["value"],
        "unit": "grid-points/s",
        "n_gpus": world,
        "steps": cb["frames"],
        "steps_requested": args.steps,
        "warmup": min(args.warmup, 1),
        "ms_per_step": cb["ms_per_frame"],
        "ms_per_frame": cb["ms_per_frame"],
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (SURVEY 8d config 3)",
        "config": {"workload": WORKLOAD, "grid": N_GRID, "cascades": len(LENGTHS),
                   "depth_slices": DEPTHS, "fdm_grid": FDM_N, "parallelism": "host CPU"},
        "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
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
    ap.add_argument("--config", type=int, default=3, choices=[3, 4, 5],
                    help="3: the BASELINE metric frame (default); 4: 64 batched 512^2 instances; "
                         "5: single 16384^2 grid, slab FFT + all-to-all across ranks")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
