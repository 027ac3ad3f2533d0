"""Slab-decomposed single grid across ranks.

Rank r owns spectrum rows and output columns [r R, (r+1) R), R = N / ranks.
One frame = ocn_slab_rows (evolve + packed coefficients + row FFTs straight
into the all-to-all send layout) -> all-to-all of the R x R tiles -> ocn_slab_cols
(column FFTs + sign + Re/Im split into the column slab).

The exchange is the only collective of the path: `exchange()` runs it with
torch.distributed.all_to_all_single (NCCL over NVLink on B200 boxes; gloo in the
CPU tests). `emulated_frame()` runs R ranks' slabs on one GPU with the tile
exchange done as device copies: the same kernels and layouts, for testing the
decomposition without several GPUs (no rank ever waits on another).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _abi
from ._abi import check, lib
from ._types import SpectrumParams


def tile_layout(rows: int, ranks: int):
    """Send / receive layout: [peer][pair 0..3][row in R][column in R] complex64.
    Returns (elements per peer tile block, total elements)."""
    per_peer = 4 * rows * rows
    return per_peer, per_peer * ranks


class SlabSurface:
    def __init__(self, n: int, ranks: int, rank: int, length: float, params: SpectrumParams,
                 band_min: float = 0.0, band_max: float = 1e300, cascade_index: int = 0,
                 ctx=None):
        from .ocean import Context
        self.ctx = ctx or Context.default()
        self.n, self.ranks, self.rank = n, ranks, rank
        h = C.c_void_p()
        check(lib().ocn_slab_create(self.ctx.h, n, ranks, rank, length, band_min, band_max,
                                    cascade_index, C.byref(params), C.byref(h)), self.ctx.h, "slab")
        self.h = h
        rows, cols, nbytes = C.c_int(), C.c_int(), C.c_size_t()
        lib().ocn_slab_info(self.h, C.byref(rows), C.byref(cols), C.byref(nbytes))
        self.rows, self.cols, self.exchange_bytes = rows.value, cols.value, nbytes.value

    def rows_pass(self, t: float, send_ptr: int, choppiness: float = 1.0):
        check(lib().ocn_slab_rows(self.h, t, choppiness, C.c_void_p(send_ptr)), self.ctx.h, "rows")

    def cols_pass(self, recv_ptr: int):
        """Column pass from the receive buffer (overwritten in place for n >= 4096)."""
        check(lib().ocn_slab_cols(self.h, C.c_void_p(recv_ptr)), self.ctx.h, "cols")

    def field(self, f: int) -> np.ndarray:
        """Column slab [N][R] of surface field f (fp64 copy)."""
        out = np.zeros((self.n, self.cols))
        check(lib().ocn_slab_download(self.h, f, out.ctypes.data_as(_abi.d)), self.ctx.h, "download")
        return out

    def __del__(self):
        try:
            if self.h:
                lib().ocn_slab_destroy(self.h)
                self.h = None
        except Exception:
            pass


class Comm:
    """The library's own NCCL communicator (ocn_comm): rank 0 makes the unique
    id, `share` distributes it (e.g. torch.distributed.broadcast_object_list),
    every rank joins on its context's device."""

    def __init__(self, ctx, nranks: int, rank: int, share=None):
        uid = C.create_string_buffer(128)
        if rank == 0:
            check(lib().ocn_comm_unique_id(uid), None, "comm id")
        raw = bytes(uid.raw)
        if share is not None:
            raw = share(raw)
        self.ctx = ctx
        h = C.c_void_p()
        check(lib().ocn_comm_create(ctx.h, C.c_char_p(raw), nranks, rank, C.byref(h)), ctx.h,
              "comm")
        self.h = h

    def __del__(self):
        try:
            if self.h:
                lib().ocn_comm_destroy(self.h)
                self.h = None
        except Exception:
            pass


def frame(slab: "SlabSurface", comm, t: float, send_ptr: int, recv_ptr: int,
          choppiness: float = 1.0):
    """ocn_slab_frame: rows, per-pair exchange over NVLink, columns (async)."""
    check(lib().ocn_slab_frame(slab.h, comm.h if comm else None, t, choppiness,
                               C.c_void_p(send_ptr), C.c_void_p(recv_ptr)), slab.ctx.h, "frame")


def exchange(send, recv, group=None):
    """All-to-all of the equal R x R tile blocks (send[peer] -> rank peer)."""
    import torch.distributed as dist
    dist.all_to_all_single(recv, send, group=group)


def emulated_frame(slabs, t: float, choppiness: float = 1.0):
    """All ranks' slabs on one device: rows passes, tile exchange by device
    copies (recv[r][src] = send[src][r]), columns passes. Returns the full
    fields [8][N][N] assembled from the column slabs."""
    import torch
    R = len(slabs)
    rows = slabs[0].rows
    per_peer, total = tile_layout(rows, R)
    dev = f"cuda:{slabs[0].ctx.device}"
    send = [torch.empty(2 * total, dtype=torch.float32, device=dev) for _ in range(R)]
    recv = [torch.empty(2 * total, dtype=torch.float32, device=dev) for _ in range(R)]
    for r, s in enumerate(slabs):
        s.rows_pass(t, send[r].data_ptr(), choppiness)
        s.ctx.synchronize()
    for r in range(R):
        for src in range(R):
            recv[r][2 * per_peer * src:2 * per_peer * (src + 1)].copy_(
                send[src][2 * per_peer * r:2 * per_peer * (r + 1)])
    torch.cuda.synchronize()
    for r, s in enumerate(slabs):
        s.cols_pass(recv[r].data_ptr())
        s.ctx.synchronize()
    n = slabs[0].n
    out = np.zeros((8, n, n))
    for r, s in enumerate(slabs):
        for f in range(8):
            out[f][:, r * s.cols:(r + 1) * s.cols] = s.field(f)
    return out
