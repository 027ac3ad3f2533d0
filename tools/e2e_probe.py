"""Host time per C-ABI call of bench.py's config-3 frame in the e2e loop
(pipelined frames, report read after the next spectral step is enqueued)."""
import ctypes as C
import os
import sys
import time
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

fr = bench.Frame(0, pipelined=True)
L = fr.L
acc = defaultdict(float)


def timed(name, fn, *a):
    t0 = time.perf_counter()
    r = fn(*a)
    acc[name] += time.perf_counter() - t0
    return r


for name in ["ocn_spectral_step", "ocn_hydro_aggregate", "ocn_zone_update_stability",
             "ocn_zone_mask_from_hydro", "ocn_zone_step", "ocn_hydro_report_get"]:
    orig = getattr(L, name)
    setattr(fr, "_" + name, orig)
for _ in range(10):
    fr.step(read_report=True)
fr.finish(read_report=True)
fr.sync()
K = 200


class Wrap:
    def __init__(self, lib):
        self.lib = lib

    def __getattr__(self, name):
        f = getattr(self.lib, name)
        if not name.startswith("ocn_"):
            return f
        return lambda *a: timed(name, f, *a)


fr.L = Wrap(L)
t0 = time.perf_counter()
for _ in range(K):
    fr.step(read_report=True)
fr.finish(read_report=True)
fr.sync()
tot = time.perf_counter() - t0
print(f"e2e {tot / K * 1e3:.3f} ms/frame; per call (ms/frame):")
for k, v in sorted(acc.items(), key=lambda x: -x[1]):
    print(f"  {k:32s} {v / K * 1e3:.4f}")
