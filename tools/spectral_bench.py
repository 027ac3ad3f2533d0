"""Time the config-2 spectral step alone under kernel-variant switches
(env vars read by libocean_b200): prints ms/frame (device events)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C  # noqa: E402

import bench  # noqa: E402

fr = bench.Frame(0, pipelined=False)
L = fr.L
for _ in range(5):
    L.ocn_spectral_step(fr.maps[0].h, fr.slices[0].h, 0.1, 1.0)
fr.ctx.synchronize()
import torch  # noqa: E402
s = torch.cuda.ExternalStream(fr.ctx.stream, device="cuda:0")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
K = 50
e0.record(s)
for k in range(K):
    L.ocn_spectral_step(fr.maps[0].h, fr.slices[0].h, 0.1 + k / 60, 1.0)
e1.record(s)
fr.ctx.synchronize()
print(f"{sys.argv[1] if len(sys.argv) > 1 else 'default'}: spectral {e0.elapsed_time(e1) / K:.3f} ms/frame")
