"""Time one configuration's spectral step alone under kernel-variant switches
(env vars read by libocean_b200): prints ms per step (device events).

    python tools/spectral_bench.py LABEL [CONFIG]   (CONFIG 3 default, 4, 1 or 5)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402

cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 3
if cfg == 4:
    fr = bench.Frame4(0, 0, 1)
    step = lambda k: fr.L.ocn_surface_generate(fr.maps.h, 0.1 + k / 60, 1.0)  # noqa: E731
elif cfg == 5:
    fr = bench.Frame5(0, 0, 1, None)
    step = lambda k: fr.step()  # noqa: E731
elif cfg == 1:
    fr = bench.Frame1(0, 0, 1)
    step = lambda k: fr.L.ocn_surface_generate_batch(fr.maps.h, 0.1 + k * 10, 1 / 60, 1.0)  # noqa: E731
else:
    fr = bench.Frame(0, pipelined=False)
    step = lambda k: fr.L.ocn_spectral_step(fr.maps[0].h, fr.slices[0].h, 0.1 + k / 60, 1.0)  # noqa: E731
for k in range(5):
    step(k)
fr.ctx.synchronize()
import torch  # noqa: E402
s = torch.cuda.ExternalStream(fr.ctx.stream, device="cuda:0")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
K = 50
e0.record(s)
for k in range(K):
    step(k)
e1.record(s)
fr.ctx.synchronize()
label = sys.argv[1] if len(sys.argv) > 1 else "default"
print(f"{label} config {cfg}: spectral {e0.elapsed_time(e1) / K:.3f} ms/step")
