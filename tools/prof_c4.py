"""Run a few config-4 frames (for ncu captures; not a benchmark)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 2
fr = bench.Frame4(0, 0, 1)
for _ in range(frames):
    fr.step()
fr.sync()
print("ok", fr.ctx.kernel_launches())
