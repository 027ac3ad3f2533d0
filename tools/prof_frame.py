"""Run a few config-3 frames (for ncu captures; not a benchmark)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 3
fr = bench.Frame(0)
for _ in range(frames):
    fr.step()
fr.sync()
print("ok", sum(c.kernel_launches() for c in fr.contexts()))
