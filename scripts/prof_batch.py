"""Profiling driver for the batched system-ID evaluation (C5 shape): builds the
batch once, then runs `evals` evaluations of `frames` frames (run under ncu
with HETERODYN_NO_COND_GRAPH=1 for a per-kernel launch list).
  python scripts/prof_batch.py [samples] [frames] [evals]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2605_14526_b200 import scenes  # noqa: E402
from paper_2605_14526_b200.hd import Library  # noqa: E402

samples = int(sys.argv[1]) if len(sys.argv) > 1 else 64
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 1
evals = int(sys.argv[3]) if len(sys.argv) > 3 else 1
lib = Library(os.path.join(ROOT, "paper_2605_14526_b200", "_lib", "libheterodyn_b200.so"))
sc = lib.scene(scenes.config_scene("C2", frames=frames))
young = scenes.c5_young(samples, sc.element_count)
b = sc.batch(samples, young, threads=32)
b.set_target(np.asarray(sc.rest_positions()).reshape(-1))
for i in range(evals):
    t0 = time.time()
    r = b.evaluate(frames)
    print(f"eval {i}: {1e3 * (time.time() - t0):.1f} ms wall, {b.last_ms:.1f} ms device, "
          f"loss sum {r['loss'].sum():.6e}, solves {b.solve_count}", flush=True)
