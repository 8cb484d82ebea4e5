"""Per-step wall time, contact rows and iterations of a contact scene on the
product library (diagnostics): python scripts/time_contact_steps.py C4 8"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_14526_b200 import scenes  # noqa: E402
from paper_2605_14526_b200.hd import Library  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "C4"
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 8
lib = Library(os.path.join(ROOT, "paper_2605_14526_b200", "_lib", "libheterodyn_b200.so"))
sim = lib.scene(scenes.config_scene(tag, frames=frames)).sim()
for f in range(frames):
    t0 = time.perf_counter()
    sim.step()
    t = time.perf_counter() - t0
    tr = sim.contact_trace()
    print(f"frame {f}: {1e3 * t:8.2f} ms  iterations {sim.last_iterations:4d}  contacts {sim.last_contact_count:3d}"
          f"  frictional {tr['cone'].shape[1]:3d}", flush=True)
