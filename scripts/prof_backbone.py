"""Ablation timing of one adjoint backbone iteration on C3 (profiling only):
ms per body launch with subsets of its kernels skipped."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_14526_b200 import scenes  # noqa: E402
from paper_2605_14526_b200.hd import Library  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = Library(os.path.join(ROOT, "paper_2605_14526_b200", "_lib", "libheterodyn_b200.so"))
sim = lib.scene(scenes.config_scene(sys.argv[1] if len(sys.argv) > 1 else "C3")).sim()
sim.record(True)
sim.step()
sim.backward_canonical(download=False)
names = {0: "full body", 1: "-Bx", 2: "-gather", 4: "-solve", 8: "-dots/aasolve", 16: "-mix",
         32: "-AA tail", 64: "-rowdot", 128: "-zreduce", 256: "-coltile", 31 - 4: "solve only", 31: "empty"}
base = None
only = [int(a) for a in sys.argv[2:]]
for mask, name in names.items():
    if only and mask not in only and mask != 0:
        continue
    ms = sim.time_backbone(100, mask)
    if mask == 0:
        base = ms
    print(f"{name:16s} mask={mask:2d}  {1e3 * ms:8.2f} us/iter  (delta {1e3 * (base - ms):7.2f})")
ms, b = sim.time_solve(50)
print(f"time_solve (perm, with x-fold): {1e3 * ms:.2f} us")
