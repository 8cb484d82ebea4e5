"""Ablation timing of one multi-column contact-adjoint iteration (profiling)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_14526_b200 import scenes  # noqa: E402
from paper_2605_14526_b200.hd import Library  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = Library(os.path.join(ROOT, "paper_2605_14526_b200", "_lib", "libheterodyn_b200.so"))
sim = lib.scene(scenes.config_scene("C3")).sim()
sim.record(True)
sim.step()
sim.backward_canonical(download=False)
for name, mask in (("full", 0x10000), ("-solve", 0x10000 | (1 << 17)), ("-columns", 0x10000 | (2 << 17))):
    print(f"{name:10s} {1e3 * sim.time_backbone(30, mask):8.1f} us / 4-column iteration")
print(f"single-column backbone iteration {1e3 * sim.time_backbone(30, 0):.1f} us")
