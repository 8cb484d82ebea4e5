"""Diagnostics: the CPU oracle on the reduced C4 scene at eps_rel = 1e-12 —
per-frame iterations / convergence, and a checksum, to compare machines."""
import hashlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_2605_14526_b200.hd import Library  # noqa: E402
from test_gpu_contact import CONVERGED  # noqa: E402

orc = Library(os.path.join(ROOT, "oracle", "_build", "libheterodyn_oracle.so"))
scene, frames = CONVERGED["C4-reduced"]
sim = orc.scene(scene).sim()
for f in range(frames):
    sim.step()
    q = sim.positions()
    print(f, sim.last_iterations, sim.last_converged, hashlib.md5(q.tobytes()).hexdigest(), flush=True)
