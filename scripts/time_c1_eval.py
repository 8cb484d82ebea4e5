"""Split of one identify evaluation at C1 (profiling): set_young vs 20
recorded frames + adjoint chain."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_14526_b200 import scenes  # noqa: E402
from paper_2605_14526_b200.hd import Library  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = Library(os.path.join(ROOT, "paper_2605_14526_b200", "_lib", "libheterodyn_b200.so"))
sc = lib.scene(scenes.config_scene("C1"))
sim = sc.sim()
y = np.full(sc.element_count, 5e4)
for rep in range(3):
    t0 = time.perf_counter()
    sim.set_young(y * (1 + 0.01 * rep))
    t1 = time.perf_counter()
    sim.set_state(q=sim.positions(), v=sim.velocities())
    sim.record(False)
    sim.record(True)
    sim.step(20)
    t2 = time.perf_counter()
    sim.backward(dl_dq_final=sim.positions())
    t3 = time.perf_counter()
    print(f"set_young {1e3 * (t1 - t0):.1f} ms, 20 frames {1e3 * (t2 - t1):.1f} ms, backward {1e3 * (t3 - t2):.1f} ms")
