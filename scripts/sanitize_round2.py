"""compute-sanitizer target for the round-2 paths: the lockstep batch
(hdk_seg_* kernels) with a device refactorization (refactor.cu) and a
contact scene whose adjoint columns run eight per factor stream through the
tensor-core row-dot pass."""
import sys

import numpy as np

sys.path.insert(0, '.')
from paper_2605_14526_b200 import scenes  # noqa: E402
from paper_2605_14526_b200.hd import Library  # noqa: E402

lib = Library('paper_2605_14526_b200/_lib/libheterodyn_b200.so')
sc = lib.scene(scenes.block_scene(dims=(3, 2, 2), frames=2, gravity_z=-9.81, alpha=0.02, beta0=0.03, v0_amp=0.05))
young = scenes.c5_young(3, sc.element_count, base=5e4)
b = sc.batch(3, young)
b.set_target(np.asarray(sc.sim().positions()) + 1e-3)
b.evaluate(2)
b.set_young(young * 1.1)
r = b.evaluate(2)
print("lockstep", b.lockstep, r["loss"])
sim = lib.scene(scenes.config_scene("C4", frames=2, dims=(6, 4, 4))).sim()
sim.record(True)
sim.step(2)
q = sim.positions()
g = sim.backward(dl_dq_final=q, dl_dv_final=sim.velocities())
print("contacts", sim.last_contact_count, "adjoint iterations", g["adjoint_iterations"])
print("ok")
