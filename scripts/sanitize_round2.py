"""compute-sanitizer target for the round-2 paths: the lockstep batch
(hdk_seg_* kernels) with a device refactorization (refactor.cu), a contact
scene whose adjoint columns run by block CG eight per factor stream through
the tensor-core passes, and a three-frame backward whose backbone solves
record and then deflate with the recycled Ritz vectors (hdk_defl_*)."""
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
sim = lib.scene(scenes.block_scene(dims=(6, 4, 3), frames=3, contrast=10.0, alpha=0.02, gravity_z=-9.81)).sim()
sim.record(True)
sim.step(3)
g = sim.backward(dl_dq_final=sim.positions(), dl_dv_final=sim.velocities())
print("deflated backward, adjoint iterations", g["adjoint_iterations"])
print("ok")
