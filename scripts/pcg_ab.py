"""A/B of the adjoint backbone: Anderson (the reference's fixed point) vs
preconditioned CG (HETERODYN_ADJOINT=pcg) on one scene; prints adjoint
iterations, backward time and the gradients' difference.  Run each variant
in its own process:  python scripts/pcg_ab.py out.npz TAG"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_14526_b200 import scenes  # noqa: E402
from paper_2605_14526_b200.hd import Library  # noqa: E402

tag = sys.argv[2] if len(sys.argv) > 2 else "C3"
lib = Library(os.path.join(ROOT, "paper_2605_14526_b200", "_lib", "libheterodyn_b200.so"))
if tag.startswith("C"):
    scene = scenes.config_scene(tag, frames=3)
else:
    scene = scenes.block_scene(dims=(4, 3, 2), contrast=10.0, beta0=0.05, frames=3)
sim = lib.scene(scene).sim()
sim.record(True)
sim.step(3)
q, v = sim.positions(), sim.velocities()
t0 = time.time()
g = sim.backward(dl_dq_final=q, dl_dv_final=v)
dt = time.time() - t0
np.savez(sys.argv[1], **{k: g[k] for k in ("dl_dq0", "dl_dv0", "dl_df_ext", "dl_de", "dl_dw", "tau")},
         it=g["adjoint_iterations"])
print(f"{tag}: adjoint iterations {g['adjoint_iterations']}, backward {1e3 * dt:.1f} ms")
