"""A/B helper for the multi-column solve passes (run in a subprocess: the pass
variant is read once per process from HETERODYN_ROWDOT / HETERODYN_COLTILE).
Runs a contact scene's trajectory and adjoint chain (the adjoint's contact
columns go through hdk_apply_inverse3_multi) and saves q, v and the
gradients.   python scripts/columns_ab.py out.npz [dims]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_14526_b200 import scenes  # noqa: E402
from paper_2605_14526_b200.hd import Library  # noqa: E402

dims = tuple(int(x) for x in sys.argv[2].split(",")) if len(sys.argv) > 2 else (10, 6, 6)
lib = Library(os.path.join(ROOT, "paper_2605_14526_b200", "_lib", "libheterodyn_b200.so"))
sim = lib.scene(scenes.config_scene("C4", frames=3, dims=dims, solver={"eps_rel": 1e-12, "eps_abs": 1e-14})).sim()
sim.record(True)
sim.step(3)
q, v = sim.positions(), sim.velocities()
g = sim.backward(dl_dq_final=q, dl_dv_final=v)
np.savez(sys.argv[1], q=q, v=v, contacts=sim.last_contact_count, adjoint_iterations=g["adjoint_iterations"],
         **{k: g[k] for k in ("dl_dq0", "dl_dv0", "dl_df_ext", "dl_de", "dl_dw", "tau")})
print(f"contacts {sim.last_contact_count}, adjoint iterations {g['adjoint_iterations']}")
