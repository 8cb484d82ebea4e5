"""compute-sanitizer target: a small contact scene through forward, the
multi-column contact adjoint (two-columns-per-warp passes) and the drivers."""
import sys
sys.path.insert(0, '.')
from paper_2605_14526_b200 import scenes  # noqa: E402
from paper_2605_14526_b200.hd import Library  # noqa: E402
lib = Library('paper_2605_14526_b200/_lib/libheterodyn_b200.so')
sim = lib.scene(scenes.block_scene(dims=(3, 2, 2), floor=True, frames=2)).sim()
sim.record(True)
sim.step(2)
q = sim.positions()
g = sim.backward(dl_dq_final=q, dl_dv_final=sim.velocities())
print("contacts", sim.last_contact_count, "adjoint sweeps", sim.backward_iterations if hasattr(sim, "backward_iterations") else "-")
print(lib.builtin("ball-drop").run_simulate()["max_penetration"])
print("ok")
