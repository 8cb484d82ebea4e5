import sys
import numpy as np
sys.path.insert(0, '.')
from paper_2605_14526_b200.hd import Library
from paper_2605_14526_b200 import scenes
P = Library('paper_2605_14526_b200/_lib/libheterodyn_b200.so')
which = sys.argv[1] if len(sys.argv) > 1 else "c2"
if which == "c2":
    sd = scenes.config_scene("C2", frames=2)
else:
    sd = scenes.block_scene(dims=(3, 2, 2), frames=2, gravity_z=-9.81, alpha=0.02)
sc = P.scene(sd)
young = scenes.c5_young(2, sc.element_count, base=1e5)
ref = sc.sim(); ref.step(2); target = ref.positions()
b = sc.batch(2, young, threads=2)
b.set_target(target)
r = b.evaluate(2)
print("ok", r["loss"], np.linalg.norm(r["dl_de"]))
