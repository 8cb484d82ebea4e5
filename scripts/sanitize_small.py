import sys
sys.path.insert(0, '.')
from paper_2605_14526_b200 import scenes
from paper_2605_14526_b200.hd import Library
lib = Library('paper_2605_14526_b200/_lib/libheterodyn_b200.so')
sim = lib.scene(scenes.block_scene(dims=(4, 3, 2), contrast=10.0)).sim()
sim.record(True)
sim.step()
g = sim.backward_canonical(download=False)
print("ok")
