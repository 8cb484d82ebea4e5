import sys, time
import numpy as np
sys.path.insert(0, '.')
from paper_2605_14526_b200.hd import Library, HdError
from paper_2605_14526_b200 import scenes
P = Library('paper_2605_14526_b200/_lib/libheterodyn_b200.so')
samples, threads, frames = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
sd = scenes.config_scene("C2", frames=frames)
sc = P.scene(sd)
young = scenes.c5_young(samples, sc.element_count)
ref = sc.sim(); ref.step(frames); target = ref.positions()
b = sc.batch(samples, young, threads=threads)
b.set_target(target)
for rep in range(2):
    try:
        t = time.time(); r = b.evaluate(frames)
        print(f"samples={samples} threads={threads} rep={rep} ok wall={time.time()-t:.2f}s dev={b.last_ms:.1f}ms loss={r['loss'].sum():.6e}", flush=True)
    except HdError as e:
        print(f"samples={samples} threads={threads} rep={rep} ERR {e}", flush=True)
