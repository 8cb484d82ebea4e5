import ctypes as C, sys, time
import numpy as np
sys.path.insert(0, '.')
from paper_2605_14526_b200.hd import Library, HdError
from paper_2605_14526_b200 import scenes
P = Library('paper_2605_14526_b200/_lib/libheterodyn_b200.so')
sd = scenes.config_scene("C2", frames=10)
sc = P.scene(sd)
ne = sc.element_count
young = scenes.c5_young(64, ne)
ref = sc.sim(); ref.step(10); target = ref.positions()
D = C.POINTER(C.c_double)
bad = []
for s in range(64):
    sim = sc.sim()
    y = np.ascontiguousarray(young[s])
    P.check(P.lib.hd_sim_set_young(sim.h, y.ctypes.data_as(D), ne, 0))
    sim.record(True)
    its = []
    for f in range(10):
        sim.step(); its.append(sim.last_iterations)
    q = sim.positions()
    try:
        g = sim.backward(dl_dq_final=q - target)
        print(s, round(young[s, 0]), its, "adj", g["adjoint_iterations"], flush=True)
    except HdError as e:
        print(s, round(young[s, 0]), its, "ERR", e, flush=True)
        bad.append(s)
print("bad", bad)
for th in (1, 16):
    b = sc.batch(64, young, threads=th)
    b.set_target(target)
    try:
        t = time.time(); r = b.evaluate(10); print("batch threads", th, "ok", time.time() - t, r["loss"].sum(), b.last_ms)
    except HdError as e:
        print("batch threads", th, "ERR", e)
