import os, sys, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2605_14526_b200 import scenes
from paper_2605_14526_b200.hd import Library
prod = Library('paper_2605_14526_b200/_lib/libheterodyn_b200.so')
orc = Library('oracle/_build/libheterodyn_oracle.so')
def rel2(a,b): return np.linalg.norm(np.asarray(a)-b)/max(np.linalg.norm(b),1e-300)
def run(lib, scene, young, frames=2, sety=True):
    sim = lib.scene(scene).sim()
    if sety: sim.set_young(young)
    sim.record(True); sim.step(frames)
    q = sim.positions()
    return q, sim.velocities(), sim.backward(dl_dq_final=q, dl_dv_final=sim.velocities())
for name, scene in [("C1", scenes.config_scene("C1", frames=2)), ("pin", scenes.block_scene(dims=(5,3,2), kind="corotated", fix_x0_face=True, frames=2))]:
    ne = prod.scene(scene).element_count
    young = 3e4 * (1.0 + 0.5 * np.sin(np.arange(ne)))
    os.environ.pop("HETERODYN_HOST_REFACTOR", None)
    d = run(prod, scene, young)
    os.environ["HETERODYN_HOST_REFACTOR"] = "1"
    h = run(prod, scene, young)
    os.environ.pop("HETERODYN_HOST_REFACTOR", None)
    o = run(orc, scene, young)
    sc = dict(scene); sc["material"] = dict(sc["material"]); sc["material"]["young"] = young.tolist()
    f = run(prod, sc, young, sety=False)
    for k in ("dl_dq0","dl_dv0","dl_df_ext","dl_de","dl_dw"):
        print(name, k, "dev-orc %.2e host-orc %.2e fresh-orc %.2e" % (rel2(d[2][k], o[2][k]), rel2(h[2][k], o[2][k]), rel2(f[2][k], o[2][k])))
    print(name, "q", rel2(d[0], o[0]), rel2(h[0], o[0]), "tau", d[2]["tau"], o[2]["tau"])
