import time, sys, traceback
import numpy as np
sys.path.insert(0, ".")
from paper_2605_14526_b200.hd import Library
from paper_2605_14526_b200 import scenes
P = Library("paper_2605_14526_b200/_lib/libheterodyn_b200.so")
O = Library("oracle/_build/libheterodyn_oracle.so")

def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)

def compare(scene, frames, name):
    try:
        ps = P.scene(scene); os_ = O.scene(scene)
        t0 = time.time(); psim = ps.sim(); t1 = time.time(); osim = os_.sim()
        print(f"== {name}: nv={ps.vertex_count} ne={ps.element_count} create {t1-t0:.2f}s", flush=True)
        psim.record(); osim.record()
        for f in range(frames):
            t0 = time.time(); psim.step(); t1 = time.time(); osim.step(); t2 = time.time()
            qp, qo = psim.positions(), osim.positions()
            vp, vo = psim.velocities(), osim.velocities()
            print(f"  frame {f}: it {psim.last_iterations}/{osim.last_iterations} conv {psim.last_converged}/{osim.last_converged} "
                  f"relq {rel(qp,qo):.2e} relv {rel(vp,vo):.2e} gpu {1e3*(t1-t0):.1f}ms cpu {1e3*(t2-t1):.1f}ms", flush=True)
        qp = psim.positions(); qo = osim.positions()
        t0 = time.time(); gp = psim.backward(dl_dq_final=qo, dl_dv_final=osim.velocities()); t1 = time.time()
        go = osim.backward(dl_dq_final=qo, dl_dv_final=osim.velocities()); t2 = time.time()
        for k in ["dl_dq0", "dl_dv0", "dl_df_ext", "dl_de", "dl_dw"]:
            print(f"  {k}: rel {rel(gp[k], go[k]):.2e}")
        print(f"  tau {gp['tau']} / {go['tau']}  adj {gp['adjoint_iterations']}/{go['adjoint_iterations']} gpu {1e3*(t1-t0):.1f}ms cpu {1e3*(t2-t1):.1f}ms", flush=True)
    except Exception:
        traceback.print_exc()

compare(scenes.block_scene(), 3, "block NH")
compare(scenes.block_scene(fix_x0_face=True, kind="corotated", beta0=0.1, hook=True), 3, "block corot fixed hook")
compare(scenes.two_tets_unequal(alpha=0.01, beta0=0.05), 1, "two tets")
compare(scenes.config_scene("C1", frames=3), 3, "C1")
compare(scenes.config_scene("C2", frames=2), 2, "C2")

try:
    sc = P.scene(scenes.config_scene("C3", frames=2))
    t0=time.time(); sim = sc.sim(); print("C3 create %.2fs nnz %d"%(time.time()-t0, sim.factor_nnz), flush=True)
    sim.record()
    for f in range(2):
        t0=time.time(); sim.step(); print("C3 step %.1f ms it %d conv %d"%(1e3*(time.time()-t0), sim.last_iterations, sim.last_converged), flush=True)
    t0=time.time(); g = sim.backward(dl_dq_final=sim.positions(), dl_dv_final=sim.velocities()); print("C3 backward %.1f ms adj %d tau %s"%(1e3*(time.time()-t0), g["adjoint_iterations"], g["tau"]), flush=True)
except Exception:
    traceback.print_exc()
