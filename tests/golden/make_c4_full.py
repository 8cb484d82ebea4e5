"""Generates tests/golden/c4_full.npz (test infrastructure): the CPU oracle on
the full-size C4 scene (40 x 24 x 18 gripper pad, 103,680 tets, frictional
contact) for 3 frames at eps_rel = 1e-12 — per frame q, v, iterations and the
contact trace (rows; clamp / cone decisions as -1 / +1, 0 for round-off
ties), and the chained gradients of L = 1/2|q_T|^2 + 1/2|v_T|^2 seeds
(dl_dq_final = q_T, dl_dv_final = v_T).  Values are stored as float32 (the
parity bars are >= 1e-6 relative; float32 rounding is 6e-8).  A second run
with q0 perturbed by 1e-15 max|q0| gives the oracle's own conditioning per
quantity (entry "converged/C4-full" of contact_conditioning.json).

The oracle needs hours for this (about 100 contact rows, one adjoint
backbone each per frame); the GPU box cannot run it inside a test, so the
outputs are committed.

Run: python tests/golden/make_c4_full.py run  /tmp/c4a.npz
     python tests/golden/make_c4_full.py run  /tmp/c4b.npz 1e-15
     python tests/golden/make_c4_full.py merge /tmp/c4a.npz /tmp/c4b.npz"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
GOLDEN = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from paper_2605_14526_b200 import scenes  # noqa: E402

FRAMES = 3
GRADS = ("dl_dq0", "dl_dv0", "dl_df_ext", "dl_de", "dl_dw")
TIE = 1e-9


def c4_full_scene():
    return scenes.config_scene("C4", frames=FRAMES, solver={"eps_rel": 1e-12, "eps_abs": 1e-14, "k_max": 5000})


def decisions(tr):
    cl, co = tr["clamp"], tr["cone"]
    scale = max(np.abs(cl).max(initial=0.0), 1e-300)
    dc = np.where(np.abs(cl) <= TIE * scale, 0, np.where(cl < 0, 1, -1)).astype(np.int8)
    dk = np.where((np.abs(co) <= TIE), 0, np.where(co > 0, 1, -1)).astype(np.int8)
    return dc, dk


def do_run(out, perturb):
    from paper_2605_14526_b200.hd import Library
    orc = Library(os.path.join(ROOT, "oracle", "_build", "libheterodyn_oracle.so"))
    sim = orc.scene(c4_full_scene()).sim()
    if perturb:
        q = sim.positions()
        sim.set_state(q + perturb * np.abs(q).max() * np.sin(np.arange(q.size)), sim.velocities(), 0.0)
    sim.record(True)
    rec = {}
    t0 = time.time()
    for f in range(FRAMES):
        sim.step()
        tr = sim.contact_trace()
        dc, dk = decisions(tr)
        rec[f"q{f}"], rec[f"v{f}"] = sim.positions(), sim.velocities()
        rec[f"it{f}"] = np.array([sim.last_iterations, sim.last_converged])
        rec[f"vertex{f}"], rec[f"obstacle{f}"] = tr["vertex"], tr["obstacle"]
        rec[f"clamp{f}"], rec[f"cone{f}"] = dc, dk
        print(f"frame {f}: {sim.last_iterations} iterations, {tr['vertex'].size} contacts, {time.time() - t0:.0f} s",
              flush=True)
    g = sim.backward(dl_dq_final=rec[f"q{FRAMES - 1}"], dl_dv_final=rec[f"v{FRAMES - 1}"])
    print(f"backward: {time.time() - t0:.0f} s, adjoint iterations {g['adjoint_iterations']}", flush=True)
    for k in GRADS:
        rec[k] = g[k]
    rec["tau"] = g["tau"]
    np.savez(out, **rec)


def rel2(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def merge(a_path, b_path):
    a, b = np.load(a_path), np.load(b_path)
    out = {}
    for k in a.files:
        x = a[k]
        out[k] = x.astype(np.float32) if x.dtype == np.float64 and k not in ("tau",) else x
    np.savez_compressed(os.path.join(GOLDEN, "c4_full.npz"), **out)
    cond = {"q": [rel2(b[f"q{f}"], a[f"q{f}"]) for f in range(FRAMES)],
            "v": [rel2(b[f"v{f}"], a[f"v{f}"]) for f in range(FRAMES)],
            "iterations": [int(a[f"it{f}"][0]) for f in range(FRAMES)],
            "iterations_perturbed": [int(b[f"it{f}"][0]) for f in range(FRAMES)]}
    for k in GRADS:
        cond[k] = rel2(b[k], a[k])
    p = os.path.join(GOLDEN, "contact_conditioning.json")
    allc = json.load(open(p)) if os.path.exists(p) else {}
    allc["converged/C4-full"] = cond
    json.dump(allc, open(p, "w"), indent=1)
    print(json.dumps(cond))


if __name__ == "__main__":
    if sys.argv[1] == "run":
        do_run(sys.argv[2], float(sys.argv[3]) if len(sys.argv) > 3 else 0.0)
    else:
        merge(sys.argv[2], sys.argv[3])
