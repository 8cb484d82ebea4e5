"""Diagnostics: product vs oracle on one contact case of tests/test_gpu_contact.py —
per frame iterations, |dq|, and the first clamp / cone decision that differs."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_2605_14526_b200.hd import Library  # noqa: E402
from test_gpu_contact import CONVERGED, FIXED, fixed_iterations, rel2, run  # noqa: E402

prod = Library(os.path.join(ROOT, "paper_2605_14526_b200", "_lib", "libheterodyn_b200.so"))
orc = Library(os.path.join(ROOT, "oracle", "_build", "libheterodyn_oracle.so"))
kind, name = sys.argv[1], sys.argv[2]
if kind == "fixed":
    scene, frames, k = FIXED[name]
    scene = fixed_iterations(scene, k)
else:
    scene, frames = CONVERGED[name]
tp, trp, gp = run(prod, scene, frames)
to, tro, go = run(orc, scene, frames)
for f in range(frames):
    a, b = trp[f], tro[f]
    print(f"frame {f}: iters {a['iterations']} / {b['iterations']}  rel dq {rel2(tp[f][0], to[f][0]):.2e}  "
          f"rows equal {np.array_equal(a['vertex'], b['vertex'])}")
    n = min(a["iterations"], b["iterations"])
    dc = np.argwhere((a["clamp"][:n] < 0) != (b["clamp"][:n] < 0))
    dk = np.argwhere((a["cone"][:n] > 0) != (b["cone"][:n] > 0))
    for lab, d, A, B in (("clamp", dc, a["clamp"], b["clamp"]), ("cone", dk, a["cone"], b["cone"])):
        if len(d):
            it, i = d[0]
            print(f"   {lab}: {len(d)} differ; first at iteration {it} entry {i}: product {A[it, i]:.3e} oracle {B[it, i]:.3e}"
                  f"  (oracle row {np.array2string(B[it], precision=2, max_line_width=200)})")
