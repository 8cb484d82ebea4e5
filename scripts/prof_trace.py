"""In-graph timeline of the adjoint backbone kernels on C3 (profiling only):
per kernel, when its first CTA was resident, passed its PDL dependency wait,
and when its last CTA ended, relative to the iteration's first kernel."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_14526_b200 import scenes  # noqa: E402
from paper_2605_14526_b200.hd import Library  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = Library(os.path.join(ROOT, "paper_2605_14526_b200", "_lib", "libheterodyn_b200.so"))
sim = lib.scene(scenes.config_scene(sys.argv[1] if len(sys.argv) > 1 else "C3")).sim()
sim.record(True)
sim.step()
sim.backward_canonical(download=False)
names = ["Bx", "gather", "rowdot", "zfold", "coltile", "dots", "mix"]
tr = sim.trace_backbone(12)
per = []
for it in range(4, 12):
    t = tr[it] / 1e3
    base = t[0, 1]
    nxt = tr[it + 1][0, 1] / 1e3 if it + 1 < 12 else None
    per.append((nxt - base) if nxt is not None else np.nan)
    if it in (6, 7):
        print(f"iteration {it}: (us from B x start)  resident / start / end / busy")
        for k, nm in enumerate(names):
            print(f"  {nm:8s} {t[k, 0] - base:8.2f} {t[k, 1] - base:8.2f} {t[k, 2] - base:8.2f}  {t[k, 2] - t[k, 1]:7.2f}")
        print("  AA dots: loop done %.2f  partials %.2f  | tail entry %.2f  folded %.2f  solved %.2f" %
              (t[10, 2] - base, t[11, 2] - base, t[7, 2] - base, t[8, 2] - base, t[9, 2] - base))
print("iteration period (us):", " ".join(f"{p:.1f}" for p in per if p == p))

# the real WHILE loop (unrolled body, conditional node)
tl = sim.trace_loop()
print(f"real loop: {len(tl)} traced iterations")
starts = [tl[i][0, 1] / 1e3 for i in range(len(tl))]
print("iteration period (us):", " ".join(f"{b - a:.1f}" for a, b in zip(starts, starts[1:])))
for it in (len(tl) - 3, len(tl) - 2):
    t = tl[it] / 1e3
    base = t[0, 1]
    print(f"loop iteration {it}: resident / start / end / busy")
    for k, nm in enumerate(names):
        print(f"  {nm:8s} {t[k, 0] - base:8.2f} {t[k, 1] - base:8.2f} {t[k, 2] - base:8.2f}  {t[k, 2] - t[k, 1]:7.2f}")
for it in (len(tl) - 3, len(tl) - 2):
    t = tl[it] / 1e3
    base = t[0, 1]
    print(f"loop iteration {it}: AA solve kernel resident {t[7, 0] - base:.2f} start {t[7, 1] - base:.2f} fold {t[8, 2] - base:.2f}  bookkeeping {t[12, 2] - base:.2f}  LDLT {t[13, 2] - base:.2f}  end {t[7, 2] - base:.2f}")
