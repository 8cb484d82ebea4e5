"""Generates tests/golden/contact_conditioning.json (test infrastructure): the
CPU oracle's own sensitivity on every contact case of tests/test_gpu_contact.py
— the relative change of q and v per frame and of every gradient when every
coordinate of q0 is perturbed by 1e-15 max|q0| (sin pattern).  It measures the reference algorithm's
conditioning: where the dual gate fires (eps_rel = 1e-12) or where a run of
fixed length stops inside the linearly converging NCP / Anderson iteration is
decided at round-off level, and the contact adjoint's lifted reduced system
can amplify rounding.  No implementation can agree with the oracle below this
floor; the tests hold each quantity to max(1e-6, 10 x its entry).

Run: python tests/golden/make_contact_conditioning.py   (a few minutes, 8 cores)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from paper_2605_14526_b200.hd import Library  # noqa: E402
from test_gpu_contact import CONVERGED, FIXED, GRADS, fixed_iterations, rel2, run  # noqa: E402

orc = Library(os.path.join(ROOT, "oracle", "_build", "libheterodyn_oracle.so"))


def measure(scene, frames):
    a = run(orc, scene, frames)
    b = run(orc, scene, frames, perturb=1e-15)
    rec = {"q": [rel2(b[0][f][0], a[0][f][0]) for f in range(frames)],
           "v": [rel2(b[0][f][1], a[0][f][1]) for f in range(frames)],
           "iterations": [int(a[0][f][2]) for f in range(frames)],
           "iterations_perturbed": [int(b[0][f][2]) for f in range(frames)]}
    for k in GRADS:
        rec[k] = rel2(b[2][k], a[2][k])
    return rec


out = {}
for name, (scene, frames, k) in FIXED.items():
    out["fixed/" + name] = measure(fixed_iterations(scene, k), frames)
    print("fixed/" + name, json.dumps(out["fixed/" + name]), flush=True)
for name, (scene, frames) in CONVERGED.items():
    out["converged/" + name] = measure(scene, frames)
    print("converged/" + name, json.dumps(out["converged/" + name]), flush=True)
with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "contact_conditioning.json"), "w") as f:
    json.dump(out, f, indent=1)
