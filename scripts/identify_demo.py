"""hd_run_identify on a C1-sized scene (device engine): wall time per
evaluation (refactorization + frames forward + adjoint chain)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_14526_b200 import scenes  # noqa: E402
from paper_2605_14526_b200.hd import Library  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = Library(os.path.join(ROOT, "paper_2605_14526_b200", "_lib", "libheterodyn_b200.so"))
for tag, frames in (("C1", 20), ("C2", 10)):
    scene = dict(scenes.config_scene(tag))
    scene["frames"] = frames
    problem = {"scene": scene, "design": {"variable": "young", "initial": 4e4}, "true": 6e4,
               "loss": {"kind": "trajectory"}, "optimizer": {"max_evals": 12, "grad_tol": 1e-14}}
    t = time.perf_counter()
    r, stalled = lib.run_identify(problem)
    dt = time.perf_counter() - t
    print(f"{tag}: {frames} frames, {r['evaluations']} evaluations in {dt:.2f} s "
          f"({1e3 * dt / r['evaluations']:.0f} ms each), recovered {r['recovered'][0]:.6g} "
          f"(true 6e4, rel err {r['rel_errors'][0]:.2e}), factorizations {r['factorizations']}")
