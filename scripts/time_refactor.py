"""Refactorization time (hd_sim_set_young) for C2 and C3: the device path
(assembly + multifrontal LDL^T + S' values on the GPU) against the host path
(HETERODYN_HOST_REFACTOR=1: host assembly and up-looking LDL^T, S' values on
the device), and for the C5 lockstep batch (64 C2 samples in one engine).
Wall time per set_young after one warm-up refactorization (profiling)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_14526_b200 import scenes  # noqa: E402
from paper_2605_14526_b200.hd import Library  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = Library(os.path.join(ROOT, "paper_2605_14526_b200", "_lib", "libheterodyn_b200.so"))
for tag in ("C2", "C3"):
    for host in ("0", "1"):
        os.environ["HETERODYN_HOST_REFACTOR"] = host
        sc = lib.scene(scenes.config_scene(tag))
        sim = sc.sim()
        young = np.full(sc.element_count, 2e5)
        sim.set_young(young)
        t0 = time.perf_counter()
        for k in range(3):
            sim.set_young(young * (1.1 + 0.1 * k))
        dt = (time.perf_counter() - t0) / 3
        print(f"{tag} set_young ({'host' if host == '1' else 'device'} refactorization): {1e3 * dt:.1f} ms", flush=True)
os.environ["HETERODYN_HOST_REFACTOR"] = "0"
sc = lib.scene(scenes.config_scene("C2"))
young = scenes.c5_young(64, sc.element_count)
b = sc.batch(64, young, threads=32)
b.set_young(young * 1.01)
t0 = time.perf_counter()
for k in range(3):
    b.set_young(young * (1.02 + 0.01 * k))
print(f"C5 lockstep batch (64 x C2) set_young: {1e3 * (time.perf_counter() - t0) / 3:.1f} ms", flush=True)
