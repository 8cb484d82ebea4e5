"""Refactorization time (hd_sim_set_young: host symbolic + numeric LDL^T, S'
values on the device or the host) for C2 and C3 (profiling)."""
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
        os.environ["HETERODYN_HOST_FACTOR_VALUES"] = host
        sc = lib.scene(scenes.config_scene(tag))
        sim = sc.sim()
        young = np.full(sc.element_count, 2e5)
        sim.set_young(young)
        t0 = time.perf_counter()
        for _ in range(3):
            sim.set_young(young * (1.1 + 0.1 * _))
        dt = (time.perf_counter() - t0) / 3
        print(f"{tag} set_young ({'host' if host == '1' else 'device'} S' values): {1e3 * dt:.0f} ms, "
              f"factor stats phases {sc.factor_stats()['factor_phase_millis']}")
