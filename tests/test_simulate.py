"""Simulate driver (hd_run_simulate; reference drivers.cpp:238-365): the
summary JSON and the trajectory.jsonl / metrics.csv / summary.json bundle,
host logic over the public ABI shared by both libraries (csrc/drivers.cpp).
CPU: the reference's own test (test_capi.cpp:194-238) through the oracle, and
the region displacement ratio against an independent numpy Kabsch fit.  The
device path is test_gpu_parity.py::test_simulate_matches_oracle.  CPU only."""
import json

import numpy as np


def test_simulate_writes_a_parsable_bundle(orc, tmp_path):
    """test_capi.cpp:194-238, case for case."""
    d = tmp_path / "simulate"
    s = orc.builtin("two-tet").run_simulate(str(d))
    assert s["frames"] == 3 and s["all_converged"] and len(s["iterations"]) == 3 and s["refactorizations"] >= 1
    lines = [json.loads(l) for l in open(d / "trajectory.jsonl") if l.strip()]
    assert len(lines) == 3
    for rec in lines:
        assert {"time", "iterations", "converged", "contact_count"} <= set(rec)
        assert len(rec["q"]) == 15 and len(rec["v"]) == 15
    rows = [l for l in open(d / "metrics.csv").read().splitlines() if l]
    assert len(rows) == 4 and rows[0].startswith("frame,time,iterations")
    assert json.load(open(d / "summary.json"))["frames"] == 3


def kabsch_residual(verts, rest, q):
    r = rest[verts] - rest[verts].mean(0)
    x = q[verts] - q[verts].mean(0)
    u, _, vt = np.linalg.svd(r.T @ x)
    rot = vt.T @ u.T
    if np.linalg.det(rot) < 0:
        vt[2] *= -1
        rot = vt.T @ u.T
    return np.linalg.norm(x - r @ rot.T, axis=1).max()


def test_displacement_ratio_matches_numpy_kabsch(orc, tmp_path):
    """displacement_ratio = softest / stiffest region's worst rigid-fit
    residual over the run (drivers.cpp:250-290, 115-145)."""
    sc = orc.builtin("cantilever3")
    s = sc.run_simulate(str(tmp_path))
    region, young, el = sc.regions(), sc.young_moduli(), sc.elements()
    rest = sc.rest_positions().reshape(-1, 3)
    means = np.array([young[region == r].mean() for r in range(sc.region_count)])
    soft = [r for r in range(sc.region_count) if means[r] <= means.min() * (1 + 1e-9)]
    stiff = [r for r in range(sc.region_count) if means[r] >= means.max() * (1 - 1e-9)]
    verts = {r: np.unique(el[region == r].ravel()) for r in range(sc.region_count)}
    sd = td = 0.0
    for line in open(tmp_path / "trajectory.jsonl"):
        q = np.array(json.loads(line)["q"]).reshape(-1, 3)
        sd = max([sd] + [kabsch_residual(verts[r], rest, q) for r in soft])
        td = max([td] + [kabsch_residual(verts[r], rest, q) for r in stiff])
    assert abs(s["displacement_ratio"] - sd / td) <= 1e-9 * sd / td


def test_penetration_and_contact_metrics(orc, tmp_path):
    """max_penetration and the per-frame FB residual of a contact scene."""
    sc = orc.builtin("ball-drop")
    s = sc.run_simulate(str(tmp_path))
    m = np.loadtxt(tmp_path / "metrics.csv", delimiter=",", skiprows=1)
    assert m.shape == (sc.frame_count, 7)
    assert np.isclose(s["max_penetration"], m[:, 6].max(), rtol=1e-5, atol=0)
    assert (m[:, 4] > 0).any() and m[:, 5].max() < 1e-6
