"""System-identification driver (hd_run_identify; reference drivers.cpp:570-979,
lbfgs.cpp:40-143).  The driver (csrc/drivers.cpp) is host logic over the
public ABI, linked into both libraries: on CPU it is checked through the
oracle against the reference's own test (test_capi.cpp:241-284) and the
other design variables by inverse-crime recovery; the product's problem
validation (host only, before any device work) is checked here too.  The
device path against the oracle is in test_gpu_parity.py.  CPU only."""
import json
import os

import numpy as np
import pytest

from paper_2605_14526_b200.hd import HdError

TWO_TET = {"mesh": {"generator": "two-tet"}}


def test_identify_recovers_uniform_initial_velocity(orc, tmp_path):
    """test_capi.cpp:241-284, case for case."""
    problem = {"scene": TWO_TET, "design": {"variable": "v0", "initial": [0, 0, 0]}, "true": [0.3, -0.1, 0.2],
               "loss": {"kind": "trajectory"}, "optimizer": {"max_evals": 60, "grad_tol": 1e-12}}
    out = tmp_path / "identify"
    r, stalled = orc.run_identify(problem, str(out))
    assert not stalled
    assert r["variable"] == "v0"
    assert np.max(np.abs(np.array(r["recovered"]) - [0.3, -0.1, 0.2])) <= 1e-5
    assert r["converged"]
    assert r["factorizations"] == 1 and r["material_updates"] == 1  # the design never touches the material
    assert r["evaluations"] <= 60
    assert json.load(open(out / "result.json"))["variable"] == "v0"
    rows = open(out / "loss_curve.csv").read().splitlines()
    assert rows[0] == "evaluation,loss,best_so_far" and len(rows) == r["evaluations"] + 1
    with pytest.raises(HdError) as e:
        orc.run_identify("{ nope")
    assert e.value.code == 1


@pytest.mark.parametrize("design,initial,truth,loss", [
    ("young", 3e5, 1e6, {"kind": "final_pose"}),
    ("young_regions", [5e5, 5e5], [1e6, 2e5], {"kind": "trajectory"}),
    ("orientation", [0, 0, 0], [0.1, -0.2, 0.05], {"kind": "trajectory"}),
])
def test_identify_recovers_design_variables(orc, design, initial, truth, loss):
    """Inverse crime on every design variable (drivers.cpp:710-803): the
    adjoint gradients drive L-BFGS back to the generating parameters."""
    problem = {"scene": TWO_TET, "design": {"variable": design, "initial": initial}, "true": truth, "loss": loss,
               "optimizer": {"max_evals": 60, "grad_tol": 1e-14}}
    r, stalled = orc.run_identify(problem)
    assert r["converged"] and not stalled, r
    assert max(r["rel_errors"]) <= 1e-6, r
    material = design.startswith("young")
    # a material design refactors on every evaluation (material.cpp:75-86 bumps the version)
    assert r["factorizations"] == (r["evaluations"] if material else 1)
    assert r["material_updates"] == (r["evaluations"] if material else 1)


def test_identify_target_com(orc):
    """LossKind::TargetCom at an intermediate frame (drivers.cpp:888-905):
    the centre of mass of frame 2 reaches the target."""
    target = [0.3, 0.2, 0.1]
    problem = {"scene": TWO_TET, "design": {"variable": "v0", "initial": [0, 0, 0]},
               "loss": {"kind": "target_com", "target": target, "frame": 2},
               "optimizer": {"max_evals": 60, "grad_tol": 1e-12}}
    r, _ = orc.run_identify(problem)
    assert r["converged"] and r["loss"] <= 1e-20
    assert "true" not in r and "rel_errors" not in r
    sc = orc.builtin("two-tet")
    sim = sc.sim()
    sim.set_state(v=np.tile(r["recovered"], sc.vertex_count))
    sim.step(2)
    m = sc.vertex_masses()
    com = (m[:, None] * sim.positions().reshape(-1, 3)).sum(0) / m.sum()
    assert np.allclose(com, target, atol=1e-9)


@pytest.mark.parametrize("lib", ["orc", "prod"])
def test_identify_problem_validation(lib, request, tmp_path):
    """parse_identify_problem (drivers.cpp:570-708): parse errors, the
    validation list, and file I/O errors surface with the reference's codes.
    Nothing here reaches the device, so the product is checked on CPU too."""
    L = request.getfixturevalue(lib)
    cases = [
        ({"design": {"variable": "v0", "initial": [0, 0, 0]}, "true": [0, 0, 0]}, 2, "expected \"scene\""),
        ({"scene": TWO_TET, "design": {"variable": "mass", "initial": 1}, "true": 1}, 2, "design.variable"),
        ({"scene": TWO_TET, "design": {"variable": "young", "initial": -1}, "true": 1}, 2, "positive modulus"),
        ({"scene": TWO_TET, "design": {"variable": "young_regions", "initial": [1e5]}, "true": [1e5]}, 2,
         "one modulus per region (2)"),
        ({"scene": TWO_TET, "design": {"variable": "v0", "initial": [0, 0]}, "true": [0, 0]}, 2, "3-vector"),
        ({"scene": TWO_TET, "design": {"variable": "v0", "initial": [0, 0, 0]}}, 2, "true: required"),
        ({"scene": TWO_TET, "design": {"variable": "v0", "initial": [0, 0, 0]}, "loss": {"kind": "target_com"}},
         2, "loss.target: required"),
        ({"scene": TWO_TET, "design": {"variable": "v0", "initial": [0, 0, 0]}, "true": [0, 0, 0],
          "loss": {"frame": 99}}, 2, "loss.frame: out of range"),
        ({"scene": TWO_TET, "design": {"variable": "v0", "initial": [0, 0, 0]}, "true": [0, 0, 0],
          "loss": {"kind": "energy"}}, 2, "loss.kind"),
    ]
    for problem, code, needle in cases:
        with pytest.raises(HdError) as e:
            L.run_identify(problem)
        assert e.value.code == code and needle in str(e.value), (problem, str(e.value))
    with pytest.raises(HdError) as e:
        L.run_identify("{ nope")
    assert e.value.code == 1
    with pytest.raises(HdError) as e:
        L.run_identify_file(str(tmp_path / "missing.json"))
    assert e.value.code == 12
    bad = tmp_path / "bad.json"
    bad.write_text(json.dumps({"scene_file": str(tmp_path / "none.json"), "design": {"variable": "v0"}}))
    with pytest.raises(HdError) as e:
        L.run_identify_file(str(bad))
    assert e.value.code == 12  # the scene file is missing


def test_scene_data_accessors_agree(orc, prod):
    """hd_scene_regions / rest positions / vertex masses: both libraries
    build the same scene data from the same JSON."""
    for name in ("two-tet", "cantilever3"):
        a, b = orc.builtin(name), prod.builtin(name)
        assert a.region_count == b.region_count
        assert np.array_equal(a.regions(), b.regions())
        assert np.array_equal(a.rest_positions(), b.rest_positions())
        assert np.allclose(a.vertex_masses(), b.vertex_masses(), rtol=1e-14, atol=0)


def test_scene_and_problem_files(orc, prod, tmp_path):
    """hd_scene_load and hd_run_identify_file read real files inside a Python
    process (stdio readers; the libraries carry their own libstdc++)."""
    scene_path = tmp_path / "scene.json"
    scene_path.write_text(json.dumps(TWO_TET))
    for L in (orc, prod):
        sc = L.load(str(scene_path))
        assert (sc.vertex_count, sc.element_count) == (5, 2)
    problem = {"scene_file": str(scene_path), "design": {"variable": "v0", "initial": [0, 0, 0]},
               "true": [0.1, 0.0, 0.0], "optimizer": {"max_evals": 40, "grad_tol": 1e-12}}
    path = tmp_path / "problem.json"
    path.write_text(json.dumps(problem))
    r, stalled = orc.run_identify_file(str(path), str(tmp_path / "out" / "nested"))
    assert r["converged"] and not stalled
    assert abs(r["recovered"][0] - 0.1) <= 1e-8
    assert (tmp_path / "out" / "nested" / "result.json").exists()
