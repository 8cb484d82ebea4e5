"""Finite-difference gradient-check driver (hd_run_gradcheck; reference
drivers.cpp:367-531, capi.cpp:260-277), host logic over the public ABI
linked into both libraries (csrc/drivers.cpp).  CPU: the reference's own
test through the oracle (test_capi.cpp:157-192), the f_ext setter, and the
product's host-side argument checks.  The device path against the oracle is
test_gpu_parity.py::test_gradcheck_matches_oracle.  CPU only."""
import json

import numpy as np
import pytest

from paper_2605_14526_b200 import scenes
from paper_2605_14526_b200.hd import HdError, _ptr


def test_gradcheck_passes_on_the_smallest_scene(orc, tmp_path):
    """test_capi.cpp:157-183, case for case."""
    out = tmp_path / "gradcheck" / "report.json"
    rep, ok = orc.builtin("two-tet").run_gradcheck("q0,v0", str(out))
    assert ok and rep["pass"]
    assert rep["fd_check"]["max_rel_err"] <= 2e-3
    assert rep["vars"] == ["q0", "v0"]
    assert json.load(open(out))["pass"]
    assert len(rep["tau"]) == len(rep["rho"]) == len(rep["iterations"]) == 3


def test_gradcheck_all_variables(orc):
    """Every variable, default list (capi.cpp:269) and "w" (norm only)."""
    sc = orc.scene(scenes.block_scene(dims=(3, 2, 2), kind="corotated", fix_x0_face=True, frames=2))
    rep, ok = sc.run_gradcheck()
    assert rep["vars"] == ["q0", "v0", "f_ext", "E"] and ok
    assert set(rep["fd_check"]["per_var_max_rel_err"]) == {"q0", "v0", "f_ext", "E"}
    rep, ok = orc.builtin("two-tet").run_gradcheck("w, E")
    assert rep["vars"] == ["w", "E"] and "w" in rep["grad_norms"] and ok
    assert "w" not in rep["fd_check"]["per_var_max_rel_err"]


@pytest.mark.parametrize("lib", ["orc", "prod"])
def test_gradcheck_rejects_unknown_variables(lib, request):
    """run_gradcheck raises ErrorCode::InvalidArgument for an unknown name
    (drivers.cpp:370-376; the reference test at test_capi.cpp:187-189 expects
    Validation, which its own code does not return — we follow the code).
    Checked before any device work, so the product is covered on CPU."""
    L = request.getfixturevalue(lib)
    with pytest.raises(HdError) as e:
        L.builtin("two-tet").run_gradcheck("q0,bogus")
    assert e.value.code == 13 and "bogus" in str(e.value)


def test_external_force_roundtrip(orc):
    """hd_sim_external_force / hd_sim_set_external_force: the sim starts from
    the scene's gravity + point forces and steps with a replaced f_ext."""
    sc = orc.builtin("two-tet")
    sim = sc.sim()
    f0 = sim.external_force()
    assert f0.shape == (3 * sc.vertex_count,) and np.linalg.norm(f0) > 0
    sim.set_external_force(2.0 * f0)
    np.testing.assert_array_equal(sim.external_force(), 2.0 * f0)
    bad = np.zeros(3)
    assert orc.lib.hd_sim_set_external_force(sim.h, _ptr(bad), 3) == 13
