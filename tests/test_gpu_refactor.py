"""Device refactorization (engine_refactor.cpp,
refactor.cu): a same-pattern hd_sim_set_young re-assembles A, re-factors
LDL^T (multifrontal over the supernodal elimination tree) and rebuilds S' on
the GPU.  Checks:

* bitwise: the device A values equal the host assembly (factor.cpp assemble
  order), and the device fronts' L and D equal the CPU reference of the same
  algorithm (refactor.cpp mf_factor_host) — HETERODYN_MF_VERIFY=1 makes the
  engine compare them after every device refactorization;
* the CPU reference itself agrees with the host up-looking LDL^T to rounding
  (factor_stats "mf_check", CPU test below);
* the refactored sim steps and differentiates like one refactored on the host
  (HETERODYN_HOST_REFACTOR=1) and like the oracle;
* Dirichlet scenes (A_fd / A_df values re-assembled too), corotated, and a
  lockstep batch (the combined block-diagonal factor).
(C1 is left to test_gpu_fullsize.py: at the default tolerance its corotated
gradients move by ~1e-3 under rounding-level changes in every path — device,
host and a fresh build alike, scripts/rfdiag.py.)"""
import numpy as np
import pytest

from paper_2605_14526_b200 import scenes

GRADS = ("dl_dq0", "dl_dv0", "dl_df_ext", "dl_de", "dl_dw")


def rel2(a, b):
    return np.linalg.norm(np.asarray(a) - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("tag", ["C1", "C2"])
def test_multifrontal_reference_matches_host_ldlt(prod, monkeypatch, tag):
    monkeypatch.setenv("HETERODYN_MF_CHECK", "1")
    st = prod.scene(scenes.config_scene(tag)).factor_stats()["mf_check"]
    assert st["lx_max_abs_diff_rel"] <= 1e-13 and st["dis_max_rel_diff"] <= 1e-13, st
    assert st["levels"] < 100 and st["supernodes"] > 0


def run(lib, scene, young, frames=2):
    sim = lib.scene(scene).sim()
    sim.set_young(young)
    sim.record(True)
    sim.step(frames)
    q = sim.positions()
    return q, sim.velocities(), sim.backward(dl_dq_final=q, dl_dv_final=sim.velocities())


CASES = {
    "contrast-damped": scenes.block_scene(dims=(4, 3, 2), contrast=10.0, beta0=0.05, alpha=0.02, frames=2),
    "pinned-corotated": scenes.block_scene(dims=(5, 3, 2), kind="corotated", fix_x0_face=True, frames=2),
    "pinned-contrast-nh": scenes.block_scene(dims=(8, 6, 5), contrast=10.0, fix_x0_face=True, alpha=0.02, beta0=0.02,
                                             frames=2),
}


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(CASES))
def test_device_refactor_bitwise_and_parity(prod, orc, monkeypatch, name):
    scene = CASES[name]
    ne = prod.scene(scene).element_count
    young = 3e4 * (1.0 + 0.5 * np.sin(np.arange(ne)))
    monkeypatch.setenv("HETERODYN_MF_VERIFY", "1")
    qd, vd, gd = run(prod, scene, young)
    monkeypatch.delenv("HETERODYN_MF_VERIFY")
    monkeypatch.setenv("HETERODYN_HOST_REFACTOR", "1")
    qh, vh, gh = run(prod, scene, young)
    monkeypatch.delenv("HETERODYN_HOST_REFACTOR")
    qo, vo, go = run(orc, scene, young)
    assert rel2(qd, qh) <= 1e-12 and rel2(vd, vh) <= 1e-10
    assert rel2(qd, qo) <= 1e-10
    np.testing.assert_array_equal(gd["tau"], go["tau"])
    for k in GRADS:
        if np.linalg.norm(go[k]) > 0:
            assert rel2(gd[k], gh[k]) <= 1e-9, (k, rel2(gd[k], gh[k]))
            assert rel2(gd[k], go[k]) <= 1e-6, (k, rel2(gd[k], go[k]))


@pytest.mark.gpu
def test_lockstep_batch_refactors_on_device(prod, orc, monkeypatch):
    scene = scenes.block_scene(dims=(4, 3, 2), frames=2, gravity_z=-9.81, alpha=0.02, beta0=0.03, v0_amp=0.05)
    sp, so = prod.scene(scene), orc.scene(scene)
    ne = sp.element_count
    young = scenes.c5_young(4, ne, base=5e4)
    target = np.asarray(so.sim().positions()) + 1e-3
    young2 = young * np.linspace(0.7, 1.3, 4)[:, None] * (1 + 0.2 * np.sin(np.arange(ne)))[None, :]
    monkeypatch.setenv("HETERODYN_MF_VERIFY", "1")
    bp = sp.batch(4, young)
    bp.set_target(target)
    bp.set_young(young2)
    rp = bp.evaluate(2)
    bo = so.batch(4, young2)
    bo.set_target(target)
    ro = bo.evaluate(2)
    assert rel2(rp["loss"], ro["loss"]) <= 1e-6
    assert rel2(rp["dl_de"], ro["dl_de"]) <= 1e-6
