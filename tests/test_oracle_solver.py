"""Solver-level property tests of the CPU oracle through the hd_* ABI,
mirroring the reference's test_forward.cpp / test_backward.cpp /
test_factor.cpp / test_scene.cpp / test_capi.cpp.  CPU only."""
import json

import numpy as np
import pytest

from paper_2605_14526_b200 import scenes


def test_builtin_table(orc):
    """test_scene.cpp:30-47 and test_capi.cpp:37-39."""
    rows = {"two-tet": (5, 2, 3), "cantilever3": (208, 648, 60), "twist-bar": (208, 648, 40),
            "ball-drop": (13, 20, 50), "resting-box": (27, 48, 30), "slab-on-sphere": (162, 384, 60)}
    for name, (nv, ne, fr) in rows.items():
        sc = orc.builtin(name)
        assert (sc.vertex_count, sc.element_count, sc.frame_count) == (nv, ne, fr)
        assert sc.name == name


def test_ballistic_closed_form(orc):
    """test_forward.cpp:284-332: uniform translation under gravity is symplectic Euler."""
    s = scenes.block_scene(alpha=0.0, beta0=0.0, v0_amp=0.0, gravity_z=-2.0, eps_rel=1e-4, eps_abs=1e-9)
    sim = orc.scene(s).sim()
    q0 = sim.positions()
    sim.step(3)
    q, v = sim.positions(), sim.velocities()
    h, g, N = 0.01, -2.0, 3
    np.testing.assert_allclose(q[2::3], q0[2::3] + g * h * h * N * (N + 1) / 2, rtol=1e-10)
    np.testing.assert_allclose(v[2::3], N * h * g, rtol=1e-10)
    np.testing.assert_allclose(q[0::3], q0[0::3], rtol=1e-12, atol=1e-14)
    assert sim.last_converged and sim.last_iterations <= 3


def test_pinned_bitwise(orc):
    """test_forward.cpp:334-359"""
    s = scenes.block_scene(fix_x0_face=True, v0_amp=0.0, gravity_z=-2.0, eps_rel=1e-6, eps_abs=1e-10)
    sim = orc.scene(s).sim()
    q0 = sim.positions()
    sim.step(3)
    q, v = sim.positions(), sim.velocities()
    fixed = [d["vertex"] for d in s["dirichlet"]]
    for vtx in fixed:
        assert np.array_equal(q[3 * vtx:3 * vtx + 3], q0[3 * vtx:3 * vtx + 3])
        assert np.all(v[3 * vtx:3 * vtx + 3] == 0.0)
    assert np.abs(q[2::3] - q0[2::3]).max() > 1e-6


def test_iteration_cap_advances(orc):
    """test_forward.cpp:361-378"""
    s = scenes.block_scene(fix_x0_face=True, v0_amp=0.0, gravity_z=-9.81)
    s["solver"]["k_max"] = 1
    sim = orc.scene(s).sim()
    sim.step()
    assert not sim.last_converged and sim.last_iterations == 1


def test_solve_exact_inverse(orc):
    """test_factor.cpp:57-68 analogue: the explicit inverse factor solves A x = b."""
    s = scenes.block_scene(dims=(3, 2, 2), contrast=10.0, alpha=0.02, beta0=0.1)
    sim = orc.scene(s).sim()
    rng = np.random.default_rng(1000)
    b = rng.standard_normal(sim.n)
    x1 = sim.solve_free(b)
    x2 = sim.solve_free(2 * b)
    np.testing.assert_allclose(x2, 2 * x1, rtol=1e-12, atol=1e-300)


def one_step_loss(orc, scene, q, v, young=None):
    sim = orc.scene(scene).sim()
    if young is not None:
        sim.set_young(young, freeze_means=False)
    sim.set_state(q, v, 0.0)
    sim.step()
    rest = np.asarray(scene_rest(scene))
    qn, vn = sim.positions(), sim.velocities()
    return 0.5 * np.sum((qn - rest) ** 2) + 0.5 * np.sum(vn ** 2)


def scene_rest(scene):
    m = scene["mesh"]
    if "vertices" in m:
        return np.asarray(m["vertices"], dtype=float).ravel()
    g = m["grid"]
    return scenes.grid_vertices(g["dims"], g["spacing"]).ravel()


def test_one_step_gradients_fd(orc):
    """test_backward.cpp:245-332: contact-free one-step gradients vs central FD (1e-4)."""
    sc = scenes.two_tets_unequal(alpha=0.01, beta0=0.05)
    rest = scene_rest(sc)
    n = rest.size
    q_t = rest + 0.01 * np.sin(0.7 * np.arange(n) + 0.2)
    v_t = 0.2 * np.sin(0.7 * np.arange(n) + 1.0)
    sc["gravity"] = [0.0, 0.0, -2.0]
    sim = orc.scene(sc).sim()
    sim.set_state(q_t, v_t, 0.0)
    sim.record(True)
    sim.step()
    q1, v1 = sim.positions(), sim.velocities()
    g = sim.backward(dl_dq_final=q1 - rest, dl_dv_final=v1)
    eps = 1e-6
    for i in (0, 5, 14):
        for key, base in (("dl_dq0", "q"), ("dl_dv0", "v")):
            qp, qm, vp, vm = q_t.copy(), q_t.copy(), v_t.copy(), v_t.copy()
            if base == "q":
                qp[i] += eps
                qm[i] -= eps
            else:
                vp[i] += eps
                vm[i] -= eps
            fd = (one_step_loss(orc, sc, qp, vp) - one_step_loss(orc, sc, qm, vm)) / (2 * eps)
            an = g[key][i]
            assert abs(fd - an) <= 1e-4 * max(abs(fd), abs(an), 1e-6), (key, i, fd, an)
    young = np.array([4e4, 9e4])
    for e in range(2):
        yp, ym = young.copy(), young.copy()
        yp[e] *= 1 + 1e-6
        ym[e] *= 1 - 1e-6
        fd = (one_step_loss(orc, sc, q_t, v_t, yp) - one_step_loss(orc, sc, q_t, v_t, ym)) / (2e-6 * young[e])
        an = g["dl_de"][e]
        assert abs(fd - an) <= 1e-4 * max(abs(fd), abs(an), 1e-10), (e, fd, an)


def test_zero_seed_zero_gradient(orc):
    """test_backward.cpp:182-221"""
    sim = orc.scene(scenes.block_scene()).sim()
    sim.record(True)
    sim.step()
    g = sim.backward()
    for k in ("dl_dq0", "dl_dv0", "dl_df_ext", "dl_de"):
        assert np.linalg.norm(g[k]) == 0.0


def test_capi_error_surface(orc):
    """test_capi.cpp:28-90: error codes through the C surface."""
    from paper_2605_14526_b200.hd import HdError
    with pytest.raises(HdError) as e:
        orc.builtin("no-such-scene")
    assert e.value.code == 2
    with pytest.raises(HdError) as e:
        orc.scene("{ not json")
    assert e.value.code == 1
    with pytest.raises(HdError) as e:
        orc.load("/nonexistent/path/scene.json")
    assert e.value.code == 12
    sc = orc.scene({"mesh": {"grid": {"dims": [1, 1, 1], "spacing": 0.1}}, "material": {"young": 5e4, "poisson": 0.4},
                    "frames": 2})
    assert (sc.vertex_count, sc.element_count, sc.frame_count) == (8, 6, 2)


def test_batch_objective_matches_finite_differences(orc):
    """The batched system-ID objective (hd_batch_evaluate, config C5): the
    summed dL/dE agrees with central differences of sum_s L_s under a uniform
    relative perturbation of every sample's moduli."""
    import numpy as np
    from paper_2605_14526_b200 import scenes
    sc = orc.scene(scenes.block_scene(dims=(2, 1, 1), frames=2, gravity_z=-9.81))
    ne = sc.element_count
    young = scenes.c5_young(3, ne, base=5e4)
    target = np.asarray(sc.sim().positions()) + 1e-3
    def total(y):
        b = sc.batch(3, y)
        b.set_target(target)
        r = b.evaluate(2)
        return r["loss"].sum(), r
    _, r = total(young)
    eps = 1e-6
    lp, _ = total(young * (1 + eps))
    lm, _ = total(young * (1 - eps))
    fd = (lp - lm) / (2 * eps)
    # d/d(eps) sum_s L_s(E_s (1 + eps)) = sum_s sum_e dL_s/dE_e E_s,e; samples are uniform per row
    an = sum(float(np.dot(bb, yy)) for bb, yy in zip(_per_sample(sc, young, target), young))
    assert abs(fd - an) <= 1e-4 * abs(fd), (fd, an)
    assert np.isfinite(r["dl_de"]).all()


def _per_sample(sc, young, target):
    out = []
    for y in young:
        b = sc.batch(1, y[None, :])
        b.set_target(target)
        out.append(b.evaluate(2)["dl_de"])
    return out
