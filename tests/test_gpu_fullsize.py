"""Parity at the configurations' real sizes (SURVEY.md §8 configs C1, C3, C4,
C5), product against the CPU oracle through the hd_* C ABI.

* C1 — 5,184-tet corotated cantilever, x = 0 face pinned: 3 frames at
  eps_rel = 1e-12, q / v per frame and all five gradients.  Corotated
  gradients depend on the SVD basis at (near-)repeated singular values through
  the ProxDifferential floors (localstep.cpp:305-357), so each gradient's bar
  is max(1e-6, 10 x the oracle's own change under a 1e-15 perturbation of q0),
  measured here.
* C3 — 103,680-tet 100x-contrast Neo-Hookean crab, default tolerance: 3
  frames, identical forward iteration counts and tau per frame, q / v and the
  gradients to a flat 1e-6.
* C5 — batched system-ID at C2 size (29,952 tets): 4 parameter samples
  E_s = 1e5 exp(0.5 z_s), 3 frames each; per-sample losses and the
  sample-ordered dL/dE sum to 1e-6.
* C4 — full 40 x 24 x 18 gripper pad with frictional contact, 3 frames at
  eps_rel = 1e-12: the oracle needs hours for it, so its outputs are the
  committed fixture tests/golden/c4_full.npz (tests/golden/make_c4_full.py);
  contact rows exact, decisions exact outside round-off ties, q / v / gradients
  within max(1e-6, 10 x the oracle's conditioning)."""
import json
import os

import numpy as np
import pytest

from paper_2605_14526_b200 import scenes

pytestmark = pytest.mark.gpu

GRADS = ("dl_dq0", "dl_dv0", "dl_df_ext", "dl_de", "dl_dw")
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def rel2(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def run(lib, scene, frames, perturb=0.0):
    sim = lib.scene(scene).sim()
    if perturb:
        q = sim.positions()
        sim.set_state(q + perturb * np.abs(q).max() * np.sin(np.arange(q.size)), sim.velocities(), 0.0)
    sim.record(True)
    traj, traces = [], []
    for _ in range(frames):
        sim.step()
        traj.append((sim.positions(), sim.velocities(), sim.last_iterations, sim.last_converged))
        traces.append(sim.contact_trace())
    g = sim.backward(dl_dq_final=traj[-1][0], dl_dv_final=traj[-1][1])
    return traj, traces, g


def test_c1_full_size(prod, orc):
    scene = scenes.config_scene("C1", frames=3, solver={"eps_rel": 1e-12, "eps_abs": 1e-14})
    tp, _, gp = run(prod, scene, 3)
    to, _, go = run(orc, scene, 3)
    ts, _, gs = run(orc, scene, 3, perturb=1e-15)
    for f, ((qp, vp, ip, cp), (qo, vo, io, co), (qs, vs, _, _)) in enumerate(zip(tp, to, ts)):
        assert cp == co, (f, cp, co)
        assert rel2(qp, qo) <= max(1e-6, 10 * rel2(qs, qo)), (f, rel2(qp, qo))
        assert rel2(vp, vo) <= max(1e-6, 10 * rel2(vs, vo)), (f, rel2(vp, vo))
    np.testing.assert_array_equal(gp["tau"], go["tau"])
    for k in GRADS:
        bar = max(1e-6, 10 * rel2(gs[k], go[k]))
        assert rel2(gp[k], go[k]) <= bar, (k, rel2(gp[k], go[k]), bar)


def test_c3_full_size_three_frames(prod, orc):
    scene = scenes.config_scene("C3", frames=3)
    tp, _, gp = run(prod, scene, 3)
    to, _, go = run(orc, scene, 3)
    for f, ((qp, vp, ip, cp), (qo, vo, io, co)) in enumerate(zip(tp, to)):
        assert ip == io and cp == co, (f, ip, io)  # default tolerance: iteration counts agree exactly
        assert rel2(qp, qo) <= 1e-6 and rel2(vp, vo) <= 1e-6, (f, rel2(qp, qo), rel2(vp, vo))
    np.testing.assert_array_equal(gp["tau"], go["tau"])
    for k in GRADS:
        assert rel2(gp[k], go[k]) <= 1e-6, (k, rel2(gp[k], go[k]))


def test_c5_four_samples_at_c2_size(prod, orc):
    scene = scenes.config_scene("C2", frames=3)
    sp, so = prod.scene(scene), orc.scene(scene)
    ne = sp.element_count
    young = scenes.c5_young(4, ne)
    ref = so.sim()
    ref.step(3)
    target = ref.positions()
    bo = so.batch(4, young)
    bo.set_target(target)
    ro = bo.evaluate(3)
    bp = sp.batch(4, young, threads=4)
    bp.set_target(target)
    rp = bp.evaluate(3)
    assert rel2(rp["loss"], ro["loss"]) <= 1e-6, rel2(rp["loss"], ro["loss"])
    assert rel2(rp["dl_de"], ro["dl_de"]) <= 1e-6, rel2(rp["dl_de"], ro["dl_de"])


C4_FIXTURE = os.path.join(GOLDEN, "c4_full.npz")


@pytest.mark.skipif(not os.path.exists(C4_FIXTURE), reason="tests/golden/c4_full.npz not generated yet")
def test_c4_full_size_against_committed_oracle_run(prod):
    import sys
    sys.path.insert(0, GOLDEN)
    from make_c4_full import FRAMES, c4_full_scene, decisions
    gold = np.load(C4_FIXTURE)
    with open(os.path.join(GOLDEN, "contact_conditioning.json")) as f:
        cond = json.load(f)["converged/C4-full"]
    bar = lambda c: max(1e-6, 10 * c)  # noqa: E731
    tp, trp, gp = run(prod, c4_full_scene(), FRAMES)
    for f in range(FRAMES):
        np.testing.assert_array_equal(trp[f]["vertex"], gold[f"vertex{f}"], err_msg=f"frame {f} contact vertices")
        np.testing.assert_array_equal(trp[f]["obstacle"], gold[f"obstacle{f}"], err_msg=f"frame {f} obstacles")
        dc, dk = decisions(trp[f])
        gc, gk = gold[f"clamp{f}"], gold[f"cone{f}"]
        n = min(dc.shape[0], gc.shape[0])
        sure = lambda a, b: (a != 0) & (b != 0)  # noqa: E731  round-off ties (0) exempt
        assert np.array_equal(dc[:n][sure(dc[:n], gc[:n])], gc[:n][sure(dc[:n], gc[:n])]), f"frame {f} clamp"
        assert np.array_equal(dk[:n][sure(dk[:n], gk[:n])], gk[:n][sure(dk[:n], gk[:n])]), f"frame {f} cone"
        qp, vp = tp[f][0], tp[f][1]
        assert rel2(qp, gold[f"q{f}"]) <= bar(cond["q"][f]), (f, rel2(qp, gold[f"q{f}"]))
        assert rel2(vp, gold[f"v{f}"]) <= bar(cond["v"][f]), (f, rel2(vp, gold[f"v{f}"]))
    np.testing.assert_array_equal(gp["tau"], gold["tau"])
    for k in GRADS:
        assert rel2(gp[k], gold[k]) <= bar(cond[k]), (k, rel2(gp[k], gold[k]), cond[k])
