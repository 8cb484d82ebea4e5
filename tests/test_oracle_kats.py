"""Pins the CPU oracle (oracle/) against the known answers and property checks
of the reference's own unit tests (/root/reference/proj/tests).  CPU only."""
import ctypes as C

import numpy as np
import pytest

D = C.POINTER(C.c_double)


def arr(*vals):
    a = np.ascontiguousarray(vals if len(vals) > 1 else vals[0], dtype=np.float64)
    return a, a.ctypes.data_as(D)


def colmajor(m):
    return np.ascontiguousarray(np.asarray(m, dtype=np.float64).T.ravel())


BENT = np.array([[1.10, 0.20, -0.10], [0.05, 0.85, 0.15], [-0.20, 0.10, 1.25]])  # test_util.hpp:59-65


def test_lame_kat(oracle_unit):
    """test_material.cpp:10-19"""
    mu, la = C.c_double(), C.c_double()
    assert oracle_unit.ho_lame(1e6, 0.4, C.byref(mu), C.byref(la)) == 0
    assert mu.value == pytest.approx(357142.85714285716, rel=1e-13)
    assert la.value == pytest.approx(1428571.4285714286, rel=1e-13)
    assert oracle_unit.ho_lame(2e5, 0.0, C.byref(mu), C.byref(la)) == 0
    assert mu.value == pytest.approx(1e5, rel=1e-13) and la.value == 0.0


@pytest.mark.parametrize("bad", [0.5, 0.7, -1.0, -1.2])
def test_poisson_rejected(oracle_unit, bad):
    """test_material.cpp:21-32: InvalidPoisson (4)."""
    mu, la = C.c_double(), C.c_double()
    assert oracle_unit.ho_lame(1e6, bad, C.byref(mu), C.byref(la)) == 4


def test_nh_energy_kat(oracle_unit):
    """test_material.cpp:34-43"""
    out = C.c_double()
    f, fp = arr(colmajor(2 * np.eye(3)))
    assert oracle_unit.ho_nh_energy(fp, 1.0, 0.0, C.byref(out)) == 0
    assert out.value == pytest.approx(2.4205584583201643, rel=1e-14)
    assert oracle_unit.ho_nh_energy(fp, 0.0, 2.0, C.byref(out)) == 0
    assert out.value == pytest.approx(4.324077125263812, rel=1e-14)
    i, ip = arr(colmajor(np.eye(3)))
    assert oracle_unit.ho_nh_energy(ip, 3.0, 7.0, C.byref(out)) == 0
    assert abs(out.value) < 1e-15


def test_min_eigen_kat(oracle_unit):
    """test_localstep.cpp:122-130: lambda_min(H((2,2,2); 1, 4))."""
    s, sp = arr(2.0, 2.0, 2.0)
    o, op = arr(np.zeros(3))
    assert oracle_unit.ho_stretch_hessian_eigs(sp, 1.0, 4.0, op) == 0
    assert o.min() == pytest.approx(-0.8294415416798357, abs=1e-12)


def test_prox_means_volume_weighted(oracle_unit):
    """test_material.cpp:100-113: means 2e5 / 2e5."""
    from paper_2605_14526_b200 import scenes
    import json
    sc = scenes.two_tets_unequal(young=(3e5, 6e5), poisson=0.25)
    o, op = arr(np.zeros(3))
    assert oracle_unit.ho_prox_means(json.dumps(sc).encode(), op) == 0
    assert o[0] == pytest.approx(2e5, rel=1e-12)
    assert o[1] == pytest.approx(2e5, rel=1e-12)
    assert o[2] == pytest.approx(2 * o[0] + o[1], rel=1e-13)


@pytest.mark.parametrize("f", [BENT, np.diag([1.3, 0.7, 1.1]), np.diag([1.0, 1.0, -1.0]) @ BENT,
                               np.array([[0.2, 1.1, 0.0], [-1.0, 0.3, 0.4], [0.1, 0.0, 0.9]])])
def test_signed_svd(oracle_unit, f):
    """test_localstep.cpp:62-81: reconstruction 1e-12, proper rotations, ordering, sign fold."""
    fa, fp = arr(colmajor(f))
    u, up = arr(np.zeros(9))
    s, sp = arr(np.zeros(3))
    v, vp = arr(np.zeros(9))
    assert oracle_unit.ho_signed_svd(fp, up, sp, vp) == 0
    U, V = u.reshape(3, 3).T, v.reshape(3, 3).T
    assert np.abs(U @ np.diag(s) @ V.T - f).max() <= 1e-12
    assert np.linalg.det(U) == pytest.approx(1.0, abs=1e-10)
    assert np.linalg.det(V) == pytest.approx(1.0, abs=1e-10)
    assert np.abs(U.T @ U - np.eye(3)).max() <= 1e-12
    assert s[0] >= s[1] >= abs(s[2])
    assert (s[2] < 0) == (np.linalg.det(f) < 0)


def test_nh_prox_stationarity(oracle_unit):
    """test_localstep.cpp:174-189: |k(s*-sf) + grad psi(s*)| <= 1.001e-10 k."""
    mu, la = 2.0e4, 8.0e4
    k = 2 * mu + la
    f, fp = arr(colmajor(BENT))
    p, pp = arr(np.zeros(9))
    ss, ssp = arr(np.zeros(3))
    sf, sfp = arr(np.zeros(3))
    assert oracle_unit.ho_project(0, fp, mu, la, k, pp, ssp, sfp) == 0
    L = np.log(ss.prod())
    grad = mu * (ss - 1 / ss) + la * L / ss
    assert np.abs(k * (ss - sf) + grad).max() <= 1.001e-10 * k
    assert ss.min() > 0


def test_volume_projection_unit_det(oracle_unit):
    """test_localstep.cpp:156-172"""
    f, fp = arr(colmajor(BENT))
    p, pp = arr(np.zeros(9))
    ss, ssp = arr(np.zeros(3))
    sf, sfp = arr(np.zeros(3))
    assert oracle_unit.ho_project(1, fp, 0, 0, 0, pp, ssp, sfp) == 0
    assert np.linalg.det(p.reshape(3, 3).T) == pytest.approx(1.0, abs=1e-10)
    assert ss.prod() == pytest.approx(1.0, abs=1e-10)


def test_rest_is_fixed_by_every_projection(oracle_unit):
    """test_localstep.cpp:191-202"""
    f, fp = arr(colmajor(np.eye(3)))
    p, pp = arr(np.zeros(9))
    ss, ssp = arr(np.zeros(3))
    sf, sfp = arr(np.zeros(3))
    for kind in (0, 1, 3):
        assert oracle_unit.ho_project(kind, fp, 1e4, 4e4, 6e4, pp, ssp, sfp) == 0
        assert np.abs(p.reshape(3, 3).T - np.eye(3)).max() <= 1e-12


@pytest.mark.parametrize("kind", [0, 1, 2, 3])
def test_differential_fd_and_symmetry(oracle_unit, kind):
    """test_localstep.cpp:284-331: differential vs FD (2e-5), 9x9 symmetric."""
    mu, la = 1.0e4, 3.0e4
    k = 2 * mu + la
    f, fp = arr(colmajor(BENT))
    d9, dp = arr(np.zeros(81))
    assert oracle_unit.ho_prox_differential(kind, fp, mu, la, k, 1.0, dp) == 0
    Dm = d9.reshape(9, 9).T  # column-major storage
    if kind != 0:  # NH with tau = 1 filters the Hessian; compare unfiltered below
        assert np.abs(Dm - Dm.T).max() <= 1e-12 * max(1.0, np.abs(Dm).max())
    d0, dp0 = arr(np.zeros(81))
    assert oracle_unit.ho_prox_differential(kind, fp, mu, la, k, 0.0, dp0) == 0
    D0 = d0.reshape(9, 9).T
    eps = 1e-6
    p, pp = arr(np.zeros(9))
    q, qp = arr(np.zeros(9))
    s1, s1p = arr(np.zeros(3))
    s2, s2p = arr(np.zeros(3))
    for c in range(9):
        fplus = colmajor(BENT).copy()
        fplus[c] += eps
        fminus = colmajor(BENT).copy()
        fminus[c] -= eps
        a, ap = arr(fplus)
        b, bp = arr(fminus)
        assert oracle_unit.ho_project(kind, ap, mu, la, k, pp, s1p, s2p) == 0
        assert oracle_unit.ho_project(kind, bp, mu, la, k, qp, s1p, s2p) == 0
        fd = (p - q) / (2 * eps)
        assert np.abs(fd - D0[:, c]).max() <= 2e-5 * max(1.0, np.abs(D0).max())


def test_tr_blend_clamp_and_reflect(oracle_unit):
    """test_localstep.cpp:253-282: tau 1/2 clamps, tau 1 reflects negative eigenvalues."""
    s, sp = arr(2.0, 2.0, 2.0)
    h, hp = arr(np.zeros(9))
    mu, la, k = 1.0, 4.0, 0.5
    w, wp = arr(np.zeros(3))
    assert oracle_unit.ho_stretch_hessian_eigs(sp, mu, la, wp) == 0
    kap = w + k
    assert oracle_unit.ho_tr_blend(sp, mu, la, k, 0.5, hp) == 0
    assert np.linalg.eigvalsh(h.reshape(3, 3)).min() >= -1e-12 * np.abs(h).max()
    assert np.allclose(np.sort(np.linalg.eigvalsh(h.reshape(3, 3))), np.sort(np.maximum(kap, 0)), atol=1e-10)
    assert oracle_unit.ho_tr_blend(sp, mu, la, k, 1.0, hp) == 0
    assert np.allclose(np.sort(np.linalg.eigvalsh(h.reshape(3, 3))), np.sort(np.abs(kap)), atol=1e-10)


def test_contact_scalar_update_kat(oracle_unit):
    """test_contact.cpp:273-305"""
    out = C.c_double()
    m = 0.8 * 2.5 * 0.8 + 0.15
    step = (0.6 - 0.8 * 0.25) / (m + 1e-10 * m)
    assert oracle_unit.ho_contact_scalar(2.5, 0.8, 0.15, 0.6, 0.25, 0.1, C.byref(out)) == 0
    assert out.value == pytest.approx(0.1 + step, rel=1e-12)
    assert oracle_unit.ho_contact_scalar(2.5, 0.8, 0.15, -5.0, 0.25, 0.1, C.byref(out)) == 0
    assert out.value == 0.0


def test_cone_projection_kat(oracle_unit):
    """test_contact.cpp:151-173: ||(3,4)|| > 0.5*2 -> (0.6, 0.8); negative normal -> 0."""
    lin, lp = arr(2.0, 3.0, 4.0)
    lout, lop = arr(np.zeros(3))
    assert oracle_unit.ho_cone_project(0.5, lp, lop) == 0
    assert lout[1] == pytest.approx(0.6, rel=1e-14) and lout[2] == pytest.approx(0.8, rel=1e-14)
    lin2, lp2 = arr(-3.0, 3.0, 4.0)
    assert oracle_unit.ho_cone_project(0.5, lp2, lop) == 0
    assert tuple(lout) == (0.0, 0.0, 0.0)
    lin3, lp3 = arr(2.0, 0.3, 0.4)
    assert oracle_unit.ho_cone_project(0.5, lp3, lop) == 0
    assert lout[1] == pytest.approx(0.3) and lout[2] == pytest.approx(0.4)
