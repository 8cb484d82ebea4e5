"""Procedural scene JSON for the benchmark configurations and the parity tests.

Every scene is a document in the reference's scene schema
(/root/reference/proj/src/scene.cpp:255-680): ``grid`` meshes follow the Kuhn
hex split of ``ingest_hex_grid`` (mesh.cpp:100-140), so per-element fields
(heterogeneous Young's moduli) are addressed in the reference's element
order.  Both the product library and the CPU oracle consume the same bytes.

Configurations (BASELINE.json ``configs``):
  C1  cantilever 36x6x4, corotated, x=0 face pinned             (5,184 tets)
  C2  24x16x13 Neo-Hookean, nu=0.45, wiggle initial velocity    (29,952 tets)
  C3  40x24x18 crab-like Neo-Hookean, 100x stiffness contrast,
      Rayleigh damping, gravity + point pull                     (103,680 tets)
  C4  soft gripper pad: C3-sized Neo-Hookean block (stiff core, soft pad,
      100x contrast) pressed onto a rigid rounded cube edge (sphere
      obstacle, friction 0.5)                                    (103,680 tets)
  C5  batched system-ID: samples of C2 with E_s = 1e5 exp(0.5 z_s),
      z_s ~ N(0, 1) from std::mt19937_64 seed 2605            (c5_young)
"""
from __future__ import annotations

import json
import math

import numpy as np

KUHN = ((0, 1, 3, 7), (0, 3, 2, 7), (0, 2, 6, 7), (0, 6, 4, 7), (0, 4, 5, 7), (0, 5, 1, 7))


def grid_vertices(dims, spacing):
    nx, ny, nz = dims
    k, j, i = np.meshgrid(np.arange(nz + 1), np.arange(ny + 1), np.arange(nx + 1), indexing="ij")
    return np.stack([i.ravel() * spacing, j.ravel() * spacing, k.ravel() * spacing], axis=1)


def grid_elements(dims):
    """Element vertex ids in ingest_hex_grid order (orientation fix applied)."""
    nx, ny, nz = dims
    sx, sy = nx + 1, ny + 1
    out = []
    for k in range(nz):
        for j in range(ny):
            for i in range(nx):
                odd = (i + j + k) & 1
                corner = []
                for c in range(8):
                    bx, by, bz = c & 1, (c >> 1) & 1, (c >> 2) & 1
                    if odd:
                        bx = 1 - bx
                    corner.append((i + bx) + sx * ((j + by) + sy * (k + bz)))
                for t in KUHN:
                    out.append([corner[t[0]], corner[t[1]], corner[t[2]], corner[t[3]]])
    el = np.array(out, dtype=np.int64)
    # orientation: swap 2,3 where the signed volume is negative (mesh.cpp:130-133)
    x = grid_vertices(dims, 1.0)
    d = np.stack([x[el[:, 1]] - x[el[:, 0]], x[el[:, 2]] - x[el[:, 0]], x[el[:, 3]] - x[el[:, 0]]], axis=2)
    neg = np.linalg.det(d) < 0
    el[neg, 2], el[neg, 3] = el[neg, 3].copy(), el[neg, 2].copy()
    return el


def element_centroids(dims, spacing):
    x = grid_vertices(dims, spacing)
    el = grid_elements(dims)
    return x[el].mean(axis=1)


def wiggle(n, amp, phase=0.0):
    """test_util.hpp:51-55: amp * sin(0.7 i + phase)."""
    return amp * np.sin(0.7 * np.arange(n) + phase)


def _solver(**kw):
    base = {"h": 0.01}
    base.update(kw)
    return base


def config_scene(tag: str, frames: int | None = None, solver: dict | None = None, ordering: str | None = None,
                 dims: tuple | None = None) -> dict:
    """Scene dict for configuration C1..C4 (SURVEY.md §8(d) synthetic inputs).
    `dims` shrinks C4's grid for parity tests (same construction)."""
    tag = tag.upper()
    if tag == "C1":
        dims, h = (36, 6, 4), 0.05
        s = {
            "name": "C1-cantilever",
            "mesh": {"grid": {"dims": list(dims), "spacing": h, "density": 1000.0}},
            "material": {"energy": "corotated", "young": 5e4, "poisson": 0.35, "alpha": 0.02, "beta0": 0.01},
            "fix_region": {"min": [-1.0, -1.0, -1.0], "max": [1e-3, 10.0, 10.0]},
            "gravity": [0.0, 0.0, -9.81],
            "solver": _solver(),
            "frames": 100,
        }
    elif tag == "C2":
        dims, h = (24, 16, 13), 0.02
        nv = (dims[0] + 1) * (dims[1] + 1) * (dims[2] + 1)
        s = {
            "name": "C2-bunny-block",
            "mesh": {"grid": {"dims": list(dims), "spacing": h, "density": 1000.0}},
            "material": {"energy": "neo-hookean", "young": 1e5, "poisson": 0.45, "alpha": 0.01, "beta0": 0.0},
            "gravity": [0.0, 0.0, -9.81],
            "initial": {"velocity": wiggle(3 * nv, 0.05).tolist()},
            "solver": _solver(),
            "frames": 100,
        }
    elif tag == "C3":
        dims, h = (40, 24, 18), 0.01
        c = element_centroids(dims, h)
        ext = np.array(dims, dtype=float) * h
        # carapace: ellipsoid around the upper centre; legs/soft tissue elsewhere
        centre = np.array([0.5, 0.5, 0.6]) * ext
        radii = np.array([0.38, 0.36, 0.34]) * ext
        inside = (((c - centre) / radii) ** 2).sum(axis=1) <= 1.0
        young = np.where(inside, 5e6, 5e4)
        nx, ny, nz = dims
        pull_vertex = nx + (nx + 1) * (ny // 2 + (ny + 1) * (nz // 2))  # +x face centre
        nv = (nx + 1) * (ny + 1) * (nz + 1)
        s = {
            "name": "C3-crab-heterogeneous",
            "mesh": {"grid": {"dims": list(dims), "spacing": h, "density": 1000.0}},
            "material": {"energy": "neo-hookean", "young": young.tolist(), "poisson": 0.4, "alpha": 0.05, "beta0": 0.01},
            "gravity": [0.0, 0.0, -9.81],
            "f_ext": [{"vertex": int(pull_vertex), "force": [0.01, 0.0, 0.005]}],
            "initial": {"velocity": wiggle(3 * nv, 0.05).tolist()},
            "solver": _solver(),
            "frames": 100,
        }
    elif tag == "C4":
        dims = tuple(dims) if dims else (40, 24, 18)
        h = 0.01
        nx, ny, nz = dims
        c = element_centroids(dims, h)
        ext = np.array(dims, dtype=float) * h
        # stiff core (the gripper's skeleton) above a soft contact pad
        core = (np.abs(c[:, 0] - 0.5 * ext[0]) <= 0.3 * ext[0]) & (np.abs(c[:, 1] - 0.5 * ext[1]) <= 0.3 * ext[1]) \
            & (c[:, 2] >= 0.4 * ext[2])
        young = np.where(core, 5e6, 5e4)
        radius = 0.05
        # rigid cube edge, rounded: its top touches the pad's bottom-face centre vertex
        centre = [0.5 * ext[0], 0.5 * ext[1], -radius - 2e-4]
        s = {
            "name": "C4-gripper-pad",
            "mesh": {"grid": {"dims": list(dims), "spacing": h, "density": 1000.0}},
            "material": {"energy": "neo-hookean", "young": young.tolist(), "poisson": 0.4, "alpha": 0.05, "beta0": 0.01},
            "gravity": [0.0, 0.0, -9.81],
            "obstacles": [{"type": "sphere", "center": centre, "radius": radius, "friction": 0.5}],
            "initial": {"velocity": [0.0, 0.0, -0.05]},
            "solver": _solver(),
            "frames": 100,
        }
    else:
        raise ValueError(f"unknown config {tag}")
    if frames is not None:
        s["frames"] = frames
    if solver:
        s["solver"].update(solver)
    if ordering:
        s["factor"] = {"ordering": ordering}
    return s


class MT19937_64:
    """std::mt19937_64 (the 64-bit Mersenne Twister of <random>), so the C5
    sample parameters are reproducible from any language."""

    def __init__(self, seed: int = 5489):
        m = (1 << 64) - 1
        self.mt = [0] * 312
        self.mt[0] = seed & m
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & m
        self.i = 312

    def __call__(self) -> int:
        m = (1 << 64) - 1
        if self.i >= 312:
            up, lo = 0xFFFFFFFF80000000, 0x7FFFFFFF
            for k in range(312):
                x = (self.mt[k] & up) | (self.mt[(k + 1) % 312] & lo)
                xa = x >> 1
                if x & 1:
                    xa ^= 0xB5026F5AA96619E9
                self.mt[k] = self.mt[(k + 156) % 312] ^ xa
            self.i = 0
        x = self.mt[self.i]
        self.i += 1
        x ^= (x >> 29) & 0x5555555555555555
        x ^= (x << 17) & 0x71D67FFFEDA60000
        x ^= (x << 37) & 0xFFF7EEE000000000
        x ^= x >> 43
        return x & m


def c5_normals(samples: int, seed: int = 2605) -> np.ndarray:
    """z_s ~ N(0, 1): Box-Muller on pairs of 53-bit uniforms (u = (x >> 11) 2^-53)
    drawn from std::mt19937_64(seed); the cosine branch, one z per pair."""
    g = MT19937_64(seed)
    z = np.empty(samples)
    for s in range(samples):
        u1 = (g() >> 11) * 2.0 ** -53
        u2 = (g() >> 11) * 2.0 ** -53
        z[s] = math.sqrt(-2.0 * math.log1p(-u1)) * math.cos(2.0 * math.pi * u2)
    return z


def c5_young(samples: int, element_count: int, base: float = 1e5, seed: int = 2605) -> np.ndarray:
    """Per-sample Young's moduli of the batched system-ID configuration C5
    (SURVEY.md §8(d)): sample s uses E_s = base exp(0.5 z_s) on every element.
    Returns a (samples, element_count) array."""
    z = c5_normals(samples, seed)
    return np.repeat((base * np.exp(0.5 * z))[:, None], element_count, axis=1)


def block_scene(dims=(2, 2, 2), spacing=0.1, kind="neo-hookean", young_base=5e4, contrast=1.0, poisson=0.4,
                alpha=0.01, beta0=0.0, floor=False, friction=0.4, gravity_z=-2.0, frames=3, v0_amp=0.05,
                fix_x0_face=False, hook=False, eps_rel=1e-12, eps_abs=1e-14) -> dict:
    """The reference test fixture testutil::block_scene (test_util.hpp:68-143)."""
    x = grid_vertices(dims, spacing)
    nv = x.shape[0]
    c = element_centroids(dims, spacing)
    zmid = 0.5 * (x[:, 2].min() + x[:, 2].max())
    young = np.full(c.shape[0], young_base)
    if contrast != 1.0:
        young[c[:, 2] > zmid] = contrast * young_base
    v0 = wiggle(3 * nv, v0_amp)
    fixed = [int(v) for v in range(nv) if x[v, 0] <= 1e-12] if fix_x0_face else []
    for v in fixed:
        v0[3 * v:3 * v + 3] = 0.0
    s = {
        "name": "block",
        "mesh": {"grid": {"dims": list(dims), "spacing": spacing, "density": 1000.0}},
        "material": {"energy": kind, "young": young.tolist(), "poisson": poisson, "alpha": alpha, "beta0": beta0},
        "gravity": [0.0, 0.0, gravity_z],
        "solver": {"h": 0.01, "eps_rel": eps_rel, "eps_abs": eps_abs},
        "frames": frames,
        "initial": {"velocity": v0.tolist()},
    }
    if fixed:
        s["dirichlet"] = [{"vertex": v} for v in fixed]
    if floor:
        s["obstacles"] = [{"type": "halfspace", "normal": [0, 0, 1], "offset": 0.0, "friction": friction}]
    if hook:
        s["f_state"] = {"point_spring": {"vertex": nv - 1,
                                         "anchor": (x[nv - 1] + np.array([0.02, -0.01, 0.05])).tolist(),
                                         "stiffness": 2e3, "damping": 5.0}}
    return s


def two_tets_unequal(young=(4e4, 9e4), kind="neo-hookean", poisson=0.35, alpha=0.0, beta0=0.0, barrier=False) -> dict:
    """test_util.hpp:37-47: two tets sharing a face, volumes 1/6 and 1/3."""
    return {
        "name": "two-tets-unequal",
        "mesh": {"vertices": [[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [0, 0, -2]],
                 "elements": [[0, 1, 2, 3], [0, 2, 1, 4]], "density": 1000.0},
        "material": {"energy": kind, "young": list(young), "poisson": poisson, "alpha": alpha, "beta0": beta0,
                     "log_barrier": barrier},
        "solver": {"h": 0.01, "eps_rel": 1e-12, "eps_abs": 1e-14},
        "frames": 1,
    }


def dumps(scene: dict) -> str:
    return json.dumps(scene)
