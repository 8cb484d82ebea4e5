"""ctypes binding of the ``hd_*`` C ABI declared in ``include/heterodyn.h``.

Host-side mirror of the reference's public interface
(/root/reference/proj/include/heterodyn/heterodyn.h:30-141) plus the B200
extensions (backward chain, state control, counters).  The binding is
library-agnostic: ``Library(path)`` wraps any shared object exporting the
header — the product (``paper_2605_14526_b200/_lib/libheterodyn_b200.so``)
or, in the tests only, the CPU oracle.  Error behaviour follows the
reference: a non-OK ``hd_status`` raises :class:`HdError` carrying the code
and ``hd_last_error()`` message.
"""
from __future__ import annotations

import ctypes as C
import json
import os

import numpy as np

HD_STATUS = {
    0: "OK", 1: "PARSE", 2: "VALIDATION", 3: "DEGENERATE_ELEMENT", 4: "INVALID_POISSON",
    5: "NON_POSITIVE_JACOBIAN", 6: "PROX_DIVERGED", 7: "SINGULAR_FILTERED_HESSIAN",
    8: "NOT_POSITIVE_DEFINITE", 9: "SINGULAR_CONTACT_SYSTEM", 10: "ADJOINT_DIVERGED",
    11: "LINE_SEARCH_FAILED", 12: "IO", 13: "INVALID_ARGUMENT",
}

_D = C.POINTER(C.c_double)
_VP = C.c_void_p

# name -> (restype, argtypes); mirrors include/heterodyn.h
SIGNATURES = {
    "hd_last_error": (C.c_char_p, []),
    "hd_last_error_code": (C.c_int, []),
    "hd_string_free": (None, [_VP]),
    "hd_scene_load": (_VP, [C.c_char_p]),
    "hd_scene_parse": (_VP, [C.c_char_p]),
    "hd_scene_builtin": (_VP, [C.c_char_p]),
    "hd_scene_free": (None, [_VP]),
    "hd_scene_vertex_count": (C.c_int, [_VP]),
    "hd_scene_element_count": (C.c_int, [_VP]),
    "hd_scene_frame_count": (C.c_int, [_VP]),
    "hd_scene_name": (C.c_char_p, [_VP]),
    "hd_scene_region_count": (C.c_int, [_VP]),
    "hd_scene_regions": (C.c_int, [_VP, C.POINTER(C.c_int), C.c_size_t]),
    "hd_scene_rest_positions": (C.c_int, [_VP, _D, C.c_size_t]),
    "hd_scene_vertex_masses": (C.c_int, [_VP, _D, C.c_size_t]),
    "hd_scene_young_moduli": (C.c_int, [_VP, _D, C.c_size_t]),
    "hd_scene_elements": (C.c_int, [_VP, C.POINTER(C.c_int), C.c_size_t]),
    "hd_sim_last_fb_residual": (C.c_double, [_VP]),
    "hd_sim_contact_trace": (C.c_int, [_VP, C.POINTER(C.c_int), C.POINTER(C.c_int), C.c_size_t,
                                      _D, C.c_size_t, _D, C.c_size_t, C.POINTER(C.c_int)]),
    "hd_sim_penetration": (C.c_double, [_VP]),
    "hd_sim_external_force": (C.c_int, [_VP, _D, C.c_size_t]),
    "hd_sim_set_external_force": (C.c_int, [_VP, _D, C.c_size_t]),
    "hd_sim_create": (_VP, [_VP]),
    "hd_sim_free": (None, [_VP]),
    "hd_sim_step": (C.c_int, [_VP]),
    "hd_sim_time": (C.c_double, [_VP]),
    "hd_sim_dof_count": (C.c_int, [_VP]),
    "hd_sim_positions": (C.c_int, [_VP, _D, C.c_size_t]),
    "hd_sim_velocities": (C.c_int, [_VP, _D, C.c_size_t]),
    "hd_sim_last_iterations": (C.c_int, [_VP]),
    "hd_sim_last_converged": (C.c_int, [_VP]),
    "hd_sim_last_contact_count": (C.c_int, [_VP]),
    "hd_run_simulate": (C.c_int, [_VP, C.c_char_p, C.POINTER(_VP)]),
    "hd_run_gradcheck": (C.c_int, [_VP, C.c_char_p, C.c_char_p, C.POINTER(_VP), C.POINTER(C.c_int)]),
    "hd_run_identify": (C.c_int, [C.c_char_p, C.c_char_p, C.POINTER(_VP), C.POINTER(C.c_int)]),
    "hd_run_identify_file": (C.c_int, [C.c_char_p, C.c_char_p, C.POINTER(_VP), C.POINTER(C.c_int)]),
    "hd_factor_stats": (C.c_int, [_VP, C.POINTER(_VP)]),
    "hd_sim_record": (C.c_int, [_VP, C.c_int]),
    "hd_sim_recorded_frames": (C.c_int, [_VP]),
    "hd_sim_set_state": (C.c_int, [_VP, _D, _D, C.c_double]),
    "hd_sim_backward": (C.c_int, [_VP, _D, _D, _D, _D, _D, _D, _D, _D, C.c_size_t]),
    "hd_sim_backward_tau": (C.c_int, [_VP, _D, _D, C.c_size_t]),
    "hd_sim_backward_iterations": (C.c_int, [_VP]),
    "hd_sim_solve_free": (C.c_int, [_VP, _D, _D, _D]),
    "hd_sim_set_young": (C.c_int, [_VP, _D, C.c_size_t, C.c_int]),
    "hd_sim_set_deflation": (C.c_int, [_VP, C.c_int]),
    "hd_sim_factor_nnz": (C.c_longlong, [_VP]),
    "hd_sim_free_count": (C.c_int, [_VP]),
    "hd_sim_solve_count": (C.c_longlong, [_VP]),
    "hd_sim_factor_streams": (C.c_longlong, [_VP]),
    "hd_sim_a_spmv_count": (C.c_longlong, [_VP]),
    "hd_sim_refactor_count": (C.c_longlong, [_VP]),
    "hd_sim_backward_canonical": (C.c_int, [_VP, _D, _D, _D, _D, _D, C.c_size_t]),
    "hd_sim_stream": (_VP, [_VP]),
    "hd_sim_kernel_launches": (C.c_longlong, [_VP]),
    "hd_sim_time_solve": (C.c_int, [_VP, C.c_int, _D, _D]),
    "hd_batch_time_solve": (C.c_int, [_VP, C.c_int, _D, _D]),
    "hd_batch_lockstep": (C.c_int, [_VP]),
    "hd_sim_time_backbone": (C.c_int, [_VP, C.c_int, C.c_uint, _D]),
    "hd_sim_trace_backbone": (C.c_int, [_VP, C.c_int, _D, C.c_size_t]),
    "hd_sim_trace_loop": (C.c_int, [_VP, _D, C.c_size_t, C.POINTER(C.c_int)]),
    "hd_batch_create": (_VP, [_VP, C.c_int, _D, C.c_size_t, C.c_int]),
    "hd_batch_free": (None, [_VP]),
    "hd_batch_sample_count": (C.c_int, [_VP]),
    "hd_batch_set_target": (C.c_int, [_VP, _D, C.c_size_t]),
    "hd_batch_evaluate": (C.c_int, [_VP, C.c_int, _D, C.c_size_t, _D, C.c_size_t, _VP]),
    "hd_batch_last_ms": (C.c_double, [_VP]),
    "hd_batch_kernel_launches": (C.c_longlong, [_VP]),
    "hd_batch_solve_count": (C.c_longlong, [_VP]),
    "hd_batch_set_young": (C.c_int, [_VP, _D, C.c_size_t, C.c_int]),
    "hd_batch_solve_bytes": (C.c_double, [_VP]),
}


class HdError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(f"[{HD_STATUS.get(code, code)}] {message}")
        self.code = code
        self.name = HD_STATUS.get(code, str(code))


def _ptr(a):
    if a is None:
        return None
    return a.ctypes.data_as(_D)


def _f64(a, n=None):
    if a is None:
        return None
    a = np.ascontiguousarray(a, dtype=np.float64)
    if n is not None and a.size != n:
        raise ValueError(f"expected {n} doubles, got {a.size}")
    return a


class Library:
    """A loaded ``hd_*`` library (product or oracle)."""

    def __init__(self, path: str):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.path = path
        self.lib = C.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(self.lib, name)
            fn.restype = res
            fn.argtypes = args

    def check(self, status: int):
        if status != 0:
            raise HdError(self.lib.hd_last_error_code(), self.lib.hd_last_error().decode())

    def _take_string(self, p: C.c_void_p) -> str:
        s = C.cast(p, C.c_char_p).value.decode()
        self.lib.hd_string_free(p)
        return s

    # scenes
    def scene(self, text_or_dict) -> "Scene":
        text = text_or_dict if isinstance(text_or_dict, str) else json.dumps(text_or_dict)
        h = self.lib.hd_scene_parse(text.encode())
        if not h:
            raise HdError(self.lib.hd_last_error_code(), self.lib.hd_last_error().decode())
        return Scene(self, h)

    def builtin(self, name: str) -> "Scene":
        h = self.lib.hd_scene_builtin(name.encode())
        if not h:
            raise HdError(self.lib.hd_last_error_code(), self.lib.hd_last_error().decode())
        return Scene(self, h)

    def run_identify(self, problem, out_dir: str | None = None) -> tuple[dict, bool]:
        """hd_run_identify: L-BFGS system identification (drivers.cpp:805-979);
        returns (result, stalled)."""
        text = problem if isinstance(problem, str) else json.dumps(problem)
        p, st = _VP(), C.c_int(-1)
        self.check(self.lib.hd_run_identify(text.encode(), out_dir.encode() if out_dir else None,
                                            C.byref(p), C.byref(st)))
        return json.loads(self._take_string(p)), bool(st.value)

    def run_identify_file(self, path: str, out_dir: str | None = None) -> tuple[dict, bool]:
        p, st = _VP(), C.c_int(-1)
        self.check(self.lib.hd_run_identify_file(path.encode(), out_dir.encode() if out_dir else None,
                                                 C.byref(p), C.byref(st)))
        return json.loads(self._take_string(p)), bool(st.value)

    def load(self, path: str) -> "Scene":
        h = self.lib.hd_scene_load(path.encode())
        if not h:
            raise HdError(self.lib.hd_last_error_code(), self.lib.hd_last_error().decode())
        return Scene(self, h)


class Scene:
    def __init__(self, lib: Library, handle):
        self.L = lib
        self.h = handle

    def __del__(self):
        try:
            if self.h:
                self.L.lib.hd_scene_free(self.h)
                self.h = None
        except Exception:
            pass

    @property
    def vertex_count(self):
        return self.L.lib.hd_scene_vertex_count(self.h)

    @property
    def element_count(self):
        return self.L.lib.hd_scene_element_count(self.h)

    @property
    def frame_count(self):
        return self.L.lib.hd_scene_frame_count(self.h)

    @property
    def name(self):
        return self.L.lib.hd_scene_name(self.h).decode()

    @property
    def region_count(self):
        return self.L.lib.hd_scene_region_count(self.h)

    def regions(self):
        out = np.zeros(self.element_count, dtype=np.int32)
        self.L.check(self.L.lib.hd_scene_regions(self.h, out.ctypes.data_as(C.POINTER(C.c_int)), out.size))
        return out

    def rest_positions(self):
        out = np.zeros(3 * self.vertex_count)
        self.L.check(self.L.lib.hd_scene_rest_positions(self.h, _ptr(out), out.size))
        return out

    def vertex_masses(self):
        out = np.zeros(self.vertex_count)
        self.L.check(self.L.lib.hd_scene_vertex_masses(self.h, _ptr(out), out.size))
        return out

    def factor_stats(self) -> dict:
        p = _VP()
        self.L.check(self.L.lib.hd_factor_stats(self.h, C.byref(p)))
        return json.loads(self.L._take_string(p))

    def run_simulate(self, out_dir: str | None = None) -> dict:
        p = _VP()
        self.L.check(self.L.lib.hd_run_simulate(self.h, out_dir.encode() if out_dir else None, C.byref(p)))
        return json.loads(self.L._take_string(p))

    def run_gradcheck(self, variables: str | None = None, out_path: str | None = None) -> tuple[dict, bool]:
        """hd_run_gradcheck: adjoint vs central differences (drivers.cpp:367-515);
        returns (report, pass)."""
        p, ok = _VP(), C.c_int(-1)
        self.L.check(self.L.lib.hd_run_gradcheck(self.h, variables.encode() if variables is not None else None,
                                                 out_path.encode() if out_path else None, C.byref(p), C.byref(ok)))
        return json.loads(self.L._take_string(p)), bool(ok.value)

    def elements(self):
        out = np.zeros((self.element_count, 4), dtype=np.int32)
        self.L.check(self.L.lib.hd_scene_elements(self.h, out.ctypes.data_as(C.POINTER(C.c_int)), out.size))
        return out

    def young_moduli(self):
        out = np.zeros(self.element_count)
        self.L.check(self.L.lib.hd_scene_young_moduli(self.h, _ptr(out), out.size))
        return out

    def batch(self, samples: int, young=None, threads: int = 8) -> "Batch":
        """hd_batch_create: `samples` parameter samples of this scene; young is a
        (samples, element_count) array of per-element Young's moduli or None."""
        y = None
        cnt = 0
        if young is not None:
            y = np.ascontiguousarray(young, dtype=np.float64).reshape(-1)
            cnt = y.size
        h = self.L.lib.hd_batch_create(self.h, samples, _ptr(y), cnt, threads)
        if not h:
            raise HdError(self.L.lib.hd_last_error_code(), self.L.lib.hd_last_error().decode())
        return Batch(self, h, y)

    def sim(self) -> "Sim":
        h = self.L.lib.hd_sim_create(self.h)
        if not h:
            raise HdError(self.L.lib.hd_last_error_code(), self.L.lib.hd_last_error().decode())
        return Sim(self, h)


class Sim:
    def __init__(self, scene: Scene, handle):
        self.scene = scene  # keeps the scene alive (the sim borrows it)
        self.L = scene.L
        self.h = handle
        self.n = self.L.lib.hd_sim_dof_count(handle)

    def __del__(self):
        try:
            if self.h:
                self.L.lib.hd_sim_free(self.h)
                self.h = None
        except Exception:
            pass

    def step(self, frames: int = 1):
        for _ in range(frames):
            self.L.check(self.L.lib.hd_sim_step(self.h))

    @property
    def time(self):
        return self.L.lib.hd_sim_time(self.h)

    def positions(self):
        out = np.empty(self.n)
        self.L.check(self.L.lib.hd_sim_positions(self.h, _ptr(out), out.size))
        return out

    def velocities(self):
        out = np.empty(self.n)
        self.L.check(self.L.lib.hd_sim_velocities(self.h, _ptr(out), out.size))
        return out

    @property
    def last_iterations(self):
        return self.L.lib.hd_sim_last_iterations(self.h)

    @property
    def last_converged(self):
        return bool(self.L.lib.hd_sim_last_converged(self.h))

    @property
    def last_contact_count(self):
        return self.L.lib.hd_sim_last_contact_count(self.h)

    def contact_trace(self) -> dict:
        """Last step's contact rows and per-iteration decision values
        (hd_sim_contact_trace): vertex, obstacle (nc,), clamp (iterations, nc:
        clamped iff < 0), cone (iterations, nf: projected iff > 0)."""
        lib = self.L.lib
        cnt = (C.c_int * 3)()
        self.L.check(lib.hd_sim_contact_trace(self.h, None, None, 0, None, 0, None, 0, cnt))
        nc, nf, it = cnt[0], cnt[1], cnt[2]
        v = np.zeros(max(nc, 1), dtype=np.int32)
        o = np.zeros(max(nc, 1), dtype=np.int32)
        cl = np.zeros(max(it * nc, 1))
        co = np.zeros(max(it * nf, 1))
        ip = C.POINTER(C.c_int)
        self.L.check(lib.hd_sim_contact_trace(self.h, v.ctypes.data_as(ip), o.ctypes.data_as(ip), v.size,
                                              _ptr(cl), cl.size, _ptr(co), co.size, cnt))
        return {"vertex": v[:nc], "obstacle": o[:nc], "clamp": cl[:it * nc].reshape(it, nc),
                "cone": co[:it * nf].reshape(it, nf), "iterations": it}

    def record(self, enable: bool = True):
        self.L.check(self.L.lib.hd_sim_record(self.h, 1 if enable else 0))

    @property
    def recorded_frames(self):
        return self.L.lib.hd_sim_recorded_frames(self.h)

    def set_state(self, q=None, v=None, time: float = 0.0):
        q = _f64(q, self.n)
        v = _f64(v, self.n)
        self.L.check(self.L.lib.hd_sim_set_state(self.h, _ptr(q), _ptr(v), time))

    def backward(self, dl_dq_final=None, dl_dv_final=None, dl_dq_direct=None) -> dict:
        ne = self.scene.element_count
        frames = self.recorded_frames
        direct = None
        if dl_dq_direct is not None:
            direct = _f64(dl_dq_direct, (frames + 1) * self.n)
        qf = _f64(dl_dq_final, self.n)
        vf = _f64(dl_dv_final, self.n)
        out = {k: np.zeros(self.n) for k in ("dl_dq0", "dl_dv0", "dl_df_ext")}
        out["dl_de"] = np.zeros(ne)
        dw = np.zeros(2 * ne)
        self.L.check(self.L.lib.hd_sim_backward(
            self.h, _ptr(direct), _ptr(qf), _ptr(vf), _ptr(out["dl_dq0"]), _ptr(out["dl_dv0"]),
            _ptr(out["dl_df_ext"]), _ptr(out["dl_de"]), _ptr(dw), dw.size))
        out["dl_dw"] = dw
        tau = np.zeros(max(frames, 1))
        rho = np.zeros(max(frames, 1))
        self.L.check(self.L.lib.hd_sim_backward_tau(self.h, _ptr(tau), _ptr(rho), tau.size))
        out["tau"] = tau[:frames]
        out["rho"] = rho[:frames]
        out["adjoint_iterations"] = self.L.lib.hd_sim_backward_iterations(self.h)
        return out

    def backward_canonical(self, download: bool = False) -> dict | None:
        """Adjoint chain of L = 1/2|q_T - rest|^2 + 1/2|v_T|^2 seeded in device memory."""
        if not download:
            self.L.check(self.L.lib.hd_sim_backward_canonical(self.h, None, None, None, None, None, 0))
            return None
        ne = self.scene.element_count
        out = {k: np.zeros(self.n) for k in ("dl_dq0", "dl_dv0", "dl_df_ext")}
        out["dl_de"] = np.zeros(ne)
        dw = np.zeros(2 * ne)
        self.L.check(self.L.lib.hd_sim_backward_canonical(
            self.h, _ptr(out["dl_dq0"]), _ptr(out["dl_dv0"]), _ptr(out["dl_df_ext"]), _ptr(out["dl_de"]),
            _ptr(dw), dw.size))
        out["dl_dw"] = dw
        return out

    @property
    def stream(self) -> int:
        return self.L.lib.hd_sim_stream(self.h) or 0

    @property
    def kernel_launches(self) -> int:
        return self.L.lib.hd_sim_kernel_launches(self.h)

    def time_solve(self, reps: int = 20):
        ms = C.c_double()
        b = C.c_double()
        self.L.check(self.L.lib.hd_sim_time_solve(self.h, reps, C.byref(ms), C.byref(b)))
        return ms.value, b.value

    def time_backbone(self, reps: int = 50, skip_mask: int = 0) -> float:
        """ms per adjoint backbone iteration (profiling; see heterodyn.h)."""
        ms = C.c_double()
        self.L.check(self.L.lib.hd_sim_time_backbone(self.h, reps, skip_mask, C.byref(ms)))
        return ms.value

    def trace_backbone(self, reps: int = 8):
        """Per-iteration kernel timeline (profiling; see heterodyn.h): array
        [reps, 14, 3] of ns (first resident, first past wait, last end)."""
        import numpy as np
        out = np.full(reps * 14 * 3, -1.0)
        self.L.check(self.L.lib.hd_sim_trace_backbone(self.h, reps, out.ctypes.data_as(_D), out.size))
        return out.reshape(reps, 14, 3)

    def trace_loop(self):
        """Records of the real backbone loop's last iterations (profiling)."""
        import numpy as np
        out = np.full(16 * 14 * 3, -1.0)
        k = C.c_int()
        self.L.check(self.L.lib.hd_sim_trace_loop(self.h, out.ctypes.data_as(_D), out.size, C.byref(k)))
        return out[: k.value * 42].reshape(k.value, 14, 3)

    def solve_free(self, rhs, fixed_q=None):
        rhs = _f64(rhs, self.n)
        fq = _f64(fixed_q, self.n)
        out = np.empty(self.n)
        self.L.check(self.L.lib.hd_sim_solve_free(self.h, _ptr(rhs), _ptr(fq), _ptr(out)))
        return out

    def external_force(self):
        out = np.zeros(self.n)
        self.L.check(self.L.lib.hd_sim_external_force(self.h, _ptr(out), out.size))
        return out

    def set_external_force(self, f):
        f = _f64(f, self.n)
        self.L.check(self.L.lib.hd_sim_set_external_force(self.h, _ptr(f), f.size))

    def set_young(self, young, freeze_means: bool = False):
        y = _f64(young)
        self.L.check(self.L.lib.hd_sim_set_young(self.h, _ptr(y), y.size, 1 if freeze_means else 0))

    def set_deflation(self, on: bool):
        self.L.check(self.L.lib.hd_sim_set_deflation(self.h, 1 if on else 0))

    @property
    def factor_nnz(self):
        return self.L.lib.hd_sim_factor_nnz(self.h)

    @property
    def free_count(self):
        return self.L.lib.hd_sim_free_count(self.h)

    @property
    def solve_count(self):
        return self.L.lib.hd_sim_solve_count(self.h)

    @property
    def factor_streams(self):
        return self.L.lib.hd_sim_factor_streams(self.h)

    @property
    def a_spmv_count(self):
        return self.L.lib.hd_sim_a_spmv_count(self.h)

    @property
    def refactor_count(self):
        return self.L.lib.hd_sim_refactor_count(self.h)


class Batch:
    """hd_batch_*: one process's share of a batched system-ID evaluation."""

    def __init__(self, scene: Scene, handle, young):
        self.scene = scene
        self.L = scene.L
        self.h = handle
        self._young = young
        self.samples = self.L.lib.hd_batch_sample_count(handle)

    def __del__(self):
        try:
            if self.h:
                self.L.lib.hd_batch_free(self.h)
                self.h = None
        except Exception:
            pass

    def set_target(self, q):
        q = np.ascontiguousarray(q, dtype=np.float64)
        self.L.check(self.L.lib.hd_batch_set_target(self.h, _ptr(q), q.size))

    def evaluate(self, frames: int, device_out: int | None = None, want_host: bool = True) -> dict:
        """Returns {"loss": per-sample losses, "dl_de": sum over samples} (host)
        and/or writes [sum L, sum dL/dE] to the device pointer device_out."""
        ne = self.scene.element_count
        loss = np.zeros(self.samples) if want_host else None
        grad = np.zeros(ne) if want_host else None
        self.L.check(self.L.lib.hd_batch_evaluate(
            self.h, frames, _ptr(loss), self.samples, _ptr(grad), ne,
            C.c_void_p(device_out) if device_out else None))
        return {"loss": loss, "dl_de": grad}

    @property
    def last_ms(self) -> float:
        return self.L.lib.hd_batch_last_ms(self.h)

    @property
    def kernel_launches(self) -> int:
        return self.L.lib.hd_batch_kernel_launches(self.h)

    def set_young(self, young, freeze_means: bool = False):
        """One system-ID parameter update: every sample refactors."""
        y = _f64(young)
        self.L.check(self.L.lib.hd_batch_set_young(self.h, _ptr(y), y.size, 1 if freeze_means else 0))

    @property
    def solve_count(self) -> int:
        return self.L.lib.hd_batch_solve_count(self.h)

    @property
    def lockstep(self) -> bool:
        return bool(self.L.lib.hd_batch_lockstep(self.h))

    def time_solve(self, reps: int = 20):
        """(ms per solve, algorithmic bytes per solve) of the batch's solve path."""
        ms, b = C.c_double(0.0), C.c_double(0.0)
        self.L.check(self.L.lib.hd_batch_time_solve(self.h, reps, C.byref(ms), C.byref(b)))
        return ms.value, b.value

    @property
    def solve_bytes(self) -> float:
        return self.L.lib.hd_batch_solve_bytes(self.h)
