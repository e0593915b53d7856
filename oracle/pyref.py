"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes binding of oracle/_ref/libeqsref.so: the UNMODIFIED reference sources
(/root/reference/proj/src) compiled against oracle/ref_shim (an Eigen-API
shim) plus oracle/ref_driver.cpp, a C API over the reference's public
functions. Built here by ``make -C oracle ref`` (needs /root/reference); the
built .so travels to the GPU box with the repo snapshot, where
/root/reference does not exist.

Used to (1) generate the reference-made golden fixtures under tests/golden/
(tests/golden/make_ref_fixtures.py), (2) check the restatement in oracle/
against the reference itself (tests/test_ref_pinning.py), and (3) time the
reference's own CPU path in bench.py (``--impl reference`` and the
``cpu_baseline`` leg). The product package never imports it.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libeqsref.so")
_lib = None

ERRORS = {1: "ConfigError", 2: "NumericalError", 3: "GeometryError", 4: "InvalidArgument", 7: "Error"}


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code
        self.kind = ERRORS.get(code, str(code))


def available() -> bool:
    return os.path.exists(LIB_PATH)


def build() -> str:
    """Compile the reference (only possible where /root/reference exists)."""
    subprocess.run(["make", "-C", _HERE, "-j8", "ref"], check=True, stdout=subprocess.DEVNULL)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not available():
            build()
        L = C.CDLL(LIB_PATH)
        P, I, D = C.c_void_p, C.c_int, C.c_double
        dp, ip, lp = C.POINTER(C.c_double), C.POINTER(C.c_int), C.POINTER(C.c_long)
        L.ref_last_error.restype = C.c_char_p
        L.ref_create.argtypes = [C.c_char_p, D, C.c_uint, C.POINTER(P)]
        L.ref_destroy.argtypes = [P]
        L.ref_destroy.restype = None
        L.ref_sizes.argtypes = [P, lp]
        L.ref_mesh.argtypes = [P, dp, ip, ip]
        L.ref_free_dofs.argtypes = [P, ip]
        L.ref_colors.argtypes = [P, ip]
        L.ref_mass_free.argtypes = [P, ip, ip, dp]
        L.ref_aggregate.argtypes = [P, ip]
        L.ref_amg_levels.argtypes = [P, ip, lp, lp, lp, I]
        L.ref_amg_level_csr.argtypes = [P, I, ip, ip, dp]
        L.ref_kx_apply.argtypes = [P, dp, dp, dp]
        L.ref_mass_apply.argtypes = [P, dp, dp]
        L.ref_eval_residual.argtypes = [P, D, dp, dp]
        L.ref_eval_rhs.argtypes = [P, D, dp, dp]
        L.ref_lift_full.argtypes = [P, D, dp, dp]
        L.ref_spectral_radius.argtypes = [P, D, dp, dp]
        L.ref_set_state.argtypes = [P, D, dp, D]
        L.ref_get_state.argtypes = [P, dp, dp, dp]
        L.ref_rkc_advance_fixed.argtypes = [P, D, I, I]
        L.ref_rkc_step.argtypes = [P, D, dp]
        L.ref_euler_step.argtypes = [P, D]
        L.ref_stats.argtypes = [P, lp, dp]
        L.ref_run_scenario.argtypes = [C.c_char_p, C.c_char_p, lp, dp, dp, I]
        _lib = L
    return _lib


def _p(a, ctype=C.c_double):
    return None if a is None else a.ctypes.data_as(C.POINTER(ctype))


def _check(rc):
    if rc != 0:
        raise RefError(rc, lib().ref_last_error().decode())


def _config_text(config) -> tuple[str, float, int]:
    """The reference parser ignores unknown keys; the additive `jitter` box key
    is applied by the driver (same rule as oracle/mesh_dof.cpp)."""
    cfg = json.loads(config) if isinstance(config, str) else config
    box = cfg.get("mesh", {}).get("box", {})
    return json.dumps(cfg), float(box.get("jitter", 0.0)), int(box.get("jitter_seed", 1612))


class RefProblem:
    """Mesh + DofMap + FemSystem of the reference, built as run_scenario does."""

    def __init__(self, config, workers: int | None = None):
        cfg = json.loads(config) if isinstance(config, str) else dict(config)
        if workers is not None:
            cfg["workers"] = int(workers)
        text, jit, seed = _config_text(cfg)
        h = C.c_void_p()
        _check(lib().ref_create(text.encode(), C.c_double(jit), C.c_uint(seed), C.byref(h)))
        self._h = h
        s = np.zeros(8, dtype=np.int64)
        _check(lib().ref_sizes(h, _p(s, C.c_long)))
        (self.n_nodes, self.n_tets, self.n_dofs, self.n_free, self.n_fixed, self.nnz_ii, self.n_colors,
         self.workers) = (int(v) for v in s)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None:
            _lib.ref_destroy(h)
            self._h = None

    def mesh(self):
        nodes = np.zeros((self.n_nodes, 3))
        tets = np.zeros((self.n_tets, 4), dtype=np.int32)
        region = np.zeros(self.n_tets, dtype=np.int32)
        _check(lib().ref_mesh(self._h, _p(nodes), _p(tets, C.c_int), _p(region, C.c_int)))
        return nodes, tets, region

    def free_dofs(self):
        f = np.zeros(self.n_free, dtype=np.int32)
        _check(lib().ref_free_dofs(self._h, _p(f, C.c_int)))
        return f

    def colors(self):
        c = np.zeros(self.n_tets, dtype=np.int32)
        lib().ref_colors(self._h, _p(c, C.c_int))
        return c

    def mass_free(self):
        rp = np.zeros(self.n_free + 1, dtype=np.int32)
        ci = np.zeros(self.nnz_ii, dtype=np.int32)
        v = np.zeros(self.nnz_ii)
        _check(lib().ref_mass_free(self._h, _p(rp, C.c_int), _p(ci, C.c_int), _p(v)))
        return rp, ci, v

    def aggregate(self):
        a = np.zeros(self.n_free, dtype=np.int32)
        _check(lib().ref_aggregate(self._h, _p(a, C.c_int)))
        return a

    def amg_levels(self):
        n = C.c_int()
        rows, nnz_a, nnz_p = (np.zeros(16, dtype=np.int64) for _ in range(3))
        _check(lib().ref_amg_levels(self._h, C.byref(n), _p(rows, C.c_long), _p(nnz_a, C.c_long),
                                    _p(nnz_p, C.c_long), C.c_int(16)))
        k = n.value
        return rows[:k].tolist(), nnz_a[:k].tolist(), nnz_p[:k].tolist()

    def amg_level_csr(self, level: int):
        rows, nnz_a, _ = self.amg_levels()
        rp = np.zeros(rows[level] + 1, dtype=np.int32)
        ci = np.zeros(nnz_a[level], dtype=np.int32)
        v = np.zeros(nnz_a[level])
        _check(lib().ref_amg_level_csr(self._h, C.c_int(level), _p(rp, C.c_int), _p(ci, C.c_int), _p(v)))
        return rp, ci, v

    def kx_apply(self, x_full, v_full):
        y = np.zeros(self.n_dofs)
        _check(lib().ref_kx_apply(self._h, _p(np.ascontiguousarray(x_full, float)),
                                  _p(np.ascontiguousarray(v_full, float)), _p(y)))
        return y

    def mass_apply(self, v):
        y = np.zeros(self.n_free)
        _check(lib().ref_mass_apply(self._h, _p(np.ascontiguousarray(v, float)), _p(y)))
        return y

    def eval_residual(self, t, x):
        r = np.zeros(self.n_free)
        _check(lib().ref_eval_residual(self._h, C.c_double(t), _p(np.ascontiguousarray(x, float)), _p(r)))
        return r

    def eval_rhs(self, t, x):
        f = np.zeros(self.n_free)
        _check(lib().ref_eval_rhs(self._h, C.c_double(t), _p(np.ascontiguousarray(x, float)), _p(f)))
        return f

    def lift_full(self, t, x):
        f = np.zeros(self.n_dofs)
        _check(lib().ref_lift_full(self._h, C.c_double(t), _p(np.ascontiguousarray(x, float)), _p(f)))
        return f

    def spectral_radius(self, t, x):
        rho = np.zeros(1)
        _check(lib().ref_spectral_radius(self._h, C.c_double(t), _p(np.ascontiguousarray(x, float)), _p(rho)))
        return float(rho[0])

    def set_state(self, t, x, dt=0.0):
        _check(lib().ref_set_state(self._h, C.c_double(t), _p(np.ascontiguousarray(x, float)), C.c_double(dt)))

    def get_state(self):
        x = np.zeros(self.n_free)
        t, dt = np.zeros(1), np.zeros(1)
        _check(lib().ref_get_state(self._h, _p(t), _p(x), _p(dt)))
        return x, float(t[0]), float(dt[0])

    def rkc_advance_fixed(self, dt, s, steps=1):
        _check(lib().ref_rkc_advance_fixed(self._h, C.c_double(dt), C.c_int(s), C.c_int(steps)))

    def rkc_step(self, pinned_rho=0.0):
        a = np.zeros(7)
        _check(lib().ref_rkc_step(self._h, C.c_double(pinned_rho), _p(a)))
        return dict(t_start=a[0], dt=a[1], accepted=bool(a[2]), stages=int(a[3]), error=a[4], rho=a[5],
                    dt_next=a[6])

    def euler_step(self, dt):
        _check(lib().ref_euler_step(self._h, C.c_double(dt)))

    def stats(self):
        s = np.zeros(9, dtype=np.int64)
        tm = np.zeros(4)
        _check(lib().ref_stats(self._h, _p(s, C.c_long), _p(tm)))
        keys = ("m_solves", "pcg_iterations", "rho_solves", "rho_pcg_iterations", "newton_linear_solves",
                "newton_pcg_iterations", "precond_setups", "assemblies", "svd_count")
        d = dict(zip(keys, (int(v) for v in s)))
        d["timers"] = dict(zip(("setup", "residual", "solve", "estimator"), tm.tolist()))
        return d


def run_scenario(config, out_dir: str = "", n_free: int = 0):
    """run_scenario (scenario.cpp:217-383) of the reference; returns
    (exit_code, accepted, rejected, m_solves, pcg_iterations, final_t, final_x)."""
    text, jit, _ = _config_text(config)
    if jit:
        raise ValueError("run_scenario: jittered meshes go through RefProblem")
    counts = np.zeros(6, dtype=np.int64)
    t = np.zeros(1)
    x = np.zeros(max(n_free, 1))
    _check(lib().ref_run_scenario(text.encode(), out_dir.encode(), _p(counts, C.c_long), _p(t),
                                  _p(x) if n_free else None, C.c_int(n_free)))
    return dict(exit_code=int(counts[0]), accepted=int(counts[1]), rejected=int(counts[2]),
                m_solves=int(counts[3]), pcg_iterations=int(counts[4]), final_t=float(t[0]),
                final_x=x if n_free and counts[5] == n_free else None, error=lib().ref_last_error().decode())
