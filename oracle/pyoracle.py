"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes binding of the CPU restatement of the reference hot path
(oracle/liboracle.so, built from oracle/*.cpp by oracle/Makefile). Only
tests/, __graft_entry__.smoke() and bench.py's CPU-baseline /
``--impl reference`` legs may import this module. The product package
(paper_1612_09447_b200) never imports it.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

ERRORS = {1: "ConfigError", 2: "NumericalError", 3: "GeometryError",
          4: "InvalidArgument", 5: "ParseError", 7: "Error"}


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code
        self.kind = ERRORS.get(code, str(code))


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB_PATH):
        subprocess.run(["make", "-C", _HERE, "-j8"], check=True,
                       stdout=subprocess.DEVNULL)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        P, I, D, L_ = C.c_void_p, C.c_int, C.c_double, C.c_long
        dp, ip, lp = C.POINTER(C.c_double), C.POINTER(C.c_int), C.POINTER(C.c_long)
        L.ora_last_error.restype = C.c_char_p
        L.ora_create.argtypes = [C.c_char_p, I, C.POINTER(P)]
        L.ora_destroy.argtypes = [P]
        L.ora_destroy.restype = None
        L.ora_rkc_amplification.restype = D
        L.ora_rkc_amplification.argtypes = [I, D]
        L.ora_kappa_of_e.restype = D
        L.ora_kappa_of_e.argtypes = [D, I, D, D, D, D, D]
        for name in ("ora_eval_rhs", "ora_eval_residual", "ora_lift_full",
                     "ora_spectral_radius", "ora_rkc_advance_fixed", "ora_euler_step"):
            getattr(L, name).argtypes = None
        _lib = L
    return _lib


def _ptr(a, ctype=C.c_double):
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(ctype))


def _check(rc):
    if rc != 0:
        raise OracleError(rc, lib().ora_last_error().decode())


def random_vec(n: int, seed: int) -> np.ndarray:
    """proj/tests/support/test_helpers.hpp:15-21 (mt19937 + uniform[-1,1))."""
    out = np.empty(n)
    _check(lib().ora_random_vec(C.c_int(n), C.c_uint(seed), _ptr(out)))
    return out


def rkc_amplification(s: int, z: float) -> float:
    return lib().ora_rkc_amplification(s, z)


def rkc_coefficients(s: int) -> dict:
    out = np.zeros(3 + 5 * (s + 1))
    _check(lib().ora_rkc_coefficients(C.c_int(s), _ptr(out)))
    o = out[3:].reshape(5, s + 1)
    return dict(w0=out[0], w1=out[1], mu1_tilde=out[2], c=o[0], mu=o[1], nu=o[2],
                mu_tilde=o[3], gamma_tilde=o[4])


def kappa_of_e(material: dict, e: float) -> float:
    c = material["conductivity"]
    if c["kind"] == "constant":
        return lib().ora_kappa_of_e(material["eps_r"], 0, c["kappa"], 0, 0, 0, e)
    return lib().ora_kappa_of_e(material["eps_r"], 1, c.get("kappa_lo", 1e-10), c.get("kappa_hi", 1e-4),
                                c.get("e_switch", 5e5), c.get("width", 5e4), e)


def element_laplacian(coords, order: int, coeff_at_qp) -> np.ndarray:
    n = 4 if order == 1 else 10
    c = np.ascontiguousarray(coords, dtype=np.float64).reshape(12)
    q = np.ascontiguousarray(coeff_at_qp, dtype=np.float64)
    S = np.zeros((n, n))
    _check(lib().ora_element_laplacian(_ptr(c), C.c_int(order), _ptr(q), _ptr(S)))
    return S


def run_scenario(config, out_dir: str = "", x_cap: int = 0):
    """Drop-in run (proj/src/scenario.cpp:217-383); returns dict of totals."""
    text = json.dumps(config) if not isinstance(config, str) else config
    x = np.zeros(max(x_cap, 1))
    totals = np.zeros(8, dtype=np.int64)
    ft = C.c_double()
    wall = C.c_double()
    _check(lib().ora_run_scenario(text.encode(), out_dir.encode(), _ptr(x), C.c_long(x_cap),
                                  _ptr(totals, C.c_long), C.byref(ft), C.byref(wall)))
    n = int(totals[7])
    return dict(accepted=int(totals[0]), rejected=int(totals[1]), stages=int(totals[2]),
                m_solves=int(totals[3]), pcg_iterations=int(totals[4]), rho_solves=int(totals[5]),
                precond_setups=int(totals[6]), n_free=n, final_t=ft.value, wall=wall.value,
                x=x[:n].copy() if x_cap >= n else None)


class Problem:
    """Mesh + dofmap + FemSystem built from a reference-schema JSON config."""

    def __init__(self, config, workers: int = 0):
        text = json.dumps(config) if not isinstance(config, str) else config
        h = C.c_void_p()
        _check(lib().ora_create(text.encode(), C.c_int(workers), C.byref(h)))
        self._h = h
        s = np.zeros(10, dtype=np.int64)
        _check(lib().ora_sizes(h, _ptr(s, C.c_long)))
        (self.n_nodes, self.n_tets, self.n_dofs, self.n_free, self.n_fixed, self.n_local,
         self.order, self.n_colors, self.nnz_ii, self.nnz_ib) = (int(v) for v in s)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None:
            _lib.ora_destroy(h)
            self._h = None

    # --- data
    def mesh(self):
        nodes = np.zeros((self.n_nodes, 3))
        tets = np.zeros((self.n_tets, 4), dtype=np.int32)
        region = np.zeros(self.n_tets, dtype=np.int32)
        _check(lib().ora_get_mesh(self._h, _ptr(nodes), _ptr(tets, C.c_int), _ptr(region, C.c_int)))
        return nodes, tets, region

    def dofs(self):
        ed = np.zeros((self.n_tets, self.n_local), dtype=np.int32)
        fr = np.zeros(self.n_free, dtype=np.int32)
        fx = np.zeros(self.n_fixed, dtype=np.int32)
        fs = np.zeros(self.n_dofs, dtype=np.int32)
        _check(lib().ora_get_dofs(self._h, _ptr(ed, C.c_int), _ptr(fr, C.c_int), _ptr(fx, C.c_int),
                                  _ptr(fs, C.c_int)))
        return ed, fr, fx, fs

    def colors(self):
        c = np.zeros(self.n_tets, dtype=np.int32)
        _check(lib().ora_get_colors(self._h, _ptr(c, C.c_int)))
        return c

    def mass(self, which: int = 0):
        nnz = self.nnz_ii if which == 0 else self.nnz_ib
        rp = np.zeros(self.n_free + 1, dtype=np.int32)
        ci = np.zeros(nnz, dtype=np.int32)
        v = np.zeros(nnz)
        _check(lib().ora_get_mass(self._h, C.c_int(which), _ptr(rp, C.c_int), _ptr(ci, C.c_int), _ptr(v)))
        return rp, ci, v

    # --- operators
    def kx_apply(self, x_state, v):
        y = np.zeros(self.n_dofs)
        _check(lib().ora_kx_apply(self._h, _ptr(np.ascontiguousarray(x_state, float)),
                                  _ptr(np.ascontiguousarray(v, float)), _ptr(y)))
        return y

    def kx_residual(self, x_full, b_mass):
        r = np.zeros(self.n_free)
        _check(lib().ora_kx_residual(self._h, _ptr(np.ascontiguousarray(x_full, float)),
                                     _ptr(np.ascontiguousarray(b_mass, float)), _ptr(r)))
        return r

    def assembled_k_apply(self, x_full, v):
        y = np.zeros(self.n_dofs)
        _check(lib().ora_assembled_k_apply(self._h, _ptr(np.ascontiguousarray(x_full, float)),
                                           _ptr(np.ascontiguousarray(v, float)), _ptr(y)))
        return y

    def eval_residual(self, t, x):
        r = np.zeros(self.n_free)
        _check(lib().ora_eval_residual(self._h, C.c_double(t), _ptr(np.ascontiguousarray(x, float)), _ptr(r)))
        return r

    def eval_rhs(self, t, x):
        f = np.zeros(self.n_free)
        _check(lib().ora_eval_rhs(self._h, C.c_double(t), _ptr(np.ascontiguousarray(x, float)), _ptr(f)))
        return f

    def lift_full(self, t, x):
        f = np.zeros(self.n_dofs)
        _check(lib().ora_lift_full(self._h, C.c_double(t), _ptr(np.ascontiguousarray(x, float)), _ptr(f)))
        return f

    def mass_apply(self, v):
        y = np.zeros(self.n_free)
        _check(lib().ora_mass_apply(self._h, _ptr(np.ascontiguousarray(v, float)), _ptr(y)))
        return y

    def mass_solve(self, b, x0=None, tol=1e-12, max_iter=500):
        x = np.zeros(self.n_free)
        it, conv = C.c_int(), C.c_int()
        rel = C.c_double()
        x0p = None if x0 is None else _ptr(np.ascontiguousarray(x0, float))
        _check(lib().ora_mass_solve(self._h, _ptr(np.ascontiguousarray(b, float)), x0p, C.c_double(tol),
                                    C.c_int(max_iter), _ptr(x), C.byref(it), C.byref(rel), C.byref(conv)))
        return x, it.value, rel.value, bool(conv.value)

    def amg_levels(self):
        n = C.c_int()
        rn = np.zeros(40, dtype=np.int64)
        _check(lib().ora_amg_levels(self._h, C.byref(n), _ptr(rn, C.c_long)))
        return [(int(rn[2 * i]), int(rn[2 * i + 1])) for i in range(n.value)]

    def amg_aggregates(self, level: int):
        rows = self.amg_levels()[level][0]
        a = np.zeros(rows, dtype=np.int32)
        _check(lib().ora_amg_aggregates(self._h, C.c_int(level), _ptr(a, C.c_int)))
        return a

    def spectral_radius(self, t, x):
        rho = C.c_double()
        _check(lib().ora_spectral_radius(self._h, C.c_double(t), _ptr(np.ascontiguousarray(x, float)),
                                         C.byref(rho)))
        return rho.value

    def rkc_advance_fixed(self, t, x, dt, s, nsteps=1):
        x = np.array(x, dtype=np.float64, copy=True)
        _check(lib().ora_rkc_advance_fixed(self._h, C.c_double(t), _ptr(x), C.c_double(dt), C.c_int(s),
                                           C.c_int(nsteps)))
        return x

    def rkc_step_pinned(self, t, x, dt, rho, rtol=1e-2, atol=1e-8, max_stages=200):
        """rkc_step with the rho cache pinned; returns (x_new, attempt dict)."""
        x = np.array(x, dtype=np.float64, copy=True)
        out = np.zeros(7)
        _check(lib().ora_rkc_step_pinned(self._h, C.c_double(t), _ptr(x), C.c_double(dt), C.c_double(rho),
                                         C.c_double(rtol), C.c_double(atol), C.c_int(max_stages), _ptr(out)))
        d = dict(zip(("accepted", "stages", "dt", "error", "rho", "dt_next", "t"), out.tolist()))
        d["accepted"] = bool(d["accepted"])
        d["stages"] = int(d["stages"])
        return x, d

    def shifted_solve(self, t, z, gdt, rhs, refresh_precond=True):
        """FemSystem::shifted_solve (fem_system.cpp:124-145)."""
        z = np.ascontiguousarray(z, dtype=np.float64)
        rhs = np.ascontiguousarray(rhs, dtype=np.float64)
        d = np.zeros_like(rhs)
        _check(lib().ora_shifted_solve(self._h, C.c_double(t), _ptr(z), C.c_double(gdt), _ptr(rhs), _ptr(d),
                                       C.c_int(1 if refresh_precond else 0)))
        return d

    def sdirk_advance_fixed(self, t, x, dt, nsteps=1):
        """sdirk_advance_fixed (integrators.cpp:329-341)."""
        x = np.array(x, dtype=np.float64, copy=True)
        _check(lib().ora_sdirk_advance_fixed(self._h, C.c_double(t), _ptr(x), C.c_double(dt), C.c_int(nsteps)))
        return x

    def euler_step(self, t, x, dt):
        x = np.array(x, dtype=np.float64, copy=True)
        _check(lib().ora_euler_step(self._h, C.c_double(t), _ptr(x), C.c_double(dt)))
        return x

    def estimator_next(self, b):
        """StartVectorEstimator::next(M_II, b) -> (x0, current_rank) (start_vector.cpp:84-109)."""
        b = np.ascontiguousarray(b, dtype=np.float64)
        x0 = np.zeros_like(b)
        rank = C.c_int(0)
        _check(lib().ora_estimator_next(self._h, _ptr(b), _ptr(x0), C.byref(rank)))
        return x0, rank.value

    def estimator_feedback(self, x, iterations: int):
        """StartVectorEstimator::feedback (start_vector.cpp:152-187)."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        _check(lib().ora_estimator_feedback(self._h, _ptr(x), C.c_int(int(iterations))))

    def estimator_stats(self) -> dict:
        s = np.zeros(3, dtype=np.int64)
        _check(lib().ora_estimator_stats(self._h, _ptr(s, C.c_long)))
        return dict(zip(("svd_count", "appends", "spe_fallbacks"), (int(v) for v in s)))

    def stats(self):
        s = np.zeros(8, dtype=np.int64)
        tm = np.zeros(4)
        _check(lib().ora_stats(self._h, _ptr(s, C.c_long), _ptr(tm)))
        keys = ("m_solves", "pcg_iterations", "rho_solves", "rho_pcg_iterations", "precond_setups",
                "assemblies", "applies", "svd_count")
        d = {k: int(v) for k, v in zip(keys, s)}
        d["timers"] = dict(zip(("residual", "solve", "setup", "estimator"), tm.tolist()))
        return d


def pod_build(snapshots, rank: int):
    """pod_build (start_vector.cpp:64-71): snapshots [k][n] -> (basis [keep][n], sigma [k])."""
    S = np.ascontiguousarray(snapshots, dtype=np.float64)
    k, n = S.shape
    U = np.zeros((min(rank, k), n))
    sig = np.zeros(k)
    keep = C.c_int(0)
    _check(lib().ora_pod_build(C.c_int(n), C.c_int(k), _ptr(S), C.c_int(rank), _ptr(U), C.byref(keep), _ptr(sig)))
    return U[:keep.value].copy(), sig


def amg_level_csr(problem: "Problem", level: int, which: int = 0):
    """(rows, cols, row_ptr, col_idx, values) of A (0), P (1) or R (2) at a level."""
    dims = np.zeros(3, dtype=np.int32)
    _check(lib().ora_amg_level_csr(problem._h, C.c_int(level), C.c_int(which), _ptr(dims, C.c_int),
                                   None, None, None))
    rows, cols, nnz = (int(v) for v in dims)
    rp = np.zeros(rows + 1, dtype=np.int32)
    ci = np.zeros(nnz, dtype=np.int32)
    v = np.zeros(nnz)
    _check(lib().ora_amg_level_csr(problem._h, C.c_int(level), C.c_int(which), _ptr(dims, C.c_int),
                                   _ptr(rp, C.c_int), _ptr(ci, C.c_int), _ptr(v)))
    return rows, cols, rp, ci, v


def step_controller(err: float, dt: float, order: int):
    out = np.zeros(2)
    lib().ora_step_controller(C.c_double(err), C.c_double(dt), C.c_int(order), _ptr(out))
    return bool(out[0]), float(out[1])


class DiagonalSystem:
    """proj/tests/support/test_helpers.hpp:37-87 with drive b(t) = c1 sin(w1 t) + c2 cos(w2 t)."""

    def __init__(self, mass, stiffness, c1=0.0, w1=0.0, c2=0.0, w2=0.0):
        m = np.ascontiguousarray(mass, float)
        k = np.ascontiguousarray(stiffness, float)
        L = lib()
        L.ora_diag_create.restype = C.c_void_p
        L.ora_diag_destroy.argtypes = [C.c_void_p]
        L.ora_diag_spectral_radius.restype = C.c_double
        L.ora_diag_spectral_radius.argtypes = [C.c_void_p]
        self.n = len(m)
        self._h = C.c_void_p(L.ora_diag_create(C.c_int(self.n), _ptr(m), _ptr(k), C.c_double(c1), C.c_double(w1),
                                               C.c_double(c2), C.c_double(w2)))

    def __del__(self):
        if getattr(self, "_h", None) is not None and _lib is not None:
            _lib.ora_diag_destroy(self._h)
            self._h = None

    def advance(self, method: str, x, dt, nsteps=1, s=2, t=0.0):
        x = np.array(x, dtype=float, copy=True)
        code = {"euler": 0, "rkc": 1, "sdirk": 2}[method]
        rc = lib().ora_diag_advance(self._h, C.c_int(code), C.c_int(s), C.c_double(t),
                                    C.c_double(dt), C.c_int(nsteps), _ptr(x))
        if rc:
            raise OracleError(rc, lib().ora_diag_last_error().decode())
        return x

    def rkc_step(self, x, dt, rtol=1e-2, atol=1e-8, max_stages=200, t=0.0):
        x = np.array(x, dtype=float, copy=True)
        out = np.zeros(7)
        rc = lib().ora_diag_rkc_step(self._h, C.c_double(t), C.c_double(dt), C.c_double(rtol), C.c_double(atol),
                                     C.c_int(max_stages), _ptr(x), _ptr(out))
        if rc:
            raise OracleError(rc, lib().ora_diag_last_error().decode())
        keys = ("accepted", "stages", "dt", "error", "rho", "dt_next", "t")
        d = dict(zip(keys, out.tolist()))
        d["accepted"] = bool(d["accepted"])
        d["stages"] = int(d["stages"])
        return x, d

    def sdirk_step(self, x, dt, rtol=1e-2, atol=1e-8, t=0.0):
        x = np.array(x, dtype=float, copy=True)
        out = np.zeros(7)
        rc = lib().ora_diag_sdirk_step(self._h, C.c_double(t), C.c_double(dt), C.c_double(rtol), C.c_double(atol),
                                       _ptr(x), _ptr(out))
        if rc:
            raise OracleError(rc, lib().ora_diag_last_error().decode())
        d = dict(zip(("accepted", "newton_iterations", "dt", "error", "dt_next", "t", "precond_setups"),
                     out.tolist()))
        d["accepted"] = bool(d["accepted"])
        d["newton_iterations"] = int(d["newton_iterations"])
        d["precond_setups"] = int(d["precond_setups"])
        return x, d

    def spectral_radius(self):
        return lib().ora_diag_spectral_radius(self._h)
