"""ctypes front-end of the fp64 CPU oracle — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package.  The product path
(``paper_1908_01762_b200``) never imports it, and the two share no code.

The arithmetic lives in ``sisph_oracle.c`` (plain C, fp64, -ffp-contract=off);
this module only compiles it, marshals arrays and names the entry points.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sisph_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (-O2 -ffp-contract=off -fopenmp)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "sisph_oracle.h"))):
        cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
               "-fPIC", "-shared", "-Wall", "-Wno-unknown-pragmas", "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


class Cfg(C.Structure):
    _fields_ = [
        ("dim", C.c_int),
        ("lo", C.c_double * 3), ("hi", C.c_double * 3),
        ("periodic", C.c_int * 3),
        ("h", C.c_double),
        ("rho0", C.c_double), ("nu", C.c_double), ("g", C.c_double * 3),
        ("alpha", C.c_double), ("c_ref", C.c_double), ("omega", C.c_double),
        ("eta", C.c_double), ("fs_ratio", C.c_double),
        ("h_tilde_factor", C.c_double), ("p_ref", C.c_double),
        ("pgrad", C.c_int), ("pref_external", C.c_int), ("ustar_noslip", C.c_int),
        ("clamp_wall_p", C.c_int), ("K", C.c_int), ("min_iter", C.c_int),
        ("max_iter", C.c_int), ("tol", C.c_double),
        ("wall_rho_summation", C.c_int),
        ("ppe_mean_free", C.c_int),
        ("conv_mean", C.c_int),
        ("open_x", C.c_int),
        ("x_inlet", C.c_double), ("x_outlet", C.c_double), ("x_end", C.c_double), ("inlet_length", C.c_double),
        ("pref_auto", C.c_int),
    ]


class Report(C.Structure):
    _fields_ = [("iters", C.c_int), ("residual", C.c_double), ("lambda_", C.c_double)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        dp, ip64, i32p = C.POINTER(C.c_double), C.POINTER(C.c_int64), C.POINTER(C.c_int32)
        L.or_W.restype = C.c_double
        L.or_W.argtypes = [C.c_int, C.c_double, C.c_double]
        L.or_dWdr.restype = C.c_double
        L.or_dWdr.argtypes = [C.c_int, C.c_double, C.c_double]
        L.or_cell_geometry.argtypes = [C.POINTER(Cfg), C.POINTER(C.c_int), dp]
        L.or_cell_order.argtypes = [C.POINTER(Cfg), C.c_int64, dp, ip64, ip64]
        for f in (L.or_neighbors_cell, L.or_neighbors_brute):
            f.restype = C.c_int64
            f.argtypes = [C.POINTER(Cfg), C.c_int64, dp, C.c_int64, ip64, ip64, ip64, C.c_int64]
        L.or_create.restype = C.c_void_p
        L.or_create.argtypes = [C.POINTER(Cfg), C.c_int64, dp, dp, dp, dp, dp, i32p]
        L.or_destroy.argtypes = [C.c_void_p]
        L.or_get.argtypes = [C.c_void_p, C.c_char_p, dp]
        L.or_set.argtypes = [C.c_void_p, C.c_char_p, dp]
        L.or_predict.argtypes = [C.c_void_p, C.c_double]
        L.or_predict_stage2.argtypes = [C.c_void_p, C.c_double]
        L.or_solve.argtypes = [C.c_void_p, C.c_double, C.c_int, C.POINTER(Report)]
        L.or_correct.argtypes = [C.c_void_p, C.c_double]
        L.or_step.argtypes = [C.c_void_p, C.c_double, C.POINTER(Report)]
        L.or_pass_density.argtypes = [C.c_void_p]
        L.or_pass_ghost_velocity.argtypes = [C.c_void_p]
        L.or_pass_wall_pressure.argtypes = [C.c_void_p, dp, dp]
        L.or_pass_sweep.argtypes = [C.c_void_p, dp, C.c_int64, ip64, dp]
        L.or_num_pairs.restype = C.c_int64
        L.or_num_pairs.argtypes = [C.c_void_p, C.c_int]
        L.or_next_dt.argtypes = [C.c_void_p, dp, dp, dp]
        L.or_get_tags.argtypes = [C.c_void_p, i32p]
        L.or_get_tags.restype = None
        L.or_error.argtypes = [C.c_void_p]
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _ip(a):
    return a.ctypes.data_as(C.POINTER(C.c_int64))


def _x3(x):
    x = np.asarray(x, dtype=np.float64)
    out = np.zeros((x.shape[0], 3))
    out[:, : x.shape[1]] = x
    return np.ascontiguousarray(out)


def make_cfg(dim, lo, hi, periodic, h, params: dict | None = None) -> Cfg:
    p = dict(params or {})
    c = Cfg()
    c.dim = dim
    for a in range(3):
        c.lo[a] = float(lo[a]) if a < len(lo) else 0.0
        c.hi[a] = float(hi[a]) if a < len(hi) else 0.0
        c.periodic[a] = int(periodic[a]) if a < len(periodic) else 0
    c.h = float(h)
    c.rho0 = p.get("rho0", 1.0)
    c.nu = p.get("nu", 0.0)
    g = list(p.get("g", [0.0, 0.0, 0.0])) + [0.0] * 3
    for a in range(3):
        c.g[a] = g[a]
    c.alpha = p.get("alpha", 0.0)
    c.c_ref = p.get("c_ref", 0.0)
    c.omega = p.get("omega", 0.5)
    c.eta = p.get("eta", 0.01)
    c.fs_ratio = p.get("fs_ratio", 0.8)
    c.h_tilde_factor = p.get("h_tilde_factor", 1.0)
    c.p_ref = p.get("p_ref", 0.0)
    c.pgrad = p.get("pgrad", 0)
    c.pref_external = p.get("pref_external", 0)
    c.ustar_noslip = p.get("ustar_noslip", 0)
    c.clamp_wall_p = p.get("clamp_wall_p", 0)
    c.K = p.get("K", 10)
    c.min_iter = p.get("min_iter", 2)
    c.max_iter = p.get("max_iter", 1000)
    c.tol = p.get("tol", 1e-2)
    c.wall_rho_summation = p.get("wall_rho_summation", 0)
    c.ppe_mean_free = p.get("ppe_mean_free", 0)
    c.conv_mean = p.get("conv_mean", 1)   # reading R12b
    c.open_x = p.get("open_x", 0)
    c.x_inlet = p.get("x_inlet", 0.0)
    c.x_outlet = p.get("x_outlet", 0.0)
    c.x_end = p.get("x_end", 0.0)
    c.inlet_length = p.get("inlet_length", 0.0)
    c.pref_auto = p.get("pref_auto", 0)
    return c


def case_cfg(case) -> Cfg:
    return make_cfg(case.dim, case.lo, case.hi, case.periodic, case.h, case.params)


def W(dim, r, h):
    return lib().or_W(dim, float(r), float(h))


def dWdr(dim, r, h):
    return lib().or_dWdr(dim, float(r), float(h))


def cell_geometry(cfg):
    nc = (C.c_int * 3)()
    cl = np.zeros(3)
    lib().or_cell_geometry(C.byref(cfg), nc, _dp(cl))
    return [nc[0], nc[1], nc[2]], cl


def cell_order(cfg, x):
    x3 = _x3(x)
    n = x3.shape[0]
    order = np.zeros(n, np.int64)
    keys = np.zeros(n, np.int64)
    lib().or_cell_order(C.byref(cfg), n, _dp(x3), _ip(order), _ip(keys))
    return order, keys


def neighbors(cfg, x, dests=None, brute=False):
    """CSR (offsets, ids) of N(i) for each dest (all particles by default)."""
    x3 = _x3(x)
    n = x3.shape[0]
    d = None if dests is None else np.ascontiguousarray(dests, dtype=np.int64)
    nd = n if d is None else d.size
    off = np.zeros(nd + 1, np.int64)
    fn = lib().or_neighbors_brute if brute else lib().or_neighbors_cell
    dptr = _ip(d) if d is not None else None
    total = fn(C.byref(cfg), n, _dp(x3), nd, dptr, _ip(off), None, 0)
    if total < 0:
        total = int(off[-1])
    nbr = np.zeros(max(total, 1), np.int64)
    fn(C.byref(cfg), n, _dp(x3), nd, dptr, _ip(off), _ip(nbr), nbr.size)
    return off, nbr[:total]


class Sim:
    """The oracle's simulation state, kept in creation-id order."""

    VEC = ("x", "u", "ut", "xs", "us", "normal", "xk", "ftot", "uwall")

    def __init__(self, case=None, *, cfg=None, x=None, u=None, m=None, rho=None, p=None, tag=None):
        if case is not None:
            cfg = case_cfg(case)
            x, u, m, rho, p, tag = case.x, case.u, case.m, case.rho, case.p, case.tag
        self.cfg = cfg
        self.dim = cfg.dim
        x3, u3 = _x3(x), _x3(u)
        self.n = x3.shape[0]
        m = np.ascontiguousarray(m, np.float64)
        rho = np.ascontiguousarray(rho, np.float64)
        p = np.ascontiguousarray(np.zeros(self.n) if p is None else p, np.float64)
        tag = np.ascontiguousarray(tag, np.int32)
        self._h = lib().or_create(C.byref(cfg), self.n, _dp(x3), _dp(u3), _dp(m), _dp(rho),
                                  _dp(p), tag.ctypes.data_as(C.POINTER(C.c_int32)))
        self.tag = tag

    def __del__(self):
        if getattr(self, "_h", None):
            lib().or_destroy(self._h)
            self._h = None

    def get(self, f):
        if f == "lambda":
            out = np.zeros(1)
            lib().or_get(self._h, b"lambda", _dp(out))
            return float(out[0])
        out = np.zeros((self.n, 3)) if f in self.VEC else np.zeros(self.n)
        if lib().or_get(self._h, f.encode(), _dp(out)) != 0:
            raise KeyError(f)
        return out[:, : self.dim] if f in self.VEC else out

    def tags(self):
        """current tags (open boundaries change them: R34)"""
        out = np.zeros(self.n, np.int32)
        lib().or_get_tags(self._h, out.ctypes.data_as(C.POINTER(C.c_int32)))
        return out

    def error(self):
        return int(lib().or_error(self._h))

    def set(self, f, v):
        if f in self.VEC:
            buf = _x3(v)
        elif f == "lambda":
            buf = np.array([float(v)])
        else:
            buf = np.ascontiguousarray(v, np.float64)
        if lib().or_set(self._h, f.encode(), _dp(buf)) != 0:
            raise KeyError(f)

    def predict(self, dt):
        lib().or_predict(self._h, float(dt))

    def predict_stage2(self, dt):
        """A9-A11 again from the current xs (e.g. a working-precision handle's r*)."""
        lib().or_predict_stage2(self._h, float(dt))

    def solve(self, tol, max_iter):
        r = Report()
        lib().or_solve(self._h, float(tol), int(max_iter), C.byref(r))
        return r.iters, r.residual, r.lambda_

    def correct(self, dt):
        lib().or_correct(self._h, float(dt))

    def next_dt(self):
        """Adaptive time step of the next step: (dt, dt_cfl, dt_force)."""
        a, b, c = C.c_double(), C.c_double(), C.c_double()
        if lib().or_next_dt(self._h, C.byref(a), C.byref(b), C.byref(c)) != 0:
            raise RuntimeError("next_dt before any completed step")
        return a.value, b.value, c.value

    def step(self, dt):
        r = Report()
        lib().or_step(self._h, float(dt), C.byref(r))
        return r.iters, r.residual, r.lambda_

    def density(self):
        lib().or_pass_density(self._h)

    def ghost_velocity(self):
        lib().or_pass_ghost_velocity(self._h)

    def wall_pressure(self, pk):
        pk = np.ascontiguousarray(pk, np.float64).copy()
        lib().or_pass_wall_pressure(self._h, _dp(pk), _dp(pk))
        return pk

    def sweep(self, pk, dests=None):
        pk = np.ascontiguousarray(pk, np.float64)
        if dests is None:
            out = np.zeros(int((self.tag == 0).sum()))
            lib().or_pass_sweep(self._h, _dp(pk), 0, None, _dp(out))
        else:
            d = np.ascontiguousarray(dests, np.int64)
            out = np.zeros(d.size)
            lib().or_pass_sweep(self._h, _dp(pk), d.size, _ip(d), _dp(out))
        return out

    def num_pairs(self, which):
        return lib().or_num_pairs(self._h, which)
