"""Thin ctypes binding of libsisph.so (include/sisph.h).

Argument marshalling only: every step of the hot path runs in the CUDA
kernels behind the C ABI.  There is no CPU fallback — if the library is
missing or CUDA is unavailable the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# SISPH_LIB: an A/B variant of the library built in-tree (build.py --out); default libsisph.so
LIB_PATH = os.environ.get("SISPH_LIB") or os.path.join(_HERE, "libsisph.so")

SISPH_OK, SISPH_EINVAL, SISPH_ENOMEM, SISPH_ECUDA, SISPH_ENCCL, SISPH_ENONFINITE, SISPH_EOVERFLOW = range(7)
ERROR_NAMES = {1: "SISPH_EINVAL", 2: "SISPH_ENOMEM", 3: "SISPH_ECUDA", 4: "SISPH_ENCCL",
               5: "SISPH_ENONFINITE", 6: "SISPH_EOVERFLOW"}

FIELDS = dict(POSITION=0, VELOCITY=1, TRANSPORT_VELOCITY=2, PRESSURE=3, DENSITY=4, MASS=5,
              USTAR=6, RSTAR=7, RHS=8, DIAG=9, NORMAL=10, FREE_SURFACE=11, TAG=12, WALL_VELOCITY=13)
VECTOR_FIELDS = {"POSITION", "VELOCITY", "TRANSPORT_VELOCITY", "USTAR", "RSTAR", "NORMAL", "WALL_VELOCITY"}

EXPORTED = ["sisph_params_default", "sisph_create", "sisph_destroy", "sisph_build_neighbors",
            "sisph_predict", "sisph_ppe_solve", "sisph_correct", "sisph_step", "sisph_get_field",
            "sisph_set_field", "sisph_get_field_f32", "sisph_set_field_f32", "sisph_stage_field",
            "sisph_stage_field_f32", "sisph_commit_staged", "sisph_fetch_field", "sisph_fetch_field_f32",
            "sisph_fetch_wait", "sisph_get_order", "sisph_get_neighbors", "sisph_get_neighbors_of",
            "sisph_get_counts", "sisph_get_owned_counts", "sisph_nccl_unique_id", "sisph_local_group_create",
            "sisph_local_group_destroy", "sisph_slab_bounds", "sisph_slab_owner", "sisph_create_dist", "sisph_next_dt", "sisph_sweep_timing",
            "sisph_set_timing", "sisph_sync", "sisph_last_error"]


class sisph_domain(C.Structure):
    _fields_ = [("dim", C.c_int), ("lo", C.c_double * 3), ("hi", C.c_double * 3),
                ("periodic", C.c_int * 3)]


class sisph_params(C.Structure):
    _fields_ = [
        ("precision", C.c_int), ("rho0", C.c_double), ("nu", C.c_double), ("g", C.c_double * 3),
        ("alpha", C.c_double), ("c_ref", C.c_double), ("omega", C.c_double), ("eta", C.c_double),
        ("fs_ratio", C.c_double), ("h_tilde_factor", C.c_double), ("p_ref", C.c_double),
        ("pgrad", C.c_int), ("pref_external", C.c_int), ("ustar_noslip", C.c_int),
        ("clamp_wall_p", C.c_int), ("K", C.c_int), ("min_iter", C.c_int), ("max_iter", C.c_int),
        ("tol", C.c_double), ("wall_rho_summation", C.c_int), ("nbr_cap", C.c_int),
        ("device", C.c_int), ("stream", C.c_void_p), ("rebuild_mode", C.c_int),
        ("matrix_free", C.c_int), ("ppe_loop", C.c_int), ("ppe_mean_free", C.c_int),
        ("conv_mean", C.c_int), ("open_x", C.c_int), ("x_inlet", C.c_double), ("x_outlet", C.c_double),
        ("x_end", C.c_double), ("inlet_length", C.c_double), ("pref_auto", C.c_int),
    ]


class sisph_step_report(C.Structure):
    _fields_ = [("dt", C.c_double), ("iters", C.c_int), ("residual", C.c_double),
                ("lambda_", C.c_double), ("ms_predict", C.c_double), ("ms_solve", C.c_double),
                ("ms_correct", C.c_double), ("pairs", C.c_int64), ("max_neighbors", C.c_int),
                ("ms_sweeps", C.c_double), ("sweeps_timed", C.c_int), ("launches", C.c_int64),
                ("single_build", C.c_int), ("skin_radius", C.c_double), ("n_owned_fluid", C.c_int64),
                ("n_ghost_fluid", C.c_int64), ("halo_bytes", C.c_int64), ("ms_build", C.c_double),
                ("ms_filter", C.c_double), ("ms_rhs", C.c_double), ("ms_ppe", C.c_double)]


class sisph_dist(C.Structure):
    _fields_ = [("nranks", C.c_int), ("rank", C.c_int), ("slab_axis", C.c_int), ("nccl_id", C.c_uint8 * 128),
                ("nccl_lib", C.c_char_p), ("local_group", C.c_void_p), ("always_slab", C.c_int)]


class SisphError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{ERROR_NAMES.get(code, code)}: {msg}")
        self.code = code


_lib = None


def lib():
    """Load libsisph.so; raise loudly if it is missing (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_1908_01762_b200.build`")
        L = C.CDLL(LIB_PATH)
        dp, i64p = C.POINTER(C.c_double), C.POINTER(C.c_int64)
        L.sisph_params_default.argtypes = [C.POINTER(sisph_params)]
        L.sisph_create.argtypes = [dp, dp, dp, dp, C.POINTER(C.c_int32), C.c_int64, C.c_double,
                                   C.POINTER(sisph_domain), C.POINTER(sisph_params), C.POINTER(C.c_void_p)]
        L.sisph_destroy.argtypes = [C.c_void_p]
        L.sisph_build_neighbors.argtypes = [C.c_void_p]
        L.sisph_predict.argtypes = [C.c_void_p, C.c_double]
        L.sisph_ppe_solve.argtypes = [C.c_void_p, C.c_double, C.c_int, C.POINTER(C.c_int), dp]
        L.sisph_correct.argtypes = [C.c_void_p, C.c_double]
        L.sisph_step.argtypes = [C.c_void_p, C.c_double, C.POINTER(sisph_step_report)]
        L.sisph_get_field.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int64]
        L.sisph_set_field.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int64]
        L.sisph_stage_field.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int64]
        L.sisph_stage_field_f32.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int64]
        L.sisph_commit_staged.argtypes = [C.c_void_p]
        L.sisph_fetch_field.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int64]
        L.sisph_fetch_field_f32.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int64]
        L.sisph_fetch_wait.argtypes = [C.c_void_p]
        L.sisph_get_order.argtypes = [C.c_void_p, i64p, C.c_int64]
        L.sisph_get_neighbors.argtypes = [C.c_void_p, i64p, i64p, C.c_int64, i64p]
        L.sisph_get_neighbors_of.argtypes = [C.c_void_p, i64p, C.c_int64, i64p, i64p, C.c_int64, i64p]
        L.sisph_get_counts.argtypes = [C.c_void_p, i64p, i64p, i64p]
        L.sisph_get_owned_counts.argtypes = [C.c_void_p, i64p, i64p]
        L.sisph_next_dt.argtypes = [C.c_void_p, dp, dp, dp]
        L.sisph_sweep_timing.argtypes = [C.c_void_p, dp, C.POINTER(C.c_int)]
        L.sisph_nccl_unique_id.argtypes = [C.c_char_p, C.POINTER(C.c_uint8)]
        L.sisph_local_group_create.argtypes = [C.c_int, C.POINTER(C.c_void_p)]
        L.sisph_local_group_destroy.argtypes = [C.c_void_p]
        L.sisph_slab_bounds.argtypes = [C.POINTER(sisph_domain), C.c_int, C.c_int, C.c_int, dp, dp]
        L.sisph_slab_owner.argtypes = [C.POINTER(sisph_domain), C.c_int, C.c_int, C.c_double]
        L.sisph_create_dist.argtypes = [dp, dp, dp, dp, C.POINTER(C.c_int32), C.c_int64, C.c_double,
                                        C.POINTER(sisph_domain), C.POINTER(sisph_params), C.POINTER(sisph_dist),
                                        C.POINTER(C.c_void_p)]
        L.sisph_set_timing.argtypes = [C.c_void_p, C.c_int]
        L.sisph_sync.argtypes = [C.c_void_p]
        L.sisph_last_error.argtypes = [C.c_void_p]
        L.sisph_last_error.restype = C.c_char_p
        _lib = L
    return _lib


def _check(rc, h=None):
    if rc != SISPH_OK:
        msg = lib().sisph_last_error(h)
        raise SisphError(rc, msg.decode() if msg else "")


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def params_from_dict(d: dict) -> sisph_params:
    p = sisph_params()
    lib().sisph_params_default(C.byref(p))
    for k, v in d.items():
        if k == "g":
            g = list(v) + [0.0] * 3
            for a in range(3):
                p.g[a] = float(g[a])
        elif k == "stream":
            p.stream = int(v) if v else None
        elif hasattr(p, k):
            setattr(p, k, type(getattr(p, k))(v))
    return p


def domain(dim, lo, hi, periodic) -> sisph_domain:
    d = sisph_domain()
    d.dim = dim
    for a in range(3):
        d.lo[a] = float(lo[a]) if a < len(lo) else 0.0
        d.hi[a] = float(hi[a]) if a < len(hi) else 0.0
        d.periodic[a] = int(periodic[a]) if a < len(periodic) else 0
    return d


def default_nccl_lib():
    """The NCCL library torch itself loads (nvidia-nccl wheel), else None (loader search)."""
    try:
        import nvidia.nccl
        for d in nvidia.nccl.__path__:
            p = os.path.join(d, "lib", "libnccl.so.2")
            if os.path.exists(p):
                return p
    except ImportError:
        pass
    return None


def nccl_unique_id(nccl_lib=None) -> bytes:
    """sisph_nccl_unique_id: 128 bytes to broadcast to every rank."""
    buf = (C.c_uint8 * 128)()
    _check(lib().sisph_nccl_unique_id(nccl_lib.encode() if nccl_lib else None, buf), None)
    return bytes(buf)


def slab_bounds(dom: sisph_domain, axis: int, nranks: int, rank: int):
    lo, hi = C.c_double(), C.c_double()
    _check(lib().sisph_slab_bounds(C.byref(dom), axis, nranks, rank, C.byref(lo), C.byref(hi)), None)
    return lo.value, hi.value


class LocalGroup:
    """sisph_local_group_create: ranks as threads of this process on one GPU (tests)."""

    def __init__(self, nranks):
        self._g = C.c_void_p()
        _check(lib().sisph_local_group_create(int(nranks), C.byref(self._g)), None)
        self.nranks = nranks

    def close(self):
        if getattr(self, "_g", None):
            lib().sisph_local_group_destroy(self._g)
            self._g = None

    __del__ = close


def slab_owner(dom: sisph_domain, axis: int, nranks: int, y: float) -> int:
    return lib().sisph_slab_owner(C.byref(dom), axis, nranks, float(y))


def make_dist(nranks, rank, axis, nccl_id: bytes | None = None, nccl_lib=None, local_group: LocalGroup | None = None,
              always_slab=False):
    d = sisph_dist()
    d.nranks, d.rank, d.slab_axis = int(nranks), int(rank), int(axis)
    d.always_slab = 1 if always_slab else 0
    if nccl_id is not None:
        for k in range(128):
            d.nccl_id[k] = nccl_id[k]
    d.nccl_lib = nccl_lib.encode() if nccl_lib else None
    d.local_group = local_group._g if local_group is not None else None
    d._keep = (local_group, nccl_lib)
    return d


class Simulation:
    """Owns one sisph_t handle.  Methods map 1:1 onto the C entry points.
    With dist (make_dist(...)), the handle is one rank of a slab-decomposed
    simulation (sisph_create_dist): every rank passes the same global arrays."""

    def __init__(self, x, u, m, rho, tag, h, dom: sisph_domain, params: sisph_params, dist=None):
        L = lib()
        self.dim = dom.dim
        x = np.ascontiguousarray(x, np.float64)
        u = np.ascontiguousarray(u, np.float64)
        m = np.ascontiguousarray(m, np.float64)
        rho = np.ascontiguousarray(rho, np.float64)
        tag = np.ascontiguousarray(tag, np.int32)
        self.n = int(x.shape[0])
        h_out = C.c_void_p()
        self.dist = dist
        if dist is None:
            rc = L.sisph_create(_dp(x), _dp(u), _dp(m), _dp(rho), tag.ctypes.data_as(C.POINTER(C.c_int32)),
                                self.n, float(h), C.byref(dom), C.byref(params), C.byref(h_out))
        else:
            rc = L.sisph_create_dist(_dp(x), _dp(u), _dp(m), _dp(rho), tag.ctypes.data_as(C.POINTER(C.c_int32)),
                                     self.n, float(h), C.byref(dom), C.byref(params), C.byref(dist),
                                     C.byref(h_out))
        _check(rc, None)
        self._h = h_out
        nn, nf, nw = C.c_int64(), C.c_int64(), C.c_int64()
        L.sisph_get_counts(self._h, C.byref(nn), C.byref(nf), C.byref(nw))
        self.n_fluid, self.n_wall = nf.value, nw.value

    @classmethod
    def from_case(cls, case, dist=None, **overrides):
        prm = dict(case.params)
        prm.update(overrides)
        sim = cls(case.x, case.u, case.m, case.rho, case.tag, case.h,
                  domain(case.dim, case.lo, case.hi, case.periodic), params_from_dict(prm), dist=dist)
        if np.any(case.p != 0):
            sim.set("PRESSURE", case.p)
        return sim

    def next_dt(self):
        """sisph_next_dt: (dt_next, dt_cfl, dt_force) of the paper's adaptive rule."""
        a, b, c = C.c_double(), C.c_double(), C.c_double()
        _check(lib().sisph_next_dt(self._h, C.byref(a), C.byref(b), C.byref(c)), self._h)
        return a.value, b.value, c.value

    def sweep_timing(self):
        """(device ms, launches) of the bracketed sweep launches of the last solve."""
        ms, n = C.c_double(), C.c_int()
        _check(lib().sisph_sweep_timing(self._h, C.byref(ms), C.byref(n)), self._h)
        return ms.value, n.value

    def owned_counts(self):
        nf, nw = C.c_int64(), C.c_int64()
        _check(lib().sisph_get_owned_counts(self._h, C.byref(nf), C.byref(nw)), self._h)
        return nf.value, nw.value

    def close(self):
        if getattr(self, "_h", None):
            lib().sisph_destroy(self._h)
            self._h = None

    __del__ = close

    # --- entry points -------------------------------------------------------
    def build_neighbors(self):
        _check(lib().sisph_build_neighbors(self._h), self._h)

    def predict(self, dt):
        _check(lib().sisph_predict(self._h, float(dt)), self._h)

    def ppe_solve(self, tol, max_iter):
        it, res = C.c_int(), C.c_double()
        _check(lib().sisph_ppe_solve(self._h, float(tol), int(max_iter), C.byref(it), C.byref(res)), self._h)
        return it.value, res.value

    def correct(self, dt):
        _check(lib().sisph_correct(self._h, float(dt)), self._h)

    def step(self, dt):
        rep = sisph_step_report()
        _check(lib().sisph_step(self._h, float(dt), C.byref(rep)), self._h)
        return rep

    def set_timing(self, on=True):
        _check(lib().sisph_set_timing(self._h, 1 if on else 0), self._h)

    def sync(self):
        _check(lib().sisph_sync(self._h), self._h)

    def get(self, field: str, out: np.ndarray | None = None, dtype=np.float64):
        """sisph_get_field (float64) or sisph_get_field_f32 (dtype / out float32)."""
        nc = self.dim if field in VECTOR_FIELDS else 1
        if out is None:
            out = np.empty((self.n, nc) if nc > 1 else self.n, dtype)
        fn = lib().sisph_get_field_f32 if out.dtype == np.float32 else lib().sisph_get_field
        if out.dtype not in (np.float32, np.float64) or not out.flags.c_contiguous:
            raise ValueError("out must be a C-contiguous float32 or float64 array")
        _check(fn(self._h, FIELDS[field], out.ctypes.data, out.size), self._h)
        return out

    def set(self, field: str, value):
        """sisph_set_field; float32 arrays go through sisph_set_field_f32."""
        if isinstance(value, np.ndarray) and value.dtype == np.float32:
            v = np.ascontiguousarray(value)
            _check(lib().sisph_set_field_f32(self._h, FIELDS[field], v.ctypes.data, v.size), self._h)
            return
        v = np.ascontiguousarray(value, np.float64)
        _check(lib().sisph_set_field(self._h, FIELDS[field], v.ctypes.data, v.size), self._h)

    def set_ptr(self, field: str, ptr: int, count: int, f32: bool = False):
        """set_field from a raw host pointer (e.g. pinned torch memory); f32: float buffer."""
        fn = lib().sisph_set_field_f32 if f32 else lib().sisph_set_field
        _check(fn(self._h, FIELDS[field], C.c_void_p(ptr), count), self._h)

    def stage_ptr(self, field: str, ptr: int, count: int, f32: bool = False):
        """sisph_stage_field(_f32): enqueue the upload of a field's next value from a raw host
        pointer (pinned memory overlaps the running step); applied by commit_staged()."""
        fn = lib().sisph_stage_field_f32 if f32 else lib().sisph_stage_field
        _check(fn(self._h, FIELDS[field], C.c_void_p(ptr), count), self._h)

    def commit_staged(self):
        """sisph_commit_staged: the staged fields become the handle's state (stream-ordered)."""
        _check(lib().sisph_commit_staged(self._h), self._h)

    def fetch_ptr(self, field: str, ptr: int, count: int, f32: bool = False):
        """sisph_fetch_field(_f32): enqueue the read of a field into a raw host pointer (pinned
        memory overlaps the handle's next work); the data is there after fetch_wait()."""
        fn = lib().sisph_fetch_field_f32 if f32 else lib().sisph_fetch_field
        _check(fn(self._h, FIELDS[field], C.c_void_p(ptr), count), self._h)

    def fetch_wait(self):
        """sisph_fetch_wait: block until the pending fetch's copy has landed."""
        _check(lib().sisph_fetch_wait(self._h), self._h)

    def get_ptr(self, field: str, ptr: int, count: int, f32: bool = False):
        fn = lib().sisph_get_field_f32 if f32 else lib().sisph_get_field
        _check(fn(self._h, FIELDS[field], C.c_void_p(ptr), count), self._h)

    def order(self):
        ids = np.empty(self.n, np.int64)
        _check(lib().sisph_get_order(self._h, ids.ctypes.data_as(C.POINTER(C.c_int64)), self.n), self._h)
        return ids

    def neighbors(self):
        off = np.zeros(self.n + 1, np.int64)
        tot = C.c_int64()
        L = lib()
        rc = L.sisph_get_neighbors(self._h, off.ctypes.data_as(C.POINTER(C.c_int64)), None, 0, C.byref(tot))
        ids = np.empty(max(tot.value, 1), np.int64)
        _check(L.sisph_get_neighbors(self._h, off.ctypes.data_as(C.POINTER(C.c_int64)),
                                     ids.ctypes.data_as(C.POINTER(C.c_int64)), ids.size, C.byref(tot)), self._h)
        del rc
        return off, ids[: tot.value]

    def neighbors_of(self, which):
        """Neighbour sets (sorted ids) of the particles with creation ids `which`."""
        which = np.ascontiguousarray(which, np.int64)
        m = which.size
        off = np.zeros(m + 1, np.int64)
        tot = C.c_int64()
        L = lib()
        wp = which.ctypes.data_as(C.POINTER(C.c_int64))
        L.sisph_get_neighbors_of(self._h, wp, m, off.ctypes.data_as(C.POINTER(C.c_int64)), None, 0, C.byref(tot))
        ids = np.empty(max(tot.value, 1), np.int64)
        _check(L.sisph_get_neighbors_of(self._h, wp, m, off.ctypes.data_as(C.POINTER(C.c_int64)),
                                        ids.ctypes.data_as(C.POINTER(C.c_int64)), ids.size, C.byref(tot)), self._h)
        return off, ids[: tot.value]
