"""The C-ABI library builds, loads and exports every symbol include/sisph.h declares;
argument validation (no GPU needed: it runs before any CUDA call)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def sl():
    from paper_1908_01762_b200 import build, sisph
    build.build()
    return sisph


def header_functions():
    src = open(os.path.join(ROOT, "include", "sisph.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sisph_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol(sl):
    names = header_functions()
    assert len(names) >= 15
    L = sl.lib()
    for n in names:
        assert hasattr(L, n), n
    assert sorted(sl.EXPORTED) == names


def test_library_is_sm100a(sl):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", sl.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_params_default(sl):
    p = sl.sisph_params()
    sl.lib().sisph_params_default(C.byref(p))
    assert p.precision == 64 and p.omega == 0.5 and p.eta == 0.01 and p.fs_ratio == 0.8
    assert p.min_iter == 2 and p.max_iter == 1000 and p.K == 10 and p.tol == 1e-2


def _create(sl, x, u, m, rho, tag, h, dom, prm=None):
    out = C.c_void_p()
    dp = lambda a: np.ascontiguousarray(a, np.float64).ctypes.data_as(C.POINTER(C.c_double))
    keep = [np.ascontiguousarray(a, np.float64) for a in (x, u, m, rho)]
    t = np.ascontiguousarray(tag, np.int32)
    rc = sl.lib().sisph_create(*(k.ctypes.data_as(C.POINTER(C.c_double)) for k in keep),
                               t.ctypes.data_as(C.POINTER(C.c_int32)), len(t), h, C.byref(dom),
                               C.byref(prm) if prm is not None else None, C.byref(out))
    del dp
    return rc, sl.lib().sisph_last_error(None).decode()


@pytest.mark.parametrize("case", ["h", "dim", "tag", "mass", "nan", "periodic_cells", "outside", "nofluid",
                                  "precision", "open_tag_without_open_x", "open_x_periodic", "open_x_order"])
def test_create_rejects_invalid_arguments(sl, case):
    n = 16
    x = np.random.default_rng(0).uniform(0.1, 0.9, (n, 2))
    u = np.zeros((n, 2))
    m = np.ones(n)
    rho = np.ones(n)
    tag = np.zeros(n, np.int32)
    h = 0.05
    dom = sl.domain(2, [0, 0], [1, 1], [1, 1])
    prm = None
    if case == "h":
        h = -1.0
    elif case == "dim":
        dom.dim = 4
    elif case == "tag":
        tag[3] = 7
    elif case == "mass":
        m[2] = 0.0
    elif case == "nan":
        x[5, 1] = np.nan
    elif case == "periodic_cells":
        h = 0.2  # 3h = 0.6 -> 1 cell on a periodic axis
    elif case == "outside":
        x[0, 0] = 1.5  # outside [lo, hi) on a periodic axis
    elif case == "nofluid":
        tag[:] = 1
    elif case == "precision":
        prm = sl.params_from_dict({"precision": 16})
    elif case == "open_tag_without_open_x":
        tag[4] = 2           # an inlet tag needs open_x (R34)
    elif case == "open_x_periodic":
        prm = sl.params_from_dict({"open_x": 1, "inlet_length": 0.1, "x_inlet": 0.1, "x_outlet": 0.8, "x_end": 0.9})
    elif case == "open_x_order":
        dom = sl.domain(2, [0, 0], [1, 1], [0, 1])
        prm = sl.params_from_dict({"open_x": 1, "inlet_length": 0.1, "x_inlet": 0.8, "x_outlet": 0.2, "x_end": 0.9})
    rc, msg = _create(sl, x, u, m, rho, tag, h, dom, prm)
    assert rc == sl.SISPH_EINVAL, (rc, msg)
    assert msg


def test_null_handle_calls_fail_cleanly(sl):
    L = sl.lib()
    assert L.sisph_build_neighbors(None) == sl.SISPH_EINVAL
    assert L.sisph_step(None, 1e-3, None) == sl.SISPH_EINVAL
    L.sisph_destroy(None)
