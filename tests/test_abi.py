"""C-ABI checks that need no GPU: libei.so loads, exports every function include/ei.h declares,
and rejects bad arguments synchronously (before any CUDA call), per include/ei.h."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2202_08627_b200 import build as ei_build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ei():
    ei_build.build()
    from paper_2202_08627_b200 import ei as mod
    return mod


def header_functions():
    txt = open(os.path.join(ROOT, "include", "ei.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(ei_[a-z_0-9]+)\s*\(", txt)))


def test_exports_every_declared_symbol(ei):
    names = header_functions()
    assert {"ei_plan_create", "ei_forward", "ei_cost_grad", "ei_backproject", "ei_project"} <= set(names)
    lib = ctypes.CDLL(ei.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(ei.SYMBOLS)


def test_error_strings_and_version(ei):
    assert ei.ei_error_string(0) == "ok"
    assert "shape" in ei.ei_error_string(2)
    assert ei.ei_error_string(99) == "unknown error code"
    assert ei.ei_version().startswith("libei sm_100a")


def _create(ei, **kw):
    g = dict(n_slices=1, n=8, n_angles=4, n_det=12, n_mask=3, pixel=1.0, det_pitch=1.0, z=1.0)
    g.update(kw)
    ang = kw.pop("angles", None)
    if ang is None:
        ang = np.linspace(0, np.pi, g["n_angles"], endpoint=False)
    g.pop("angles", None)
    return ei.Plan(angles=ang, **g)


@pytest.mark.parametrize("kw,code", [
    (dict(n=1), 2), (dict(n_det=2), 2), (dict(n_mask=0), 2), (dict(n_slices=0), 2),
    (dict(n_angles=0, angles=np.zeros(0)), 2), (dict(n_det=20000), 2),
    (dict(pixel=0.0), 3), (dict(z=-1.0), 3), (dict(det_pitch=0.5), 3), (dict(pixel=float("nan")), 3),
    (dict(angles=np.array([0.0, np.inf, 1.0, 2.0])), 3),
])
def test_plan_argument_errors(ei, kw, code):
    with pytest.raises(ei.EIError) as e:
        _create(ei, **kw)
    assert e.value.code == code


def test_null_arguments(ei):
    lib = ctypes.CDLL(ei.LIB_PATH)
    lib.ei_plan_create.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    out = ctypes.c_void_p()
    assert lib.ei_plan_create(None, None, ctypes.byref(out)) == 1
    assert lib.ei_plan_create(None, None, None) == 1
    for fn in ("ei_project", "ei_backproject"):
        f = getattr(lib, fn)
        f.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
        assert f(None, None, 3, None, None) == 1
    lib.ei_plan_stats.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
    assert lib.ei_plan_stats(None, None) == 1


def test_null_arguments_extended_entry_points(ei):
    """The NEXT-2/3/4 entry points reject a NULL plan or array synchronously (EI_ERR_NULL = 1)."""
    lib = ctypes.CDLL(ei.LIB_PATH)
    vp, f, i = ctypes.c_void_p, ctypes.c_float, ctypes.c_int
    lib.ei_cost_grad_drift.argtypes = [vp] * 8 + [f] + [vp] * 6 + [vp]
    assert lib.ei_cost_grad_drift(*([None] * 8), 0.0, *([None] * 6), None) == 1
    lib.ei_forward_h.argtypes = [vp, vp, f] + [vp] * 4 + [vp]
    assert lib.ei_forward_h(None, None, 5.0, None, None, None, None, None) == 1
    lib.ei_cost_grad_h.argtypes = [vp, vp, f] + [vp] * 4 + [f] + [vp] * 4 + [vp]
    assert lib.ei_cost_grad_h(None, None, 5.0, None, None, None, None, 0.0, None, None, None, None, None) == 1
    lib.ei_forward_hs.argtypes = [vp, vp, f, vp, i] + [vp] * 3 + [vp]
    assert lib.ei_forward_hs(None, None, 5.0, None, 33, None, None, None, None) == 1
    lib.ei_cost_grad_hs.argtypes = [vp, vp, f, vp, i] + [vp] * 3 + [f] + [vp] * 4 + [vp]
    assert lib.ei_cost_grad_hs(None, None, 5.0, None, 33, None, None, None, 0.0, None, None, None, None,
                               None) == 1
    lib.ei_plan_info.argtypes = [vp, vp]
    assert lib.ei_plan_info(None, None) == 1


def test_binding_fails_loudly_without_library(tmp_path):
    """No CPU fallback: the binding raises at import when libei.so is absent."""
    import shutil
    import subprocess
    import sys
    src = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2202_08627_b200")
    pkg = tmp_path / "nolib_pkg"
    pkg.mkdir()
    (pkg / "__init__.py").write_text("")
    shutil.copy(os.path.join(src, "ei.py"), pkg / "ei.py")
    r = subprocess.run([sys.executable, "-c", "import nolib_pkg.ei"], cwd=tmp_path, capture_output=True, text=True)
    assert r.returncode != 0 and "ImportError" in r.stderr and "no CPU fallback" in r.stderr
