"""C-ABI library checks that need no GPU: it loads, exports every symbol include/itlumm.h
declares, and host-side validation returns the documented status codes."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2207_05808_b200 import _lib, build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    build.build()
    return _lib.load()


def header_symbols():
    src = open(os.path.join(ROOT, "include", "itlumm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(itlumm_[a-z_]+)\s*\(", src)))


def test_exports_every_header_symbol(lib):
    syms = header_symbols()
    assert set(syms) == set(_lib.EXPORTS), syms
    for s in syms:
        assert hasattr(lib, s), s
    assert lib.itlumm_abi_version() == 5


def test_sm100a_only_binary():
    """The library carries sm_100a SASS (built with -gencode arch=compute_100a,code=sm_100a)."""
    import subprocess
    r = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                       capture_output=True, text=True)
    assert r.returncode == 0 and "sm_100a" in r.stdout, r.stdout + r.stderr


def _params(D=8, C=2, M=3, **over):
    arr = dict(perm=np.arange(D, dtype=np.int32), boundaries=None,
               split_dim=np.zeros((C, 4), np.int32), thresholds=np.zeros((C, 15), np.float32),
               lut=np.zeros((C, 16, M), np.uint8), scale=np.ones(M, np.float32),
               offset=np.zeros(M, np.float32), bias=None)
    arr.update(over)
    keep = {k: (None if v is None else np.ascontiguousarray(v)) for k, v in arr.items()}
    ptr = lambda a: None if a is None else a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    p = _lib.Params(D, C, M, ptr(keep["perm"]), ptr(keep["boundaries"]), ptr(keep["split_dim"]),
                    ptr(keep["thresholds"]), ptr(keep["lut"]), ptr(keep["scale"]),
                    ptr(keep["offset"]), ptr(keep["bias"]))
    return p, keep


@pytest.mark.parametrize("case,over,msg", [
    ("perm_dup", dict(perm=np.array([0, 0, 2, 3, 4, 5, 6, 7], np.int32)), "bijection"),
    ("perm_range", dict(perm=np.array([0, 1, 2, 3, 4, 5, 6, 8], np.int32)), "bijection"),
    ("split_range", dict(split_dim=np.full((2, 4), 4, np.int32)), "split_dim"),
    ("nan_thr", dict(thresholds=np.full((2, 15), np.nan, np.float32)), "NaN"),
    ("inf_scale", dict(scale=np.array([1, np.inf, 1], np.float32)), "finite"),
    ("bad_bnd", dict(boundaries=np.array([0, 5, 5], np.int32)), "boundaries"),
])
def test_plan_create_validation(lib, case, over, msg):
    p, keep = _params(**over)
    h = ctypes.c_void_p()
    st = lib.itlumm_plan_create(ctypes.byref(p), 0, ctypes.byref(h))
    assert st == _lib.EINVAL, case
    assert msg in lib.itlumm_last_error().decode()
    assert not h.value


def test_plan_create_shape_errors(lib):
    for D, C, M in [(0, 1, 1), (4, 5, 1), (4, 1, 0)]:
        p, keep = _params(D=max(D, 1), C=max(min(C, 4), 1), M=max(M, 1))
        p.D, p.C, p.M = D, C, M
        h = ctypes.c_void_p()
        assert lib.itlumm_plan_create(ctypes.byref(p), 0, ctypes.byref(h)) == _lib.EINVAL
    assert lib.itlumm_plan_create(None, 0, None) == _lib.EINVAL


def test_calls_reject_null_plan(lib):
    assert lib.itlumm_amm(None, None, 0, 8, 1, None, 3, 0, None) == _lib.EINVAL
    assert lib.itlumm_encode(None, None, 0, 8, 1, None, 1, None) == _lib.EINVAL
    assert lib.itlumm_lut_accumulate(None, None, 1, 1, None, 3, None, 3, 0, None) == _lib.EINVAL
    assert lib.itlumm_amm_host(None, None, 0, 8, 1, None, 3, 0, None) == _lib.EINVAL
    assert lib.itlumm_plan_set_algo(None, 0) == _lib.EINVAL
    assert lib.itlumm_plan_set_summation(None, 1) == _lib.EINVAL
    assert lib.itlumm_plan_destroy(None) == _lib.OK
    assert lib.itlumm_mlp_forward(None, None, 0, 8, 1, None, 3, None) == _lib.EINVAL
    assert lib.itlumm_mlp_info(None, None, None) == _lib.EINVAL
    assert lib.itlumm_mlp_destroy(None) == _lib.OK
    assert lib.itlumm_mlp_create(None, None, 0, 0, None) == _lib.EINVAL


def test_no_cpu_fallback_in_product_path():
    """The product package never imports the oracle, and the binding has no numpy compute path."""
    pkg = os.path.join(ROOT, "paper_2207_05808_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            src = open(os.path.join(pkg, fn)).read()
            assert "import oracle" not in src and "from oracle" not in src, fn


def _build_c_smoke(tmp_path):
    import subprocess
    exe = str(tmp_path / "c_abi_smoke")
    lib_dir = os.path.dirname(_lib.LIB_PATH)
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "tests", "c_abi_smoke.c"), "-L", lib_dir, "-litlumm",
                        f"-Wl,-rpath,{lib_dir}", "-o", exe], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_header_is_plain_c_and_links(tmp_path):
    """include/itlumm.h compiles as C99 and the library links from C (no torch, no GPU needed)."""
    import subprocess
    r = subprocess.run([_build_c_smoke(tmp_path)], capture_output=True, text=True)
    assert r.returncode == 0 and r.stdout.startswith("ok 5"), (r.returncode, r.stdout, r.stderr)


@pytest.mark.gpu
def test_c_program_pushes_data_through_a_plan(tmp_path):
    """From plain C on the GPU: plan_create -> amm_host and a 1-layer mlp_forward_host give the
    hand-worked outputs in tests/c_abi_smoke.c bit for bit; lda < D is ESHAPE."""
    import subprocess
    r = subprocess.run([_build_c_smoke(tmp_path)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip() == "ok 5 gpu", (r.returncode, r.stdout, r.stderr)
