"""ORACLE for the ITLUMM hot path — TEST INFRASTRUCTURE, NOT PRODUCT CODE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg (and
``bench.py --impl reference``) may import, call, link or execute anything under ``oracle/``.
The product library (``paper_2207_05808_b200``) never imports it, and this package never
imports the product library: the two share no code, headers, tables or constant generators.
Only ``synth`` (seeded raw inputs, no method arithmetic) serves both.

Contents
  fit.py    offline fit in fp64: partition, depth-4 trees, prototypes, LUT, uint8 quantisation
  infer.c   inference in plain C: permute -> slice -> 4 compares -> integer sum -> fmaf dequant
Pins: tests/test_oracle_pins.py (-m "not gpu").  Parity unpinned: the tree-fit rule at
BASELINE scale (readings R3-R5, no printed values anywhere) — see DESIGN.md.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

from . import fit  # noqa: F401  (re-export)

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "infer.c")
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle_itlumm.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile infer.c with gcc (-O2 -ffp-contract=off: fmaf is the only fused op)."""
    os.makedirs(os.path.dirname(_LIB_PATH), exist_ok=True)
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11",
                               "-shared", "-fPIC", "-pthread", _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            P = ctypes.c_void_p
            lib.oracle_amm.argtypes = [ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                       P, ctypes.c_int, ctypes.c_int64, P, P, P, P, P, P, P, P,
                                       ctypes.c_int, P, P, P, ctypes.c_int]
            lib.oracle_amm.restype = ctypes.c_int
            lib.oracle_amm2.argtypes = lib.oracle_amm.argtypes + [ctypes.c_int]
            lib.oracle_amm2.restype = ctypes.c_int
            _lib = lib
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def amm(params: dict, A: np.ndarray, relu: bool, dtype: str = "f32", want_codes: bool = False,
        want_acc: bool = False, want_y: bool = True, nthreads: int = 1, summation: str = "exact"):
    """Run the oracle inference on rows A (N x lda; fp32, or uint16 bf16 bits when dtype='bf16').
    summation: "exact" (reading R7) or "avg16" (MADDNESS rounded averaging tree, reading R22).

    Returns dict(codes=[N][C] uint8 or None, acc=[N][M] int64 or None, y=[N][M] fp32 or None)."""
    lib = _load()
    A = np.ascontiguousarray(A)
    N = A.shape[0]
    D, C, M = int(params["D"]), int(params["C"]), int(params["M"])
    lda = A.shape[1] if A.ndim == 2 else D
    if dtype == "f32":
        A = A.astype(np.float32, copy=False)
        dt = 0
    else:
        A = A.astype(np.uint16, copy=False)
        dt = 1
    perm = np.ascontiguousarray(params["perm"], dtype=np.int32)
    bnd = np.ascontiguousarray(params["boundaries"], dtype=np.int32)
    sd = np.ascontiguousarray(params["split_dim"], dtype=np.int32)
    thr = np.ascontiguousarray(params["thresholds"], dtype=np.float32)
    lut = np.ascontiguousarray(params["lut"], dtype=np.uint8)
    scale = np.ascontiguousarray(params["scale"], dtype=np.float32)
    off = np.ascontiguousarray(params["offset"], dtype=np.float32)
    bias = params.get("bias")
    bias = None if bias is None else np.ascontiguousarray(bias, dtype=np.float32)
    codes = np.zeros((N, C), dtype=np.uint8) if want_codes else None
    acc = np.zeros((N, M), dtype=np.int64) if want_acc else None
    y = np.zeros((N, M), dtype=np.float32) if want_y else None
    st = lib.oracle_amm2(N, D, C, M, _ptr(A), dt, lda, _ptr(perm), _ptr(bnd), _ptr(sd), _ptr(thr),
                         _ptr(lut), _ptr(scale), _ptr(off), _ptr(bias), int(bool(relu)),
                         _ptr(codes), _ptr(acc), _ptr(y), int(nthreads),
                         {"exact": 0, "avg16": 1}[summation])
    if st != 0:
        raise RuntimeError(f"oracle_amm failed with status {st}")
    return dict(codes=codes, acc=acc, y=y)


def fit_mlp(A_train: np.ndarray, Bs: list, Cs: list, perms: list, biases: list, relus: list,
            a_is_bf16: bool = False, nthreads: int = 8) -> list:
    """Fit an MLP whose linear layers are all ITLUMM (BASELINE configs[3]): layer l+1
    is fit on layer l's ITLUMM outputs of the training rows, computed by this
    oracle's inference."""
    X = np.asarray(A_train)
    layers = []
    for l, (B, C, perm, bias, relu) in enumerate(zip(Bs, Cs, perms, biases, relus)):
        bf = a_is_bf16 and l == 0
        p = fit.fit(X, B, C, perm, bias, a_is_bf16=bf)
        layers.append(p)
        if l + 1 < len(Bs):
            X = amm(p, X, relu=relu, dtype="bf16" if bf else "f32", nthreads=nthreads)["y"]
    return layers


def mlp_forward(layers: list, relus: list, A: np.ndarray, a_is_bf16: bool = False, nthreads: int = 8):
    """Every layer computed in full, output fed to the next (O9)."""
    X = A
    for l, (p, relu) in enumerate(zip(layers, relus)):
        X = amm(p, X, relu=relu, dtype="bf16" if (a_is_bf16 and l == 0) else "f32", nthreads=nthreads)["y"]
    return X
