"""ctypes loader for libitlumm.so (the C ABI of include/itlumm.h).

Fails loudly: there is no CPU fallback for any step of the hot path."""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libitlumm.so")
# developer A/B runs only (tools/): another build of the same library; never set by the tests or bench
LIB_PATH = os.environ.get("ITLUMM_DEV_LIB", LIB_PATH)

OK, EINVAL, ESHAPE, EUNSUPPORTED, ECUDA, ENOMEM = range(6)
STATUS_NAMES = {0: "OK", 1: "EINVAL", 2: "ESHAPE", 3: "EUNSUPPORTED", 4: "ECUDA", 5: "ENOMEM"}
F32, BF16 = 0, 1
EPI_NONE, EPI_RELU = 0, 1
ALGO = {"auto": 0, "simt": 1, "tc": 2, "tc_pipe": 3}
SUMMATION = {"exact": 0, "avg16": 1}
ONEHOT = {"auto": 0, "dense": 1, "sparse24": 2}

# every symbol include/itlumm.h declares (checked by tests/test_abi.py against the header)
EXPORTS = [
    "itlumm_plan_create", "itlumm_plan_destroy", "itlumm_plan_set_algo", "itlumm_plan_set_summation",
    "itlumm_plan_set_onehot", "itlumm_plan_info",
    "itlumm_encode", "itlumm_lut_accumulate", "itlumm_amm", "itlumm_amm_host",
    "itlumm_mlp_create", "itlumm_mlp_destroy", "itlumm_mlp_info", "itlumm_mlp_forward", "itlumm_mlp_forward_host",
    "itlumm_last_launch_count", "itlumm_last_error", "itlumm_abi_version",
]


class ItlummError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class Params(ctypes.Structure):
    _fields_ = [("D", ctypes.c_int32), ("C", ctypes.c_int32), ("M", ctypes.c_int32),
                ("perm", ctypes.c_void_p), ("boundaries", ctypes.c_void_p),
                ("split_dim", ctypes.c_void_p), ("thresholds", ctypes.c_void_p),
                ("lut", ctypes.c_void_p), ("scale", ctypes.c_void_p),
                ("offset", ctypes.c_void_p), ("bias", ctypes.c_void_p)]


_lib = None


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2207_05808_b200.build` "
                          "(nvcc, sm_100a). There is no CPU fallback.")
    lib = ctypes.CDLL(LIB_PATH)
    V, I64, I32, S = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int
    sig = {
        "itlumm_plan_create": ([ctypes.POINTER(Params), S, ctypes.POINTER(V)], S),
        "itlumm_plan_destroy": ([V], S),
        "itlumm_plan_set_algo": ([V, S], S),
        "itlumm_plan_set_summation": ([V, S], S),
        "itlumm_plan_set_onehot": ([V, S], S),
        "itlumm_plan_info": ([V, V, V, V, V], S),
        "itlumm_encode": ([V, V, S, I64, I64, V, I64, V], S),
        "itlumm_lut_accumulate": ([V, V, I64, I64, V, I64, V, I64, S, V], S),
        "itlumm_amm": ([V, V, S, I64, I64, V, I64, S, V], S),
        "itlumm_amm_host": ([V, V, S, I64, I64, V, I64, S, V], S),
        "itlumm_mlp_create": ([V, V, I32, S, ctypes.POINTER(V)], S),
        "itlumm_mlp_destroy": ([V], S),
        "itlumm_mlp_info": ([V, V, V], S),
        "itlumm_mlp_forward": ([V, V, S, I64, I64, V, I64, V], S),
        "itlumm_mlp_forward_host": ([V, V, S, I64, I64, V, I64, V], S),
        "itlumm_last_launch_count": ([], I32),
        "itlumm_last_error": ([], ctypes.c_char_p),
        "itlumm_abi_version": ([], I32),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes, fn.restype = args, res
    _lib = lib
    return lib


def check(status: int):
    if status != OK:
        raise ItlummError(status, load().itlumm_last_error().decode())
