"""Thin Python binding over the C ABI (argument marshalling only).

torch tensors supply device memory (``data_ptr()``) and the stream
(``torch.cuda.current_stream().cuda_stream``); every step of the hot path runs in the CUDA
kernels of libitlumm.so.  Names follow include/itlumm.h."""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib

try:
    import torch
except ImportError:  # pragma: no cover
    torch = None


def _np_ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _ld(t):
    """Row stride in elements; a 1-row tensor's stride(0) is arbitrary in torch, so its row length."""
    return t.stride(0) if t.shape[0] > 1 else max(t.stride(0), t.shape[1])


def _stream(stream, device):
    """A raw cudaStream_t: `stream` (a torch.cuda.Stream or an int handle), else the current stream of
    the plan's device."""
    if stream is not None:
        return ctypes.c_void_p(int(getattr(stream, "cuda_stream", stream)))
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _check(t, name, dtypes, rows, cols, device=None):
    """Reject what the C ABI cannot detect from raw pointers: a tensor on the wrong device (or on the
    host when device memory is required), the wrong element type, too few rows or columns, or rows
    that are not unit-stride."""
    if t.dim() != 2:
        raise ValueError(f"{name} must be 2-D, got shape {tuple(t.shape)}")
    if device is None:
        if t.is_cuda:
            raise ValueError(f"{name} must be a host tensor")
    elif not t.is_cuda or t.device.index != device:
        raise ValueError(f"{name} must live on cuda:{device}, got {t.device}")
    if t.dtype not in dtypes:
        raise TypeError(f"{name} must be {' or '.join(str(d) for d in dtypes)}, got {t.dtype}")
    if t.shape[0] < rows or t.shape[1] < cols:
        raise ValueError(f"{name} is {tuple(t.shape)}, needs at least ({rows}, {cols})")
    if t.shape[0] > 1 and t.stride(1) != 1 and t.shape[1] > 1:
        raise ValueError(f"{name} rows must be contiguous (stride(1) == 1), got strides {t.stride()}")


def _dtype_code(t):
    if t.dtype == torch.float32:
        return _lib.F32
    if t.dtype in (torch.bfloat16, torch.int16, torch.uint16):
        return _lib.BF16
    raise TypeError(f"A must be float32 or bfloat16, got {t.dtype}")


def _params_struct(params: dict):
    """itlumm_params for a fitted layer dict; returns (struct, arrays kept alive)."""
    D, C, M = int(params["D"]), int(params["C"]), int(params["M"])
    keep = dict(
        perm=np.ascontiguousarray(params["perm"], np.int32) if params.get("perm") is not None else None,
        boundaries=(np.ascontiguousarray(params["boundaries"], np.int32)
                    if params.get("boundaries") is not None else None),
        split_dim=np.ascontiguousarray(params["split_dim"], np.int32),
        thresholds=np.ascontiguousarray(params["thresholds"], np.float32),
        lut=np.ascontiguousarray(params["lut"], np.uint8),
        scale=np.ascontiguousarray(params["scale"], np.float32),
        offset=np.ascontiguousarray(params["offset"], np.float32),
        bias=np.ascontiguousarray(params["bias"], np.float32) if params.get("bias") is not None else None,
    )
    p = _lib.Params(D, C, M, *[_np_ptr(keep[k]) for k in
                               ("perm", "boundaries", "split_dim", "thresholds", "lut", "scale",
                                "offset", "bias")])
    return p, keep


def _a_dtypes():
    return (torch.float32, torch.bfloat16, torch.int16, torch.uint16)


class Plan:
    """An immutable ITLUMM layer on one GPU (itlumm_plan)."""

    def __init__(self, params: dict, device: int = 0, algo: str = "auto"):
        self._lib = _lib.load()
        D, C, M = int(params["D"]), int(params["C"]), int(params["M"])
        p, keep = _params_struct(params)
        h = ctypes.c_void_p()
        _lib.check(self._lib.itlumm_plan_create(ctypes.byref(p), int(device), ctypes.byref(h)))
        self._h = h
        self.D, self.C, self.M, self.device = D, C, M, int(device)
        self.summation, self.onehot = "exact", "auto"
        self.set_algo(algo)

    def close(self):
        if getattr(self, "_h", None):
            self._lib.itlumm_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_algo(self, algo: str):
        _lib.check(self._lib.itlumm_plan_set_algo(self._h, _lib.ALGO[algo]))
        self.algo = algo

    def set_summation(self, summation: str):
        """"exact" (default) or "avg16" (MADDNESS rounded averaging tree; C % 16 == 0)."""
        _lib.check(self._lib.itlumm_plan_set_summation(self._h, _lib.SUMMATION[summation]))
        self.summation = summation

    def set_onehot(self, onehot: str):
        """"auto" (default: the library's choice), "dense" or "sparse24": the one-hot operand of
        the tensor-core paths (tcgen05.mma.sp for the 2:4-sparse form); bit-identical
        results."""
        _lib.check(self._lib.itlumm_plan_set_onehot(self._h, _lib.ONEHOT[onehot]))
        self.onehot = onehot

    @property
    def last_launch_count(self) -> int:
        return int(self._lib.itlumm_last_launch_count())

    # ------------------------------------------------------------------ device-pointer calls
    def encode(self, A, codes=None, stream=None):
        """a1+a2: A [N, lda>=D] fp32/bf16 on the plan's device -> packed codes [N, ceil(C/2)] u8."""
        N = A.shape[0]
        _dtype_code(A)
        _check(A, "A", _a_dtypes(), 0, self.D, self.device)
        if codes is None:
            codes = torch.empty((N, (self.C + 1) // 2), dtype=torch.uint8, device=A.device)
        _check(codes, "codes", (torch.uint8,), N, (self.C + 1) // 2, self.device)
        _lib.check(self._lib.itlumm_encode(self._h, ctypes.c_void_p(A.data_ptr()), _dtype_code(A),
                                           _ld(A), N, ctypes.c_void_p(codes.data_ptr()),
                                           _ld(codes), _stream(stream, self.device)))
        return codes

    def lut_accumulate(self, codes, out=None, acc=None, relu=False, want_out=True, stream=None):
        """a3(+a4): packed codes -> fp32 out [N, M] (and/or int32 acc [N, M])."""
        N = codes.shape[0]
        _check(codes, "codes", (torch.uint8,), 0, (self.C + 1) // 2, self.device)
        if out is None and want_out:
            out = torch.empty((N, self.M), dtype=torch.float32, device=codes.device)
        if out is not None:
            _check(out, "out", (torch.float32,), N, self.M, self.device)
        if acc is not None:
            _check(acc, "acc", (torch.int32,), N, self.M, self.device)
        _lib.check(self._lib.itlumm_lut_accumulate(
            self._h, ctypes.c_void_p(codes.data_ptr()), _ld(codes), N,
            ctypes.c_void_p(acc.data_ptr()) if acc is not None else None,
            _ld(acc) if acc is not None else self.M,
            ctypes.c_void_p(out.data_ptr()) if out is not None else None,
            _ld(out) if out is not None else self.M,
            _lib.EPI_RELU if relu else _lib.EPI_NONE, _stream(stream, self.device)))
        return out, acc

    def amm(self, A, out=None, relu=False, stream=None):
        """Fused a1..a4: A [N, lda>=D] -> out [N, M] fp32 (codes never reach HBM)."""
        N = A.shape[0]
        _dtype_code(A)
        _check(A, "A", _a_dtypes(), 0, self.D, self.device)
        if out is None:
            out = torch.empty((N, self.M), dtype=torch.float32, device=A.device)
        _check(out, "out", (torch.float32,), N, self.M, self.device)
        _lib.check(self._lib.itlumm_amm(self._h, ctypes.c_void_p(A.data_ptr()), _dtype_code(A),
                                        _ld(A), N, ctypes.c_void_p(out.data_ptr()),
                                        _ld(out), _lib.EPI_RELU if relu else _lib.EPI_NONE,
                                        _stream(stream, self.device)))
        return out

    # ------------------------------------------------------------------ host-buffer call
    def amm_host(self, A, out=None, relu=False, stream=None):
        """End-to-end: HOST rows (torch CPU tensor, pinned is fastest) -> HOST out [N, M] fp32.
        Blocking; H2D / kernel / D2H are pipelined inside the library."""
        N = A.shape[0]
        _dtype_code(A)
        _check(A, "A", _a_dtypes(), 0, self.D)
        if out is None:
            out = torch.empty((N, self.M), dtype=torch.float32, pin_memory=A.is_pinned())
        _check(out, "out", (torch.float32,), N, self.M)
        _lib.check(self._lib.itlumm_amm_host(self._h, ctypes.c_void_p(A.data_ptr()), _dtype_code(A),
                                             _ld(A), N, ctypes.c_void_p(out.data_ptr()),
                                             _ld(out), _lib.EPI_RELU if relu else _lib.EPI_NONE,
                                             _stream(stream, self.device)))
        return out


class Mlp:
    """A chain of ITLUMM layers on one GPU (itlumm_mlp): each hidden layer computes only the output
    columns the next layer splits on (include/itlumm.h "Whole-network chaining")."""

    def __init__(self, layers: list, relus: list, device: int = 0):
        self._lib = _lib.load()
        structs, keeps = zip(*[_params_struct(p) for p in layers])
        arr = (_lib.Params * len(structs))(*structs)
        epis = (ctypes.c_int * len(relus))(*[_lib.EPI_RELU if r else _lib.EPI_NONE for r in relus])
        h = ctypes.c_void_p()
        _lib.check(self._lib.itlumm_mlp_create(ctypes.cast(arr, ctypes.c_void_p), ctypes.cast(epis, ctypes.c_void_p),
                                               len(structs), int(device), ctypes.byref(h)))
        self._h = h
        self.n_layers = len(structs)
        self.D, self.M, self.device = int(layers[0]["D"]), int(layers[-1]["M"]), int(device)

    def widths(self) -> list:
        w = (ctypes.c_int32 * self.n_layers)()
        _lib.check(self._lib.itlumm_mlp_info(self._h, None, ctypes.cast(w, ctypes.c_void_p)))
        return list(w)

    @property
    def last_launch_count(self) -> int:
        return int(self._lib.itlumm_last_launch_count())

    def forward(self, A, out=None, stream=None):
        N = A.shape[0]
        _dtype_code(A)
        _check(A, "A", _a_dtypes(), 0, self.D, self.device)
        if out is None:
            out = torch.empty((N, self.M), dtype=torch.float32, device=A.device)
        _check(out, "out", (torch.float32,), N, self.M, self.device)
        _lib.check(self._lib.itlumm_mlp_forward(self._h, ctypes.c_void_p(A.data_ptr()), _dtype_code(A),
                                                _ld(A), N, ctypes.c_void_p(out.data_ptr()),
                                                _ld(out), _stream(stream, self.device)))
        return out

    def forward_host(self, A, out=None, stream=None):
        """End-to-end: HOST rows (pinned is fastest) -> HOST logits; blocking, the library pipelines
        H2D / forward / D2H (itlumm_mlp_forward_host)."""
        N = A.shape[0]
        _dtype_code(A)
        _check(A, "A", _a_dtypes(), 0, self.D)
        if out is None:
            out = torch.empty((N, self.M), dtype=torch.float32, pin_memory=A.is_pinned())
        _check(out, "out", (torch.float32,), N, self.M)
        _lib.check(self._lib.itlumm_mlp_forward_host(self._h, ctypes.c_void_p(A.data_ptr()), _dtype_code(A),
                                                     _ld(A), N, ctypes.c_void_p(out.data_ptr()),
                                                     _ld(out), _stream(stream, self.device)))
        return out

    def close(self):
        if getattr(self, "_h", None):
            self._lib.itlumm_mlp_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
