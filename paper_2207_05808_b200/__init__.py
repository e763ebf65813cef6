"""B200-native ITLUMM / MADDNESS inference hot path (arXiv 2207.05808).

  Plan        — an ITLUMM layer on one GPU (C ABI: include/itlumm.h, libitlumm.so)
  fit_layer   — offline host fit of trees + uint8 LUT (fit-time, not the hot path)
  dist        — row sharding over ranks and the one-time parameter broadcast
"""
from .api import Plan, Mlp  # noqa: F401
from .fit import fit_layer, fit_mlp, chunk_bounds, split_packed  # noqa: F401
from . import _lib  # noqa: F401

__all__ = ["Plan", "Mlp", "fit_layer", "fit_mlp", "chunk_bounds", "split_packed"]
