"""paper_2409_15053_b200 — B200-native filtered Lanczos eigensolver (filter-and-Lanczos hot path).

The product is ``libflz.so`` (hand-written sm_100a CUDA behind the C ABI of include/flz.h plus
the C++ host solver mirroring the reference's ``speig`` API).  This package only binds it.
"""
from . import _lib  # noqa: F401
from ._lib import FlzConfig, FlzError, FlzStats, build, lib  # noqa: F401
from .device import Basis, Context, DeviceMatrix, LoopHub  # noqa: F401

__all__ = ["Basis", "Context", "DeviceMatrix", "LoopHub", "FlzConfig", "FlzError", "FlzStats", "build", "lib"]
