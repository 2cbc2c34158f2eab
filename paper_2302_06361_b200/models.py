"""Deterministic synthetic models (host only, no GPU needed).

The builders live in the product library (engine.cpp ``models::build``) so
that the weights are drawn exactly as the reference's
``tests/support/test_models.hpp:21-145`` draws them (std::mt19937 +
std::uniform_int_distribution<int>): model_a, model_c, model_d, model_f_dims,
model_tiny, plus the benchmark configurations of SURVEY.md §8(d): ``lenet5``
(LeNet-5 restated in reference ops), ``minionn`` (paper Model F, ReLU) and
single-layer ``relu<N>`` / ``sign<N>`` / ``dense<N>`` sweeps.
"""
from __future__ import annotations

import ctypes
import os

from .circuit import Circuit, CircuitDesc
from .engine import LIB_PATH, _declare, CudaError

_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise CudaError(f"{LIB_PATH} is not built; run __graft_entry__.build()")
        _lib = ctypes.CDLL(LIB_PATH)
        _declare(_lib)
    return _lib


def build(name: str, seed: int, k: int = 8, private: bool = False) -> Circuit:
    L = _load()
    h = ctypes.c_void_p()
    rc = L.dashgpu_model_build(name.encode(), seed, k, 1 if private else 0, ctypes.byref(h))
    if rc:
        raise RuntimeError(L.dashgpu_last_error().decode())
    try:
        d = CircuitDesc()
        rc = L.dashgpu_circuit_desc_view(h, ctypes.byref(d))
        if rc:
            raise RuntimeError(L.dashgpu_last_error().decode())
        return Circuit.from_desc(d)
    finally:
        L.dashgpu_circuit_destroy(h)
