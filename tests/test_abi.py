"""The C-ABI boundary: libdashgpu.so loads, exports every entry point that
include/dashgpu.h declares, refuses to run without a GPU (no CPU fallback),
and its host-only services (model builders, layout, tape) work on any machine.
"""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import CUDA_LIB, ROOT
from helpers import models


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "dashgpu.h")).read()
    return sorted(set(re.findall(r"\b(dashgpu_\w+)\s*\(", text)))


def test_header_declares_the_reference_api():
    syms = declared_symbols()
    for s in ["dashgpu_garble", "dashgpu_garble_inputs", "dashgpu_evaluate", "dashgpu_decode_outputs",
              "dashgpu_export_gc", "dashgpu_export_encoding", "dashgpu_export_decoding", "dashgpu_export_bundle",
              "dashgpu_import_bundle", "dashgpu_import_gc", "dashgpu_infer", "dashgpu_circuit_create"]:
        assert s in syms


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(CUDA_LIB)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2302_06361_b200.engine import CudaError, Dash

    with pytest.raises(CudaError):
        Dash(0)


def test_host_only_model_builders_and_layout():
    # circuit_layout / count_circuit (garble.cpp:16-42, circuit.cpp:127-142)
    # are host logic: the numbers below are the reference's.
    from paper_2302_06361_b200.engine import _declare, CircuitInfo

    lib = ctypes.CDLL(CUDA_LIB)
    _declare(lib)
    for name, seed, k, cts in [("model_a", 1001, 8, 426752), ("model_tiny", 1000, 8, 101007),
                               ("lenet5", 2001, 8, 7808228)]:
        h = ctypes.c_void_p()
        assert lib.dashgpu_model_build(name.encode(), seed, k, 0, ctypes.byref(h)) == 0
        info = CircuitInfo()
        assert lib.dashgpu_circuit_info_get(h, ctypes.byref(info)) == 0
        assert info.cts == cts, name
        assert list(info.radices[: info.sign_t]) == [110, 8, 7, 7, 6, 6, 5, 5]
        assert info.act_uc_cts == 1667 and info.act_eval_rows == 170
        lib.dashgpu_circuit_destroy(h)


def test_model_builders_match_reference_draws():
    # model_a's first weights, drawn by std::mt19937(1001) +
    # uniform_int_distribution<int>(-2, 2) exactly as test_models.hpp:31-42
    c = models.build("model_a", 1001, 8)
    assert c.layers[0].q_weights[:10].tolist() == [-1, -1, -1, 0, -2, -1, 0, 0, -2, 0]
    assert [l.kind for l in models.build("lenet5", 2001, 8).layers] == [2, 3, 2, 2, 3, 2, 5, 1, 3, 1, 3, 1]


def test_bad_circuits_raise_data_error():
    from paper_2302_06361_b200.circuit import Circuit, dense, relu
    from paper_2302_06361_b200.engine import _declare

    lib = ctypes.CDLL(CUDA_LIB)
    _declare(lib)
    bad = Circuit([4], 8, [dense(5, 3, np.zeros(15), np.zeros(3)), relu()])  # shape mismatch
    h = ctypes.c_void_p()
    desc = bad.to_desc()
    assert lib.dashgpu_circuit_create(ctypes.byref(desc), ctypes.byref(h)) == 3
    bad = Circuit([4], 17, [relu()])  # k out of range
    desc = bad.to_desc()
    assert lib.dashgpu_circuit_create(ctypes.byref(desc), ctypes.byref(h)) == 3


def test_bad_extension_circuits_raise_data_error(oracle):
    # Pad2d / Add / DAG inputs (include/dash_circuit_desc.h) are validated by
    # the engine and the oracle alike
    from paper_2302_06361_b200.circuit import Circuit, add, dense, pad2d, relu
    from paper_2302_06361_b200.engine import _declare
    from pyoracle import CheckerError

    lib = ctypes.CDLL(CUDA_LIB)
    _declare(lib)
    cases = [
        Circuit([4], 8, [pad2d(1)]),                                     # pad needs [C][H][W]
        Circuit([4], 8, [relu(), add(3)]),                               # add operand from a later layer
        Circuit([4], 8, [dense(4, 3, np.zeros(12), np.zeros(3)), add(-1)]),  # add shapes differ (3 vs 4)
        Circuit([4], 8, [relu(src=2)]),                                  # input from a later layer
    ]
    for bad in cases:
        h = ctypes.c_void_p()
        desc = bad.to_desc()
        assert lib.dashgpu_circuit_create(ctypes.byref(desc), ctypes.byref(h)) == 3, bad
        with pytest.raises(CheckerError):
            oracle.circuit(bad)


def test_import_gc_rejects_bad_arguments_without_a_device():
    # argument and file checks come before any device work (host-only path)
    lib = ctypes.CDLL(CUDA_LIB)
    vp = ctypes.c_void_p
    out = vp()
    assert lib.dashgpu_import_gc(None, None, 1, ctypes.byref(out)) == 3  # DASHGPU_ERR_DATA
    data = ctypes.c_char_p(b"DASH\x01\x00\x02" + bytes(64))          # wrong file kind
    ptrs = (ctypes.c_char_p * 1)(data)
    lens = (ctypes.c_size_t * 1)(71)
    assert lib.dashgpu_import_gc(ptrs, lens, 0, ctypes.byref(out)) == 3  # empty batch
    assert lib.dashgpu_import_gc(ptrs, lens, 1, ctypes.byref(out)) == 3
    lib.dashgpu_last_error.restype = ctypes.c_char_p
    assert b"kind" in lib.dashgpu_last_error()
    assert lib.dashgpu_network_circuit(None, ctypes.byref(out)) == 3


def test_emulation_library_is_refused_by_the_product_api():
    """Dash() only runs the CUDA engine: the tests' CPU emulation of the
    device code (tests/emu) loads only with the explicit test flag."""
    from conftest import EMU_LIB
    from paper_2302_06361_b200.engine import CudaError, Dash

    if not os.path.exists(EMU_LIB):
        pytest.skip("emulation library not built")
    with pytest.raises(CudaError, match="not the CUDA engine"):
        Dash(lib_path=EMU_LIB)
    assert Dash(lib_path=EMU_LIB, emulation=True).lib.dashgpu_backend() == 2
