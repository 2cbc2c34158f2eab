"""Drop-in proof: the dash::gpu shim (integration/garble_gpu.cpp, the code
INTEGRATION.md tells a maintainer to add to proj/core) compiled against the
reference's own headers and linked with the unmodified reference sources
plus libdashgpu.so (oracle/Makefile target `shim` -> oracle/_ref/shim_check).

CPU: the binary exists, links libdashgpu.so, and without a GPU fails loudly
(no CPU fallback).  GPU: every check of integration/shim_check.cpp passes:
dash::gpu::garble artifacts byte-identical to dash::garble, dash::gpu::evaluate
equal to dash::evaluate, decode == circuit_plain_forward, AuthenticityError /
DataError through the shim.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHIM = os.path.join(ROOT, "oracle", "_ref", "shim_check")

need_shim = pytest.mark.skipif(not os.path.exists(SHIM), reason="oracle/_ref/shim_check not built "
                                                                 "(needs /root/reference at build time)")


@need_shim
def test_shim_links_the_engine_and_the_reference():
    out = subprocess.run(["ldd", SHIM], capture_output=True, text=True).stdout
    assert "libdashgpu.so" in out and "not found" not in out
    syms = subprocess.run(["nm", "-C", SHIM], capture_output=True, text=True).stdout
    # the reference's own garble / evaluate / parsers are linked in, next to the shim
    for s in ("dash::garble(", "dash::evaluate(", "dash::parse_garbled_circuit(", "dash::gpu::garble(",
              "dash::gpu::evaluate("):
        assert s in syms, s


@need_shim
def test_shim_without_gpu_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    r = subprocess.run([SHIM], capture_output=True, text=True, timeout=300)
    assert r.returncode != 0
    assert "FAIL" in r.stdout


@pytest.mark.gpu
@need_shim
def test_shim_is_a_drop_in_for_the_reference_api():
    r = subprocess.run([SHIM], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "shim check: all passed" in r.stdout
    for m in ("model_tiny", "model_tiny_priv", "model_a", "model_c", "model_d", "model_tiny_batch", "malformed_gc"):
        assert f"ok {m}" in r.stdout
