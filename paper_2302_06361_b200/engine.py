"""Python mirror of the reference's whole-network API over the C ABI.

Names and argument meaning follow ``dash::garble`` / ``garble_inputs`` /
``evaluate`` / ``decode_outputs`` (reference
``proj/core/include/dash/garble.hpp:93-112``); errors follow
``proj/core/include/dash/errors.hpp:9-34`` (``DataError``, ``OverflowError``
(a DataError), ``AuthenticityError``).  Every call is batched over
independent inferences, one 16-byte seed each.

The compute path is libdashgpu.so (CUDA, sm_100a).  There is no CPU fallback:
constructing ``Dash()`` without the built library or without a CUDA device
raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

from .circuit import PRIMES, Circuit, CircuitDesc

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libdashgpu.so")

vp = ctypes.c_void_p
u8p = ctypes.POINTER(ctypes.c_uint8)
u16p = ctypes.POINTER(ctypes.c_uint16)


def _n_digits(m: int) -> int:
    """Digits of a label mod m (reference label.cpp:15-29): largest n with m^n <= 2^128."""
    n, v = 0, 1
    while v * m <= (1 << 128):
        v *= m
        n += 1
    return n
u64p = ctypes.POINTER(ctypes.c_uint64)
i64p = ctypes.POINTER(ctypes.c_int64)
f64p = ctypes.POINTER(ctypes.c_double)


class Error(RuntimeError):
    """dash::Error"""


class DataError(Error):
    """dash::DataError (CLI exit 3)"""


class OverflowError_(DataError):
    """dash::OverflowError"""


class AuthenticityError(Error):
    """dash::AuthenticityError (CLI exit 4)"""


class CudaError(Error):
    """CUDA runtime failure (no device, launch failure, out of memory)."""


_CODES = {1: Error, 2: CudaError, 3: DataError, 4: AuthenticityError, 5: OverflowError_}


class CircuitInfo(ctypes.Structure):
    _fields_ = [
        ("k", ctypes.c_int32),
        ("n_layers", ctypes.c_uint32),
        ("n_in", ctypes.c_uint64),
        ("n_out", ctypes.c_uint64),
        ("cts", ctypes.c_uint64),
        ("gates", ctypes.c_uint64),
        ("wires", ctypes.c_uint64),
        ("sign_t", ctypes.c_uint32),
        ("radices", ctypes.c_uint16 * 32),
        ("relu_elements", ctypes.c_uint64),
        ("linear_macs", ctypes.c_uint64),
        ("act_uc_cts", ctypes.c_uint64),
        ("act_eval_rows", ctypes.c_uint64),
        ("max_slots", ctypes.c_uint32),
    ]


# dashgpu_gc_sink: (user, inference, data, len) -> 0 to continue
GC_SINK = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_uint32, ctypes.POINTER(ctypes.c_uint8),
                           ctypes.c_size_t)


class Timing(ctypes.Structure):
    _fields_ = [
        ("ms_garble", ctypes.c_double),
        ("ms_encode", ctypes.c_double),
        ("ms_evaluate", ctypes.c_double),
        ("ms_decode", ctypes.c_double),
        ("ms_total", ctypes.c_double),
        ("h2d_bytes", ctypes.c_uint64),
        ("d2h_bytes", ctypes.c_uint64),
        ("sub_batches", ctypes.c_uint32),
        ("layerwise", ctypes.c_uint32),
    ]


KERNEL_KINDS = ["act_garble", "act_eval", "linear", "priv_garble", "priv_eval", "setup", "encode", "decode", "misc"]


def _declare(L):
    L.dashgpu_last_error.restype = ctypes.c_char_p
    L.dashgpu_backend.restype = ctypes.c_int
    L.dashgpu_init.argtypes = [ctypes.c_int]
    L.dashgpu_set_stream.argtypes = [vp]
    L.dashgpu_use.argtypes = [ctypes.c_int, vp]
    L.dashgpu_network_release_gc.argtypes = [vp]
    L.dashgpu_circuit_create.argtypes = [vp, ctypes.POINTER(vp)]
    L.dashgpu_circuit_destroy.argtypes = [vp]
    L.dashgpu_circuit_info_get.argtypes = [vp, ctypes.POINTER(CircuitInfo)]
    L.dashgpu_model_build.argtypes = [ctypes.c_char_p, ctypes.c_uint32, ctypes.c_int, ctypes.c_int,
                                      ctypes.POINTER(vp)]
    L.dashgpu_circuit_desc_view.argtypes = [vp, ctypes.POINTER(CircuitDesc)]
    L.dashgpu_random_input.argtypes = [vp, ctypes.c_uint32, ctypes.c_int, ctypes.c_int, i64p]
    L.dashgpu_plain_forward.argtypes = [vp, i64p, i64p]
    L.dashgpu_garble.argtypes = [vp, u8p, ctypes.c_uint32, ctypes.POINTER(vp)]
    L.dashgpu_network_destroy.argtypes = [vp]
    L.dashgpu_garble_inputs.argtypes = [vp, i64p, ctypes.POINTER(vp)]
    L.dashgpu_evaluate.argtypes = [vp, vp, ctypes.POINTER(vp)]
    L.dashgpu_decode_outputs.argtypes = [vp, vp, i64p]
    L.dashgpu_bundle_destroy.argtypes = [vp]
    for n in ("dashgpu_export_gc", "dashgpu_export_encoding", "dashgpu_export_decoding", "dashgpu_export_bundle"):
        getattr(L, n).argtypes = [vp, ctypes.c_uint32, u8p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]
    L.dashgpu_import_bundle.argtypes = [vp, u8p, ctypes.c_size_t, ctypes.c_int, ctypes.POINTER(vp)]
    L.dashgpu_import_gc.argtypes = [ctypes.POINTER(u8p), ctypes.POINTER(ctypes.c_size_t), ctypes.c_uint32,
                                    ctypes.POINTER(vp)]
    L.dashgpu_import_gc_host.argtypes = L.dashgpu_import_gc.argtypes
    L.dashgpu_network_circuit.argtypes = [vp, ctypes.POINTER(vp)]
    L.dashgpu_tamper_ct.argtypes = [vp, ctypes.c_uint32, ctypes.c_uint64, u8p]
    L.dashgpu_infer.argtypes = [vp, vp, ctypes.c_uint32, vp, vp, ctypes.c_int, ctypes.POINTER(Timing)]
    L.dashgpu_garble_digest.argtypes = [vp, u8p, ctypes.c_uint32, u8p]
    L.dashgpu_network_digest.argtypes = [vp, ctypes.c_uint32, u8p]
    L.dashgpu_garble_stream.argtypes = [vp, u8p, ctypes.c_uint32, GC_SINK, vp, ctypes.POINTER(vp)]
    L.dashgpu_infer_stream.argtypes = [vp, vp, ctypes.c_uint32, vp, vp, ctypes.c_uint64, vp, ctypes.POINTER(Timing)]
    L.dashgpu_infer_stream_range.argtypes = [vp, vp, ctypes.c_uint32, vp, vp, ctypes.c_uint64, ctypes.c_uint64,
                                             ctypes.c_uint64, vp, ctypes.POINTER(Timing)]
    L.dashgpu_network_setup.argtypes = [vp, u8p, ctypes.c_uint32, ctypes.POINTER(vp)]
    L.dashgpu_input_base.argtypes = [vp, ctypes.POINTER(vp)]
    L.dashgpu_layer_garble.argtypes = [vp, ctypes.c_uint32, vp, vp, ctypes.POINTER(vp)]
    L.dashgpu_layer_eval.argtypes = [vp, ctypes.c_uint32, vp, vp, ctypes.POINTER(vp)]
    L.dashgpu_network_finish.argtypes = [vp, vp]
    L.dashgpu_layer_count.argtypes = [vp, ctypes.c_uint32, u64p]
    L.dashgpu_bundle_info.argtypes = [vp, ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_uint64)]
    L.dashgpu_bundle_from_labels.argtypes = [vp, ctypes.c_uint64, ctypes.POINTER(u16p), ctypes.c_int,
                                             ctypes.POINTER(vp)]
    L.dashgpu_bundle_labels.argtypes = [vp, ctypes.c_int, u16p]
    L.dashgpu_proj_garble.argtypes = [u8p, ctypes.c_uint32, ctypes.c_int, ctypes.c_int, u8p, u64p, u64p, u64p,
                                      u64p, u64p, u64p]
    L.dashgpu_proj_eval.argtypes = [ctypes.c_uint32, ctypes.c_int, ctypes.c_int, u64p, u64p, u64p, u64p]
    L.dashgpu_proj_ctx_create.argtypes = [u8p, ctypes.c_int, ctypes.c_int, u8p, ctypes.POINTER(vp)]
    L.dashgpu_proj_ctx_destroy.argtypes = [vp]
    L.dashgpu_proj_garble_dev.argtypes = [vp, ctypes.c_uint32, vp, vp, vp, vp, vp]
    L.dashgpu_proj_eval_dev.argtypes = [vp, ctypes.c_uint32, vp, vp, vp, vp]
    L.dashgpu_profile.argtypes = [ctypes.c_int]
    L.dashgpu_profile_read.argtypes = [f64p, u64p, ctypes.c_int]
    L.dashgpu_last_act_launch.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_uint32)]
    L.dashgpu_prim.argtypes = [ctypes.c_int, ctypes.c_uint32, ctypes.c_int, ctypes.c_int, u64p, u64p, u16p, u8p,
                               u64p, ctypes.c_uint64]


class Dash:
    """Handle to the device engine (one CUDA device)."""

    def __init__(self, device: int = 0, lib_path: Optional[str] = None, emulation: bool = False):
        """lib_path / DASHGPU_LIB: another build of libdashgpu.so (A/B of kernel
        variants).  Whatever is loaded must be the CUDA engine
        (dashgpu_backend() == 1); only the tests pass emulation=True to load
        their CPU emulation of the device code (tests/emu)."""
        path = lib_path or os.environ.get("DASHGPU_LIB") or LIB_PATH
        if not os.path.exists(path):
            raise CudaError(f"{path} is not built; run __graft_entry__.build()")
        self.lib = ctypes.CDLL(path)
        _declare(self.lib)
        if self.lib.dashgpu_backend() != 1 and not emulation:
            raise CudaError(f"{path} is not the CUDA engine (backend {self.lib.dashgpu_backend()}); "
                            "there is no CPU fallback")
        self._check(self.lib.dashgpu_init(device))

    def _check(self, rc: int):
        if rc:
            raise _CODES.get(rc, Error)(self.lib.dashgpu_last_error().decode())

    def set_stream(self, stream_ptr: int):
        """Stream of the calling host thread (thread-local in the library)."""
        self.lib.dashgpu_set_stream(vp(stream_ptr))

    def use(self, device: int, stream_ptr: int = 0):
        """Per-call device and stream for the calling host thread (dashgpu_use)."""
        self._check(self.lib.dashgpu_use(device, vp(stream_ptr)))

    # ---- circuits ----
    def circuit(self, c: Circuit) -> "GpuCircuit":
        desc = c.to_desc()
        h = vp()
        self._check(self.lib.dashgpu_circuit_create(ctypes.byref(desc), ctypes.byref(h)))
        return GpuCircuit(self, h)

    def model(self, name: str, seed: int, k: int = 8, private: bool = False) -> "GpuCircuit":
        h = vp()
        self._check(self.lib.dashgpu_model_build(name.encode(), seed, k, 1 if private else 0, ctypes.byref(h)))
        return GpuCircuit(self, h)

    # ---- whole-network API (garble.hpp:93-112), batched ----
    def garble(self, c: "GpuCircuit", seeds: bytes) -> "GarbledNetwork":
        if len(seeds) == 0 or len(seeds) % 16:
            raise DataError("seeds must be a non-empty multiple of 16 bytes")
        h = vp()
        buf = (ctypes.c_uint8 * len(seeds)).from_buffer_copy(seeds)
        self._check(self.lib.dashgpu_garble(c.h, buf, len(seeds) // 16, ctypes.byref(h)))
        return GarbledNetwork(self, h, c, len(seeds) // 16)

    def garble_digest(self, c: "GpuCircuit", seeds: bytes) -> np.ndarray:
        """Digest parity mode of streamed garbling: [batch][n_layers][32] tree
        SHA-256 of each layer's ciphertexts in the reference's cts order,
        garbled through a one-layer window (csrc/sha256.hpp)."""
        if len(seeds) == 0 or len(seeds) % 16:
            raise DataError("seeds must be a non-empty multiple of 16 bytes")
        batch = len(seeds) // 16
        buf = (ctypes.c_uint8 * len(seeds)).from_buffer_copy(seeds)
        out = np.zeros((batch, c.info.n_layers, 32), np.uint8)
        self._check(self.lib.dashgpu_garble_digest(c.h, buf, batch,
                                                   out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))))
        return out

    def garble_stream(self, c: "GpuCircuit", seeds: bytes, sink) -> "GarbledNetwork":
        """Streamed serialize_garbled_circuit: sink(b, chunk: bytes) receives
        inference b's GC bytes in order (their concatenation == export_gc(b));
        the device holds one layer's ciphertexts at a time.  Returns the
        network with encoding / decoding (its GC already released).  A sink
        that returns a truthy value or raises aborts the stream (DataError)."""
        if len(seeds) == 0 or len(seeds) % 16:
            raise DataError("seeds must be a non-empty multiple of 16 bytes")
        failure = []

        def cb(_user, b, data, n):
            try:
                return 1 if sink(int(b), ctypes.string_at(data, n)) else 0
            except BaseException as e:  # noqa: BLE001 -- re-raised below, never across the C frame
                failure.append(e)
                return 1

        fn = GC_SINK(cb)
        buf = (ctypes.c_uint8 * len(seeds)).from_buffer_copy(seeds)
        h = vp()
        rc = self.lib.dashgpu_garble_stream(c.h, buf, len(seeds) // 16, fn, None, ctypes.byref(h))
        if failure:
            raise failure[0]
        self._check(rc)
        return GarbledNetwork(self, h, c, len(seeds) // 16)

    def garble_inputs(self, net: "GarbledNetwork", values) -> "Bundle":
        v = np.ascontiguousarray(values, np.int64).reshape(net.batch, net.circuit.info.n_in)
        h = vp()
        self._check(self.lib.dashgpu_garble_inputs(net.h, v.ctypes.data_as(i64p), ctypes.byref(h)))
        return Bundle(self, h, net, False)

    def evaluate(self, net: "GarbledNetwork", inputs: "Bundle") -> "Bundle":
        h = vp()
        self._check(self.lib.dashgpu_evaluate(net.h, inputs.h, ctypes.byref(h)))
        return Bundle(self, h, net, True)

    def decode_outputs(self, net: "GarbledNetwork", outputs: "Bundle") -> np.ndarray:
        out = np.zeros((net.batch, net.circuit.info.n_out), np.int64)
        self._check(self.lib.dashgpu_decode_outputs(net.h, outputs.h, out.ctypes.data_as(i64p)))
        return out

    # ---- layer level (layer.hpp:79-97) ----
    def network_setup(self, c: "GpuCircuit", seeds: bytes) -> "GarbledNetwork":
        """garble()'s environment without any layer: offsets, multiples, zero / input base labels."""
        h = vp()
        buf = (ctypes.c_uint8 * len(seeds)).from_buffer_copy(seeds)
        self._check(self.lib.dashgpu_network_setup(c.h, buf, len(seeds) // 16, ctypes.byref(h)))
        return GarbledNetwork(self, h, c, len(seeds) // 16)

    def input_base(self, net: "GarbledNetwork") -> "Bundle":
        h = vp()
        self._check(self.lib.dashgpu_input_base(net.h, ctypes.byref(h)))
        return Bundle(self, h, net, False)

    def layer_garble(self, net: "GarbledNetwork", layer: int, inp: "Bundle", inp2: "Bundle" = None) -> "Bundle":
        """garble_layer: base labels in -> base labels out; rows into the network's GC."""
        h = vp()
        self._check(self.lib.dashgpu_layer_garble(net.h, layer, inp.h, inp2.h if inp2 else None, ctypes.byref(h)))
        return Bundle(self, h, net, False)

    def layer_eval(self, net: "GarbledNetwork", layer: int, inp: "Bundle", inp2: "Bundle" = None) -> "Bundle":
        """eval_layer: active labels in -> active labels out."""
        h = vp()
        self._check(self.lib.dashgpu_layer_eval(net.h, layer, inp.h, inp2.h if inp2 else None, ctypes.byref(h)))
        return Bundle(self, h, net, True)

    def network_finish(self, net: "GarbledNetwork", final_base: "Bundle"):
        self._check(self.lib.dashgpu_network_finish(net.h, final_base.h))

    def layer_count(self, c: "GpuCircuit", layer: int):
        out = (ctypes.c_uint64 * 3)()
        self._check(self.lib.dashgpu_layer_count(c.h, layer, out))
        return tuple(int(v) for v in out)

    def bundle_from_labels(self, net: "GarbledNetwork", lanes, output: bool = False) -> "Bundle":
        """LabelTensor images (per lane [batch][elements][n_p] u16 digits) -> device bundle."""
        arrs = [np.ascontiguousarray(a, np.uint16) for a in lanes]
        if len(arrs) != net.circuit.info.k:
            raise DataError("one label image per CRT lane expected")
        ptrs = (u16p * len(arrs))(*[a.ctypes.data_as(u16p) for a in arrs])
        h = vp()
        self._check(self.lib.dashgpu_bundle_from_labels(net.h, arrs[0].shape[1], ptrs, 1 if output else 0,
                                                        ctypes.byref(h)))
        return Bundle(self, h, net, output)

    def import_bundle(self, net: "GarbledNetwork", payload: bytes, output: bool) -> "Bundle":
        h = vp()
        buf = (ctypes.c_uint8 * len(payload)).from_buffer_copy(payload)
        self._check(self.lib.dashgpu_import_bundle(net.h, buf, len(payload), 1 if output else 0, ctypes.byref(h)))
        return Bundle(self, h, net, output)

    def import_gc(self, gcs, host_resident: bool = False) -> "GarbledNetwork":
        """parse_garbled_circuit (garble.cpp:368-403) on the evaluator side:
        serialized GCs of one circuit -> an evaluator network, inference b
        evaluating gcs[b] (EvaluatorService GC_TRANSFER, protocol.cpp:309).
        host_resident: ciphertexts stay in pinned host memory and move to the
        GPU one layer at a time during evaluate (GCs larger than HBM)."""
        if isinstance(gcs, (bytes, bytearray)):
            gcs = [gcs]
        gcs = [bytes(g) for g in gcs]  # no copy for bytes; pointers into them (kept alive below)
        ptrs = (u8p * len(gcs))(*[ctypes.cast(ctypes.c_char_p(g), u8p) for g in gcs])
        lens = (ctypes.c_size_t * len(gcs))(*[len(g) for g in gcs])
        h = vp()
        fn = self.lib.dashgpu_import_gc_host if host_resident else self.lib.dashgpu_import_gc
        self._check(fn(ptrs, lens, len(gcs), ctypes.byref(h)))
        ch = vp()
        self._check(self.lib.dashgpu_network_circuit(h, ctypes.byref(ch)))
        net = GarbledNetwork(self, h, GpuCircuit(self, ch, owned=False), len(gcs))
        return net

    def infer(self, c: "GpuCircuit", seeds, inputs, outputs=None, on_device: bool = False):
        """garble + garble_inputs + evaluate + decode_outputs for every inference.

        Host mode: seeds bytes / numpy inputs.  Device mode: pass raw device
        pointers (ints) for seeds, inputs and outputs."""
        t = Timing()
        if on_device:
            batch = outputs[1]
            self._check(self.lib.dashgpu_infer(c.h, vp(seeds), batch, vp(inputs), vp(outputs[0]), 1, ctypes.byref(t)))
            return None, t
        batch = len(seeds) // 16
        sbuf = (ctypes.c_uint8 * len(seeds)).from_buffer_copy(seeds)
        x = np.ascontiguousarray(inputs, np.int64).reshape(batch, c.info.n_in)
        out = np.zeros((batch, c.info.n_out), np.int64)
        self._check(self.lib.dashgpu_infer(c.h, ctypes.cast(sbuf, vp), batch, vp(x.ctypes.data),
                                           vp(out.ctypes.data), 0, ctypes.byref(t)))
        return out, t

    def infer_stream(self, c: "GpuCircuit", seeds: bytes, inputs, chunk: int, want_gc: bool = False,
                     u_range=None):
        """Streamed garble + garble_inputs + evaluate + decode_outputs of a
        single activation-layer circuit in element chunks (the label-ops
        sweep).  u_range = (begin, end): only those elements (a rank's shard,
        SURVEY 8(e)); outputs / gc keep full-layer indexing.  Returns
        (outputs, timing, gc) with gc the per-inference ciphertext blobs when
        want_gc."""
        t = Timing()
        batch = len(seeds) // 16
        sbuf = (ctypes.c_uint8 * len(seeds)).from_buffer_copy(seeds)
        x = np.ascontiguousarray(inputs, np.int64).reshape(batch, c.info.n_in)
        out = np.zeros((batch, c.info.n_out), np.int64)
        gc = np.zeros(batch * c.info.cts * 16, np.uint8) if want_gc else None
        u0, u1 = u_range if u_range is not None else (0, c.info.n_in)
        self._check(self.lib.dashgpu_infer_stream_range(c.h, ctypes.cast(sbuf, vp), batch, vp(x.ctypes.data),
                                                        vp(out.ctypes.data), chunk, u0, u1,
                                                        vp(gc.ctypes.data) if want_gc else None, ctypes.byref(t)))
        gcs = [gc[b * c.info.cts * 16:(b + 1) * c.info.cts * 16].tobytes() for b in range(batch)] if want_gc else None
        return out, t, gcs

    # ---- profiling ----
    def profile(self, enable: bool):
        self._check(self.lib.dashgpu_profile(1 if enable else 0))

    def profile_read(self):
        ms = (ctypes.c_double * 16)()
        n = (ctypes.c_uint64 * 16)()
        k = self.lib.dashgpu_profile_read(ms, n, 16)
        return {KERNEL_KINDS[i]: (ms[i], int(n[i])) for i in range(max(k, 0))}

    ACT_SHAPES = {0: "none", 1: "lane-group eval", 2: "level-parallel garble", 3: "lane-group garble",
                  4: "per-thread"}

    def last_act_launch(self, garble: bool = True) -> dict:
        """Launch shape of the most recent activation launch (kernels_act.cu)."""
        o = (ctypes.c_uint32 * 5)()
        self._check(self.lib.dashgpu_last_act_launch(1 if garble else 0, o))
        return {"variant": self.ACT_SHAPES.get(o[0], str(o[0])), "nchunks": o[1], "grid": o[2], "items": o[3],
                "group": o[4]}

    # ---- t_proj primitive (gadgets.hpp:146-176) ----
    def proj_garble(self, seed: bytes, p: int, q: int, phi, labels, gates, wires):
        """n projection gates: labels = compressed base labels mod p (list of ints).
        Returns (rows [n][p] ints, out0 [n] ints, (R_p, R_q))."""
        n = len(labels)
        ia = np.array([[v & (2**64 - 1), v >> 64] for v in labels], np.uint64).reshape(n, 2)
        ph = np.ascontiguousarray(phi, np.uint8)
        g = np.ascontiguousarray(gates, np.uint64)
        w = np.ascontiguousarray(wires, np.uint64)
        rows = np.zeros((n, p, 2), np.uint64)
        out0 = np.zeros((n, 2), np.uint64)
        offs = np.zeros(4, np.uint64)
        self._check(self.lib.dashgpu_proj_garble((ctypes.c_uint8 * 16)(*seed), n, p, q, ph.ctypes.data_as(u8p),
                                                 ia.ctypes.data_as(u64p), g.ctypes.data_as(u64p),
                                                 w.ctypes.data_as(u64p), rows.ctypes.data_as(u64p),
                                                 out0.ctypes.data_as(u64p), offs.ctypes.data_as(u64p)))
        j = lambda a: int(a[0]) | (int(a[1]) << 64)  # noqa: E731
        return ([[j(r) for r in rr] for rr in rows], [j(o) for o in out0], (j(offs[:2]), j(offs[2:])))

    def proj_eval(self, p: int, q: int, labels, gates, rows):
        n = len(labels)
        ia = np.array([[v & (2**64 - 1), v >> 64] for v in labels], np.uint64).reshape(n, 2)
        g = np.ascontiguousarray(gates, np.uint64)
        ra = np.array([[[v & (2**64 - 1), v >> 64] for v in rr] for rr in rows], np.uint64).reshape(n, p, 2)
        out = np.zeros((n, 2), np.uint64)
        self._check(self.lib.dashgpu_proj_eval(n, p, q, ia.ctypes.data_as(u64p), g.ctypes.data_as(u64p),
                                               ra.ctypes.data_as(u64p), out.ctypes.data_as(u64p)))
        return [int(o[0]) | (int(o[1]) << 64) for o in out]

    def proj_ctx(self, seed: bytes, p: int, q: int, phi) -> "ProjCtx":
        """Device-resident t_proj (dashgpu_proj_ctx_*): buffers are device
        pointers (ints), work goes on this thread's stream without a sync."""
        ph = np.ascontiguousarray(phi, np.uint8)
        h = vp()
        self._check(self.lib.dashgpu_proj_ctx_create((ctypes.c_uint8 * 16)(*seed), p, q, ph.ctypes.data_as(u8p),
                                                     ctypes.byref(h)))
        return ProjCtx(self, h, p, q)

    # ---- primitives (parity tests) ----
    def prim(self, op: int, m: int, q: int = 0, inp=None, out=None, key: bytes = None, wires=None, gate: int = 0,
             n: int = None):
        n = n if n is not None else (len(inp) if inp is not None else len(wires))
        ia = np.zeros((n, 2), np.uint64) if inp is None else np.ascontiguousarray(inp, np.uint64).reshape(n, 2)
        oa = np.zeros((n, 2), np.uint64) if out is None else np.ascontiguousarray(out, np.uint64).reshape(n, 2).copy()
        dg = np.zeros((n, 128), np.uint16)
        kb = (ctypes.c_uint8 * 16)(*key) if key is not None else None
        wa = None if wires is None else np.ascontiguousarray(wires, np.uint64)
        self._check(self.lib.dashgpu_prim(op, n, m, q, ia.ctypes.data_as(u64p), oa.ctypes.data_as(u64p),
                                          dg.ctypes.data_as(u16p), kb,
                                          None if wa is None else wa.ctypes.data_as(u64p), gate))
        return oa, dg


class ProjCtx:
    def __init__(self, eng: Dash, h, p: int, q: int):
        self.eng, self.h, self.p, self.q = eng, h, p, q

    def __del__(self):
        try:
            self.eng.lib.dashgpu_proj_ctx_destroy(self.h)
        except Exception:
            pass

    def garble(self, n: int, labels: int, gates: int, wires: int, rows: int, out0: int):
        self.eng._check(self.eng.lib.dashgpu_proj_garble_dev(self.h, n, vp(labels), vp(gates), vp(wires), vp(rows),
                                                             vp(out0)))

    def eval(self, n: int, labels: int, gates: int, rows: int, out: int):
        self.eng._check(self.eng.lib.dashgpu_proj_eval_dev(self.h, n, vp(labels), vp(gates), vp(rows), vp(out)))


class GpuCircuit:
    def __init__(self, eng: Dash, h, owned: bool = True):
        self.eng, self.h, self.owned = eng, h, owned
        self.info = CircuitInfo()
        eng._check(eng.lib.dashgpu_circuit_info_get(h, ctypes.byref(self.info)))

    def __del__(self):
        try:
            if self.owned:
                self.eng.lib.dashgpu_circuit_destroy(self.h)
        except Exception:
            pass

    def to_circuit(self) -> Circuit:
        d = CircuitDesc()
        self.eng._check(self.eng.lib.dashgpu_circuit_desc_view(self.h, ctypes.byref(d)))
        return Circuit.from_desc(d)

    def random_input(self, seed: int, lo: int = -7, hi: int = 7) -> np.ndarray:
        out = np.zeros(self.info.n_in, np.int64)
        self.eng._check(self.eng.lib.dashgpu_random_input(self.h, seed, lo, hi, out.ctypes.data_as(i64p)))
        return out

    def plain_forward(self, x) -> np.ndarray:
        x = np.ascontiguousarray(x, np.int64)
        out = np.zeros(self.info.n_out, np.int64)
        self.eng._check(self.eng.lib.dashgpu_plain_forward(self.h, x.ctypes.data_as(i64p), out.ctypes.data_as(i64p)))
        return out

    @property
    def radices(self):
        return list(self.info.radices[: self.info.sign_t])


class GarbledNetwork:
    def __init__(self, eng: Dash, h, circuit: GpuCircuit, batch: int):
        self.eng, self.h, self.circuit, self.batch = eng, h, circuit, batch

    def __del__(self):
        try:
            self.eng.lib.dashgpu_network_destroy(self.h)
        except Exception:
            pass

    def _export(self, fn, b: int) -> bytes:
        n = ctypes.c_size_t()
        self.eng._check(fn(self.h, b, None, 0, ctypes.byref(n)))
        out = bytearray(n.value)
        buf = (ctypes.c_uint8 * n.value).from_buffer(out)
        self.eng._check(fn(self.h, b, buf, n.value, ctypes.byref(n)))
        del buf  # release the export lock on `out`
        return bytes(out)

    def digest(self, b: int = 0) -> np.ndarray:
        """[n_layers][32] tree SHA-256 of inference b's layer ciphertexts
        (dashgpu_network_digest; the same digests as Dash.garble_digest)."""
        out = np.zeros((self.circuit.info.n_layers, 32), np.uint8)
        self.eng._check(self.eng.lib.dashgpu_network_digest(self.h, b,
                                                            out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))))
        return out

    def export_gc(self, b: int = 0) -> bytes:
        """serialize_garbled_circuit (garble.cpp:347-370) of inference b."""
        return self._export(self.eng.lib.dashgpu_export_gc, b)

    def export_encoding(self, b: int = 0) -> bytes:
        return self._export(self.eng.lib.dashgpu_export_encoding, b)

    def export_decoding(self, b: int = 0) -> bytes:
        return self._export(self.eng.lib.dashgpu_export_decoding, b)

    def release_gc(self):
        """Garbler side after export_gc: free ciphertexts / slots / layer planes
        (dashgpu_network_release_gc); garble_inputs and decode_outputs still work."""
        self.eng._check(self.eng.lib.dashgpu_network_release_gc(self.h))

    def tamper(self, b: int, index: int, mask: bytes):
        self.eng._check(self.eng.lib.dashgpu_tamper_ct(self.h, b, index, (ctypes.c_uint8 * 16)(*mask)))


class Bundle:
    def __init__(self, eng: Dash, h, net: GarbledNetwork, output: bool):
        self.eng, self.h, self.net, self.output = eng, h, net, output

    def __del__(self):
        try:
            self.eng.lib.dashgpu_bundle_destroy(self.h)
        except Exception:
            pass

    def labels(self, lane: int) -> np.ndarray:
        """LabelTensor image of CRT lane `lane`: [batch][elements][n_p] u16 digits."""
        B, E = ctypes.c_uint32(), ctypes.c_uint64()
        self.eng._check(self.eng.lib.dashgpu_bundle_info(self.h, ctypes.byref(B), ctypes.byref(E)))
        p = PRIMES[lane]
        nd = _n_digits(p)
        out = np.zeros((B.value, E.value, nd), np.uint16)
        self.eng._check(self.eng.lib.dashgpu_bundle_labels(self.h, lane, out.ctypes.data_as(u16p)))
        return out

    def payload(self, b: int = 0) -> bytes:
        """bundle_payload (garble.cpp:465-472) of inference b."""
        fn = self.eng.lib.dashgpu_export_bundle
        n = ctypes.c_size_t()
        self.eng._check(fn(self.h, b, None, 0, ctypes.byref(n)))
        out = bytearray(n.value)
        buf = (ctypes.c_uint8 * n.value).from_buffer(out)
        self.eng._check(fn(self.h, b, buf, n.value, ctypes.byref(n)))
        del buf  # release the export lock on `out`
        return bytes(out)
