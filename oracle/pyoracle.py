"""TEST INFRASTRUCTURE ONLY — Python bindings for the two CPU checkers.

* ``Oracle``: oracle/liboracle.so, the plain-C restatement (dash_oracle.c).
* ``RefLib``: oracle/_ref/libdashref.so, the unmodified reference sources
  compiled in place (only where /root/reference existed at build time).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu-baseline /
``--impl reference`` legs import this module.  The product package never
does.
"""
from __future__ import annotations

import ctypes
import os
from typing import List, Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libdashref.so")

u64p = ctypes.POINTER(ctypes.c_uint64)
u16p = ctypes.POINTER(ctypes.c_uint16)
i64p = ctypes.POINTER(ctypes.c_int64)
u8p = ctypes.POINTER(ctypes.c_uint8)
vp = ctypes.c_void_p

MASK64 = (1 << 64) - 1


def _u128(v: int):
    return (ctypes.c_uint64 * 2)(v & MASK64, (v >> 64) & MASK64)


def _int(a) -> int:
    return int(a[0]) | (int(a[1]) << 64)


def n_digits(m: int) -> int:
    """n_m = max{n : m^n <= 2^128} (reference label.cpp:15-29)."""
    n, acc = 0, 1
    while acc * m <= (1 << 128):
        acc *= m
        n += 1
    return n


class CheckerError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class _Base:
    prefix = ""

    def __init__(self, path):
        self.path = path
        self.lib = ctypes.CDLL(path)
        self._proto()

    def f(self, name):
        return getattr(self.lib, self.prefix + name)

    def err(self):
        fn = self.f("last_error")
        fn.restype = ctypes.c_char_p
        return fn().decode()

    # ----- primitives (identical signatures in both libraries) -----
    def _proto(self):
        L = self.lib
        P = self.prefix
        for name, args, res in [
            ("aes_fixed", [u64p, u64p], None),
            ("aes_key", [u8p, u64p, u64p], None),
            ("davies_meyer", [u64p, u64p], None),
            ("n_digits", [ctypes.c_int], ctypes.c_int),
            ("compress", [ctypes.c_int, u16p, u64p], None),
            ("decompress_mod", [u64p, ctypes.c_int, u16p], None),
            ("prf_label", [u8p, ctypes.c_uint64, ctypes.c_int, u16p], None),
            ("prf_offset", [u8p, ctypes.c_int, u16p], None),
            ("pad_bits", [ctypes.c_int, u16p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, u64p], None),
            ("pad_bits2", [ctypes.c_int, u16p, ctypes.c_int, u16p, ctypes.c_uint64, ctypes.c_uint32,
                           ctypes.c_uint32, u64p], None),
            ("encrypt_label", [ctypes.c_int, u16p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                               ctypes.c_int, u16p, u64p], None),
            ("decrypt_label", [ctypes.c_int, u16p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                               u64p, ctypes.c_int, u16p], None),
            ("choose_mixed_radix", [ctypes.c_int, ctypes.c_double, u16p], ctypes.c_int),
            ("element_cost", [ctypes.c_int, ctypes.c_double, ctypes.c_int, u64p], ctypes.c_int),
        ]:
            fn = getattr(L, P + name)
            fn.argtypes = args
            fn.restype = res

    @staticmethod
    def _digits(d, m):
        n = n_digits(m)
        arr = (ctypes.c_uint16 * 128)()
        for i in range(n):
            arr[i] = int(d[i])
        return arr

    def n_digits(self, m: int) -> int:
        return self.f("n_digits")(m)

    def aes_fixed(self, x: int) -> int:
        o = (ctypes.c_uint64 * 2)()
        self.f("aes_fixed")(_u128(x), o)
        return _int(o)

    def aes_key(self, key: bytes, x: int) -> int:
        o = (ctypes.c_uint64 * 2)()
        self.f("aes_key")((ctypes.c_uint8 * 16)(*key), _u128(x), o)
        return _int(o)

    def davies_meyer(self, x: int) -> int:
        o = (ctypes.c_uint64 * 2)()
        self.f("davies_meyer")(_u128(x), o)
        return _int(o)

    def compress(self, m: int, d) -> int:
        o = (ctypes.c_uint64 * 2)()
        self.f("compress")(m, self._digits(d, m), o)
        return _int(o)

    def decompress_mod(self, c: int, m: int) -> List[int]:
        o = (ctypes.c_uint16 * 128)()
        self.f("decompress_mod")(_u128(c), m, o)
        return list(o[: n_digits(m)])

    def prf_label(self, seed: bytes, wire: int, m: int) -> List[int]:
        o = (ctypes.c_uint16 * 128)()
        self.f("prf_label")((ctypes.c_uint8 * 16)(*seed), wire, m, o)
        return list(o[: n_digits(m)])

    def prf_offset(self, seed: bytes, m: int) -> List[int]:
        o = (ctypes.c_uint16 * 128)()
        self.f("prf_offset")((ctypes.c_uint8 * 16)(*seed), m, o)
        return list(o[: n_digits(m)])

    def pad_bits(self, m, key, gate, row, slot) -> int:
        o = (ctypes.c_uint64 * 2)()
        self.f("pad_bits")(m, self._digits(key, m), gate, row, slot, o)
        return _int(o)

    def pad_bits2(self, m1, k1, m2, k2, gate, row, slot) -> int:
        o = (ctypes.c_uint64 * 2)()
        self.f("pad_bits2")(m1, self._digits(k1, m1), m2, self._digits(k2, m2), gate, row, slot, o)
        return _int(o)

    def encrypt_label(self, mk, key, gate, row, slot, mq, msg) -> int:
        o = (ctypes.c_uint64 * 2)()
        self.f("encrypt_label")(mk, self._digits(key, mk), gate, row, slot, mq, self._digits(msg, mq), o)
        return _int(o)

    def decrypt_label(self, mk, key, gate, row, slot, ct, q) -> List[int]:
        o = (ctypes.c_uint16 * 128)()
        self.f("decrypt_label")(mk, self._digits(key, mk), gate, row, slot, _u128(ct), q, o)
        return list(o[: n_digits(q)])

    def choose_mixed_radix(self, k: int, target: float = 1.0) -> List[int]:
        o = (ctypes.c_uint16 * 32)()
        t = self.f("choose_mixed_radix")(k, target, o)
        if t < 0:
            raise CheckerError(-t, self.err())
        return list(o[:t])

    def element_cost(self, k: int, target: float, kind: int):
        o = (ctypes.c_uint64 * 3)()
        rc = self.f("element_cost")(k, target, kind, o)
        if rc:
            raise CheckerError(rc, self.err())
        return tuple(int(x) for x in o)


class Net:
    """A garbled network held by a checker library."""

    def __init__(self, lib, handle, circuit):
        self.lib, self.h, self.circuit = lib, handle, circuit

    def __del__(self):
        try:
            self.lib.f("net_free")(self.h)
        except Exception:
            pass

    def _bytes(self, name) -> bytes:
        fn = self.lib.f(name)
        fn.restype = ctypes.c_size_t
        fn.argtypes = [vp, u8p, ctypes.c_size_t]
        n = fn(self.h, None, 0)
        buf = (ctypes.c_uint8 * n)()
        fn(self.h, buf, n)
        return bytes(buf)

    def gc_bytes(self) -> bytes:
        return self._bytes("net_gc_bytes")

    def enc_bytes(self) -> bytes:
        return self._bytes("net_enc_bytes")

    def dec_bytes(self) -> bytes:
        return self._bytes("net_dec_bytes")

    def cts(self) -> np.ndarray:
        cnt = self.lib.f("net_cts_count")
        cnt.restype = ctypes.c_uint64
        cnt.argtypes = [vp]
        n = cnt(self.h)
        out = np.zeros((n, 2), np.uint64)
        fn = self.lib.f("net_cts")
        fn.argtypes = [vp, u64p]
        fn(self.h, out.ctypes.data_as(u64p))
        return out

    def layer_ct_base(self) -> List[int]:
        out = (ctypes.c_uint64 * 260)()
        fn = self.lib.f("net_layer_ct_base")
        fn.argtypes = [vp, u64p]
        n = fn(self.h, out)
        return list(out[:n])

    def stats(self):
        out = (ctypes.c_uint64 * 3)()
        fn = self.lib.f("net_stats")
        fn.argtypes = [vp, u64p]
        fn(self.h, out)
        return tuple(int(x) for x in out)


class Bundle:
    def __init__(self, lib, handle):
        self.lib, self.h = lib, handle

    def __del__(self):
        try:
            self.lib.f("bundle_free")(self.h)
        except Exception:
            pass

    def payload(self) -> bytes:
        fn = self.lib.f("bundle_payload")
        fn.restype = ctypes.c_size_t
        fn.argtypes = [vp, u8p, ctypes.c_size_t]
        n = fn(self.h, None, 0)
        buf = (ctypes.c_uint8 * n)()
        fn(self.h, buf, n)
        return bytes(buf)


class Oracle(_Base):
    """The plain-C restatement (oracle/dash_oracle.c)."""

    prefix = "orc_"

    def __init__(self, path=ORACLE_SO):
        super().__init__(path)
        L = self.lib
        L.orc_circuit_new.argtypes = [vp, ctypes.POINTER(vp)]
        L.orc_garble.argtypes = [vp, u8p, ctypes.POINTER(vp)]
        L.orc_garble_inputs.argtypes = [vp, i64p, ctypes.c_size_t, ctypes.POINTER(vp)]
        L.orc_evaluate.argtypes = [vp, vp, ctypes.POINTER(vp)]
        L.orc_decode.argtypes = [vp, vp, i64p]
        L.orc_plain_forward.argtypes = [vp, i64p, i64p]
        L.orc_circuit_free.argtypes = [vp]
        L.orc_net_free.argtypes = [vp]
        L.orc_bundle_free.argtypes = [vp]
        L.orc_bundle_from_payload.argtypes = [vp, u8p, ctypes.c_size_t, ctypes.c_int, ctypes.POINTER(vp)]
        L.orc_bench_infer.argtypes = [vp, ctypes.c_int, u8p, i64p, i64p, ctypes.c_int]
        L.orc_bench_infer.restype = ctypes.c_double
        L.orc_seed_from_string.argtypes = [ctypes.c_char_p, u8p]

    def seed_from_string(self, s: str) -> bytes:
        o = (ctypes.c_uint8 * 16)()
        if self.lib.orc_seed_from_string(s.encode(), o):
            raise CheckerError(3, self.err())
        return bytes(o)

    def circuit(self, c):
        desc = c.to_desc()
        h = vp()
        rc = self.lib.orc_circuit_new(ctypes.byref(desc), ctypes.byref(h))
        if rc:
            raise CheckerError(rc, self.err())
        return _CircuitHandle(self, h, c)

    def garble(self, c, seed: bytes) -> Net:
        ch = c if isinstance(c, _CircuitHandle) else self.circuit(c)
        h = vp()
        rc = self.lib.orc_garble(ch.h, (ctypes.c_uint8 * 16)(*seed), ctypes.byref(h))
        if rc:
            raise CheckerError(rc, self.err())
        n = Net(self, h, ch)
        return n

    def garble_inputs(self, net: Net, values) -> Bundle:
        v = np.ascontiguousarray(values, np.int64)
        h = vp()
        rc = self.lib.orc_garble_inputs(net.h, v.ctypes.data_as(i64p), v.size, ctypes.byref(h))
        if rc:
            raise CheckerError(rc, self.err())
        return Bundle(self, h)

    def evaluate(self, net: Net, b: Bundle) -> Bundle:
        h = vp()
        rc = self.lib.orc_evaluate(net.h, b.h, ctypes.byref(h))
        if rc:
            raise CheckerError(rc, self.err())
        return Bundle(self, h)

    def decode(self, net: Net, b: Bundle) -> np.ndarray:
        out = np.zeros(net.circuit.c.n_out, np.int64)
        rc = self.lib.orc_decode(net.h, b.h, out.ctypes.data_as(i64p))
        if rc:
            raise CheckerError(rc, self.err())
        return out

    def bundle_from_payload(self, net: Net, data: bytes, output: bool) -> Bundle:
        h = vp()
        buf = (ctypes.c_uint8 * len(data)).from_buffer_copy(data)
        rc = self.lib.orc_bundle_from_payload(net.h, buf, len(data), 1 if output else 0, ctypes.byref(h))
        if rc:
            raise CheckerError(rc, self.err())
        return Bundle(self, h)

    def plain_forward(self, c, x) -> np.ndarray:
        ch = c if isinstance(c, _CircuitHandle) else self.circuit(c)
        x = np.ascontiguousarray(x, np.int64)
        out = np.zeros(ch.c.n_out, np.int64)
        rc = self.lib.orc_plain_forward(ch.h, x.ctypes.data_as(i64p), out.ctypes.data_as(i64p))
        if rc:
            raise CheckerError(rc, self.err())
        return out

    def bench_infer(self, c, seeds: bytes, inputs: np.ndarray, threads: int):
        ch = c if isinstance(c, _CircuitHandle) else self.circuit(c)
        n = len(seeds) // 16
        out = np.zeros((n, ch.c.n_out), np.int64)
        inp = np.ascontiguousarray(inputs, np.int64)
        sec = self.lib.orc_bench_infer(ch.h, n, (ctypes.c_uint8 * len(seeds)).from_buffer_copy(seeds),
                                       inp.ctypes.data_as(i64p), out.ctypes.data_as(i64p), threads)
        if sec < 0:
            raise CheckerError(1, self.err())
        return sec, out


class _CircuitHandle:
    def __init__(self, lib, h, c):
        self.lib, self.h, self.c = lib, h, c

    def __del__(self):
        try:
            self.lib.f("circuit_free")(self.h)
        except Exception:
            pass


class RefLib(_Base):
    """The unmodified reference, compiled in place (oracle/_ref/libdashref.so)."""

    prefix = "ref_"

    def __init__(self, path=REF_SO):
        super().__init__(path)
        L = self.lib
        L.ref_circuit_from_desc.restype = vp
        L.ref_circuit_from_desc.argtypes = [vp]
        L.ref_model.restype = vp
        L.ref_model.argtypes = [ctypes.c_char_p, ctypes.c_uint32, ctypes.c_int, ctypes.c_int]
        L.ref_circuit_desc.restype = vp
        L.ref_circuit_desc.argtypes = [vp]
        L.ref_circuit_free.argtypes = [vp]
        L.ref_random_input.argtypes = [vp, ctypes.c_uint32, ctypes.c_int, ctypes.c_int, i64p]
        L.ref_plain_forward.argtypes = [vp, i64p, i64p]
        L.ref_garble.restype = vp
        L.ref_garble.argtypes = [vp, u8p, ctypes.c_int]
        L.ref_net_free.argtypes = [vp]
        L.ref_garble_inputs.restype = vp
        L.ref_garble_inputs.argtypes = [vp, i64p, ctypes.c_size_t]
        L.ref_evaluate.restype = vp
        L.ref_evaluate.argtypes = [vp, vp, ctypes.c_int]
        L.ref_decode.argtypes = [vp, vp, i64p]
        L.ref_bundle_free.argtypes = [vp]
        L.ref_seed_from_string.argtypes = [ctypes.c_char_p, u8p]
        L.ref_bench_infer.restype = ctypes.c_double
        L.ref_bench_infer.argtypes = [vp, ctypes.c_int, u8p, i64p, i64p, ctypes.c_int, ctypes.c_int]
        L.ref_max_threads.restype = ctypes.c_int
        L.ref_eval_gc_bytes.argtypes = [u8p, ctypes.c_size_t, vp, ctypes.c_int, ctypes.POINTER(vp)]

    def seed_from_string(self, s: str) -> bytes:
        o = (ctypes.c_uint8 * 16)()
        self.lib.ref_seed_from_string(s.encode(), o)
        return bytes(o)

    def circuit(self, c):
        desc = c.to_desc()
        h = self.lib.ref_circuit_from_desc(ctypes.byref(desc))
        if not h:  # e.g. Pad2d / Add extensions the reference does not have
            raise CheckerError(3, self.err())
        return _CircuitHandle(self, vp(h), c)

    def model(self, name: str, seed: int, k: int, priv: bool = False):
        """The reference's own tests/support builders (test_models.hpp)."""
        from paper_2302_06361_b200.circuit import Circuit, CircuitDesc

        h = self.lib.ref_model(name.encode(), seed, k, 1 if priv else 0)
        if not h:
            raise CheckerError(1, self.err())
        d = ctypes.cast(self.lib.ref_circuit_desc(h), ctypes.POINTER(CircuitDesc)).contents
        c = Circuit.from_desc(d)
        return _CircuitHandle(self, vp(h), c)

    def random_input(self, ch, seed: int, lo: int = -7, hi: int = 7) -> np.ndarray:
        out = np.zeros(ch.c.n_in, np.int64)
        self.lib.ref_random_input(ch.h, seed, lo, hi, out.ctypes.data_as(i64p))
        return out

    def garble(self, c, seed: bytes, threads: int = 0) -> Net:
        ch = c if isinstance(c, _CircuitHandle) else self.circuit(c)
        h = self.lib.ref_garble(ch.h, (ctypes.c_uint8 * 16)(*seed), threads)
        if not h:
            raise CheckerError(1, self.err())
        return Net(self, vp(h), ch)

    def garble_inputs(self, net: Net, values) -> Bundle:
        v = np.ascontiguousarray(values, np.int64)
        h = self.lib.ref_garble_inputs(net.h, v.ctypes.data_as(i64p), v.size)
        if not h:
            raise CheckerError(3, self.err())
        return Bundle(self, vp(h))

    def evaluate(self, net: Net, b: Bundle, threads: int = 0) -> Bundle:
        h = self.lib.ref_evaluate(net.h, b.h, threads)
        if not h:
            raise CheckerError(3, self.err())
        return Bundle(self, vp(h))

    def eval_gc_bytes(self, gc: bytes, b: Bundle, threads: int = 0) -> Bundle:
        """parse_garbled_circuit + evaluate (EvaluatorService, protocol.cpp:309-331)."""
        out = vp()
        buf = (ctypes.c_uint8 * len(gc)).from_buffer_copy(gc)
        rc = self.lib.ref_eval_gc_bytes(buf, len(gc), b.h, threads, ctypes.byref(out))
        if rc:
            raise CheckerError(rc, self.err())
        return Bundle(self, out)

    def decode(self, net: Net, b: Bundle) -> np.ndarray:
        out = np.zeros(net.circuit.c.n_out, np.int64)
        rc = self.lib.ref_decode(net.h, b.h, out.ctypes.data_as(i64p))
        if rc:
            raise CheckerError(rc, self.err())
        return out

    def plain_forward(self, c, x) -> np.ndarray:
        ch = c if isinstance(c, _CircuitHandle) else self.circuit(c)
        x = np.ascontiguousarray(x, np.int64)
        out = np.zeros(ch.c.n_out, np.int64)
        rc = self.lib.ref_plain_forward(ch.h, x.ctypes.data_as(i64p), out.ctypes.data_as(i64p))
        if rc:
            raise CheckerError(rc, self.err())
        return out

    def bench_infer(self, c, seeds: bytes, inputs: np.ndarray, mode: int, threads: int):
        ch = c if isinstance(c, _CircuitHandle) else self.circuit(c)
        n = len(seeds) // 16
        out = np.zeros((n, ch.c.n_out), np.int64)
        inp = np.ascontiguousarray(inputs, np.int64)
        sec = self.lib.ref_bench_infer(ch.h, n, (ctypes.c_uint8 * len(seeds)).from_buffer_copy(seeds),
                                       inp.ctypes.data_as(i64p), out.ctypes.data_as(i64p), mode, threads)
        if sec < 0:
            raise CheckerError(1, self.err())
        return sec, out


_LAYER_FIELDS = ("kind", "private_weights", "in_dim", "out_dim", "in_ch", "out_ch", "filter", "stride", "src", "src2",
                 "pad")


def save_circuit(c, path: str):
    """Circuit -> plain npz (layer scalars + int8 weights / int64 biases)."""
    arrs = {"input_shape": np.asarray(c.input_shape, np.int64), "k": np.int64(c.k),
            "sign_target": np.float64(c.sign_target), "alpha": np.float64(c.alpha),
            "layers": np.asarray([[int(getattr(l, f)) for f in _LAYER_FIELDS] for l in c.layers], np.int64)}
    for i, l in enumerate(c.layers):
        if l.q_weights is not None:
            w = np.asarray(l.q_weights, np.int64)
            assert np.abs(w).max(initial=0) < 128
            arrs[f"w{i}"] = w.astype(np.int8)
        if l.q_biases is not None:
            arrs[f"b{i}"] = np.asarray(l.q_biases, np.int64)
    np.savez_compressed(path, **arrs)


def load_circuit(path: str):
    """npz written by save_circuit -> Circuit (the pure-Python circuit types;
    no native library is loaded)."""
    from paper_2302_06361_b200.circuit import Circuit, Layer

    z = np.load(path)
    layers = []
    for i, row in enumerate(z["layers"]):
        kw = dict(zip(_LAYER_FIELDS, (int(v) for v in row)))
        kw["private_weights"] = bool(kw["private_weights"])
        l = Layer(**kw)
        if f"w{i}" in z:
            l.q_weights = z[f"w{i}"].astype(np.int64)
        if f"b{i}" in z:
            l.q_biases = z[f"b{i}"].astype(np.int64)
        layers.append(l)
    return Circuit([int(v) for v in z["input_shape"]], int(z["k"]), layers, float(z["sign_target"]),
                   float(z["alpha"]))


def have_ref() -> bool:
    return os.path.exists(REF_SO)


def seed_hex(v: int) -> bytes:
    """seed_from_string(hex(v)): big-endian 16-byte seed (prf.cpp:42-66)."""
    return int(v).to_bytes(16, "big")
