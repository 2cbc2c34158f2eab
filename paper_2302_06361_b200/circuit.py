"""Host-side mirror of the reference's circuit types.

``Layer`` / ``Circuit`` follow ``dash::Layer`` and ``dash::Circuit``
(reference ``proj/core/include/dash/layer.hpp:16-54`` and
``proj/core/include/dash/circuit.hpp:13-19``): a chain of Dense / Conv2d /
ReLU / SignAct / Flatten layers over a CRT base of ``k`` primes, with
quantized integer weights (``q_weights`` row-major ``[out][in]`` or
``[out_ch][in_ch][f][f]``).  ``to_desc()`` produces the plain-data C struct
declared in ``include/dash_circuit_desc.h`` that crosses the C ABI.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

DENSE, CONV2D, RELU, SIGNACT, FLATTEN, PAD2D, ADD = 1, 2, 3, 4, 5, 6, 7
KIND_NAMES = {DENSE: "Dense", CONV2D: "Conv2d", RELU: "ReLU", SIGNACT: "SignAct", FLATTEN: "Flatten",
              PAD2D: "Pad2d", ADD: "Add"}
PRIMES = [2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41, 43, 47, 53]


class LayerDesc(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32),
        ("private_weights", ctypes.c_int32),
        ("in_dim", ctypes.c_uint32),
        ("out_dim", ctypes.c_uint32),
        ("in_ch", ctypes.c_uint32),
        ("out_ch", ctypes.c_uint32),
        ("filter", ctypes.c_uint32),
        ("stride", ctypes.c_uint32),
        ("q_weights", ctypes.POINTER(ctypes.c_int64)),
        ("n_weights", ctypes.c_uint64),
        ("q_biases", ctypes.POINTER(ctypes.c_int64)),
        ("n_biases", ctypes.c_uint64),
        ("src", ctypes.c_int32),
        ("src2", ctypes.c_int32),
        ("pad", ctypes.c_uint32),
    ]


class CircuitDesc(ctypes.Structure):
    _fields_ = [
        ("k", ctypes.c_int32),
        ("rank", ctypes.c_uint32),
        ("input_shape", ctypes.c_uint32 * 8),
        ("sign_target", ctypes.c_double),
        ("alpha", ctypes.c_double),
        ("n_layers", ctypes.c_uint32),
        ("layers", ctypes.POINTER(LayerDesc)),
    ]


@dataclass
class Layer:
    kind: int
    private_weights: bool = False
    in_dim: int = 0
    out_dim: int = 0
    in_ch: int = 0
    out_ch: int = 0
    filter: int = 0
    stride: int = 0
    q_weights: Optional[np.ndarray] = None
    q_biases: Optional[np.ndarray] = None
    # extensions (include/dash_circuit_desc.h): DAG inputs and padding
    src: int = 0    # 0 = previous layer, j + 1 = output of layer j, -1 = circuit input
    src2: int = 0   # second operand of Add
    pad: int = 0    # Pad2d cells per side

    def linear(self) -> bool:
        return self.kind in (DENSE, CONV2D)

    def weight_count(self) -> int:
        if self.kind == DENSE:
            return self.in_dim * self.out_dim
        if self.kind == CONV2D:
            return self.out_ch * self.in_ch * self.filter * self.filter
        return 0

    def out_shape(self, shape: Sequence[int]) -> List[int]:
        """layer_out_shape (reference layer.cpp:320-344)."""
        if self.kind == DENSE:
            if list(shape) != [self.in_dim]:
                raise ValueError("dense layer input shape mismatch")
            return [self.out_dim]
        if self.kind == CONV2D:
            if len(shape) != 3 or shape[0] != self.in_ch:
                raise ValueError("conv layer input shape mismatch")
            def ext(n):
                if self.filter == 0 or self.stride == 0 or self.filter > n:
                    raise ValueError("convolution filter does not fit the input")
                return (n - self.filter) // self.stride + 1
            return [self.out_ch, ext(shape[1]), ext(shape[2])]
        if self.kind in (RELU, SIGNACT, ADD):
            return list(shape)
        if self.kind == PAD2D:
            if len(shape) != 3:
                raise ValueError("pad layer needs a [C][H][W] input")
            return [shape[0], shape[1] + 2 * self.pad, shape[2] + 2 * self.pad]
        return [int(np.prod(shape))]


@dataclass
class Circuit:
    input_shape: List[int]
    k: int = 8
    layers: List[Layer] = field(default_factory=list)
    sign_target: float = 1.0
    alpha: float = 1.0

    def shapes(self) -> List[List[int]]:
        """s[0] = input, s[j + 1] = output of layer j (inputs follow src)."""
        s = [list(self.input_shape)]
        for i, l in enumerate(self.layers):
            src = i if l.src == 0 else (0 if l.src < 0 else l.src)
            s.append(l.out_shape(s[src]))
        return s

    @property
    def n_in(self) -> int:
        return int(np.prod(self.input_shape))

    @property
    def n_out(self) -> int:
        return int(np.prod(self.shapes()[-1]))

    def to_desc(self) -> CircuitDesc:
        """C-ABI image; keeps numpy buffers alive on the returned struct."""
        keep = []
        arr = (LayerDesc * max(1, len(self.layers)))()
        for i, l in enumerate(self.layers):
            d = arr[i]
            d.kind = l.kind
            d.private_weights = 1 if l.private_weights else 0
            d.in_dim, d.out_dim = l.in_dim, l.out_dim
            d.in_ch, d.out_ch, d.filter, d.stride = l.in_ch, l.out_ch, l.filter, l.stride
            d.src, d.src2, d.pad = l.src, l.src2, l.pad
            if l.q_weights is not None:
                w = np.ascontiguousarray(l.q_weights, dtype=np.int64)
                keep.append(w)
                d.q_weights = w.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
                d.n_weights = w.size
            if l.q_biases is not None:
                b = np.ascontiguousarray(l.q_biases, dtype=np.int64)
                keep.append(b)
                d.q_biases = b.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
                d.n_biases = b.size
        desc = CircuitDesc()
        desc.k = self.k
        desc.rank = len(self.input_shape)
        for i, s in enumerate(self.input_shape):
            desc.input_shape[i] = s
        desc.sign_target = self.sign_target
        desc.alpha = self.alpha
        desc.n_layers = len(self.layers)
        desc.layers = arr
        desc._keep = (keep, arr)  # lifetime
        return desc

    @staticmethod
    def from_desc(d: CircuitDesc) -> "Circuit":
        layers = []
        for i in range(d.n_layers):
            s = d.layers[i]
            w = np.ctypeslib.as_array(s.q_weights, shape=(s.n_weights,)).copy() if s.n_weights else None
            b = np.ctypeslib.as_array(s.q_biases, shape=(s.n_biases,)).copy() if s.n_biases else None
            layers.append(Layer(s.kind, bool(s.private_weights), s.in_dim, s.out_dim, s.in_ch,
                                s.out_ch, s.filter, s.stride, w, b, s.src, s.src2, s.pad))
        return Circuit([d.input_shape[i] for i in range(d.rank)], d.k, layers, d.sign_target, d.alpha)


def dense(i, o, w, b, priv=False, src=0):
    return Layer(DENSE, priv, in_dim=i, out_dim=o, q_weights=np.asarray(w, np.int64),
                 q_biases=np.asarray(b, np.int64), src=src)


def conv2d(ic, oc, f, s, w, b, priv=False, src=0):
    return Layer(CONV2D, priv, in_ch=ic, out_ch=oc, filter=f, stride=s,
                 q_weights=np.asarray(w, np.int64), q_biases=np.asarray(b, np.int64), src=src)


def relu(src=0):
    return Layer(RELU, src=src)


def pad2d(p, src=0):
    """Extension: zero padding (pad cells = zero-wire label)."""
    return Layer(PAD2D, pad=p, src=src)


def add(src2, src=0):
    """Extension: residual add of the previous (or src) output and layer src2 - 1's output."""
    return Layer(ADD, src=src, src2=src2)


def sign_act():
    return Layer(SIGNACT)


def flatten():
    return Layer(FLATTEN)
