"""Garbler / evaluator session services over the B200 engine.

The reference's protocol layer (proj/core/include/dash/protocol.hpp,
src/protocol.cpp) is the caller of the hot path: the garbler garbles a
circuit per session and ships gNN, turns plain inputs into garbled inputs
and decodes the garbled output; the evaluator holds gNN and evaluates.  This
module keeps its frame format, payload codecs and session state machines
byte-compatible and runs every garble / garble_inputs / evaluate /
decode_outputs on the device through the C ABI:

* GarblerService keeps each session's garbled network resident in HBM
  (encoding and decoding tables never leave the device; the reference keeps
  EncodingInfo / DecodingInfo in host memory),
* EvaluatorService turns GC_TRANSFER bytes into a device network with
  ``dashgpu_import_gc`` and answers GARBLED_INPUT with one device evaluation.

Transport: frames are plain bytes (``encode_frame`` / ``FrameDecoder``); the
in-process loopback ``run_local_protocol`` drives both services as the
reference's does (protocol.cpp:355-435), and the TCP plumbing of the
reference (protocol.cpp:437-614) is ``serve_garbler`` / ``serve_evaluator`` /
``remote_infer`` (one thread per client connection, one locked
request/reply link from the garbler to the evaluator).
"""
from __future__ import annotations

import os
import socket
import struct
import threading
import time
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Dict, List, Optional, Sequence

import numpy as np

from .circuit import ADD, FLATTEN, Circuit, Layer
from .engine import AuthenticityError, Dash, DataError, Error, GarbledNetwork

MAX_FRAME_PAYLOAD = 1 << 30  # kMaxFramePayload (protocol.hpp:40)
_MAGIC, _VERSION, _KIND_MODEL = b"DASH", 1, 6  # garble.hpp:21-28 (FileKind::QuantizedModel)


class ProtocolError(Error):
    """dash::ProtocolError"""


class FrameType(IntEnum):  # protocol.hpp:24-32
    MODEL_UPLOAD = 1
    GC_TRANSFER = 2
    INPUT_UPLOAD = 3
    GARBLED_INPUT = 4
    GARBLED_OUTPUT = 5
    RESULT = 6
    ERROR = 7


class ErrorCode(IntEnum):  # protocol.hpp:57-61
    PROTOCOL = 1
    DATA = 2
    AUTHENTICITY = 3


class Edge(IntEnum):  # protocol.hpp:108-113
    CLIENT_TO_GARBLER = 1
    GARBLER_TO_CLIENT = 2
    GARBLER_TO_EVALUATOR = 3
    EVALUATOR_TO_GARBLER = 4


class Destination(IntEnum):  # protocol.hpp:131
    REPLY = 1
    EVALUATOR = 2


@dataclass
class Frame:
    type: FrameType
    session: int
    payload: bytes = b""


@dataclass
class Outbound:
    dest: Destination
    frame: Frame


@dataclass
class TraceEntry:
    edge: Edge
    type: FrameType
    payload_bytes: int


# ---------------------------------------------------------------- framing

def encode_frame(f: Frame) -> bytes:
    """length u32 | type u8 | session u128 | payload (protocol.cpp:21-30)."""
    if len(f.payload) > MAX_FRAME_PAYLOAD:
        raise ProtocolError("frame payload too large")
    s = f.session
    return struct.pack("<IBQQ", 17 + len(f.payload), int(f.type), s & (2**64 - 1), s >> 64) + bytes(f.payload)


class FrameDecoder:
    """Incremental frame parser for byte streams (protocol.cpp:32-60)."""

    def __init__(self):
        self._buf = bytearray()
        self._pos = 0

    def feed(self, data: bytes):
        self._buf += data

    def next(self) -> Optional[Frame]:
        if len(self._buf) - self._pos < 4:
            return None
        (length,) = struct.unpack_from("<I", self._buf, self._pos)
        if length < 17:
            raise ProtocolError("frame shorter than its header")
        if length > 17 + MAX_FRAME_PAYLOAD:
            raise ProtocolError("frame too large")
        if len(self._buf) - self._pos < 4 + length:
            return None
        t, lo, hi = struct.unpack_from("<BQQ", self._buf, self._pos + 4)
        if t < 1 or t > 7:
            raise ProtocolError("unknown frame type")
        start = self._pos + 4 + 17
        f = Frame(FrameType(t), (hi << 64) | lo, bytes(self._buf[start:self._pos + 4 + length]))
        self._pos += 4 + length
        if self._pos == len(self._buf):
            self._buf.clear()
            self._pos = 0
        elif self._pos > (1 << 20):
            del self._buf[:self._pos]
            self._pos = 0
        return f


# ---------------------------------------------------------------- payload codecs

class _Reader:
    def __init__(self, b: bytes):
        self.b, self.at = b, 0

    def take(self, fmt: str):
        n = struct.calcsize(fmt)
        if len(self.b) - self.at < n:
            raise DataError("truncated data")
        v = struct.unpack_from(fmt, self.b, self.at)
        self.at += n
        return v if len(v) > 1 else v[0]

    def remaining(self) -> int:
        return len(self.b) - self.at


def encode_error(code: ErrorCode, message: str) -> bytes:
    m = message.encode()
    return struct.pack("<BI", int(code), len(m)) + m


def decode_error(payload: bytes):
    r = _Reader(payload)
    code = r.take("<B")
    if code < 1 or code > 3:
        raise ProtocolError("bad error code")
    n = r.take("<I")
    if r.remaining() < n:
        raise DataError("truncated data")
    return ErrorCode(code), payload[r.at:r.at + n].decode(errors="replace")


def serialize_circuit(c: Circuit) -> bytes:
    """Quantized-circuit container (model_io.cpp:215-239).  Extension layers
    (Pad2d / Add / DAG inputs) flag bit 1 of the private byte and append
    src | src2 | pad, as the GC format does."""
    out = bytearray(_MAGIC + struct.pack("<HB", _VERSION, _KIND_MODEL))
    out += struct.pack("<BB", c.k, len(c.input_shape))
    out += struct.pack(f"<{len(c.input_shape)}I", *c.input_shape)
    out += struct.pack("<ddH", c.alpha, c.sign_target, len(c.layers))
    for l in c.layers:
        ext = l.kind > FLATTEN or l.src or l.src2 or l.pad
        out += struct.pack("<BB6I", l.kind, (1 if l.private_weights else 0) | (2 if ext else 0), l.in_dim,
                           l.out_dim, l.in_ch, l.out_ch, l.filter, l.stride)
        for a in (l.q_weights, l.q_biases):
            v = np.zeros(0, np.int64) if a is None else np.ascontiguousarray(a, np.int64).ravel()
            out += struct.pack("<Q", v.size) + v.astype("<i8").tobytes()
        if ext:
            out += struct.pack("<iiI", l.src, l.src2, l.pad)
    return bytes(out)


def parse_circuit(data: bytes) -> Circuit:
    """parse_circuit (model_io.cpp:241-280); validate_circuit is the engine's
    (dashgpu_circuit_create) when the garbler builds the circuit."""
    r = _Reader(data)
    if r.take("<4s") != _MAGIC:
        raise DataError("bad file magic")
    if r.take("<H") != _VERSION:
        raise DataError("unsupported format version")
    if r.take("<B") != _KIND_MODEL:
        raise DataError("wrong file kind")
    k = r.take("<B")
    if k < 1 or k > 16:
        raise DataError("bad base size")
    rank = r.take("<B")
    if rank == 0 or rank > 8:
        raise DataError("bad input rank")
    shape = [r.take("<I") for _ in range(rank)]
    alpha, target, n_layers = r.take("<ddH")
    layers = []
    for _ in range(n_layers):
        kind, flags, *dims = r.take("<BB6I")
        if kind < 1 or kind > ADD:
            raise DataError("bad layer kind")
        l = Layer(kind, bool(flags & 1), *dims)
        for name, count in (("q_weights", l.weight_count()), ("q_biases", _bias_count(l))):
            n = r.take("<Q")
            if n != 0 and n != count:
                raise DataError("bad weight count" if name == "q_weights" else "bad bias count")
            if r.remaining() < 8 * n:
                raise DataError("truncated data")
            v = np.frombuffer(data, "<i8", n, r.at).astype(np.int64) if n else None
            r.at += 8 * n
            setattr(l, name, v)
        if flags & 2:
            l.src, l.src2, l.pad = r.take("<iiI")
        layers.append(l)
    if r.remaining():
        raise DataError("trailing bytes in quantized model")
    return Circuit(shape, k, layers, target, alpha)


def _bias_count(l: Layer) -> int:
    return l.out_dim if l.kind == 1 else (l.out_ch if l.kind == 2 else 0)


def encode_model_upload(c: Circuit, owners: int) -> bytes:
    return struct.pack("<H", owners) + serialize_circuit(c)


def decode_model_upload(payload: bytes):
    if len(payload) < 2:
        raise DataError("truncated data")
    return parse_circuit(payload[2:]), struct.unpack_from("<H", payload)[0]


def encode_input_upload(owner: int, offset: int, values: Sequence[int]) -> bytes:
    """owner u16 | offset u32 | count u32 | i16 per element (protocol.cpp:98-110)."""
    v = np.asarray(values, np.int64)
    if v.size and (v.min() < -32768 or v.max() > 32767):
        raise DataError("plain input does not fit the 16-bit wire type")
    return struct.pack("<HII", owner, offset, v.size) + v.astype("<i2").tobytes()


def decode_input_upload(payload: bytes):
    r = _Reader(payload)
    owner, offset, count = r.take("<HII")
    if count * 2 != r.remaining():
        raise ProtocolError("input upload length mismatch")
    return owner, offset, np.frombuffer(payload, "<i2", count, r.at).astype(np.int64)


def encode_result(values) -> bytes:
    return np.asarray(values, np.int64).astype("<i8").tobytes()


def decode_result(payload: bytes) -> np.ndarray:
    if len(payload) % 8:
        raise ProtocolError("result payload length not a multiple of 8")
    return np.frombuffer(payload, "<i8").astype(np.int64)


@dataclass
class CommVolume:  # protocol.hpp:88-103
    garbled_in: int
    garbled_out: int
    plain_in: int
    plain_out: int

    def online_bytes(self) -> int:
        return self.garbled_in + self.garbled_out + self.plain_in + self.plain_out

    def with_overhead(self) -> int:
        return 2 * self.online_bytes()


def comm_volume(k: int, in_size: int, out_size: int) -> CommVolume:
    return CommVolume(16 * k * in_size, 16 * k * out_size, 2 * in_size, 8 * out_size)


def _code_for(e: Exception) -> ErrorCode:
    if isinstance(e, AuthenticityError):
        return ErrorCode.AUTHENTICITY
    if isinstance(e, DataError):
        return ErrorCode.DATA
    return ErrorCode.PROTOCOL


def _error_frame(session: int, e: Exception) -> Frame:
    return Frame(FrameType.ERROR, session, encode_error(_code_for(e), str(e)))


# ---------------------------------------------------------------- services

@dataclass
class GarblerConfig:  # protocol.hpp:136-140
    seed: Optional[bytes] = None  # fixed seed (tests / DASH_SEED); None = fresh per session


@dataclass
class _GarblerSession:
    net: GarbledNetwork
    owners: int
    inputs: np.ndarray
    filled: np.ndarray
    phase: str = "inputs"  # inputs -> awaiting -> done | failed
    filled_count: int = 0
    result: Optional[np.ndarray] = None
    error: str = ""
    error_code: ErrorCode = ErrorCode.PROTOCOL


class GarblerService:
    """The trusted garbling device (protocol.cpp:167-298): garbles on the GPU,
    keeps the session's encoding / decoding tables in HBM, never ships them."""

    def __init__(self, eng: Dash, cfg: GarblerConfig = None):
        self.eng, self.cfg = eng, cfg or GarblerConfig()
        self._mu = threading.Lock()
        self._sessions: Dict[int, _GarblerSession] = {}

    def handle(self, f: Frame) -> List[Outbound]:
        try:
            if f.type == FrameType.MODEL_UPLOAD:
                return [self._on_model_upload(f)]
            if f.type == FrameType.INPUT_UPLOAD:
                out = self._on_input_upload(f)
                return [out] if out else []
            if f.type == FrameType.GARBLED_OUTPUT:
                self._on_garbled_output(f)
                return []
            if f.type == FrameType.RESULT:
                return [self._on_result_request(f)]
            if f.type == FrameType.ERROR:
                code, msg = decode_error(f.payload)
                with self._mu:
                    s = self._sessions.get(f.session)
                    if s:
                        s.phase, s.error, s.error_code = "failed", msg, code
                        s.net = None
                return []
            raise ProtocolError("unexpected frame type for garbler")
        except Error as e:
            return [Outbound(Destination.REPLY, _error_frame(f.session, e))]

    def _on_model_upload(self, f: Frame) -> Outbound:
        circuit, owners = decode_model_upload(f.payload)
        if owners == 0:
            raise ProtocolError("at least one input owner required")
        n_in = circuit.n_in
        if owners > n_in:
            raise ProtocolError("more input owners than input elements")
        seed = self.cfg.seed if self.cfg.seed is not None else os.urandom(16)
        # streamed serialize_garbled_circuit: HBM holds one layer's rows at a
        # time, and the network keeps only encoding + decoding material, as the
        # reference garbler keeps only EncodingInfo / DecodingInfo
        # (protocol.cpp:211-226)
        chunks = []
        net = self.eng.garble_stream(self.eng.circuit(circuit), seed, lambda b, data: chunks.append(data))
        gc = b"".join(chunks)
        with self._mu:
            if f.session in self._sessions:
                raise ProtocolError("session already exists")
            self._sessions[f.session] = _GarblerSession(net, owners, np.zeros(n_in, np.int64),
                                                        np.zeros(n_in, bool))
        return Outbound(Destination.EVALUATOR, Frame(FrameType.GC_TRANSFER, f.session, gc))

    def _on_input_upload(self, f: Frame) -> Optional[Outbound]:
        owner, offset, values = decode_input_upload(f.payload)
        with self._mu:
            s = self._sessions.get(f.session)
            if s is None:
                raise ProtocolError("unknown session")
            if s.phase != "inputs":
                raise ProtocolError("inputs already complete for this session")
            if owner >= s.owners:
                raise ProtocolError("input owner out of range")
            end = offset + values.size
            if end > s.inputs.size:
                raise ProtocolError("input range out of bounds")
            for i in range(values.size):  # per element, as the reference (partial fills stay)
                if s.filled[offset + i]:
                    raise ProtocolError("input element uploaded twice")
                s.filled[offset + i] = True
                s.inputs[offset + i] = values[i]
            s.filled_count += values.size
            if s.filled_count < s.inputs.size:
                return None
            gin = self.eng.garble_inputs(s.net, s.inputs[None, :])
            s.phase = "awaiting"
            return Outbound(Destination.EVALUATOR, Frame(FrameType.GARBLED_INPUT, f.session, gin.payload(0)))

    def _on_garbled_output(self, f: Frame):
        with self._mu:
            s = self._sessions.get(f.session)
            if s is None:
                raise ProtocolError("unknown session")
            if s.phase != "awaiting":
                raise ProtocolError("no garbled output expected for this session")
            try:
                out = self.eng.import_bundle(s.net, f.payload, True)
                s.result = self.eng.decode_outputs(s.net, out)[0]
                s.phase = "done"
            except Error as e:
                s.phase, s.error, s.error_code = "failed", str(e), _code_for(e)
            finally:
                # single use: the session's device memory goes as soon as the
                # outcome is known; only the host-side result / error stays
                if s.phase in ("done", "failed"):
                    s.net = None

    def _on_result_request(self, f: Frame) -> Outbound:
        if f.payload:
            raise ProtocolError("result frames to the garbler must be empty")
        with self._mu:
            s = self._sessions.get(f.session)
            if s is None:
                raise ProtocolError("unknown session")
            if s.phase == "done":
                return Outbound(Destination.REPLY, Frame(FrameType.RESULT, f.session, encode_result(s.result)))
            if s.phase == "failed":
                return Outbound(Destination.REPLY, Frame(FrameType.ERROR, f.session,
                                                         encode_error(s.error_code, s.error)))
            raise ProtocolError("result not ready")

    def session_done(self, session: int) -> bool:
        with self._mu:
            s = self._sessions.get(session)
            return s is not None and s.phase in ("done", "failed")


@dataclass
class _EvalGroup:
    """Sessions whose GCs were imported together into one batched device
    network (EvaluatorService.handle_batch): evaluated in one launch once
    every member's garbled input is in."""
    net: GarbledNetwork
    sessions: List[int]
    inputs: Dict[int, bytes] = field(default_factory=dict)  # member index -> payload
    failed: set = field(default_factory=set)                # members answered with an error
    want: int = 0                                           # GARBLED_INPUT payload bytes per member
    deadline: float = float("inf")                          # time.monotonic() after which flush_expired runs it
    done: bool = False


@dataclass
class _EvaluatorSession:
    net: GarbledNetwork
    memory: int
    used: bool = False
    group: Optional[_EvalGroup] = None
    index: int = 0


class EvaluatorService:
    """The untrusted inference device (protocol.cpp:303-350): holds gNN in
    HBM only; each garbled circuit is single-use.

    batch_timeout: seconds a batched group (handle_batch) waits for its
    members' GARBLED_INPUT frames; flush_expired() then evaluates the group
    with placeholder inputs for the missing members and answers those with
    ERROR frames, so one stalled client cannot starve the others.

    host_resident_gc: keep each session's ciphertexts in pinned host memory
    and move them to the GPU one layer at a time at evaluation
    (dashgpu_import_gc_host) -- for GCs that do not fit HBM, or many pending
    sessions; the garbled outputs are the same."""

    def __init__(self, eng: Dash, batch_timeout: float = 30.0, host_resident_gc: bool = False):
        self.eng = eng
        self.batch_timeout = batch_timeout
        self.host_resident_gc = host_resident_gc
        self._mu = threading.Lock()
        self._sessions: Dict[int, _EvaluatorSession] = {}
        self._ready: List[Frame] = []  # replies of batched sessions not yet handed out

    def handle(self, f: Frame) -> Optional[Frame]:
        with self._mu:
            s = self._sessions.get(f.session) if f.type == FrameType.GARBLED_INPUT else None
        if s is not None and s.group is not None:  # member of a batched network
            replies = self.handle_batch([f])
            mine = [r for r in replies if r.session == f.session]
            with self._mu:  # the other members' replies: take_ready() / handle_all()
                self._ready.extend(r for r in replies if r.session != f.session)
            return mine[0] if mine else None
        try:
            if f.type == FrameType.GC_TRANSFER:
                net = self.eng.import_gc([f.payload], self.host_resident_gc)
                info = net.circuit.info
                mem = info.cts * 16 + info.k * 16 + 16 * info.k * info.n_in  # protocol.cpp:347-350
                with self._mu:
                    if f.session in self._sessions:
                        raise ProtocolError("session already has a circuit")
                    self._sessions[f.session] = _EvaluatorSession(net, mem)
                return None  # same-connection ordering is the ack
            if f.type == FrameType.GARBLED_INPUT:
                with self._mu:
                    s = self._sessions.get(f.session)
                    if s is None:
                        raise ProtocolError("unknown session")
                    if s.used:
                        raise ProtocolError("garbled circuit already used (single-use)")
                    s.used = True
                try:
                    gin = self.eng.import_bundle(s.net, f.payload, False)
                    gout = self.eng.evaluate(s.net, gin)
                    return Frame(FrameType.GARBLED_OUTPUT, f.session, gout.payload(0))
                finally:
                    s.net = None  # single use: free the GC's HBM now
            raise ProtocolError("unexpected frame type for evaluator")
        except Error as e:
            return _error_frame(f.session, e)

    def handle_all(self, f: Frame) -> List[Frame]:
        """handle() plus every reply that became ready because of f (other
        members of a batched group), none parked."""
        r = self.handle(f)
        return ([r] if r is not None else []) + self.take_ready()

    def take_ready(self) -> List[Frame]:
        """Replies of batched sessions completed by earlier frames."""
        with self._mu:
            out, self._ready = self._ready, []
        return out

    def flush_expired(self, now: Optional[float] = None) -> List[Frame]:
        """Evaluate every batched group whose deadline passed: present members
        get their GARBLED_OUTPUT, missing ones an ERROR frame (their circuits
        are consumed: single use)."""
        now = time.monotonic() if now is None else now
        with self._mu:
            groups = {id(s.group): s.group for s in self._sessions.values()
                      if s.group is not None and not s.group.done and s.group.deadline <= now}
        replies: List[Frame] = []
        for grp in groups.values():
            replies += self._run_group(grp, expired=True)
        return replies + self.take_ready()

    def session_memory(self, session: int) -> int:
        with self._mu:
            s = self._sessions.get(session)
            return s.memory if s else 0

    # ---- batched sessions (B200 serving: one launch for many sessions) ----
    def handle_batch(self, frames: Sequence[Frame]) -> List[Frame]:
        """Frames of many sessions at once.  GC_TRANSFER frames of one batch
        that carry the same circuit are imported into ONE device network
        (dashgpu_import_gc with B GCs); their GARBLED_INPUT frames are held
        until every member's input is in and then evaluated in one launch.
        Same rules and error frames as handle(): single use, unknown or
        duplicate sessions, malformed bundles (a failed member is answered
        with its ERROR frame; the others still get their outputs).  Returns
        every reply that became ready, in no particular session order."""
        replies: List[Frame] = []
        gcs = [f for f in frames if f.type == FrameType.GC_TRANSFER]
        rest = [f for f in frames if f.type != FrameType.GC_TRANSFER]
        if len(gcs) >= 2:
            replies += self._import_group(gcs)
        elif gcs:
            r = self.handle(gcs[0])
            if r is not None:
                replies.append(r)
        for f in rest:
            with self._mu:
                s = self._sessions.get(f.session) if f.type == FrameType.GARBLED_INPUT else None
            if s is None or s.group is None:
                r = self.handle(f)
                if r is not None:
                    replies.append(r)
                continue
            replies += self._group_input(f, s)
        with self._mu:
            replies += self._ready
            self._ready = []
        return replies

    def _import_group(self, gcs: Sequence[Frame]) -> List[Frame]:
        replies, fresh, seen = [], [], set()
        with self._mu:
            for f in gcs:
                if f.session in self._sessions or f.session in seen:
                    replies.append(_error_frame(f.session, ProtocolError("session already has a circuit")))
                else:
                    seen.add(f.session)
                    fresh.append(f)
        if len(fresh) < 2:
            return replies + [r for r in (self.handle(f) for f in fresh) if r is not None]
        try:
            net = self.eng.import_gc([f.payload for f in fresh], self.host_resident_gc)
        except Error:  # bad file or mixed circuits: per-session imports attribute the errors
            return replies + [r for r in (self.handle(f) for f in fresh) if r is not None]
        info = net.circuit.info
        mem = info.cts * 16 + info.k * 16 + 16 * info.k * info.n_in
        grp = _EvalGroup(net, [f.session for f in fresh], want=16 * info.k * info.n_in,
                         deadline=time.monotonic() + self.batch_timeout)
        with self._mu:
            for i, f in enumerate(fresh):
                self._sessions[f.session] = _EvaluatorSession(net, mem, group=grp, index=i)
        return replies

    def _group_input(self, f: Frame, s: _EvaluatorSession) -> List[Frame]:
        grp = s.group
        want = grp.want
        with self._mu:
            if s.used:
                return [_error_frame(f.session, ProtocolError("garbled circuit already used (single-use)"))]
            s.used = True
            if len(f.payload) != want:  # bundle_from_payload's size check
                grp.failed.add(s.index)
                grp.inputs[s.index] = bytes(want)
                out = [_error_frame(f.session, DataError("wire payload size mismatch"))]
            else:
                grp.inputs[s.index] = bytes(f.payload)
                out = []
            if len(grp.inputs) < len(grp.sessions):
                return out
        return out + self._run_group(grp, expired=False)

    def _run_group(self, grp: _EvalGroup, expired: bool) -> List[Frame]:
        want = grp.want
        out: List[Frame] = []
        with self._mu:
            if grp.done:
                return []
            grp.done = True
            for i, sid in enumerate(grp.sessions):
                if i not in grp.inputs:  # expired: placeholder input, member consumed
                    grp.inputs[i] = bytes(want)
                    grp.failed.add(i)
                    s = self._sessions.get(sid)
                    if s is not None:
                        s.used = True
                    out.append(_error_frame(sid, ProtocolError("garbled input not received before the batch deadline")))
            payload = b"".join(grp.inputs[i] for i in range(len(grp.sessions)))
        try:
            gout = self.eng.evaluate(grp.net, self.eng.import_bundle(grp.net, payload, False))
            out += [Frame(FrameType.GARBLED_OUTPUT, sid, gout.payload(i))
                    for i, sid in enumerate(grp.sessions) if i not in grp.failed]
        except Error as e:
            out += [_error_frame(sid, e) for i, sid in enumerate(grp.sessions) if i not in grp.failed]
        finally:
            with self._mu:  # every member is single-use: the group's GCs leave HBM
                grp.net = None
                for sid in grp.sessions:
                    s = self._sessions.get(sid)
                    if s is not None:
                        s.net = None
        return out


# ---------------------------------------------------------------- loopback

@dataclass
class LocalRunResult:
    outputs: np.ndarray = None
    trace: List[TraceEntry] = field(default_factory=list)


LOOPBACK_SESSION = (0x44415348 << 64) | 1  # make_u128(0x44415348, 1) (protocol.cpp:362)


def run_local_protocol(eng: Dash, quantized: Circuit, inputs, owners: int = 1,
                       cfg: GarblerConfig = None, host_resident_gc: bool = False) -> LocalRunResult:
    """Both services in one process (protocol.cpp:355-435): model upload ->
    gNN transfer -> per-owner input uploads -> garbled input -> evaluation ->
    garbled output -> decode -> result request."""
    x = np.asarray(inputs, np.int64).ravel()
    if x.size != quantized.n_in:
        raise DataError("input size does not match the model")
    if owners == 0:
        raise DataError("at least one input owner required")
    garbler, evaluator = GarblerService(eng, cfg), EvaluatorService(eng, host_resident_gc=host_resident_gc)
    session = LOOPBACK_SESSION
    res = LocalRunResult()

    def to_evaluator(frame: Frame):
        res.trace.append(TraceEntry(Edge.GARBLER_TO_EVALUATOR, frame.type, len(frame.payload)))
        reply = evaluator.handle(frame)
        while reply is not None:
            res.trace.append(TraceEntry(Edge.EVALUATOR_TO_GARBLER, reply.type, len(reply.payload)))
            outs = garbler.handle(reply)
            reply = None
            for o in outs:
                if o.dest == Destination.EVALUATOR:
                    reply = o.frame

    def to_garbler(frame: Frame) -> List[Frame]:
        res.trace.append(TraceEntry(Edge.CLIENT_TO_GARBLER, frame.type, len(frame.payload)))
        replies = []
        for o in garbler.handle(frame):
            if o.dest == Destination.EVALUATOR:
                to_evaluator(o.frame)
            else:
                replies.append(o.frame)
        return replies

    def fail_on_error(replies):
        for r in replies:
            if r.type == FrameType.ERROR:
                raise ProtocolError(decode_error(r.payload)[1])

    fail_on_error(to_garbler(Frame(FrameType.MODEL_UPLOAD, session, encode_model_upload(quantized, owners))))
    n = x.size
    chunk, extra = divmod(n, owners)
    offset = 0
    for o in range(owners):
        count = chunk + (1 if o < extra else 0)
        fail_on_error(to_garbler(Frame(FrameType.INPUT_UPLOAD, session,
                                       encode_input_upload(o, offset, x[offset:offset + count]))))
        offset += count
    replies = to_garbler(Frame(FrameType.RESULT, session, b""))
    if len(replies) != 1:
        raise ProtocolError("no result reply")
    res.trace.append(TraceEntry(Edge.GARBLER_TO_CLIENT, replies[0].type, len(replies[0].payload)))
    if replies[0].type == FrameType.ERROR:
        code, msg = decode_error(replies[0].payload)
        raise {ErrorCode.AUTHENTICITY: AuthenticityError, ErrorCode.DATA: DataError}.get(code, ProtocolError)(msg)
    res.outputs = decode_result(replies[0].payload)
    return res


# ---------------------------------------------------------------- TCP transport (protocol.cpp:437-614)

_RECV_CHUNK = 1 << 20  # GC_TRANSFER frames are ~10^8 bytes


def _send_frame(sock: socket.socket, f: Frame):
    try:
        sock.sendall(encode_frame(f))
    except OSError as e:
        raise ProtocolError("connection write failed") from e


def _read_frame(sock: socket.socket, dec: FrameDecoder) -> Optional[Frame]:
    """Blocking read of the next whole frame; None on clean EOF (read_frame_fd)."""
    while True:
        f = dec.next()
        if f is not None:
            return f
        try:
            data = sock.recv(_RECV_CHUNK)
        except OSError as e:
            raise ProtocolError("connection read failed") from e
        if not data:
            return None
        dec.feed(data)


def _connect(host: str, port: int) -> socket.socket:
    try:
        s = socket.create_connection((host, port))
    except OSError as e:
        raise ProtocolError(f"cannot connect to {host}:{port}") from e
    s.setsockopt(socket.IPPROTO_TCP, socket.TCP_NODELAY, 1)
    return s


def _listen(host: str, port: int) -> socket.socket:
    try:
        infos = socket.getaddrinfo(host or None, port, socket.AF_UNSPEC, socket.SOCK_STREAM, 0, socket.AI_PASSIVE)
    except OSError as e:
        raise ProtocolError(f"cannot resolve bind address {host}") from e
    for fam, typ, proto, _, addr in infos:
        s = socket.socket(fam, typ, proto)
        try:
            s.setsockopt(socket.SOL_SOCKET, socket.SO_REUSEADDR, 1)
            s.bind(addr)
            s.listen(16)
            return s
        except OSError:
            s.close()
    raise ProtocolError(f"cannot bind {host}:{port}")


class _TcpServer:
    """Accept loop with one thread per connection (the reference detaches a
    std::thread per accepted client).  ``port`` is the bound port (0 binds an
    ephemeral one); ``start()`` runs the loop in a daemon thread, ``close()``
    stops accepting and drops the open connections."""

    def __init__(self, bind_host: str, port: int):
        self._listener = _listen(bind_host, port)
        self.port = self._listener.getsockname()[1]
        self._conns: List[socket.socket] = []
        self._conns_mu = threading.Lock()
        self._closed = False
        self._thread: Optional[threading.Thread] = None

    def _serve_client(self, conn: socket.socket):  # pragma: no cover - overridden
        raise NotImplementedError

    def _client(self, conn: socket.socket):
        try:
            self._serve_client(conn)
        except Error:
            pass  # connection torn down; session state remains consistent
        finally:
            with self._conns_mu:
                if conn in self._conns:
                    self._conns.remove(conn)
            conn.close()

    def serve_forever(self):
        while not self._closed:
            try:
                conn, _ = self._listener.accept()
            except OSError:
                if self._closed:
                    return
                continue
            conn.setsockopt(socket.IPPROTO_TCP, socket.TCP_NODELAY, 1)
            with self._conns_mu:
                self._conns.append(conn)
            threading.Thread(target=self._client, args=(conn,), daemon=True).start()

    def start(self):
        self._thread = threading.Thread(target=self.serve_forever, daemon=True)
        self._thread.start()
        return self

    def close(self):
        self._closed = True
        try:
            self._listener.shutdown(socket.SHUT_RDWR)
        except OSError:
            pass
        self._listener.close()
        with self._conns_mu:
            for c in self._conns:
                try:
                    c.shutdown(socket.SHUT_RDWR)
                except OSError:
                    pass
        if self._thread is not None:
            self._thread.join(timeout=5)

    def __enter__(self):
        return self.start()

    def __exit__(self, *a):
        self.close()


class EvaluatorServer(_TcpServer):
    """serve_evaluator (protocol.cpp:585-603): answers each frame of a
    connection with EvaluatorService.handle's reply."""

    def __init__(self, eng: Dash, bind_host: str = "127.0.0.1", port: int = 0):
        super().__init__(bind_host, port)
        self.service = EvaluatorService(eng)
        self._mu = threading.Lock()  # one device evaluation at a time

    def _serve_client(self, conn: socket.socket):
        dec = FrameDecoder()
        while True:
            f = _read_frame(conn, dec)
            if f is None:
                return
            with self._mu:
                reply = self.service.handle(f)
            if reply is not None:
                _send_frame(conn, reply)


class GarblerServer(_TcpServer):
    """serve_garbler (protocol.cpp:537-583): clients speak to the garbler;
    frames for the evaluator go over one connection, written under a lock,
    and each GARBLED_INPUT is a strict request/reply pair on it."""

    def __init__(self, eng: Dash, evaluator_host: str, evaluator_port: int, bind_host: str = "127.0.0.1",
                 port: int = 0, cfg: GarblerConfig = None):
        self.service = GarblerService(eng, cfg)
        self._evaluator = _connect(evaluator_host, evaluator_port)
        self._eval_mu = threading.Lock()
        self._eval_dec = FrameDecoder()
        self._mu = threading.Lock()  # one device call at a time
        super().__init__(bind_host, port)

    def _handle(self, f: Frame) -> List[Outbound]:
        with self._mu:
            return self.service.handle(f)

    def _to_evaluator(self, frame: Frame):
        with self._eval_mu:
            while True:
                expects_reply = frame.type == FrameType.GARBLED_INPUT
                _send_frame(self._evaluator, frame)
                if not expects_reply:
                    return
                reply = _read_frame(self._evaluator, self._eval_dec)
                if reply is None:
                    raise ProtocolError("evaluator closed the connection")
                nxt = None
                for o in self._handle(reply):
                    if o.dest == Destination.EVALUATOR:
                        nxt = o.frame
                if nxt is None:
                    return
                frame = nxt

    def _serve_client(self, conn: socket.socket):
        dec = FrameDecoder()
        while True:
            f = _read_frame(conn, dec)
            if f is None:
                return
            for o in self._handle(f):
                if o.dest == Destination.EVALUATOR:
                    self._to_evaluator(o.frame)
                else:
                    _send_frame(conn, o.frame)

    def close(self):
        super().close()
        self._evaluator.close()


def serve_evaluator(eng: Dash, bind_host: str, port: int):
    """Blocking evaluator server (protocol.hpp:232-233); never returns."""
    EvaluatorServer(eng, bind_host, port).serve_forever()


def serve_garbler(eng: Dash, bind_host: str, port: int, evaluator_host: str, evaluator_port: int,
                  cfg: GarblerConfig = None):
    """Blocking garbler server (protocol.hpp:227-230); never returns."""
    GarblerServer(eng, evaluator_host, evaluator_port, bind_host, port, cfg).serve_forever()


def remote_infer(garbler_host: str, port: int, quantized: Circuit, inputs, owners: int = 1,
                 timeout: float = 120.0) -> np.ndarray:
    """Client side (protocol.cpp:616-659): upload the model and the owners'
    input slices to the garbler, then poll RESULT until it is ready."""
    x = np.asarray(inputs, np.int64).ravel()
    if x.size != quantized.n_in:
        raise DataError("input size does not match the model")
    if owners == 0:
        raise DataError("at least one input owner required")
    session = int.from_bytes(os.urandom(16), "little")
    with _connect(garbler_host, port) as conn:
        _send_frame(conn, Frame(FrameType.MODEL_UPLOAD, session, encode_model_upload(quantized, owners)))
        chunk, extra = divmod(x.size, owners)
        offset = 0
        for o in range(owners):
            count = chunk + (1 if o < extra else 0)
            _send_frame(conn, Frame(FrameType.INPUT_UPLOAD, session,
                                    encode_input_upload(o, offset, x[offset:offset + count])))
            offset += count
        dec = FrameDecoder()
        deadline = time.monotonic() + timeout
        while True:
            _send_frame(conn, Frame(FrameType.RESULT, session, b""))
            reply = _read_frame(conn, dec)
            if reply is None:
                raise ProtocolError("garbler closed the connection")
            if reply.type == FrameType.RESULT:
                return decode_result(reply.payload)
            code, msg = decode_error(reply.payload)
            if code == ErrorCode.AUTHENTICITY:
                raise AuthenticityError(msg)
            if code == ErrorCode.DATA:
                raise DataError(msg)
            if msg != "result not ready":
                raise ProtocolError(msg)
            if time.monotonic() > deadline:
                raise ProtocolError("timed out waiting for the result")
            time.sleep(0.05)
