"""Garbler / evaluator services over the engine (paper_2302_06361_b200/protocol.py).

Ports the reference's own protocol tests (proj/tests/unit/test_protocol.cpp)
case by case; the frame / codec cases need no device, the service cases run
on the CPU emulation (``emu``) and on the B200 (``cuda``, ``-m gpu``).
"""
import numpy as np
import pytest

from helpers import models, seed_hex
from paper_2302_06361_b200 import protocol as P

BACKENDS = [pytest.param("emu", id="emu"), pytest.param("cuda", id="cuda", marks=pytest.mark.gpu)]


@pytest.fixture(params=BACKENDS)
def eng(request):
    return request.getfixturevalue("emu" if request.param == "emu" else "gpu")


def tiny():
    return models.build("model_tiny", 1000, 8)


def count_type(trace, t):
    return sum(1 for e in trace if e.type == t)


# ---------------------------------------------------------------- framing (test_protocol.cpp:34-118)

def test_frames_survive_a_byte_by_byte_stream():
    frames = [P.Frame(P.FrameType.MODEL_UPLOAD, 1, b"abc"), P.Frame(P.FrameType.RESULT, (1 << 127) | 5, b""),
              P.Frame(P.FrameType.GARBLED_INPUT, 2**64 + 3, bytes(range(256)) * 3)]
    stream = b""
    for f in frames:
        b = P.encode_frame(f)
        assert len(b) == 4 + 17 + len(f.payload)
        stream += b
    dec, got = P.FrameDecoder(), []
    for i in range(len(stream)):
        dec.feed(stream[i:i + 1])
        f = dec.next()
        if f:
            got.append(f)
    assert [(f.type, f.session, f.payload) for f in got] == [(f.type, f.session, f.payload) for f in frames]
    assert dec.next() is None
    # wire layout: length | type | session (lo u64, hi u64, little-endian) | payload
    assert P.encode_frame(P.Frame(P.FrameType.ERROR, 0x0102, b"z")) == \
        bytes([18, 0, 0, 0, 7, 2, 1]) + bytes(14) + b"z"


def test_frame_length_field_is_bounded():
    dec = P.FrameDecoder()
    dec.feed(bytes([5, 0, 0, 0]))
    with pytest.raises(P.ProtocolError):
        dec.next()
    big = 17 + (1 << 30) + 1
    dec2 = P.FrameDecoder()
    dec2.feed(big.to_bytes(4, "little"))
    with pytest.raises(P.ProtocolError):
        dec2.next()
    dec3 = P.FrameDecoder()
    dec3.feed(bytes([17, 0, 0, 0, 9]) + bytes(16))
    with pytest.raises(P.ProtocolError):
        dec3.next()


def test_payload_codecs_roundtrip():
    code, msg = P.decode_error(P.encode_error(P.ErrorCode.AUTHENTICITY, "bad label"))
    assert code == P.ErrorCode.AUTHENTICITY and msg == "bad label"
    c = tiny()
    mu = P.encode_model_upload(c, 3)
    c2, owners = P.decode_model_upload(mu)
    assert owners == 3
    assert P.serialize_circuit(c2) == P.serialize_circuit(c)
    assert len(mu) == 2 + len(P.serialize_circuit(c))
    vals = [-32768, -1, 0, 1, 32767, 5]
    iu = P.encode_input_upload(4, 19, vals)
    assert len(iu) == 10 + 2 * len(vals)
    owner, offset, v = P.decode_input_upload(iu)
    assert (owner, offset, v.tolist()) == (4, 19, vals)
    with pytest.raises(P.DataError):
        P.encode_input_upload(0, 0, [32768])
    with pytest.raises(P.ProtocolError):
        P.decode_input_upload(iu[:-1])
    res = [1, -2, 2**40, -(2**62)]
    assert P.decode_result(P.encode_result(res)).tolist() == res
    assert len(P.encode_result(res)) == 8 * len(res)
    assert P.decode_result(P.encode_result([])).size == 0


def test_quantized_model_container_matches_reference_layout():
    # model_io.cpp:215-239 field by field, and the extension record round trip
    c = tiny()
    b = P.serialize_circuit(c)
    assert b[:7] == b"DASH\x01\x00\x06" and b[7] == 8 and b[8] == 3
    from test_engine import _small_dag  # noqa: E402

    d = _small_dag()
    d2 = P.parse_circuit(P.serialize_circuit(d))
    assert [(l.kind, l.src, l.src2, l.pad) for l in d2.layers] == [(l.kind, l.src, l.src2, l.pad) for l in d.layers]
    for bad in (b[:-1], b + b"\0", b[:6] + b"\x01" + b[7:]):
        with pytest.raises(P.DataError):
            P.parse_circuit(bad)


def test_communication_volume_matches_model_dimensions():
    a = P.comm_volume(8, 784, 10)  # Model A (test_protocol.cpp:120-136)
    assert (a.garbled_in, a.garbled_out, a.plain_in, a.plain_out) == (100352, 1280, 1568, 80)
    assert a.online_bytes() == 100352 + 1280 + 1568 + 80 and a.with_overhead() == 2 * a.online_bytes()
    f = P.comm_volume(9, 3072, 10)
    assert (f.garbled_in, f.garbled_out, f.plain_in, f.plain_out) == (16 * 9 * 3072, 16 * 9 * 10, 6144, 80)


# ---------------------------------------------------------------- services

def _cfg(oracle, s):
    return P.GarblerConfig(seed=oracle.seed_from_string(s))


def test_loopback_computes_plain_result_in_one_round(eng, oracle):
    c = tiny()
    x = np.random.default_rng(900).integers(-7, 8, size=c.n_in)
    run = P.run_local_protocol(eng, c, x, 2, _cfg(oracle, "90a1"))
    assert run.outputs.tolist() == oracle.plain_forward(c, x).tolist()
    T = P.FrameType
    assert count_type(run.trace, T.GARBLED_INPUT) == 1 and count_type(run.trace, T.GARBLED_OUTPUT) == 1
    assert count_type(run.trace, T.GC_TRANSFER) == 1 and count_type(run.trace, T.INPUT_UPLOAD) == 2
    assert count_type(run.trace, T.ERROR) == 0
    assert [e.type for e in run.trace] == [T.MODEL_UPLOAD, T.GC_TRANSFER, T.INPUT_UPLOAD, T.INPUT_UPLOAD,
                                           T.GARBLED_INPUT, T.GARBLED_OUTPUT, T.RESULT, T.RESULT]
    n_in = c.n_in
    assert run.trace[4].payload_bytes == 16 * c.k * n_in
    assert run.trace[5].payload_bytes == 16 * c.k * 3
    assert run.trace[6].payload_bytes == 0 and run.trace[7].payload_bytes == 8 * 3
    assert run.trace[2].payload_bytes == 10 + 2 * (n_in // 2)


def test_gc_transfer_is_the_reference_gc(eng, oracle):
    # what the GPU garbler ships is serialize_garbled_circuit of the reference
    c = tiny()
    svc = P.GarblerService(eng, _cfg(oracle, "90a9"))
    outs = svc.handle(P.Frame(P.FrameType.MODEL_UPLOAD, 3, P.encode_model_upload(c, 1)))
    assert outs[0].dest == P.Destination.EVALUATOR and outs[0].frame.type == P.FrameType.GC_TRANSFER
    assert outs[0].frame.payload == oracle.garble(c, oracle.seed_from_string("90a9")).gc_bytes()


def test_host_resident_evaluator_gives_the_same_result(eng, oracle):
    # EvaluatorService(host_resident_gc=True): GC rows in pinned host memory,
    # moved to the GPU layer by layer; same garbled output frames
    c = models.build("model_tiny", 1000, 8, private=True)
    x = np.random.default_rng(907).integers(-7, 8, size=c.n_in)
    a = P.run_local_protocol(eng, c, x, 2, _cfg(oracle, "90b1"))
    b = P.run_local_protocol(eng, c, x, 2, _cfg(oracle, "90b1"), host_resident_gc=True)
    assert b.outputs.tolist() == a.outputs.tolist() == oracle.plain_forward(c, x).tolist()
    assert [(e.type, e.payload_bytes) for e in b.trace] == [(e.type, e.payload_bytes) for e in a.trace]


def test_input_partitioning_does_not_change_garbled_input(eng, oracle):
    c = tiny()
    x = np.random.default_rng(901).integers(-7, 8, size=c.n_in)

    def upload(svc, session, owners):
        outs = svc.handle(P.Frame(P.FrameType.MODEL_UPLOAD, session, P.encode_model_upload(c, owners)))
        assert len(outs) == 1 and outs[0].frame.type == P.FrameType.GC_TRANSFER
        gc, gin = outs[0].frame.payload, b""
        chunk = x.size // owners
        for o in range(owners):
            off = o * chunk
            count = x.size - off if o + 1 == owners else chunk
            for out in svc.handle(P.Frame(P.FrameType.INPUT_UPLOAD, session,
                                          P.encode_input_upload(o, off, x[off:off + count]))):
                assert out.frame.type == P.FrameType.GARBLED_INPUT
                gin = out.frame.payload
        return gc, gin

    gc1, gin1 = upload(P.GarblerService(eng, _cfg(oracle, "90a2")), 7, 1)
    gc3, gin3 = upload(P.GarblerService(eng, _cfg(oracle, "90a2")), 7, 3)
    assert gc1 == gc3 and gin1 and gin1 == gin3


def test_garbled_circuits_are_single_use(eng, oracle):
    c = tiny()
    onet = oracle.garble(c, oracle.seed_from_string("90a3"))
    gin = oracle.garble_inputs(onet, np.random.default_rng(903).integers(-7, 8, size=c.n_in))
    ev = P.EvaluatorService(eng)
    assert ev.handle(P.Frame(P.FrameType.GC_TRANSFER, 11, onet.gc_bytes())) is None
    f = P.Frame(P.FrameType.GARBLED_INPUT, 11, gin.payload())
    first = ev.handle(f)
    assert first.type == P.FrameType.GARBLED_OUTPUT and len(first.payload) == 16 * c.k * 3
    assert first.payload == oracle.evaluate(onet, gin).payload()
    second = ev.handle(f)
    assert second.type == P.FrameType.ERROR and P.decode_error(second.payload)[0] == P.ErrorCode.PROTOCOL


def test_evaluator_rejects_foreign_sessions_and_bad_bundles(eng, oracle):
    ev = P.EvaluatorService(eng)
    orphan = ev.handle(P.Frame(P.FrameType.GARBLED_INPUT, 99, b""))
    assert orphan.type == P.FrameType.ERROR and P.decode_error(orphan.payload)[0] == P.ErrorCode.PROTOCOL
    gc = oracle.garble(tiny(), oracle.seed_from_string("90a4")).gc_bytes()
    ev.handle(P.Frame(P.FrameType.GC_TRANSFER, 12, gc))
    bad = ev.handle(P.Frame(P.FrameType.GARBLED_INPUT, 12, bytes([1, 2, 3])))
    assert bad.type == P.FrameType.ERROR and P.decode_error(bad.payload)[0] == P.ErrorCode.DATA
    dup = ev.handle(P.Frame(P.FrameType.GC_TRANSFER, 12, gc))
    assert dup is not None and dup.type == P.FrameType.ERROR
    broken = ev.handle(P.Frame(P.FrameType.GC_TRANSFER, 13, gc[:-3]))
    assert broken.type == P.FrameType.ERROR and P.decode_error(broken.payload)[0] == P.ErrorCode.DATA


def test_evaluator_session_memory(eng, oracle):
    c = tiny()
    onet = oracle.garble(c, oracle.seed_from_string("90a5"))
    ev = P.EvaluatorService(eng)
    assert ev.session_memory(13) == 0
    ev.handle(P.Frame(P.FrameType.GC_TRANSFER, 13, onet.gc_bytes()))
    assert ev.session_memory(13) == onet.cts().size // 2 * 16 + c.k * 16 + 16 * c.k * c.n_in


def test_garbler_rejects_bad_uploads(eng, oracle):
    c = tiny()
    svc = P.GarblerService(eng, _cfg(oracle, "90a6"))
    T, s = P.FrameType, 21

    def one(frame):
        outs = svc.handle(frame)
        assert len(outs) == 1
        return outs[0].frame

    f = one(P.Frame(T.MODEL_UPLOAD, s, P.encode_model_upload(c, 0)))
    assert f.type == T.ERROR and P.decode_error(f.payload)[0] == P.ErrorCode.PROTOCOL
    assert one(P.Frame(T.MODEL_UPLOAD, s, P.encode_model_upload(c, 1))).type == T.GC_TRANSFER
    assert one(P.Frame(T.MODEL_UPLOAD, s, P.encode_model_upload(c, 1))).type == T.ERROR
    f = one(P.Frame(T.RESULT, s, b""))
    assert f.type == T.ERROR and P.decode_error(f.payload)[0] == P.ErrorCode.PROTOCOL
    assert one(P.Frame(T.RESULT, s, b"\x01")).type == T.ERROR
    half = [1] * 36
    assert svc.handle(P.Frame(T.INPUT_UPLOAD, s, P.encode_input_upload(0, 0, half))) == []
    f = one(P.Frame(T.INPUT_UPLOAD, s, P.encode_input_upload(0, 0, half)))
    assert f.type == T.ERROR and P.decode_error(f.payload)[0] == P.ErrorCode.PROTOCOL
    assert one(P.Frame(T.INPUT_UPLOAD, s, P.encode_input_upload(5, 36, half))).type == T.ERROR
    assert one(P.Frame(T.INPUT_UPLOAD, s, P.encode_input_upload(0, 60, half))).type == T.ERROR
    # a model the engine cannot garble is a DATA error
    bad = tiny()
    bad.layers[0].q_weights = bad.layers[0].q_weights[:-1]
    f = one(P.Frame(T.MODEL_UPLOAD, 22, P.encode_model_upload(bad, 1)))
    assert f.type == T.ERROR and P.decode_error(f.payload)[0] == P.ErrorCode.DATA


def test_tampered_garbled_output_fails_with_authenticity(eng, oracle):
    c = tiny()
    svc, ev = P.GarblerService(eng, _cfg(oracle, "90a7")), P.EvaluatorService(eng)
    x = np.random.default_rng(907).integers(-7, 8, size=c.n_in)
    outs = svc.handle(P.Frame(P.FrameType.MODEL_UPLOAD, 31, P.encode_model_upload(c, 1)))
    assert ev.handle(outs[0].frame) is None
    outs = svc.handle(P.Frame(P.FrameType.INPUT_UPLOAD, 31, P.encode_input_upload(0, 0, x)))
    assert len(outs) == 1 and outs[0].frame.type == P.FrameType.GARBLED_INPUT
    reply = ev.handle(outs[0].frame)
    assert reply.type == P.FrameType.GARBLED_OUTPUT
    payload = bytearray(reply.payload)
    payload[5] ^= 0x10
    assert svc.handle(P.Frame(reply.type, 31, bytes(payload))) == []
    assert svc.session_done(31)
    outs = svc.handle(P.Frame(P.FrameType.RESULT, 31, b""))
    assert outs[0].frame.type == P.FrameType.ERROR
    assert P.decode_error(outs[0].frame.payload)[0] == P.ErrorCode.AUTHENTICITY


def test_loopback_honors_owner_count(eng, oracle):
    c = tiny()
    x = np.random.default_rng(908).integers(-7, 8, size=c.n_in)
    want = oracle.plain_forward(c, x).tolist()
    for owners in (1, 3, 5):
        run = P.run_local_protocol(eng, c, x, owners, _cfg(oracle, "90a8"))
        assert run.outputs.tolist() == want
        assert count_type(run.trace, P.FrameType.INPUT_UPLOAD) == owners
        assert count_type(run.trace, P.FrameType.GARBLED_INPUT) == 1


def test_loopback_private_weights_and_extension_model(eng, oracle):
    # private-weight layers travel without weights; DAG circuits carry their
    # extension records through MODEL_UPLOAD and GC_TRANSFER
    from test_engine import _small_dag

    for c in (models.build("model_tiny", 1000, 8, private=True), _small_dag()):
        x = np.random.default_rng(909).integers(-7, 8, size=c.n_in)
        run = P.run_local_protocol(eng, c, x, 2, _cfg(oracle, "90aa"))
        assert run.outputs.tolist() == oracle.plain_forward(c, x).tolist()


def test_frame_decoder_compacts_and_rejects_bad_payload_codecs():
    dec = P.FrameDecoder()
    big = P.Frame(P.FrameType.GC_TRANSFER, 9, bytes(1 << 20))
    small = P.Frame(P.FrameType.RESULT, 9, b"")
    dec.feed(P.encode_frame(big) + P.encode_frame(small) + P.encode_frame(small)[:5])
    assert dec.next().payload == big.payload
    assert dec.next().type == P.FrameType.RESULT
    assert dec.next() is None  # partial frame stays buffered
    dec.feed(P.encode_frame(small)[5:])
    assert dec.next().session == 9
    with pytest.raises(P.ProtocolError):
        P.decode_error(bytes([9]) + P.encode_error(P.ErrorCode.DATA, "x")[1:])
    with pytest.raises(P.DataError):
        P.decode_error(P.encode_error(P.ErrorCode.DATA, "hello")[:-2])
    with pytest.raises(P.ProtocolError):
        P.decode_result(b"\0" * 7)
    with pytest.raises(P.ProtocolError):
        P.encode_frame(P.Frame(P.FrameType.ERROR, 0, bytes((1 << 30) + 1)))


def test_evaluator_rejects_unexpected_frames(eng):
    ev = P.EvaluatorService(eng)
    f = ev.handle(P.Frame(P.FrameType.MODEL_UPLOAD, 5, b""))
    assert f.type == P.FrameType.ERROR and P.decode_error(f.payload)[0] == P.ErrorCode.PROTOCOL
    svc = P.GarblerService(eng)
    out = svc.handle(P.Frame(P.FrameType.GC_TRANSFER, 5, b""))
    assert out[0].frame.type == P.FrameType.ERROR and out[0].dest == P.Destination.REPLY
    # an ERROR frame from the evaluator fails the garbler's session
    c = tiny()
    svc.handle(P.Frame(P.FrameType.MODEL_UPLOAD, 6, P.encode_model_upload(c, 1)))
    assert svc.handle(P.Frame(P.FrameType.ERROR, 6, P.encode_error(P.ErrorCode.DATA, "bad bundle"))) == []
    assert svc.session_done(6)
    res = svc.handle(P.Frame(P.FrameType.RESULT, 6, b""))[0].frame
    assert res.type == P.FrameType.ERROR and P.decode_error(res.payload) == (P.ErrorCode.DATA, "bad bundle")


# ---------------------------------------------------------------- batched evaluator sessions

def _oracle_sessions(oracle, c, n, tag):
    nets = [oracle.garble(c, oracle.seed_from_string(f"{tag}{i}")) for i in range(n)]
    rng = np.random.default_rng(len(tag) + n)
    gins = [oracle.garble_inputs(o, rng.integers(-7, 8, size=c.n_in)) for o in nets]
    return nets, gins


def test_batched_sessions_evaluate_in_one_network(eng, oracle):
    c = tiny()
    nets, gins = _oracle_sessions(oracle, c, 4, "b0")
    ev = P.EvaluatorService(eng)
    T = P.FrameType
    assert ev.handle_batch([P.Frame(T.GC_TRANSFER, 100 + i, o.gc_bytes()) for i, o in enumerate(nets)]) == []
    assert ev.session_memory(101) == ev.session_memory(100) > 0
    # half of the inputs: nothing can be evaluated yet
    assert ev.handle_batch([P.Frame(T.GARBLED_INPUT, 100 + i, gins[i].payload()) for i in (2, 0)]) == []
    out = ev.handle_batch([P.Frame(T.GARBLED_INPUT, 100 + i, gins[i].payload()) for i in (1, 3)])
    assert sorted(f.session for f in out) == [100, 101, 102, 103]
    for f in out:
        i = f.session - 100
        assert f.type == T.GARBLED_OUTPUT
        assert f.payload == oracle.evaluate(nets[i], gins[i]).payload()
    again = ev.handle(P.Frame(T.GARBLED_INPUT, 101, gins[1].payload()))
    assert again.type == T.ERROR and P.decode_error(again.payload)[0] == P.ErrorCode.PROTOCOL


def test_batched_sessions_isolate_a_bad_member(eng, oracle):
    c = tiny()
    nets, gins = _oracle_sessions(oracle, c, 3, "b1")
    ev = P.EvaluatorService(eng)
    T = P.FrameType
    ev.handle_batch([P.Frame(T.GC_TRANSFER, 200 + i, o.gc_bytes()) for i, o in enumerate(nets)])
    # through handle(): member 1's malformed bundle is answered at once,
    # member 2's output arrives with the last input, member 0's stays queued
    assert ev.handle(P.Frame(T.GARBLED_INPUT, 200, gins[0].payload())) is None
    bad = ev.handle(P.Frame(T.GARBLED_INPUT, 201, b"\1\2\3"))
    assert bad.type == T.ERROR and P.decode_error(bad.payload)[0] == P.ErrorCode.DATA
    last = ev.handle(P.Frame(T.GARBLED_INPUT, 202, gins[2].payload()))
    assert last.type == T.GARBLED_OUTPUT and last.payload == oracle.evaluate(nets[2], gins[2]).payload()
    queued = ev.handle_batch([])
    assert [(f.session, f.payload) for f in queued] == [(200, oracle.evaluate(nets[0], gins[0]).payload())]


def test_batched_gc_transfer_of_mixed_circuits_falls_back(eng, oracle):
    a, b = tiny(), models.build("relu16", 0, 5)
    na, nb = oracle.garble(a, seed_hex(0xB2)), oracle.garble(b, seed_hex(0xB3))
    ev = P.EvaluatorService(eng)
    T = P.FrameType
    out = ev.handle_batch([P.Frame(T.GC_TRANSFER, 1, na.gc_bytes()), P.Frame(T.GC_TRANSFER, 2, nb.gc_bytes()),
                           P.Frame(T.GC_TRANSFER, 2, nb.gc_bytes())])
    assert [f.type for f in out] == [T.ERROR]  # the duplicate session
    gb = oracle.garble_inputs(nb, np.arange(16) - 8)
    r = ev.handle(P.Frame(T.GARBLED_INPUT, 2, gb.payload()))
    assert r.type == T.GARBLED_OUTPUT and r.payload == oracle.evaluate(nb, gb).payload()


def test_batched_group_deadline_flushes_a_stalled_member(eng, oracle):
    """a member whose GARBLED_INPUT never arrives must not starve
    the group: after the deadline the present members get their outputs and
    the missing one an ERROR frame (its circuit is consumed)."""
    c = tiny()
    nets, gins = _oracle_sessions(oracle, c, 3, "b4")
    ev = P.EvaluatorService(eng, batch_timeout=5.0)
    T = P.FrameType
    ev.handle_batch([P.Frame(T.GC_TRANSFER, 300 + i, o.gc_bytes()) for i, o in enumerate(nets)])
    assert ev.handle_all(P.Frame(T.GARBLED_INPUT, 300, gins[0].payload())) == []
    assert ev.handle_all(P.Frame(T.GARBLED_INPUT, 302, gins[2].payload())) == []
    import time
    assert ev.flush_expired(time.monotonic()) == []  # not expired yet
    out = ev.flush_expired(time.monotonic() + 10.0)
    got = {f.session: f for f in out}
    assert sorted(got) == [300, 301, 302]
    assert got[301].type == T.ERROR and P.decode_error(got[301].payload)[0] == P.ErrorCode.PROTOCOL
    for i in (0, 2):
        assert got[300 + i].type == T.GARBLED_OUTPUT
        assert got[300 + i].payload == oracle.evaluate(nets[i], gins[i]).payload()
    late = ev.handle(P.Frame(T.GARBLED_INPUT, 301, gins[1].payload()))
    assert late.type == T.ERROR  # single use
    assert ev.flush_expired(time.monotonic() + 20.0) == []


def test_handle_all_returns_every_completed_reply(eng, oracle):
    c = tiny()
    nets, gins = _oracle_sessions(oracle, c, 2, "b5")
    ev = P.EvaluatorService(eng)
    T = P.FrameType
    ev.handle_batch([P.Frame(T.GC_TRANSFER, 400 + i, o.gc_bytes()) for i, o in enumerate(nets)])
    assert ev.handle_all(P.Frame(T.GARBLED_INPUT, 400, gins[0].payload())) == []
    out = ev.handle_all(P.Frame(T.GARBLED_INPUT, 401, gins[1].payload()))
    assert sorted(f.session for f in out) == [400, 401]
    assert ev.take_ready() == []


def test_garbler_releases_the_gc_after_transfer(eng, oracle):
    """the garbler keeps only encoding / decoding material once the
    GC has been sent (dashgpu_network_release_gc); the session still encodes
    inputs and decodes the result, and its device network is dropped once
    the result is known."""
    c = tiny()
    g = P.GarblerService(eng, P.GarblerConfig(seed=seed_hex(0x77)))
    T = P.FrameType
    out = g.handle(P.Frame(T.MODEL_UPLOAD, 9, P.encode_model_upload(c, 1)))
    gc = out[0].frame.payload
    net = g._sessions[9].net
    with pytest.raises(P.DataError):
        net.export_gc(0)
    x = np.random.default_rng(5).integers(-7, 8, size=c.n_in)
    gin = g.handle(P.Frame(T.INPUT_UPLOAD, 9, P.encode_input_upload(0, 0, x)))[0].frame.payload
    on = oracle.garble(c, seed_hex(0x77))
    assert gc == on.gc_bytes()
    og = oracle.garble_inputs(on, x)
    assert gin == og.payload()
    gout = oracle.evaluate(on, og).payload()
    assert g.handle(P.Frame(T.GARBLED_OUTPUT, 9, gout)) == []
    assert g._sessions[9].net is None
    res = g.handle(P.Frame(T.RESULT, 9, b""))[0].frame
    assert res.type == T.RESULT
    assert (P.decode_result(res.payload) == oracle.decode(on, oracle.evaluate(on, og))).all()


# ---------------------------------------------------------------- TCP transport (protocol.cpp:437-659)

def test_tcp_remote_infer_matches_plain_forward(eng, oracle):
    # serve_evaluator + serve_garbler + remote_infer on loopback sockets: the
    # client gets the plain result, for several owner splits and two
    # concurrent clients on one garbler
    import threading

    c = tiny()
    with P.EvaluatorServer(eng, "127.0.0.1", 0) as ev, \
            P.GarblerServer(eng, "127.0.0.1", ev.port, "127.0.0.1", 0) as gb:
        for owners, seed in ((1, 910), (3, 911)):
            x = np.random.default_rng(seed).integers(-7, 8, size=c.n_in)
            got = P.remote_infer("127.0.0.1", gb.port, c, x, owners)
            assert got.tolist() == oracle.plain_forward(c, x).tolist()
        xs = [np.random.default_rng(920 + i).integers(-7, 8, size=c.n_in) for i in range(2)]
        res = [None, None]

        def client(i):
            res[i] = P.remote_infer("127.0.0.1", gb.port, c, xs[i], 2)

        ts = [threading.Thread(target=client, args=(i,)) for i in range(2)]
        for t in ts:
            t.start()
        for t in ts:
            t.join(60)
        assert [r.tolist() for r in res] == [oracle.plain_forward(c, x).tolist() for x in xs]
        assert all(gb.service.session_done(s) for s in list(gb.service._sessions))


def test_tcp_errors_reach_the_client(eng, oracle):
    c = tiny()
    x = np.zeros(c.n_in, np.int64)
    with pytest.raises(P.DataError):  # client-side checks (protocol.cpp:620-622)
        P.remote_infer("127.0.0.1", 1, c, x[:-1])
    with pytest.raises(P.DataError):
        P.remote_infer("127.0.0.1", 1, c, x, 0)
    with pytest.raises(P.ProtocolError):  # nothing listens there
        P.remote_infer("127.0.0.1", 1, c, x)
    with P.EvaluatorServer(eng, "127.0.0.1", 0) as ev, \
            P.GarblerServer(eng, "127.0.0.1", ev.port, "127.0.0.1", 0) as gb:
        # more owners than input elements: the garbler's ERROR reply is what the
        # client's RESULT poll reads first
        with pytest.raises(P.ProtocolError, match="more input owners"):
            P.remote_infer("127.0.0.1", gb.port, c, x, c.n_in + 1)
        # a raw client asking for an unknown session's result
        import socket

        with socket.create_connection(("127.0.0.1", gb.port)) as s:
            s.sendall(P.encode_frame(P.Frame(P.FrameType.RESULT, 77, b"")))
            f = P._read_frame(s, P.FrameDecoder())
            assert f.type == P.FrameType.ERROR and "unknown session" in P.decode_error(f.payload)[1]
