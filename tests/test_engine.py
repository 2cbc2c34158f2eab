"""Parity of the engine against the reference (golden vectors) and the CPU oracle.

Every test runs twice:
  * ``emu``  — the device code compiled for the host (tests/emu, CPU only),
  * ``cuda`` — the product, libdashgpu.so on a B200 (``-m gpu``).
Bit-exact is the bar: garbled circuits, encodings, decoding tables, garbled
inputs/outputs and decoded values must equal the reference byte for byte
(sha256 over the reference's own wire formats, garble.cpp:347-526).
"""
import numpy as np
import pytest

from helpers import PRIMES, golden_circuit, golden_input, pairs_u128, seed_hex, sha, u128_pairs

BACKENDS = [pytest.param("emu", id="emu"), pytest.param("cuda", id="cuda", marks=pytest.mark.gpu)]


@pytest.fixture(params=BACKENDS)
def eng(request):
    return request.getfixturevalue("emu" if request.param == "emu" else "gpu")


def is_emu(eng):
    return eng.lib._name.endswith("libdashemu.so")


# ---------------------------------------------------------------- primitives

def test_codec_all_moduli(eng, golden):
    rows = golden["kat"]["codec"]
    for m in range(2, 129):
        mine = [r for r in rows if r[0] == m]
        vals = [int(r[1], 16) for r in mine]
        out, dg = eng.prim(0, m, inp=u128_pairs(vals))
        for r, back, d in zip(mine, pairs_u128(out), dg):
            assert d[: len(r[2])].tolist() == r[2], m
            assert hex(back) == r[3], m


def test_aes_pi_and_keyed(eng, golden, oracle):
    rnd = np.random.default_rng(5)
    vals = [int(x) for x in rnd.integers(0, 2**62, size=64)] + [0, (1 << 128) - 1]
    out, _ = eng.prim(1, 2, inp=u128_pairs(vals))
    assert pairs_u128(out) == [oracle.aes_fixed(v) for v in vals]
    for key, x, y in golden["kat"]["aes_key"]:
        out, _ = eng.prim(2, 2, inp=u128_pairs([int(x, 16)]), key=bytes.fromhex(key))
        assert hex(pairs_u128(out)[0]) == y


def test_prf_labels_and_offsets(eng, golden):
    seed = bytes.fromhex(golden["kat"]["seed_5eed1"])
    for m, wire, d in golden["kat"]["prf"]:
        w = m if wire < 0 else wire
        _, dg = eng.prim(3, m, q=1 if wire < 0 else 0, key=seed, wires=np.array([w], np.uint64), n=1)
        got = dg[0, : len(d)].tolist()
        if wire < 0:
            got[0] = 1  # prf.hpp:28-32: the offset's colour digit is forced to 1
        assert got == d, (m, wire)


def test_row_encryption_roundtrip(eng, oracle):
    seed = seed_hex(0x77)
    rnd = np.random.default_rng(6)
    for m, q in [(7, 11), (2, 2), (110, 2), (3, 9), (33, 5), (19, 2), (8, 33), (128, 64), (53, 3)]:
        keys = [oracle.compress(m, oracle.prf_label(seed, 100 + i, m)) for i in range(16)]
        msgs_l = [oracle.prf_label(seed, 200 + i, q) for i in range(16)]
        msgs = [oracle.compress(q, l) for l in msgs_l]
        gate = int(rnd.integers(0, 2**40))
        ct, _ = eng.prim(4, m, q=q, inp=u128_pairs(keys), out=u128_pairs(msgs), gate=gate)
        cts = pairs_u128(ct)
        for i in range(16):
            kd = oracle.decompress_mod(keys[i], m)
            assert cts[i] == oracle.encrypt_label(m, kd, gate, i % 7, i % 3, q, msgs_l[i])
        _, dg = eng.prim(5, m, q=q, inp=u128_pairs(keys), out=ct, gate=gate)
        for i in range(16):
            assert dg[i, : len(msgs_l[i])].tolist() == msgs_l[i]


# ---------------------------------------------------------------- networks

def _run_golden(eng, rec, batch_extra=1):
    c = golden_circuit(rec)
    g = eng.circuit(c)
    s0 = int(rec["garble_seed"], 16)
    seeds = seed_hex(s0) + b"".join(seed_hex(s0 ^ (0xF00D + i)) for i in range(batch_extra))
    net = eng.garble(g, seeds)
    gc = net.export_gc(0)
    assert len(gc) == rec["gc_len"]
    assert sha(gc) == rec["gc"], rec["tag"]
    assert sha(net.export_encoding(0)) == rec["enc"]
    assert sha(net.export_decoding(0)) == rec["dec"]
    assert g.info.cts == rec["stats"][0] and g.info.gates == rec["stats"][1] and g.info.wires == rec["stats"][2]
    for inp in rec["inputs"]:
        x = golden_input(rec, inp, c.n_in)
        xb = np.stack([x] * (1 + batch_extra))
        bi = eng.garble_inputs(net, xb)
        assert sha(bi.payload(0)) == inp["gin"]
        bo = eng.evaluate(net, bi)
        assert sha(bo.payload(0)) == inp["gout"]
        out = eng.decode_outputs(net, bo)
        assert out[0].tolist() == inp["decoded"]
        # the other inferences of the batch used other seeds but the same
        # inputs: the decoded values must agree
        assert (out == out[0]).all()
    return g, net


def _golden_ids(golden_path):
    import json

    recs = json.load(open(golden_path))["networks"]
    return [r["tag"] for r in recs]


def pytest_generate_tests(metafunc):
    if "golden_tag" in metafunc.fixturenames:
        from conftest import GOLDEN

        metafunc.parametrize("golden_tag", _golden_ids(GOLDEN))


def test_network_golden(eng, golden, golden_tag):
    rec = next(r for r in golden["networks"] if r["tag"] == golden_tag)
    if is_emu(eng) and rec["stats"][0] > 3_000_000:
        pytest.skip("large network: GPU suite only")
    _run_golden(eng, rec)


def test_batch_composition_does_not_change_a_garbling(eng):
    g = eng.model("model_tiny", 1000, 8)
    seeds = [seed_hex(0x1000 + i) for i in range(5)]
    alone = eng.garble(g, seeds[3]).export_gc(0)
    batch = eng.garble(g, b"".join(seeds))
    assert batch.export_gc(3) == alone
    assert batch.export_gc(0) != alone


def test_decoded_equals_plain_forward(eng):
    # decode(eval(garble)) == plain_forward (test_garble.cpp:29-51)
    for name, seed, k in [("model_a", 1001, 8), ("model_tiny", 1000, 8), ("model_f_dims", 1006, 9)]:
        g = eng.model(name, seed, k)
        B = 4
        net = eng.garble(g, b"".join(seed_hex(0x5EED0000 + b) for b in range(B)))
        x = np.stack([g.random_input(4000 + b) for b in range(B)])
        out = eng.decode_outputs(net, eng.evaluate(net, eng.garble_inputs(net, x)))
        for b in range(B):
            assert out[b].tolist() == g.plain_forward(x[b]).tolist(), (name, b)


def test_private_weights_change_nothing(eng):
    # test_garble.cpp:36-43: private-weight layers compute the same values
    pub, priv = eng.model("model_tiny", 1000, 8), eng.model("model_tiny", 1000, 8, private=True)
    x = np.stack([pub.random_input(102 + i) for i in range(3)])
    seeds = b"".join(seed_hex(0x5EED2 + i) for i in range(3))
    a = eng.decode_outputs(n := eng.garble(pub, seeds), eng.evaluate(n, eng.garble_inputs(n, x)))
    b = eng.decode_outputs(m := eng.garble(priv, seeds), eng.evaluate(m, eng.garble_inputs(m, x)))
    assert (a == b).all()


def test_relu_sign_boundaries(eng):
    # ReLU(0) = 0 and sign(0) = -1 (gadgets.hpp:437-440, layer.cpp:362-371)
    from helpers import models

    k = 5
    for name in ("relu16", "sign16"):
        g = eng.circuit(models.build(name, 0, k))
        net = eng.garble(g, seed_hex(0x99))
        x = np.array([[0, 1, -1, 2, -2, 7, -7, 3, -3, 100, -100, 1154, -1155, 0, 5, -5]], np.int64)
        out = eng.decode_outputs(net, eng.evaluate(net, eng.garble_inputs(net, x)))[0]
        want = np.where(x[0] > 0, x[0], 0) if name.startswith("relu") else np.where(x[0] > 0, 1, -1)
        assert out.tolist() == want.tolist(), name


def test_tampered_output_raises_authenticity(eng):
    from paper_2302_06361_b200.engine import AuthenticityError

    g = eng.model("model_tiny", 1000, 8)
    net = eng.garble(g, seed_hex(0x31))
    bo = eng.evaluate(net, eng.garble_inputs(net, g.random_input(7)[None, :]))
    payload = bytearray(bo.payload(0))
    assert eng.decode_outputs(net, eng.import_bundle(net, bytes(payload), True)).tolist() == \
        eng.decode_outputs(net, bo).tolist()
    payload[17] ^= 0x04
    with pytest.raises(AuthenticityError):
        eng.decode_outputs(net, eng.import_bundle(net, bytes(payload), True))


def test_tampered_ciphertexts_are_detected(eng):
    # acceptance criterion 6 (acceptance_main.cpp:581-614): corrupting the
    # tables of the last activation layer corrupts every output label
    from paper_2302_06361_b200.engine import AuthenticityError

    g = eng.model("model_tiny", 1000, 8)
    net = eng.garble(g, seed_hex(0x32))
    x = g.random_input(8)[None, :]
    base = 92672  # layer_ct_base of the final ReLU of model_tiny
    for i in range(base, 101007):
        net.tamper(0, i, bytes([0x5A] * 16))
    with pytest.raises(AuthenticityError):
        eng.decode_outputs(net, eng.evaluate(net, eng.garble_inputs(net, x)))


def test_input_out_of_range_is_a_data_error(eng):
    from paper_2302_06361_b200.engine import DataError

    g = eng.model("relu4", 0, 2)  # P_2 = 6: representable [-3, 2]
    net = eng.garble(g, seed_hex(1))
    eng.garble_inputs(net, np.array([[-3, 2, 0, 1]]))
    with pytest.raises(DataError):
        eng.garble_inputs(net, np.array([[3, 0, 0, 0]]))
    with pytest.raises(DataError):
        eng.garble_inputs(net, np.array([[-4, 0, 0, 0]]))


def test_bundle_export_import_roundtrip(eng):
    g = eng.model("model_tiny", 1000, 8)
    net = eng.garble(g, seed_hex(0x41) + seed_hex(0x42))
    x = np.stack([g.random_input(1), g.random_input(2)])
    bi = eng.garble_inputs(net, x)
    payload = bi.payload(0) + bi.payload(1)
    bi2 = eng.import_bundle(net, payload, False)
    a = eng.decode_outputs(net, eng.evaluate(net, bi))
    b = eng.decode_outputs(net, eng.evaluate(net, bi2))
    assert (a == b).all()


def test_infer_pipeline_matches_stepwise(eng):
    g = eng.model("model_a", 1001, 8)
    B = 3
    seeds = b"".join(seed_hex(0x5EED0000 + b) for b in range(B))
    x = np.stack([g.random_input(4000 + b) for b in range(B)])
    out, t = eng.infer(g, seeds, x)
    net = eng.garble(g, seeds)
    ref = eng.decode_outputs(net, eng.evaluate(net, eng.garble_inputs(net, x)))
    assert (out == ref).all()
    assert t.sub_batches >= 1


# ---------------------------------------------------------------- GPU-scale

@pytest.mark.gpu
def test_lenet_batch_vs_oracle(gpu, oracle):
    g = gpu.model("lenet5", 2001, 8)
    B = 16
    seeds = b"".join(seed_hex(0x5EED0000 + b) for b in range(B))
    x = np.stack([g.random_input(4000 + b) for b in range(B)])
    out, _ = gpu.infer(g, seeds, x)
    c = g.to_circuit()
    for b in (0, 7, 15):
        onet = oracle.garble(c, seed_hex(0x5EED0000 + b))
        want = oracle.decode(onet, oracle.evaluate(onet, oracle.garble_inputs(onet, x[b])))
        assert out[b].tolist() == want.tolist(), b
    net = gpu.garble(g, seeds[16 * 7: 16 * 8])
    assert net.export_gc(0) == oracle.garble(c, seed_hex(0x5EED0007)).gc_bytes()


@pytest.mark.gpu
def test_relu_sweep_2p16_property(gpu):
    # size-independent property at sweep scale: ReLU is exact
    # for values inside the signed range
    g = gpu.model("relu65536", 0, 8)
    x = np.random.default_rng(3).integers(-4_000_000, 4_000_000, size=(1, 65536))
    out, _ = gpu.infer(g, seed_hex(0xA1), x)
    assert (out[0] == np.maximum(x[0], 0)).all()


@pytest.mark.gpu
def test_sign_sweep_k2_to_k9(gpu):
    for k in range(2, 10):
        P = int(np.prod([2, 3, 5, 7, 11, 13, 17, 19, 23][:k]))
        lo, hi = -(P // 2), (P + 1) // 2 - 1
        g = gpu.model("sign4096", 0, k)
        x = np.random.default_rng(k).integers(lo, hi + 1, size=(2, 4096))
        x[:, :3] = [0, 1, -1]
        out, _ = gpu.infer(g, seed_hex(0xB0 + k) + seed_hex(0xC0 + k), x)
        assert (out == np.where(x > 0, 1, -1)).all(), k


# ------------------------------------------------- tensor-core linear lanes

def _linear_case(kind):
    """Circuits that stress the tcgen05 GEMM tiling (tc_linear.cuh): several N
    tiles (4*out_ch > 256), many K stages, strided windows, ragged row tiles."""
    from paper_2302_06361_b200.circuit import Circuit, conv2d, dense, flatten, relu

    r = np.random.default_rng({"wide": 11, "deep": 12, "strided": 13, "ntiles": 14, "ragged": 15}[kind])
    w = lambda *s: r.integers(-2, 3, size=s)  # noqa: E731
    b = lambda n: r.integers(-10, 11, size=n)  # noqa: E731
    if kind == "wide":   # conv N = 512 (2 tiles), dense N = 280 (BN 256, 2 tiles)
        L = [conv2d(3, 128, 3, 1, w(128, 3, 3, 3), b(128)), flatten(), dense(2048, 70, w(70, 2048), b(70)), relu(),
             dense(70, 10, w(10, 70), b(10))]
        return Circuit([3, 6, 6], 9, L)
    if kind == "ntiles":  # conv N = 272 and dense N = 300: two BN = 256 column tiles each; K = 4352
        L = [conv2d(3, 272, 3, 1, w(272, 3, 3, 3), b(272)), flatten(), dense(4352, 300, w(300, 4352), b(300)),
             relu(), dense(300, 10, w(10, 300), b(10))]
        return Circuit([3, 6, 6], 8, L)
    if kind == "ragged":  # E_in % 4 != 0: the dense window goes through the offset table, not 16-byte loads
        L = [dense(1001, 40, w(40, 1001), b(40)), relu(), dense(40, 3, w(3, 40), b(3))]
        return Circuit([1001], 6, L)
    if kind == "deep":   # K = 3000 window elements: 24 K stages, zero-padded tail
        L = [dense(3000, 20, w(20, 3000), b(20)), relu(), dense(20, 3, w(3, 20), b(3))]
        return Circuit([3000], 8, L)
    # strided / non-square windows over ragged planes (E_in = 5*13*11)
    L = [conv2d(5, 7, 4, 3, w(7, 5, 4, 4), b(7)), relu(), conv2d(7, 9, 2, 1, w(9, 7, 2, 2), b(9)), flatten(),
         dense(9 * 3 * 2, 5, w(5, 54), b(5))]
    return Circuit([5, 13, 11], 7, L)


@pytest.mark.parametrize("kind", ["wide", "ntiles", "ragged", "deep", "strided"])
def test_tensor_core_linear_vs_oracle(eng, oracle, kind):
    gpu = eng
    c = _linear_case(kind)
    g = gpu.circuit(c)
    B = 5  # rows per lane = B * nw * positions: ragged 128-row tiles
    seeds = b"".join(seed_hex(0x7C0 + i) for i in range(B))
    x = np.random.default_rng(21).integers(-7, 8, size=(B, c.n_in)).astype(np.int64)
    net = gpu.garble(g, seeds)
    bo = gpu.evaluate(net, gpu.garble_inputs(net, x))
    out = gpu.decode_outputs(net, bo)
    for i in (0, B - 1):
        onet = oracle.garble(c, seed_hex(0x7C0 + i))
        assert net.export_gc(i) == onet.gc_bytes(), (kind, i)
        assert net.export_decoding(i) == onet.dec_bytes(), (kind, i)
        ob = oracle.evaluate(onet, oracle.garble_inputs(onet, x[i]))
        assert bo.payload(i) == ob.payload(), (kind, i)
        assert out[i].tolist() == oracle.decode(onet, ob).tolist()
        assert out[i].tolist() == g.plain_forward(x[i]).tolist()


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["wide", "ntiles", "deep"])
def test_tensor_core_linear_cta_pairs_vs_oracle(gpu, oracle, monkeypatch, kind):
    # the opt-in CTA-pair digit-row kernel (tcgen05.mma.cta_group::2, M = 256,
    # each CTA holding half of the weight tile) gives the same bytes
    monkeypatch.setenv("DASH_TC_CG", "2")
    test_tensor_core_linear_vs_oracle(gpu, oracle, kind)


# ------------------------------------------------------- streamed sweep layers

@pytest.mark.parametrize("name,k,chunk", [("relu3000", 4, 1024), ("sign777", 5, 100), ("relu300", 8, 300)])
def test_streamed_layer_vs_oracle(eng, oracle, name, k, chunk):
    # chunks of a single activation layer keep the reference's numbering:
    # the concatenated chunk tables are the layer's GarbledCircuit::cts
    from helpers import models

    c = models.build(name, 0, k)
    g = eng.circuit(c)
    seeds = seed_hex(0x5A0 + k) + seed_hex(0x5B0 + k)
    P = int(np.prod(PRIMES[:k]))
    x = np.random.default_rng(k).integers(-(P // 2), (P + 1) // 2, size=(2, c.n_in))
    x[:, :3] = [0, 1, -1]
    out, t, gcs = eng.infer_stream(g, seeds, x, chunk, want_gc=True)
    assert t.sub_batches == 2 * ((c.n_in + chunk - 1) // chunk)
    want = np.maximum(x, 0) if name.startswith("relu") else np.where(x > 0, 1, -1)
    assert (out == want).all()
    onet = oracle.garble(c, seed_hex(0x5B0 + k))
    assert gcs[1] == onet.cts().tobytes()
    ref, _ = eng.infer(g, seeds, x)
    assert (ref == out).all()


# ------------------------------------- extensions: Pad2d / Add / DAG (ResNet)

def _small_dag():
    """pad -> conv -> relu -> pad -> conv, + 1x1 shortcut of the input, add,
    relu, flatten, dense: a residual block whose values stay in range."""
    from paper_2302_06361_b200.circuit import Circuit, add, conv2d, dense, flatten, pad2d, relu

    r = np.random.default_rng(31)
    w = lambda *s: r.integers(-1, 2, size=s)  # noqa: E731
    b = lambda n: r.integers(-3, 4, size=n)  # noqa: E731
    L = [pad2d(1), conv2d(2, 3, 3, 1, w(3, 2, 3, 3), b(3)), relu(), pad2d(1), conv2d(3, 3, 3, 2, w(3, 3, 3, 3), b(3)),
         conv2d(2, 3, 1, 2, w(3, 2, 1, 1), b(3), src=-1), add(5), relu(), flatten(), dense(27, 4, w(4, 27), b(4))]
    return Circuit([2, 5, 5], 8, L)


def test_extension_layers_semantics(eng, oracle):
    # decode(eval(garble)) == plain_forward for the extension layers too, in
    # the oracle (pinned by restatement) and in the engine
    c = _small_dag()
    assert c.shapes()[5] == [3, 3, 3] and c.shapes()[7] == [3, 3, 3]
    x = np.random.default_rng(2).integers(-7, 8, size=(3, c.n_in))
    want = np.stack([oracle.plain_forward(c, xi) for xi in x])
    for i in range(3):
        onet = oracle.garble(c, seed_hex(0xD0 + i))
        assert oracle.decode(onet, oracle.evaluate(onet, oracle.garble_inputs(onet, x[i]))).tolist() == want[i].tolist()
    g = eng.circuit(c)
    assert (np.stack([g.plain_forward(xi) for xi in x]) == want).all()
    out, _ = eng.infer(g, b"".join(seed_hex(0xD0 + i) for i in range(3)), x)
    assert (out == want).all()


@pytest.mark.parametrize("name", ["dag", "resnet_tiny"])
def test_extension_networks_vs_oracle(eng, oracle, name):
    from helpers import models

    c = _small_dag() if name == "dag" else models.build("resnet_tiny", 2001, 8)
    g = eng.circuit(c)
    B = 2
    seeds = b"".join(seed_hex(0xE0 + i) for i in range(B))
    x = np.random.default_rng(5).integers(-7, 8, size=(B, c.n_in))
    net = eng.garble(g, seeds)
    bo = eng.evaluate(net, eng.garble_inputs(net, x))
    out = eng.decode_outputs(net, bo)
    onet = oracle.garble(c, seed_hex(0xE1))
    assert net.export_gc(1) == onet.gc_bytes()
    assert net.export_decoding(1) == onet.dec_bytes()
    ob = oracle.evaluate(onet, oracle.garble_inputs(onet, x[1]))
    assert bo.payload(1) == ob.payload()
    assert out[1].tolist() == oracle.decode(onet, ob).tolist()


def test_resnet20_shape_and_cost():
    from helpers import models

    c = models.build("resnet20", 2001, 8)
    s = c.shapes()
    assert s[0] == [3, 32, 32] and s[-1] == [10]
    relu = sum(int(np.prod(s[j + 1])) for j, l in enumerate(c.layers) if l.kind == 3)
    assert relu == 188_416  # 188,416 ReLU per inference


def test_infer_batch19_matches_stepwise(eng):
    # a larger batch through the fused call (decode finished from pinned residues)
    g = eng.model("model_tiny", 1000, 8)
    B = 19
    seeds = b"".join(seed_hex(0x7A000 + b) for b in range(B))
    x = np.stack([g.random_input(500 + b) for b in range(B)])
    out, t = eng.infer(g, seeds, x)
    assert t.sub_batches >= 1
    net = eng.garble(g, seeds)
    ref = eng.decode_outputs(net, eng.evaluate(net, eng.garble_inputs(net, x)))
    assert (out == ref).all()
    assert all(out[b].tolist() == g.plain_forward(x[b]).tolist() for b in range(B))


# ------------------------------------------------ layer level (layer.hpp:79-97)

def _layer_by_layer(eng, g, c, seeds, x):
    net = eng.network_setup(g, seeds)
    outs = [eng.input_base(net)]
    for li, l in enumerate(c.layers):
        src = li if l.src == 0 else (0 if l.src < 0 else l.src)
        src2 = None if l.kind != 7 else outs[li if l.src2 == 0 else (0 if l.src2 < 0 else l.src2)]
        outs.append(eng.layer_garble(net, li, outs[src], src2))
    eng.network_finish(net, outs[-1])
    act = [eng.garble_inputs(net, x)]
    for li, l in enumerate(c.layers):
        src = li if l.src == 0 else (0 if l.src < 0 else l.src)
        src2 = None if l.kind != 7 else act[li if l.src2 == 0 else (0 if l.src2 < 0 else l.src2)]
        act.append(eng.layer_eval(net, li, act[src], src2))
    return net, outs, act


@pytest.mark.parametrize("name", ["model_tiny_priv", "model_tiny", "dag"])
def test_layer_level_api_matches_whole_network(eng, name):
    from helpers import models

    c = _small_dag() if name == "dag" else models.build("model_tiny", 1000, 8, name.endswith("priv"))
    g = eng.circuit(c)
    seeds = seed_hex(0x1A1) + seed_hex(0x1A2)
    x = np.random.default_rng(9).integers(-7, 8, size=(2, c.n_in))
    net, outs, act = _layer_by_layer(eng, g, c, seeds, x)
    whole = eng.garble(g, seeds)
    for b in range(2):
        assert net.export_gc(b) == whole.export_gc(b)
        assert net.export_decoding(b) == whole.export_decoding(b)
        assert net.export_encoding(b) == whole.export_encoding(b)
    ref = eng.evaluate(whole, eng.garble_inputs(whole, x))
    assert act[-1].payload(1) == ref.payload(1)
    assert (eng.decode_outputs(net, act[-1]) == eng.decode_outputs(whole, ref)).all()
    assert sum(eng.layer_count(g, li)[0] for li in range(len(c.layers))) == g.info.cts


def test_label_tensor_images_roundtrip(eng):
    g = eng.model("model_tiny", 1000, 8)
    net = eng.garble(g, seed_hex(0x1B0))
    bi = eng.garble_inputs(net, g.random_input(3)[None, :])
    lanes = [bi.labels(i) for i in range(8)]
    assert lanes[0].shape == (1, g.info.n_in, 128) and lanes[1].shape == (1, g.info.n_in, 80)
    assert all((l < p).all() for l, p in zip(lanes, [2, 3, 5, 7, 11, 13, 17, 19]))
    back = eng.bundle_from_labels(net, lanes)
    assert back.payload(0) == bi.payload(0)
    out = eng.decode_outputs(net, eng.evaluate(net, back))
    assert out[0].tolist() == g.plain_forward(g.random_input(3)).tolist()


@pytest.mark.parametrize("p,q", [(3, 110), (7, 2), (2, 8), (19, 5), (110, 2)])
def test_projection_gate_primitive_vs_oracle(eng, oracle, p, q):
    # t_proj (gadgets.hpp:146-176): every garbled row equals the oracle's
    # encrypt_label of (in + aR_p) over (out0 + phi(a) R_q); evaluation of any
    # active input recovers out0 + phi(v) R_q
    seed = seed_hex(0xC0DE + p)
    rnd = np.random.default_rng(p * 1000 + q)
    n = 24
    phi = rnd.integers(0, q, size=p).tolist()
    base = [oracle.compress(p, oracle.prf_label(seed_hex(0x77), 300 + i, p)) for i in range(n)]
    gates = rnd.integers(0, 2**40, size=n).tolist()
    wires = (10_000 + np.arange(n)).tolist()
    rows, out0, (Rp, Rq) = eng.proj_garble(seed, p, q, phi, base, gates, wires)
    rp = np.array(oracle.decompress_mod(Rp, p))
    rq = np.array(oracle.decompress_mod(Rq, q))
    assert rp[0] == 1 and rq[0] == 1  # offsets have colour digit 1 (prf.hpp:28-32)
    vs = rnd.integers(0, p, size=n)
    active = []
    for i in range(n):
        x = np.array(oracle.decompress_mod(base[i], p))
        o0 = np.array(oracle.decompress_mod(out0[i], q))
        assert o0.tolist() == oracle.prf_label(seed, wires[i], q)
        c = int(x[0])
        for a in range(p):
            key = ((x + a * rp) % p).tolist()
            msg = ((o0 + phi[a] * rq) % q).tolist()
            assert rows[i][(c + a) % p] == oracle.encrypt_label(p, key, gates[i], (c + a) % p, 0, q, msg), (i, a)
        active.append(oracle.compress(p, ((x + int(vs[i]) * rp) % p).tolist()))
    got = eng.proj_eval(p, q, active, gates, rows)
    for i in range(n):
        o0 = np.array(oracle.decompress_mod(out0[i], q))
        assert got[i] == oracle.compress(q, ((o0 + phi[vs[i]] * rq) % q).tolist())


def test_streamed_layer_element_ranges_compose(eng):
    # element-range shards of one layer reproduce the whole layer
    from helpers import models

    c = models.build("relu3000", 0, 4)
    g = eng.circuit(c)
    seed = seed_hex(0x5C0)
    x = np.random.default_rng(1).integers(-100, 100, size=(1, c.n_in))
    full, _, gcf = eng.infer_stream(g, seed, x, 512, want_gc=True)
    uc = g.info.cts // c.n_in
    parts_out = np.zeros_like(full)
    gc = bytearray(len(gcf[0]))
    for a, b in [(0, 1100), (1100, 1101), (1101, 3000)]:
        o, t, gp = eng.infer_stream(g, seed, x, 512, want_gc=True, u_range=(a, b))
        parts_out[:, a:b] = o[:, a:b]
        gc[a * uc * 16:b * uc * 16] = gp[0][a * uc * 16:b * uc * 16]
    assert (parts_out == full).all()
    assert bytes(gc) == gcf[0]


# ------------------------------------------- evaluator side: GC import (protocol)

def _evaluator_session(eng, oracle, c, seeds, x):
    """EvaluatorService flow (protocol.cpp:309-331) with the GCs made by the
    oracle: GC bytes -> import -> evaluate the oracle's garbled inputs; the
    returned payload must be the oracle evaluator's, byte for byte."""
    onets = [oracle.garble(c, s) for s in seeds]
    gcs = [o.gc_bytes() for o in onets]
    ev = eng.import_gc(gcs)
    assert ev.batch == len(seeds)
    for b, g in enumerate(gcs):  # parse -> serialize is the identity
        assert ev.export_gc(b) == g
    obi = [oracle.garble_inputs(o, xi) for o, xi in zip(onets, x)]
    bi = eng.import_bundle(ev, b"".join(o.payload() for o in obi), False)
    bo = eng.evaluate(ev, bi)
    for b, o in enumerate(onets):
        ob = oracle.evaluate(o, obi[b])
        assert bo.payload(b) == ob.payload(), b
        # the garbler decodes the returned GARBLED_OUTPUT (GarblerService)
        assert oracle.decode(o, oracle.bundle_from_payload(o, bo.payload(b), True)).tolist() == \
            oracle.decode(o, ob).tolist()
    return ev


@pytest.mark.parametrize("private", [False, True])
def test_import_gc_evaluates_oracle_gcs(eng, oracle, private):
    from helpers import models

    c = models.build("model_tiny", 1000, 8, private=private)
    seeds = [seed_hex(0x1E0), seed_hex(0x1E1)]
    x = np.random.default_rng(11).integers(-7, 8, size=(2, c.n_in))
    _evaluator_session(eng, oracle, c, seeds, x)


def test_import_gc_extension_circuit(eng, oracle):
    # the extension record is flagged in the private byte, so a DAG circuit parses back
    c = _small_dag()
    x = np.random.default_rng(12).integers(-7, 8, size=(1, c.n_in))
    _evaluator_session(eng, oracle, c, [seed_hex(0x1E5)], x)


def test_import_gc_from_engine_garbler(eng):
    # garbler and evaluator both on the engine: GC bytes travel, labels do not
    from paper_2302_06361_b200.engine import DataError

    g = eng.model("model_tiny", 1000, 8, private=True)
    seeds = seed_hex(0x1F0) + seed_hex(0x1F1) + seed_hex(0x1F2)
    net = eng.garble(g, seeds)
    x = np.stack([g.random_input(30 + b) for b in range(3)])
    bi = eng.garble_inputs(net, x)
    ev = eng.import_gc([net.export_gc(b) for b in range(3)])
    bo = eng.evaluate(ev, eng.import_bundle(ev, b"".join(bi.payload(b) for b in range(3)), False))
    back = eng.import_bundle(net, b"".join(bo.payload(b) for b in range(3)), True)
    assert eng.decode_outputs(net, back).tolist() == [g.plain_forward(xi).tolist() for xi in x]
    with pytest.raises(DataError):  # the evaluator copy has no private weights
        eng.garble(ev.circuit, seed_hex(1))


def test_import_gc_rejects_bad_files(eng):
    from paper_2302_06361_b200.engine import DataError

    g = eng.model("relu4", 0, 2)
    gc = eng.garble(g, seed_hex(2)).export_gc(0)
    other = eng.garble(eng.model("relu16", 0, 2), seed_hex(2)).export_gc(0)
    bad = [gc[:-1], gc + b"\0", b"XASH" + gc[4:], gc[:6] + b"\x02" + gc[7:]]
    cut = 7 + 1 + 1 + 4 + 16 + 1  # header, k, shape, alpha/target, t
    bad.append(gc[:cut] + b"\x7f" + gc[cut + 1:])  # mixed-radix m_1 odd / out of range
    for b in bad:
        with pytest.raises(DataError):
            eng.import_gc([b])
    with pytest.raises(DataError):  # a batch must share its circuit
        eng.import_gc([gc, other])


@pytest.mark.parametrize("private", [False, True])
def test_import_gc_agrees_with_reference_parser(eng, private):
    # the compiled reference's parse_garbled_circuit + evaluate on the same
    # bytes: identical GARBLED_OUTPUT, and the same accept / reject verdicts
    import pyoracle
    from helpers import models
    from paper_2302_06361_b200.engine import DataError

    if not pyoracle.have_ref():
        pytest.skip("oracle/_ref not built")
    ref = pyoracle.RefLib()
    c = models.build("model_tiny", 1000, 8, private=private)
    seed = seed_hex(0x1A0)
    x = np.random.default_rng(13).integers(-7, 8, size=c.n_in)
    rnet = ref.garble(c, seed)
    rbi = ref.garble_inputs(rnet, x)
    gc = rnet.gc_bytes()
    ev = eng.import_gc([gc])
    bo = eng.evaluate(ev, eng.import_bundle(ev, rbi.payload(), False))
    assert bo.payload(0) == ref.eval_gc_bytes(gc, rbi).payload()
    cut = 7 + 1 + 1 + 4 * gc[8] + 16 + 1  # header, k, shape, alpha / target, t
    n_layers_at = cut + 2 * gc[cut - 1]
    for bad in (gc[:-16], gc + b"\0", gc[:4] + b"\x02\x00" + gc[6:], gc[:cut] + b"\x07" + gc[cut + 1:],
                gc[:n_layers_at + 2] + b"\x09" + gc[n_layers_at + 3:]):
        with pytest.raises(pyoracle.CheckerError) as e:
            ref.eval_gc_bytes(bad, rbi)
        assert e.value.code == 3
        with pytest.raises(DataError):
            eng.import_gc([bad])


@pytest.mark.gpu
def test_launch_shapes_agree(gpu):
    # Model A: batch 1 takes the level-parallel garbling and warp-per-label
    # PRF kernels, batch 8 the lane-group kernels, batch 160 the per-thread
    # persistent kernels; inference 0 (same seed, same input) must produce
    # the same garbled circuit, decoding tables and garbled output bytes
    g = gpu.model("model_a", 1001, 8)
    x0 = g.random_input(77)
    ref = None
    for B in (1, 8, 160):
        seeds = b"".join(seed_hex(0xAB00 + b) for b in range(B))
        x = np.stack([x0] + [g.random_input(78 + b) for b in range(1, B)])
        net = gpu.garble(g, seeds)
        bo = gpu.evaluate(net, gpu.garble_inputs(net, x))
        got = (sha(net.export_gc(0)), sha(net.export_decoding(0)), bo.payload(0),
               gpu.decode_outputs(net, bo)[0].tolist())
        if ref is None:
            ref = got
            assert got[3] == g.plain_forward(x0).tolist()
        assert got == ref, B


@pytest.mark.gpu
def test_import_gc_lenet_batch(gpu):
    # a full LeNet-5 GC (7.8 M rows, four activation layers in the device row
    # layout) exported, imported as a batch of 2 and evaluated: the imported
    # network's garbled outputs equal the garbling network's own evaluation
    g = gpu.model("lenet5", 2001, 8)
    seeds = seed_hex(0x1E70) + seed_hex(0x1E71)
    x = np.stack([g.random_input(5), g.random_input(6)])
    net = gpu.garble(g, seeds)
    bi = gpu.garble_inputs(net, x)
    bo = gpu.evaluate(net, bi)
    gcs = [net.export_gc(0), net.export_gc(1)]
    ev = gpu.import_gc(gcs)
    assert ev.export_gc(1) == gcs[1]
    bo2 = gpu.evaluate(ev, gpu.import_bundle(ev, bi.payload(0) + bi.payload(1), False))
    assert bo2.payload(0) == bo.payload(0) and bo2.payload(1) == bo.payload(1)
    out = gpu.decode_outputs(net, gpu.import_bundle(net, bo2.payload(0) + bo2.payload(1), True))
    assert out.tolist() == gpu.decode_outputs(net, bo).tolist()


def test_foreign_or_misshapen_bundles_are_data_errors(eng):
    # evaluate / decode_outputs input checks (garble.cpp:265-280, 314-322):
    # a bundle of another network, or of the wrong element count, is refused
    from paper_2302_06361_b200.engine import DataError

    g = eng.model("model_tiny", 1000, 8)
    a = eng.garble(g, seed_hex(0x51))
    b = eng.garble(g, seed_hex(0x52))
    x = g.random_input(3)[None, :]
    bi_b = eng.garble_inputs(b, x)
    with pytest.raises(DataError):
        eng.evaluate(a, bi_b)
    bo_b = eng.evaluate(b, bi_b)
    with pytest.raises(DataError):
        eng.decode_outputs(a, bo_b)
    lanes = [bo_b.labels(i) for i in range(g.info.k)]
    wrong = eng.bundle_from_labels(a, [l[:, :2] for l in lanes], output=True)  # 2 of 3 output elements
    with pytest.raises(DataError):
        eng.decode_outputs(a, wrong)
    with pytest.raises(DataError):
        eng.evaluate(a, eng.bundle_from_labels(a, [l[:, :2] for l in lanes], output=False))
    with pytest.raises(DataError):
        eng.bundle_from_labels(a, lanes[:-1], output=True)


@pytest.mark.gpu
@pytest.mark.parametrize("p,q", [(2, 2), (7, 7), (19, 19), (23, 110)])
def test_projection_ctx_device_path_matches_host_api(gpu, oracle, p, q):
    """The device-resident t_proj (dashgpu_proj_ctx_*, the raw projection
    sweep's path) over 70,000 gates (many blocks) gives the same rows / out0 /
    evaluations as the host-buffer API, which the test above pins to the
    oracle; a sample of rows is also checked against the oracle directly."""
    import torch

    gpu.set_stream(torch.cuda.current_stream().cuda_stream)
    n = 70_000
    seed = seed_hex(0xD0 + p)
    phi = [(v * v + 1) % q for v in range(p)]
    rnd = np.random.default_rng(p + q)
    lab = rnd.integers(0, 2**63, size=(n, 2), dtype=np.int64)
    gates = rnd.integers(0, 2**40, size=n).astype(np.int64)
    wires = (5_000_000 + np.arange(n)).astype(np.int64)
    dl, dg, dw = (torch.from_numpy(a).cuda() for a in (lab, gates, wires))
    rows = torch.empty((n * p, 2), dtype=torch.int64, device="cuda")
    out0 = torch.empty((n, 2), dtype=torch.int64, device="cuda")
    outv = torch.empty((n, 2), dtype=torch.int64, device="cuda")
    ctx = gpu.proj_ctx(seed, p, q, phi)
    ctx.garble(n, dl.data_ptr(), dg.data_ptr(), dw.data_ptr(), rows.data_ptr(), out0.data_ptr())
    ctx.eval(n, dl.data_ptr(), dg.data_ptr(), rows.data_ptr(), outv.data_ptr())
    torch.cuda.synchronize()
    rows_h = rows.cpu().numpy().view(np.uint64).reshape(n, p, 2)
    out0_h = out0.cpu().numpy().view(np.uint64)
    outv_h = outv.cpu().numpy().view(np.uint64)
    j = lambda a: int(a[0]) | (int(a[1]) << 64)  # noqa: E731
    sample = sorted(set(rnd.integers(0, n, size=40).tolist()) | {0, n - 1})
    labels = [j(lab[i].view(np.uint64)) for i in sample]
    hrows, hout0, (Rp, Rq) = gpu.proj_garble(seed, p, q, phi, labels, gates[sample].tolist(), wires[sample].tolist())
    hev = gpu.proj_eval(p, q, labels, gates[sample].tolist(), hrows)
    rp = np.array(oracle.decompress_mod(Rp, p))
    rq = np.array(oracle.decompress_mod(Rq, q))
    for t, i in enumerate(sample):
        assert [j(r) for r in rows_h[i]] == hrows[t]
        assert j(out0_h[i]) == hout0[t]
        assert j(outv_h[i]) == hev[t]
        x = np.array(oracle.decompress_mod(labels[t], p))
        o0 = np.array(oracle.decompress_mod(hout0[t], q))
        c = int(x[0])
        a = (t * 7) % p
        key = ((x + a * rp) % p).tolist()
        msg = ((o0 + phi[a] * rq) % q).tolist()
        assert j(rows_h[i][(c + a) % p]) == oracle.encrypt_label(p, key, int(gates[i]), (c + a) % p, 0, q, msg)
        # the base label is the active label of value 0
        assert j(outv_h[i]) == oracle.compress(q, ((o0 + phi[0] * rq) % q).tolist())


@pytest.mark.gpu
def test_linear_accumulator_wraps_like_the_reference(gpu):
    """The reference accumulates each digit sum in u32 and wraps
    (layer.cpp:116-118, acc[d] += w * digits[d]); windows with
    K (p-1)^2 >= 2^31 must still match.  Dense(1.6M -> 1), k = 16, every
    weight -1 (residue p-1) and every input digit p-1: lane p = 53 sums
    1.6M * 52^2 = 4.33e9 (wraps past 2^32), p = 47 sums 3.39e9 (bit 31 set)."""
    from paper_2302_06361_b200.circuit import Circuit, dense

    K = 1_600_000
    k = 16
    c = Circuit([K], k, [dense(K, 1, np.full((1, K), -1, np.int64), np.zeros(1, np.int64))])
    g = gpu.circuit(c)
    net = gpu.network_setup(g, seed_hex(0xACC))
    lanes = [np.full((1, K, _ndig(p)), p - 1, np.uint16) for p in PRIMES[:k]]
    out = gpu.layer_eval(net, 0, gpu.bundle_from_labels(net, lanes))
    for i, p in enumerate(PRIMES[:k]):
        acc = (K * (p - 1) * (p - 1)) % (1 << 32)
        got = out.labels(i)[0, 0]
        assert (got == acc % p).all(), (p, acc, got[:4])
    assert K * 52 * 52 >= 1 << 32 and (1 << 31) <= K * 46 * 46 < 1 << 32


@pytest.mark.gpu
def test_linear_mid_window_reduction_paths(gpu):
    """Digit-row epilogue reduction paths by window size (tc_linear.cuh,
    TcParams::nowrap): K = 100,000 at k = 16 sums below 2^31 but not below
    2^32 / p for p = 53 (the shifted 31-bit reduction), K = 4,096 below 2^32 / p
    for every lane (the shift-free one).  Weights +-1 (no zero residues),
    random input digits; the evaluator's lane is sum (w mod p) x mod p."""
    from paper_2302_06361_b200.circuit import Circuit, dense

    k = 16
    for K in (100_000, 4_096):
        assert (K + 3) * 53 * 53 < 1 << 31
        rng = np.random.default_rng(K)
        w = rng.choice([-1, 1], size=(2, K)).astype(np.int64)
        c = Circuit([K], k, [dense(K, 2, w, np.zeros(2, np.int64))])
        g = gpu.circuit(c)
        net = gpu.network_setup(g, seed_hex(0xACD))
        lanes = [rng.integers(0, p, size=(1, K, _ndig(p))).astype(np.uint16) for p in PRIMES[:k]]
        out = gpu.layer_eval(net, 0, gpu.bundle_from_labels(net, lanes))
        for i, p in enumerate(PRIMES[:k]):
            want = ((w % p) @ lanes[i][0].astype(np.int64)) % p  # [2 units][n_p digits]
            got = out.labels(i)[0]
            assert (got == want).all(), (K, p)


def _ndig(m):
    n, v = 0, 1
    while v * m <= 1 << 128:
        v *= m
        n += 1
    return n
