"""CPU oracle (oracle/dash_oracle.c) pinned against the reference.

* golden vectors in tests/golden/golden.json, produced by the UNMODIFIED
  reference compiled in place (tests/golden/gen_golden.py);
* the reference's own frozen constants (proj/tests/oracle/oracle_data.hpp:19-41)
  and SURVEY.md Appendix A known answers (FIPS-197 AES-128 zero KAT);
* direct comparison with oracle/_ref/libdashref.so when it is present.
"""
import random

import numpy as np
import pytest

from helpers import golden_circuit, golden_input, seed_hex, sha
from pyoracle import have_ref, n_digits


def test_fips197_zero_vector(oracle):
    # AES-128, all-zero key and block: 66e94bd4ef8a2c3b884cfa59ca342b2e (bytes);
    # the u128 little-endian view
    assert oracle.aes_fixed(0) == 0x2E2B34CA59FA4C883B2C8AEFD44BE966
    assert oracle.davies_meyer(0) == 0x2E2B34CA59FA4C883B2C8AEFD44BE966
    assert oracle.davies_meyer(1) == 0xD30F8EF52BBFBB59F06F1DE916187146


def test_appendix_a_vectors(oracle):
    seed = oracle.seed_from_string("5eed1")
    lab = oracle.prf_label(seed, 0, 7)
    assert len(lab) == 45 and lab[:10] == [2, 2, 5, 3, 2, 4, 6, 6, 6, 0]
    assert oracle.compress(7, lab) == 0x2E826986E657AA3741F40AE78BAF3500
    assert oracle.prf_offset(seed, 7)[:10] == [1, 5, 1, 0, 1, 4, 6, 1, 6, 5]
    assert oracle.pad_bits(7, lab, 5, 3, 0) == 0xC970265504197A945D2E9BD798B13320
    off11 = oracle.prf_offset(seed, 11)
    assert oracle.encrypt_label(7, lab, 5, 3, 0, 11, off11) == 0xF66EE3AC00A15AB95FC6B4C03A0E816D
    lab1 = oracle.prf_label(seed, 1, 7)
    assert oracle.pad_bits2(7, lab, 7, lab1, 9, 0, 1) == 0x93F13D9478AFB1D5DA95EAC34F114D5C


def test_digit_capacities(oracle):
    # oracle_data.hpp:19-21 (kPrimeDigits, kCompositeDigits)
    prime_digits = [128, 80, 55, 45, 37, 34, 31, 30, 28, 26, 25, 24, 23, 23, 23, 22]
    primes = [2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41, 43, 47, 53]
    assert [oracle.n_digits(p) for p in primes] == prime_digits
    for m, n in [(4, 64), (6, 49), (9, 40), (16, 32), (46, 23), (64, 21), (106, 19), (128, 18)]:
        assert oracle.n_digits(m) == n == n_digits(m)


def test_golden_kats(oracle, golden):
    kat = golden["kat"]
    assert hex(oracle.aes_fixed(0)) == kat["aes_pi_zero"]
    assert hex(oracle.davies_meyer(1)) == kat["davies_meyer_1"]
    assert oracle.seed_from_string("5eed1").hex() == kat["seed_5eed1"]
    for key, x, y in kat["aes_key"]:
        assert hex(oracle.aes_key(bytes.fromhex(key), int(x, 16))) == y
    for m, c, d, back in kat["codec"]:
        assert oracle.decompress_mod(int(c, 16), m) == d
        assert hex(oracle.compress(m, d)) == back
    seed = bytes.fromhex(kat["seed_5eed1"])
    for m, wire, d in kat["prf"]:
        got = oracle.prf_offset(seed, m) if wire < 0 else oracle.prf_label(seed, wire, m)
        assert got == d, (m, wire)
    for c in kat["cipher"]:
        assert hex(oracle.pad_bits(c["m"], c["key"], c["gate"], c["row"], c["slot"])) == c["pad_bits"]
        ct = oracle.encrypt_label(c["m"], c["key"], c["gate"], c["row"], c["slot"], c["q"], c["msg"])
        assert hex(ct) == c["ct"]
        assert oracle.decrypt_label(c["m"], c["key"], c["gate"], c["row"], c["slot"], ct, c["q"]) == c["msg"]
        assert hex(oracle.pad_bits2(c["m"], c["key"], c["q"], c["key2"], c["gate"], c["row"], c["slot"])) == \
            c["pad_bits2"]


def test_mixed_radix_specs(oracle, golden):
    # oracle_data.hpp:24-34 frozen by the reference's Python oracle
    assert oracle.choose_mixed_radix(8) == [110, 8, 7, 7, 6, 6, 5, 5]
    assert oracle.choose_mixed_radix(9) == [102, 7, 6, 5, 5, 5, 5, 5, 5, 5, 3]
    assert oracle.choose_mixed_radix(4) == [106, 4]
    assert oracle.choose_mixed_radix(3) == [46]
    for k, spec in golden["specs"]["full"].items():
        assert oracle.choose_mixed_radix(int(k)) == spec
    for k, tgt, spec in golden["specs"]["reduced"]:
        assert oracle.choose_mixed_radix(k, tgt) == spec, (k, tgt)


def test_gadget_costs(oracle, golden):
    # k=8 ReLU 1667 cts / 153 gates / 161 wires; SignAct 1582 cts
    assert oracle.element_cost(8, 1.0, 3) == (1667, 153, 161)
    assert oracle.element_cost(8, 1.0, 4)[0] == 1582
    for k, kind, cts, gates, wires in golden["specs"]["costs"]:
        assert oracle.element_cost(k, 1.0, kind) == (cts, gates, wires)


def _small(rec):
    return rec["stats"][0] < 3_000_000


@pytest.mark.parametrize("idx", range(29))
def test_oracle_networks_golden(oracle, golden, idx):
    if idx >= len(golden["networks"]):
        pytest.skip("no such record")
    rec = golden["networks"][idx]
    if not _small(rec):
        pytest.skip("large network: covered by the GPU suite and test_oracle_lenet")
    c = golden_circuit(rec)
    net = oracle.garble(c, seed_hex(int(rec["garble_seed"], 16)))
    gc = net.gc_bytes()
    assert len(gc) == rec["gc_len"]
    assert sha(gc) == rec["gc"]
    assert sha(net.enc_bytes()) == rec["enc"]
    assert sha(net.dec_bytes()) == rec["dec"]
    assert net.layer_ct_base() == rec["layer_ct_base"]
    assert list(net.stats()) == rec["stats"]
    for inp in rec["inputs"]:
        x = golden_input(rec, inp, c.n_in)
        bi = oracle.garble_inputs(net, x)
        assert sha(bi.payload()) == inp["gin"]
        bo = oracle.evaluate(net, bi)
        assert sha(bo.payload()) == inp["gout"]
        assert oracle.decode(net, bo).tolist() == inp["decoded"]


@pytest.mark.slow
def test_oracle_lenet(oracle, golden):
    rec = next(r for r in golden["networks"] if r["tag"] == "lenet5/s2001/k8/pub")
    c = golden_circuit(rec)
    net = oracle.garble(c, seed_hex(int(rec["garble_seed"], 16)))
    assert sha(net.gc_bytes()) == rec["gc"]
    inp = rec["inputs"][0]
    bo = oracle.evaluate(net, oracle.garble_inputs(net, golden_input(rec, inp, c.n_in)))
    assert oracle.decode(net, bo).tolist() == inp["decoded"]


def test_oracle_tamper_detected(oracle):
    # decode raises AuthenticityError on a label outside its table (garble.cpp:335-337)
    from helpers import models

    c = models.build("model_tiny", 1000, 8)
    net = oracle.garble(c, seed_hex(0xABC))
    x = np.zeros(c.n_in, np.int64)
    out = oracle.evaluate(net, oracle.garble_inputs(net, x))
    payload = bytearray(out.payload())
    payload[5] ^= 0x10
    bad = oracle.bundle_from_payload(net, bytes(payload), True)
    from pyoracle import CheckerError

    with pytest.raises(CheckerError) as e:
        oracle.decode(net, bad)
    assert e.value.code == 4


@pytest.mark.skipif(not have_ref(), reason="oracle/_ref not built (no /root/reference here)")
def test_oracle_matches_reference_randomized(oracle):
    from pyoracle import RefLib

    ref = RefLib()
    rnd = random.Random(99)
    seed = bytes(rnd.getrandbits(8) for _ in range(16))
    for _ in range(300):
        m = rnd.randrange(2, 129)
        c = rnd.getrandbits(128)
        d = ref.decompress_mod(c, m)
        assert oracle.decompress_mod(c, m) == d
        assert oracle.compress(m, d) == ref.compress(m, d)
        w = rnd.getrandbits(40)
        assert oracle.prf_label(seed, w, m) == ref.prf_label(seed, w, m)
        q = rnd.randrange(2, 129)
        msg = ref.prf_label(seed, w + 1, q)
        g, row, slot = rnd.getrandbits(48), rnd.randrange(1 << 16), rnd.randrange(3)
        assert oracle.encrypt_label(m, d, g, row, slot, q, msg) == ref.encrypt_label(m, d, g, row, slot, q, msg)


def test_reference_harness_rejects_extension_circuits():
    # Pad2d / Add / DAG inputs exist only in this repo (dash_circuit_desc.h):
    # the compiled reference must refuse them, not misread them
    import pyoracle
    from helpers import models

    if not pyoracle.have_ref():
        pytest.skip("oracle/_ref not built")
    with pytest.raises(pyoracle.CheckerError):
        pyoracle.RefLib().circuit(models.build("resnet_tiny", 2001, 8))
