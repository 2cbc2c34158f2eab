#!/usr/bin/env python3
"""Regenerates tests/golden/golden.json from the UNMODIFIED reference.

Runs only where the reference was compiled in place (oracle/_ref/libdashref.so,
built by `make -C oracle ref` from /root/reference/proj/core/src).  Every value
in the fixture is produced by the reference's own code through
oracle/ref_harness.cpp; circuit weights of the benchmark models (lenet5, ...)
come from the product's host-only model builders (the same mt19937 draw order
as the reference's tests/support/test_models.hpp), whose equality with the
reference builders is itself recorded for model_a / model_c / model_d /
model_f_dims / model_tiny.

usage: python tests/golden/gen_golden.py
"""
import hashlib
import json
import os
import random
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from pyoracle import RefLib, n_digits, seed_hex  # noqa: E402

from paper_2302_06361_b200 import models  # noqa: E402
from paper_2302_06361_b200.circuit import Circuit, Layer, RELU, SIGNACT  # noqa: E402

R = RefLib()


def h(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def kats():
    out = {}
    out["aes_pi_zero"] = hex(R.aes_fixed(0))
    out["davies_meyer_1"] = hex(R.davies_meyer(1))
    seed = R.seed_from_string("5eed1")
    out["seed_5eed1"] = seed.hex()
    rnd = random.Random(2302)
    out["aes_key"] = []
    for _ in range(8):
        key = bytes(rnd.getrandbits(8) for _ in range(16))
        x = rnd.getrandbits(128)
        out["aes_key"].append([key.hex(), hex(x), hex(R.aes_key(key, x))])
    out["codec"] = []
    for m in range(2, 129):
        for _ in range(3):
            c = rnd.getrandbits(128)
            d = R.decompress_mod(c, m)
            out["codec"].append([m, hex(c), d, hex(R.compress(m, d))])
    out["prf"] = []
    for m in [2, 3, 5, 7, 8, 9, 11, 13, 17, 19, 23, 33, 46, 53, 64, 110, 128]:
        for wire in [0, 1, 77, 12345678901]:
            out["prf"].append([m, wire, R.prf_label(seed, wire, m)])
        out["prf"].append([m, -1, R.prf_offset(seed, m)])  # offset R_m
    out["cipher"] = []
    for m, q in [(7, 11), (2, 2), (110, 2), (3, 9), (33, 5), (19, 2), (9, 2), (8, 33)]:
        k = R.prf_label(seed, 5, m)
        msg = R.prf_label(seed, 6, q)
        g, row, slot = rnd.getrandbits(40), rnd.randrange(128), rnd.randrange(3)
        pb = R.pad_bits(m, k, g, row, slot)
        ct = R.encrypt_label(m, k, g, row, slot, q, msg)
        dec = R.decrypt_label(m, k, g, row, slot, ct, q)
        assert dec == msg
        k2 = R.prf_label(seed, 9, q)
        out["cipher"].append({"m": m, "q": q, "key": k, "msg": msg, "gate": g, "row": row, "slot": slot,
                              "pad_bits": hex(pb), "ct": hex(ct),
                              "pad_bits2": hex(R.pad_bits2(m, k, q, k2, g, row, slot)), "key2": k2})
    return out


def specs():
    out = {"full": {}, "reduced": [], "costs": []}
    for k in range(1, 17):
        out["full"][str(k)] = R.choose_mixed_radix(k, 1.0)
    for k in range(2, 10):
        for tgt in (0.9999, 0.999, 0.99, 0.9):
            out["reduced"].append([k, tgt, R.choose_mixed_radix(k, tgt)])
    for k in range(1, 10):
        for kind in (RELU, SIGNACT):
            out["costs"].append([k, kind] + list(R.element_cost(k, 1.0, kind)))
    return out


def network_case(name, c: Circuit, gseed: int, input_seeds, tag):
    ch = R.circuit(c)
    net = R.garble(ch, seed_hex(gseed))
    rec = {"tag": tag, "model": name, "garble_seed": hex(gseed), "k": c.k,
           "gc": h(net.gc_bytes()), "enc": h(net.enc_bytes()), "dec": h(net.dec_bytes()),
           "gc_len": len(net.gc_bytes()), "layer_ct_base": net.layer_ct_base(), "stats": list(net.stats()),
           "inputs": []}
    P = 1
    for q in [2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41, 43, 47, 53][: c.k]:
        P *= q
    lo, hi = max(-7, -(P // 2)), min(7, (P + 1) // 2 - 1)
    rec["input_range"] = [lo, hi]
    for s in input_seeds:
        x = np.random.default_rng(s).integers(lo, hi + 1, size=c.n_in).astype(np.int64)
        bi = R.garble_inputs(net, x)
        bo = R.evaluate(net, bi)
        dec = R.decode(net, bo)
        rec["inputs"].append({"rng": s, "gin": h(bi.payload()), "gout": h(bo.payload()), "decoded": dec.tolist()})
    return rec


def networks():
    cases = []
    # the reference's own builders vs ours: identical weights
    for name, seed, k in [("model_a", 1001, 8), ("model_c", 1003, 9), ("model_d", 1004, 8),
                          ("model_f_dims", 1006, 9), ("model_tiny", 1000, 8)]:
        ref = R.model(name, seed, k)
        ours = models.build(name, seed, k)
        for a, b in zip(ref.c.layers, ours.layers):
            assert a.kind == b.kind
            if a.q_weights is not None:
                assert (a.q_weights == b.q_weights).all() and (a.q_biases == b.q_biases).all(), name
    plan = [
        ("model_tiny", 1000, 8, False, 0x5EED1, [11, 12]),
        ("model_tiny", 1000, 8, True, 0x5EED2, [13]),
        ("model_a", 1001, 8, False, 0xE2E0A1, [14, 15]),
        ("model_c", 1003, 9, False, 0xC0, [16]),
        ("model_d", 1004, 8, False, 0xD0, [17]),
        ("model_f_dims", 1006, 9, False, 0xF0, [18]),
        ("lenet5", 2001, 8, False, 0x5EED0000, [4000, 4001]),
        ("lenet5", 2001, 8, False, 0x5EED0001, [4002]),
    ]
    for k in range(2, 10):
        plan.append(("model_tiny", 1000, k, False, 0x7100 + k, [20 + k]))
        plan.append((f"relu96", 0, k, False, 0x7200 + k, [40 + k]))
    plan.append(("sign96", 0, 8, False, 0x7300, [60]))
    plan.append(("sign96", 0, 3, False, 0x7301, [61]))
    plan.append(("lenet5", 2001, 8, True, 0x7400, [62]))  # private-weight LeNet
    for name, seed, k, priv, gseed, ins in plan:
        c = models.build(name, seed, k, priv)
        cases.append(network_case(name, c, gseed, ins, f"{name}/s{seed}/k{k}/{'priv' if priv else 'pub'}"))
    # reduced-accuracy sign spec (sign_target < 1, mixed_radix.cpp:171-189)
    c = models.build("relu96", 0, 8)
    c.sign_target = 0.999
    cases.append(network_case("relu96", c, 0x7500, [63], "relu96/target0.999/k8"))
    c = models.build("model_tiny", 1000, 9)
    c.sign_target = 0.99
    cases.append(network_case("model_tiny", c, 0x7501, [64], "model_tiny/target0.99/k9"))
    return cases


def main():
    out = {"generator": "tests/golden/gen_golden.py (reference: oracle/_ref/libdashref.so)",
           "kat": kats(), "specs": specs(), "networks": networks()}
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path, os.path.getsize(path), "bytes,", len(out["networks"]), "networks")


if __name__ == "__main__":
    main()
